// gpar.cuh -- space-parallel coarse propagator G (north star item 5).
//
// In the parareal correction the coarse steps G(U^{k+1}_n) run one after the
// other; owner-G mode runs each on the GPU that owns slice n.  Space-parallel G instead cuts
// every coarse state into P bands of n/P rows and has all P GPUs advance the chain together
// (the paper's point that G is parallel in space).  For G = FIE on a 2-D
// dimensional split:
//   x stage  : (I - tau A_x) V_1 = U + tau F is row-local -- each band solves its own rows;
//   y stage  : (I - tau A_y) V_2 = V_1 couples the bands along every column.  Each band
//              composes its 64-row block tuples (lpass4.cuh) into one band tuple per column;
//              the P band tuples are all-gathered; every band then knows the y entering it and
//              the x leaving it (gp_boundary_kernel) and finishes its rows with the fused
//              correction epilogue.
// With one process the same code runs P virtual bands (the exchange is a no-op), which is
// how the partitioned solve is tested against the oracle on one GPU.
#pragma once
#include "common.cuh"
#include "lpass4.cuh"
#include "lpass5.cuh"

namespace prs {

// compose a band's nrb block tuples per column into the band tuple, tot = [5][n]
__global__ void gp_band_total_kernel(L5Args a, double *tot) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= a.n) return;
    Tup t = tup_id();
    for (int rb = 0; rb < a.nrb; ++rb) {
        const long long o = (long long)rb * a.n + col;
        t = tup_cat(t, Tup{a.tt[o], a.tt[a.tstride + o], a.tt[2 * a.tstride + o], a.tt[3 * a.tstride + o],
                           a.tt[4 * a.tstride + o]});
    }
    tot[col] = t.A;
    tot[a.n + col] = t.B;
    tot[2 * a.n + col] = t.P;
    tot[3 * a.n + col] = t.Q;
    tot[4 * a.n + col] = t.R;
}

// per column, from the P band tuples tots = [P][5][n]: y entering band b (forward composition
// of bands 0..b-1 from y = 0 at the line start) and x leaving it (backward composition of
// bands P-1..b+1 from x = 0 at the line end)
__global__ void gp_boundary_kernel(const double *tots, int P, int b, int n, double *ybeg, double *xend) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= n) return;
    constexpr int PMAX = 64;
    double yin[PMAX];
    double Y = 0.0;
    for (int q = 0; q < P; ++q) {
        yin[q] = Y;
        const double *t = tots + (long long)q * 5 * n;
        Y = fma(t[col], Y, t[n + col]);
    }
    double X = 0.0;  // x after band q (starting after the last band)
    for (int q = P - 1; q > b; --q) {
        const double *t = tots + (long long)q * 5 * n;
        X = fma(t[2 * n + col], X, fma(t[4 * n + col], yin[q], t[3 * n + col]));
    }
    ybeg[col] = yin[b];
    xend[col] = X;
}

}  // namespace prs
