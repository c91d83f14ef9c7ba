// ie.cuh -- unsplit implicit Euler, the Parareal/IE-IE baseline of PAPER.md:455 (SPEC.md:206-214,
// SURVEY.md 8(f) NEXT-4):  (I - tau A) U_{n+1} = U_n + tau F(t_{n+1}),  A the unsplit operator.
//
// Constant coefficients (kappa = 1, coef_kind 0; the paper's section-5.1 problem, D = I,
// PAPER.md:449): A = sum_d D_d - c I with D_d = h^-2 tridiag(1, -2, 1) along axis d (Dirichlet).
// The DST-I matrix S_ij = sin(pi (i+1)(j+1) h) diagonalises every D_d (S D_d S = -(n+1)/2 mu_i,
// mu_j = 4 h^-2 sin^2(j pi h / 2); the remark of PAPER.md:237-250) and S^2 = (n+1)/2 I, so the
// step is an exact direct solve in the sine basis:
//     U_{n+1} = (2 / (n+1))^dim  S^(x) ... S^(dim)  [ (S^(x) ... S^(dim) R) / (1 + tau (c + sum_d mu)) ],
//     R = U_n + tau F(t_{n+1}).
// Each S^(axis) is a dense n x n transform of every line along that axis: a batched GEMM
// Y[o][i][q] = sum_j S[i][j] X[o][j][q] (q < n^axis, o over the lines' outer index and the batch).
// These are the only flops of the step (4 dim n^(dim+1) per state), so it runs on the fp64 tensor
// cores (DMMA, mma.sync m8n8k4): 64 x 64 output tiles, k-steps of 16 through double-buffered
// shared memory (row stride 68: the m8n8k4 fragment loads are bank-conflict free), S read from
// L2 (n^2 doubles, resident).  The first forward pass forms R on its loads (source fused), the
// last forward pass applies the diagonal solve and the normalisation in its epilogue, and the
// last inverse pass carries the parareal epilogues of lpass.cuh (DELTA / CORRECT / INIT).
#pragma once
#include "common.cuh"
#include "lpass.cuh"

namespace prs {

constexpr int IE_BM = 64, IE_BN = 64, IE_BK = 16, IE_LD = 68, IE_T = 256;
constexpr int IE_SCALE = 4;  // epilogue of the last forward pass: the diagonal solve

struct IEArgs {
    const double *in;
    double *out;
    const double *S;    // n x n DST-I matrix (symmetric)
    long long vol;      // n^dim
    long long ncols;    // lines of the pass: B n^(dim-1)
    long long inner;    // n^axis: stride along the transformed axis
    int n;
    // prologue (first forward pass, axis 0): R = U + tau F, F = src_amp g(t) prod srcsin(x_d)
    int src, dim;
    double tau, src_amp;
    const double *sinpi;
    TimeArgs ta;
    // IE_SCALE: divide by 1 + tau (c + sum mu), times norm = (2 / (n+1))^dim
    const double *mu;
    double creact, norm;
    // parareal epilogues (lpass.cuh)
    const double *e_gc;
    double *e_gcache;
    const double *e_delta;
    double *e_traj;
    unsigned long long *e_red;
};

template <int PRO, int EPI>
__global__ void __launch_bounds__(IE_T) ie_axis_kernel(IEArgs a) {
    __shared__ double As[2][IE_BK][IE_LD];  // As[kk][ii] = S[k0 + kk][i0 + ii] (S symmetric)
    __shared__ double Bs[2][IE_BK][IE_LD];  // Bs[kk][cc] = X[line c0 + cc][k0 + kk]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 2, wn = warp & 3;  // warp tile: rows wm*32 .. +32, cols wn*16 .. +16
    const int n = a.n;
    // row tiles fastest: the CTAs that share a block of lines (and read it) run together (L2)
    const long long c0 = (long long)blockIdx.y * IE_BN;
    const int i0 = blockIdx.x * IE_BM;
    const bool unit = a.inner == 1;

    // this thread's four loads of each B tile: fixed lines, k rows advancing with the k-step
    int bkk[4], bcc[4];
    long long bbase[4];
    double bsrc[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int e = tid + IE_T * r;
        bkk[r] = unit ? (e & 15) : (e >> 6);  // unit stride: 16 consecutive k of one line (128 B)
        bcc[r] = unit ? (e >> 4) : (e & 63);  // strided: 64 consecutive lines of one k row
        const long long c = c0 + bcc[r];
        bbase[r] = -1;
        bsrc[r] = 0.0;
        if (c < a.ncols) {
            const long long o = c / a.inner, q = c - o * a.inner;
            bbase[r] = o * n * a.inner + q;
            if (PRO && a.src) {  // axis 0: line c = (state b, y [, z]); F = amp g(t) sy [sz] sx
                const long long per = a.vol / n, b = c / per, yz = c - b * per;
                double f = a.tau * a.src_amp * src_tf(a.ta, b) * __ldg(a.sinpi + yz % n);
                if (a.dim == 3) f *= __ldg(a.sinpi + yz / n);
                bsrc[r] = f;
            }
        }
    }
    const int nkt = (n + IE_BK - 1) / IE_BK;
    double ra[4], rb[4];
    auto gload = [&](int k0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int e = tid + IE_T * r, kk = e >> 6, ii = e & 63;
            const int k = k0 + kk, i = i0 + ii;
            ra[r] = (k < n && i < n) ? __ldg(a.S + (long long)k * n + i) : 0.0;
            const int kb = k0 + bkk[r];
            double x = 0.0;
            if (bbase[r] >= 0 && kb < n) {
                x = __ldg(a.in + bbase[r] + (long long)kb * a.inner);
                if (PRO) x = fma(bsrc[r], __ldg(a.sinpi + kb), x);
            }
            rb[r] = x;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int e = tid + IE_T * r;
            As[buf][e >> 6][e & 63] = ra[r];
            Bs[buf][bkk[r]][bcc[r]] = rb[r];
        }
    };
    double acc[4][2][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

    gload(0);
    sstore(0);
    __syncthreads();
    const int fr = lane >> 2, fk = lane & 3;
    for (int kt = 0; kt < nkt; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nkt) gload((kt + 1) * IE_BK);
#pragma unroll
        for (int ks = 0; ks < IE_BK / 4; ++ks) {
            double fa[4], fb[2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) fa[mt] = As[buf][4 * ks + fk][wm * 32 + mt * 8 + fr];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) fb[nt] = Bs[buf][4 * ks + fk][wn * 16 + nt * 8 + fr];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) dmma_f64(acc[mt][nt][0], acc[mt][nt][1], fa[mt], fb[nt]);
        }
        if (kt + 1 < nkt) sstore(buf ^ 1);
        __syncthreads();
    }

    // ---- epilogue: element (row i, line c) at base(c) + i * inner ----
    double dmax = 0.0;
    unsigned long long bad = 0;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const long long c = c0 + wn * 16 + nt * 8 + 2 * fk + h;
            if (c >= a.ncols) continue;
            const long long o = c / a.inner, q = c - o * a.inner;
            const long long base = o * n * a.inner + q;
            double cmu = 0.0;  // IE_SCALE (last axis, inner = n^(dim-1)): mu of the lower axes of q
            if (EPI == IE_SCALE) {
                cmu = __ldg(a.mu + q % n);
                if (a.dim == 3) cmu += __ldg(a.mu + q / n);
            }
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int i = i0 + wm * 32 + mt * 8 + fr;
                if (i >= n) continue;
                const long long g = base + (long long)i * a.inner;
                const double x = acc[mt][nt][h];
                if (EPI == IE_SCALE) {
                    a.out[g] = x * (a.norm / (1.0 + a.tau * (a.creact + cmu + __ldg(a.mu + i))));
                } else if (EPI == EPI_STORE) {
                    a.out[g] = x;
                } else if (EPI == EPI_DELTA) {
                    a.out[g] = x - a.e_gc[g];
                } else if (EPI == EPI_CORRECT) {
                    const double nv = x + a.e_delta[g];
                    const double ov = a.e_traj[g];
                    a.e_gcache[g] = x;
                    a.e_traj[g] = nv;
                    dmax = fmax(dmax, fabs(nv - ov));
                    if (!isfinite(nv)) bad = 1;
                } else {  // EPI_INIT
                    a.e_gcache[g] = x;
                    a.e_traj[g] = x;
                }
            }
        }
    if (EPI == EPI_CORRECT) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
            bad |= __shfl_xor_sync(0xffffffffu, bad, off);
        }
        if (lane == 0) {
            atomicMax(a.e_red, (unsigned long long)__double_as_longlong(dmax));
            if (bad) atomicOr(a.e_red + 1, 1ull);
        }
    }
}

// S_ij = sin(pi (i+1)(j+1) / (n+1)) with the integer product reduced mod 2(n+1) first (exact
// argument), mu_j = 4 h^-2 sin^2(pi (j+1) h / 2)
__global__ void ie_setup_kernel(int n, double h2inv, double *S, double *mu) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < (long long)n * n) {
        const long long i = e / n, j = e - i * n;
        const long long m = ((i + 1) * (j + 1)) % (2LL * (n + 1));
        S[e] = sinpi((double)m / (double)(n + 1));
    }
    if (e < n) {
        const double s = sinpi((double)(e + 1) / (2.0 * (double)(n + 1)));
        mu[e] = 4.0 * h2inv * s * s;
    }
}

}  // namespace prs
