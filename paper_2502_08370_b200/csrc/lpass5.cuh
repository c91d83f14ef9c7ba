// lpass5.cuh -- strided-axis line pass for long lines (n >= 2048) in three launches over
// wide tiles, for HBM page locality.
//
// A cluster-split column panel (lpass3/lpass4) reads 64-byte row segments 32 KB apart, and
// the 144 co-resident CTAs touch only ~1 KB of each 32 KB state row at a time: DRAM row
// locality, not bandwidth, then limits the pass (measured: 1.6-2.6 TB/s at n = 4096 vs
// 5.2 TB/s for the same kernel on short lines).  Here the line is cut into row blocks of
// RB = 64 rows and every CTA works on a 64 x 64 tile (512-byte row segments, tiles in
// row-major order), with the coupling along the line carried by 5-tuples (lpass4.cuh):
//   K1 lp5_tuples  : per tile and column, walk with y_in = 0 -> chunk tuples -> the block
//                    tuple (A, B, P, Q, R) of the 64 rows;                 (reads 16 B/pt)
//   K2 lp5_scan    : per column, the sequential composition over the row blocks gives the
//                    incoming y of each block and the x after it;              (~1 B/pt)
//   K3 lp5_finish  : per tile, chunk tuples again, chunk-level y / x from the block values,
//                    exact forward and backward recurrences, fused epilogue. (24 B/pt)
// 16 rows per thread in registers; loads straight from global (a warp reads one 256-byte
// row segment per instruction), several hundred bytes in flight per thread.
#pragma once
#include "common.cuh"
#include "lpass.cuh"
#include "lpass4.cuh"

namespace prs {

constexpr int L5T = 256, L5W = 64, L5RB = 64, L5CP = L5RB / LCH;  // 4 chunks per column

struct L5Args {
    const double *in;
    double *out;
    long long vol;
    int n;
    long long Sl, Sq;     // line stride, plane stride
    int nq;               // planes per state
    int nrb, ncb;         // row blocks, column blocks per plane
    long long ntiles;     // batch * nq * nrb * ncb
    long long nsq;        // batch * nq
    int order;            // tile order: 0 column block fastest; 1 state fastest (pivot tiles
                          // shared by all states are then read by co-resident CTAs: L2 hits)
    int s8, nsg8;         // lpass8: slices per CTA, slice groups
    int row0;             // global row of local row 0 (a band of the lines, space-parallel G)
    const double *ybeg, *xend;  // lp5_scan: y entering / x leaving each line (per line; NULL: 0)
    double tau, h2inv;
    CoefTab tab;
    const double *invd, *s2n, *s2f;
    double *tt;           // block tuples [5][batch*nq][nrb][n]
    double *yx;           // [2][batch*nq][nrb][n]: y before the block, x after it
    long long tstride;    // batch*nq*nrb*n
    const double *e_gc;
    double *e_gcache;
    const double *e_delta;
    double *e_traj;
    unsigned long long *e_red;
};

// per-thread chunk data of one tile: values, pivots, coefficient accessors, walk 1
template <int COEF>
struct L5Chunk {
    double v[LCH], id[LCH], sf[LCH + 1], tm[LCH], ti[LCH], tc[LCH];
    double hsx, idm1, tauh;
    __device__ __forceinline__ double af(int i) const { return -tauh * fma(hsx, sf[i], 1.0); }
    __device__ __forceinline__ double cm(int i) const {
        return COEF ? af(i) * (i == 0 ? idm1 : id[i - 1]) : tm[i];
    }
    __device__ __forceinline__ double ci(int i) const { return COEF ? id[i] : ti[i]; }
    __device__ __forceinline__ double cc(int i) const { return COEF ? af(i + 1) * id[i] : tc[i]; }
    __device__ __forceinline__ Tup walk1() const {
        double y0 = 0.0, g = 1.0, cp = 1.0, Q = 0.0, R = 0.0;
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            const double m = cm(i);
            y0 = fma(-m, y0, v[i]);
            g = -m * g;
            const double cid = cp * ci(i);
            Q = fma(cid, y0, Q);
            R = fma(cid, g, R);
            cp *= -cc(i);
        }
        return Tup{g, y0, cp, Q, R};
    }
};

struct L5Tile {
    long long sq;       // state*nq + plane
    long long base;     // element offset of (row 0, column 0) of the plane
    int rb, cb;         // row block, column block
};
__device__ __forceinline__ L5Tile l5_tile(const L5Args &a, long long tile) {
    L5Tile T;
    if (a.order) {
        T.sq = tile % a.nsq;
        const long long r = tile / a.nsq;
        T.cb = (int)(r % a.ncb);
        T.rb = (int)(r / a.ncb);
    } else {
        T.cb = (int)(tile % a.ncb);
        const long long r = tile / a.ncb;
        T.rb = (int)(r % a.nrb);
        T.sq = r / a.nrb;
    }
    const long long b = T.sq / a.nq;
    const int q = (int)(T.sq - b * a.nq);
    T.base = b * a.vol + (long long)q * a.Sq;
    return T;
}

template <int COEF>
__device__ __forceinline__ void l5_load(const L5Args &a, const L5Tile &T, int w, int t, L5Chunk<COEF> &c) {
    const int n = a.n;
    const int col = T.cb * L5W + w;
    const int lr0 = T.rb * L5RB + t * LCH;  // local row (in the state / band)
    const int r0 = a.row0 + lr0;             // global row (coefficients, line boundary)
    const double *src = a.in + T.base + (long long)lr0 * a.Sl + col;
#pragma unroll
    for (int i = 0; i < LCH; ++i) c.v[i] = src[(long long)i * a.Sl];
    c.tauh = a.tau * a.h2inv;
    if (COEF) {
        const double *pd = a.invd + (long long)r0 * n + col;
#pragma unroll
        for (int i = 0; i < LCH; ++i) c.id[i] = __ldg(pd + (long long)i * n);
        c.idm1 = (r0 > 0) ? __ldg(pd - n) : 0.0;
#pragma unroll
        for (int i = 0; i <= LCH; ++i) c.sf[i] = __ldg(a.s2f + r0 + i);
        c.hsx = 0.5 * __ldg(a.s2n + col);
    } else {
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            c.tm[i] = __ldg(a.tab.m + r0 + i);
            c.ti[i] = __ldg(a.tab.id + r0 + i);
            c.tc[i] = __ldg(a.tab.cc + r0 + i);
        }
        c.hsx = 0.0;
        c.idm1 = 0.0;
    }
}

template <int COEF>
__global__ void __launch_bounds__(L5T, 2) lp5_tuples_kernel(L5Args a) {
    __shared__ double st[5][L5CP][L5W];
    const int w = threadIdx.x % L5W, t = threadIdx.x / L5W;
    const L5Tile T = l5_tile(a, blockIdx.x);
    L5Chunk<COEF> c;
    l5_load(a, T, w, t, c);
    const Tup u = c.walk1();
    st[0][t][w] = u.A;
    st[1][t][w] = u.B;
    st[2][t][w] = u.P;
    st[3][t][w] = u.Q;
    st[4][t][w] = u.R;
    __syncthreads();
    if (t == 0) {
        Tup tot = tup_id();
#pragma unroll
        for (int q = 0; q < L5CP; ++q) tot = tup_cat(tot, Tup{st[0][q][w], st[1][q][w], st[2][q][w], st[3][q][w], st[4][q][w]});
        const long long o = (T.sq * a.nrb + T.rb) * a.n + T.cb * L5W + w;
        a.tt[o] = tot.A;
        a.tt[a.tstride + o] = tot.B;
        a.tt[2 * a.tstride + o] = tot.P;
        a.tt[3 * a.tstride + o] = tot.Q;
        a.tt[4 * a.tstride + o] = tot.R;
    }
}

// one thread per (state*plane, column): y before each block (forward), x after it (backward)
__global__ void lp5_scan_kernel(L5Args a, long long ncols) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= ncols) return;
    const long long sq = idx / a.n;
    const int col = (int)(idx - sq * a.n);
    const long long o0 = sq * a.nrb * a.n + col;
    double Y = a.ybeg ? a.ybeg[idx] : 0.0;  // y entering the first block (0 at the line start)
    for (int rb = 0; rb < a.nrb; ++rb) {
        const long long o = o0 + (long long)rb * a.n;
        a.yx[o] = Y;
        Y = fma(a.tt[o], Y, a.tt[a.tstride + o]);
    }
    double X = a.xend ? a.xend[idx] : 0.0;  // x after the last block (0 at the line end)
    for (int rb = a.nrb - 1; rb >= 0; --rb) {
        const long long o = o0 + (long long)rb * a.n;
        a.yx[a.tstride + o] = X;
        // x at the first row of block rb, from its tuple and its incoming y
        X = fma(a.tt[2 * a.tstride + o], X, fma(a.tt[4 * a.tstride + o], a.yx[o], a.tt[3 * a.tstride + o]));
    }
}

template <int COEF, int EPI>
__global__ void __launch_bounds__(L5T, 2) lp5_finish_kernel(L5Args a) {
    __shared__ double st[5][L5CP][L5W];
    const int w = threadIdx.x % L5W, t = threadIdx.x / L5W;
    const L5Tile T = l5_tile(a, blockIdx.x);
    const long long ob = (T.sq * a.nrb + T.rb) * a.n + T.cb * L5W + w;
    const double Yblk = a.yx[ob], Xblk = a.yx[a.tstride + ob];
    L5Chunk<COEF> c;
    l5_load(a, T, w, t, c);
    const Tup u = c.walk1();
    st[0][t][w] = u.A;
    st[1][t][w] = u.B;
    st[2][t][w] = u.P;
    st[3][t][w] = u.Q;
    st[4][t][w] = u.R;
    __syncthreads();
    // y before this chunk: block input through the chunks before it
    double Y = Yblk;
#pragma unroll
    for (int q = 0; q < L5CP; ++q)
        if (q < t) Y = fma(st[0][q][w], Y, st[1][q][w]);
    const double Ylast = fma(u.A, Y, u.B);
    // x after this chunk: chunks after it, then the block's outgoing x
    Tup s = tup_id();
#pragma unroll
    for (int q = L5CP - 1; q >= 0; --q)
        if (q > t) s = tup_cat(Tup{st[0][q][w], st[1][q][w], st[2][q][w], st[3][q][w], st[4][q][w]}, s);
    const double X = fma(s.P, Xblk, fma(s.R, Ylast, s.Q));
    double y = Y;
#pragma unroll
    for (int i = 0; i < LCH; ++i) {
        y = fma(-c.cm(i), y, c.v[i]);
        c.v[i] = y;
    }
    double x = X;
#pragma unroll
    for (int i = LCH - 1; i >= 0; --i) {
        x = fma(-c.cc(i), x, c.ci(i) * c.v[i]);
        c.v[i] = x;
    }
    // ---- store + fused epilogue ----
    const int col = T.cb * L5W + w;
    const long long g0 = T.base + (long long)(T.rb * L5RB + t * LCH) * a.Sl + col;  // local rows
    double dmax = 0.0;
    unsigned long long bad = 0;
#pragma unroll
    for (int i = 0; i < LCH; ++i) {
        const long long gi = g0 + (long long)i * a.Sl;
        const double xv = c.v[i];
        if (EPI == EPI_STORE) {
            a.out[gi] = xv;
        } else if (EPI == EPI_DELTA) {
            a.out[gi] = xv - a.e_gc[gi];
        } else if (EPI == EPI_CORRECT) {
            const double nv = xv + a.e_delta[gi];
            const double ov = a.e_traj[gi];
            a.e_gcache[gi] = xv;
            a.e_traj[gi] = nv;
            dmax = fmax(dmax, fabs(nv - ov));
            if (!isfinite(nv)) bad = 1;
        } else {
            a.e_gcache[gi] = xv;
            a.e_traj[gi] = xv;
        }
    }
    if (EPI == EPI_CORRECT) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
            bad |= __shfl_xor_sync(0xffffffffu, bad, off);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMax(a.e_red, (unsigned long long)__double_as_longlong(dmax));
            if (bad) atomicOr(a.e_red + 1, 1ull);
        }
    }
}

}  // namespace prs
