// lpass8.cuh -- the long strided-line kernels of lpass5.cuh (block tuples K1, finish K3 over
// 64 x 64 tiles) made persistent over the slices of the batch, 2-D.
//
// Every slice of a fine sweep uses the same stage matrices, so the per-point pivots of a tile
// (and the face / node sines) are the same for all of them.  A CTA here owns one tile
// position and a group of S consecutive slices: it loads the tile's coefficients into
// registers once, then streams the slices' state tiles through a shared-memory ring with
// cp.async (3 slots at two CTAs per SM for the tuple kernel; 4 slots, also carrying each
// tile's boundary values, for the finish at one CTA per SM with the whole register file).
// DRAM traffic per point drops from state + pivots to state + pivots / S, and the copies in
// flight no longer depend on the per-thread register loads of the compute (lp5 with
// slice-fastest order became latency-bound exactly there: profiles/r01_fused_notes.md).  The arithmetic per tile is
// lpass5's (walk, 4-chunk tuple composition, exact forward / backward recurrences, fused
// parareal epilogue).
#pragma once
#include "common.cuh"
#include "lpass5.cuh"
#include "xpass3.cuh"

namespace prs {

constexpr int L8TILE = L5RB * L5W;     // doubles per state tile
constexpr int L8SLOT = L8TILE + 2 * L5W;  // + (finish) the tile's y entering / x leaving per column

// WIDE = 0: 2 CTAs per SM (128 registers), 3-slot ring; WIDE = 1: 1 CTA per SM with the whole
// register file (no spills of the coefficient registers) and a 4-slot ring
template <int WIDE>
struct L8Cfg {
    static constexpr int SLOTS = WIDE ? 4 : 3;
    static constexpr int MINB = WIDE ? 1 : 2;
};
inline size_t lpass8_smem_bytes(int wide) { return sizeof(double) * (size_t)(wide ? 4 : 3) * L8SLOT; }

// coefficients of one thread's column chunk (rows r0 .. r0+15 of column col)
template <int COEF>
__device__ __forceinline__ void l8_load_coef(const L5Args &a, int col, int r0, L5Chunk<COEF> &c) {
    const int n = a.n;
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

// MODE 0: block tuples (lp5_tuples_kernel); MODE 1: finish + epilogue (lp5_finish_kernel).
// Grid: (row block, column block, slice group) with the slice group fastest; a.s8 slices per
// group.  a.vol is the slice stride.
template <int COEF, int EPI, int MODE, int WIDE = 0>
__global__ void __launch_bounds__(L5T, L8Cfg<WIDE>::MINB) lp8_kernel(L5Args a) {
    constexpr int L8SLOTS = L8Cfg<WIDE>::SLOTS;
    extern __shared__ __align__(16) double ring[];
    __shared__ double st[5][L5CP][L5W];
    const int tid = threadIdx.x;
    const int w = tid % L5W, t = tid / L5W;
    const int n = a.n;
    const long long pos = blockIdx.x / a.nsg8;
    const int sg = (int)(blockIdx.x - pos * a.nsg8);
    const int cb = (int)(pos % a.ncb), rb = (int)(pos / a.ncb);
    const long long b0 = (long long)sg * a.s8;
    const long long b1 = min((long long)a.nsq, b0 + a.s8);
    const int col = cb * L5W + w;
    const int r0 = rb * L5RB + t * LCH;
    L5Chunk<COEF> c;
    l8_load_coef<COEF>(a, col, r0, c);

    const long long tile_off = (long long)(rb * L5RB) * n + cb * L5W;
    auto issue = [&](long long b, int slot) {
        const double *src = a.in + b * a.vol + tile_off;
        double *dst = ring + slot * L8SLOT;
#pragma unroll
        for (int q = 0; q < L8TILE / 2 / L5T; ++q) {  // 8 16-byte pieces per thread
            const int p = tid + q * L5T;
            const int row = p >> 5, u = p & 31;
            cp_async16(dst + row * L5W + 2 * u, src + (long long)row * n + 2 * u);
        }
        if (MODE == 1 && tid < L5W) {  // the block's boundary values ride along (2 x 64 doubles)
            const long long ob = (b * a.nrb + rb) * n + cb * L5W;
            const int h = tid >> 5, u = tid & 31;  // h = 0: y entering, 1: x leaving
            cp_async16(dst + L8TILE + h * L5W + 2 * u, a.yx + h * a.tstride + ob + 2 * u);
        }
    };
#pragma unroll
    for (int q = 0; q < L8SLOTS - 1; ++q) {
        if (b0 + q < b1) issue(b0 + q, q);
        cp_async_commit();
    }

    double dmax = 0.0;
    unsigned long long bad = 0;
    int slot = 0;
    for (long long b = b0; b < b1; ++b) {
        {
            int s2 = slot + L8SLOTS - 1;
            if (s2 >= L8SLOTS) s2 -= L8SLOTS;
            if (b + L8SLOTS - 1 < b1) issue(b + L8SLOTS - 1, s2);
            cp_async_commit();
        }
        cp_async_wait<L8SLOTS - 1>();
        __syncthreads();
        const double *tile = ring + slot * L8SLOT;
#pragma unroll
        for (int i = 0; i < LCH; ++i) c.v[i] = tile[(t * LCH + i) * L5W + w];
        const Tup u = c.walk1();
        if (MODE == 0) {
            st[0][t][w] = u.A;
            st[1][t][w] = u.B;
            st[2][t][w] = u.P;
            st[3][t][w] = u.Q;
            st[4][t][w] = u.R;
            __syncthreads();
            if (t == 0) {
                Tup tot = tup_id();
#pragma unroll
                for (int q = 0; q < L5CP; ++q)
                    tot = tup_cat(tot, Tup{st[0][q][w], st[1][q][w], st[2][q][w], st[3][q][w], st[4][q][w]});
                const long long o = (b * a.nrb + rb) * n + col;
                a.tt[o] = tot.A;
                a.tt[a.tstride + o] = tot.B;
                a.tt[2 * a.tstride + o] = tot.P;
                a.tt[3 * a.tstride + o] = tot.Q;
                a.tt[4 * a.tstride + o] = tot.R;
            }
        } else {
            const double Yblk = tile[L8TILE + w], Xblk = tile[L8TILE + L5W + w];
            st[0][t][w] = u.A;
            st[1][t][w] = u.B;
            st[2][t][w] = u.P;
            st[3][t][w] = u.Q;
            st[4][t][w] = u.R;
            __syncthreads();
            double Y = Yblk;
#pragma unroll
            for (int q = 0; q < L5CP; ++q)
                if (q < t) Y = fma(st[0][q][w], Y, st[1][q][w]);
            const double Ylast = fma(u.A, Y, u.B);
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
            const long long g0 = b * a.vol + (long long)r0 * n + col;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                const long long gi = g0 + (long long)i * n;
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
        }
        __syncthreads();  // ring slot and tuple scratch free for the next slice
        slot = (slot + 1 == L8SLOTS) ? 0 : slot + 1;
    }
    cp_async_wait<0>();
    if (MODE == 1 && EPI == EPI_CORRECT) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
            bad |= __shfl_xor_sync(0xffffffffu, bad, off);
        }
        if ((tid & 31) == 0) {
            atomicMax(a.e_red, (unsigned long long)__double_as_longlong(dmax));
            if (bad) atomicOr(a.e_red + 1, 1ull);
        }
    }
}

}  // namespace prs
