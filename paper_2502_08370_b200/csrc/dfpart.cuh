// dfpart.cuh -- full-tensor DD block solves (section 5.2; c5, SURVEY.md 8(f)
// NEXT-3) as a row-partitioned block Thomas on the fp64 tensor cores.
//
// A block of colour j (W columns x n rows) is block tridiagonal over rows (ddfull.cuh):
//     D_l u_l + B_l u_{l-1} + C_l u_{l+1} = r_l,   factors E_l = B_l P_{l-1}^{-1}, P_l^{-1} (global,
//     precomputed per tau by df_factor_kernel), and the block Thomas recurrences
//     y_l = r_l - E_l y_{l-1},        x_l = P_l^{-1} (y_l - C_l x_{l+1}).
// Both are linear recurrences with data-independent matrix coefficients, so their application
// is split into partitions of DFP_M rows that run in parallel, with a scan over the partitions
// (the W x W analogue of the tuple scan of the kappa = 1 DD stage, dd.cuh):
//   over partition p (rows a..b):  y_b = A_p y_{a-1} + (y_b with y_{a-1} = 0),  A_p = (-E_b)..(-E_a)
//                                  x_a = Pp_p x_{b+1} + (x_a with x_{b+1} = 0), Pp_p = (-G_a)..(-G_b),
//                                  G_l = P_l^{-1} C_l
// (A_p, Pp_p precomputed per tau by running the same sweeps on unit columns).  A stage is
//   dfp_fwd (y_in = 0: the partition's y_b)  ->  dfp_scan forward (y_in of every partition)
//   -> dfp_fwd (exact y of every row, stored)  ->  dfp_bwd (x_in = 0: the partition's x_a)
//   -> dfp_scan backward (x_in of every partition)  ->  dfp_bwd (exact x, fused epilogue),
// each sweep one CTA per (block, partition, group of DFP_S states), every row step a W x W by
// W x DFP_S product on DMMA (m8n8k4 f64; the matrix fragments stream from L2, the right-hand
// sides sit in shared memory).  Per row and state 4 W^2 FMA (twice the sequential block Thomas)
// buy n / DFP_M-fold row parallelism and DFP_S-fold reuse of every streamed factor.
// The stage logic and the parareal epilogues are those of df_stage_kernel (ddfull.cuh).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "ddfull.cuh"

namespace prs {

constexpr int DFP_M = 64;             // rows per partition (default; dfp_rows in dd.cuh)
constexpr int DFP_S = 16;             // right-hand sides per CTA (two n-tiles of 8)
constexpr int DFP_SP = DFP_S + 4;     // shared row stride of a W x S tile (conflict-free fragments)
constexpr int DFP_NW = DF_WMAX / 16;  // 9 warps: m-tiles w and w + 9 of the W <= 144 rows
constexpr int DFP_T = 32 * DFP_NW;    // 288 threads
constexpr int DFP_PF = 8;             // k-steps of matrix fragments in flight per warp
constexpr int DFP_TILE = DF_WMAX * DFP_SP;

struct DFPArgs {
    // the stage (pass kernels): batch in / out, stage colour, operators, epilogue (df_stage_kernel)
    const double *U;
    double *V;
    long long vol;
    int n, B, stage, nblk, ngrp, P;  // P = partitions per block, ngrp = state groups (of DFP_S)
    int M;                           // rows per partition (dfp_rows: DFP_M, shortened to fill the SMs)
    const int *bi0, *bW;
    const double *const *ET, *const *PI;   // per block: E_l^T and P_l^{-1} (n W^2 each)
    const double *const *AT, *const *PpT;  // per block: A_p^T and Pp_p^T (P W^2 each)
    double tau, c;
    DFOp op_me, op_ot;
    double src_amp;
    const double *sinpi;
    TimeArgs ta;
    int epi;
    const double *e_gc;
    double *e_gcache;
    const double *e_delta;
    double *e_traj;
    unsigned long long *e_red;
    // scratch, tiles of W x DFP_S doubles ([i][s], stride DFP_S; tile pitch DF_WMAX x DFP_S): per (block, group, partition)
    // tl (the partition's y_b or x_a with zero inflow), bnd_y / bnd_x (y_in / x_in); per
    // (block, group) ys: the exact y of every row [n][W][DFP_S]
    double *tl, *bnd_y, *bnd_x, *ys;
    // setup mode: write A_p^T / Pp_p^T of this colour (unit columns instead of states)
    double *const *setup_out;
    int setup;
};

// -------------------------------------------------------------------- the row step ------
// D = R + sgn M Y on DMMA for W <= 144 rows and DFP_S columns: M given transposed in global
// memory (MT[k W + i] = M[i][k]); Y, R (= D on entry) and D are shared [i][DFP_SP] tiles
// (D may alias R, not Y).  Warp w owns m-tiles w and w + 9 for both n-tiles.  The first DFP_PF
// k-steps of matrix fragments are loaded by dfp_mpre (before the barrier that publishes Y, so
// that their latency overlaps it).
struct DFPFrag {
    double a[DFP_PF][2];
};
__device__ __forceinline__ void dfp_mload(const double *__restrict__ MT, int W, int ks, double &a0, double &a1) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = 4 * ks + (lane & 3), r0 = 8 * warp + (lane >> 2), r1 = r0 + 72;
    const bool kin = k < W;
    a0 = (kin && r0 < W) ? __ldg(MT + (long long)k * W + r0) : 0.0;
    a1 = (kin && r1 < W) ? __ldg(MT + (long long)k * W + r1) : 0.0;
}
__device__ __forceinline__ void dfp_mpre(DFPFrag &f, const double *MT, int W) {
#pragma unroll
    for (int q = 0; q < DFP_PF; ++q) dfp_mload(MT, W, q, f.a[q][0], f.a[q][1]);
}
__device__ __forceinline__ void dfp_rowstep(DFPFrag &f, const double *__restrict__ MT, int W, const double *Y,
                                            double *D, double sgn) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane >> 2, fk = lane & 3;
    const int r0 = 8 * warp + fr, r1 = r0 + 72;  // the thread's C rows (m-tiles w, w + 9)
    double acc[2][2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
        const int col = 8 * nt + 2 * fk;
        acc[0][nt][0] = r0 < W ? D[r0 * DFP_SP + col] : 0.0;
        acc[0][nt][1] = r0 < W ? D[r0 * DFP_SP + col + 1] : 0.0;
        acc[1][nt][0] = r1 < W ? D[r1 * DFP_SP + col] : 0.0;
        acc[1][nt][1] = r1 < W ? D[r1 * DFP_SP + col + 1] : 0.0;
    }
    const int nks = (W + 3) / 4;
    for (int ks0 = 0; ks0 < nks; ks0 += DFP_PF) {
#pragma unroll
        for (int q = 0; q < DFP_PF; ++q) {
            const int ks = ks0 + q;
            if (ks < nks) {
                const double a0 = sgn * f.a[q][0], a1 = sgn * f.a[q][1];
                if (ks + DFP_PF < nks) dfp_mload(MT, W, ks + DFP_PF, f.a[q][0], f.a[q][1]);
                const int k = 4 * ks + fk;
                const double b0 = k < W ? Y[k * DFP_SP + fr] : 0.0, b1 = k < W ? Y[k * DFP_SP + 8 + fr] : 0.0;
                dmma_f64(acc[0][0][0], acc[0][0][1], a0, b0);
                dmma_f64(acc[0][1][0], acc[0][1][1], a0, b1);
                dmma_f64(acc[1][0][0], acc[1][0][1], a1, b0);
                dmma_f64(acc[1][1][0], acc[1][1][1], a1, b1);
            }
        }
    }
    __syncthreads();  // every read of R (= D) done before it is overwritten
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
        const int col = 8 * nt + 2 * fk;
        if (r0 < W) {
            D[r0 * DFP_SP + col] = acc[0][nt][0];
            D[r0 * DFP_SP + col + 1] = acc[0][nt][1];
        }
        if (r1 < W) {
            D[r1 * DFP_SP + col] = acc[1][nt][0];
            D[r1 * DFP_SP + col + 1] = acc[1][nt][1];
        }
    }
    __syncthreads();
}

// The same row step with the matrix streamed through shared memory: its rows k < KS and k >= KS
// (KS = 4 ceil(nks / 2)) are two contiguous halves, each filled by one bulk copy (TMA engine,
// completing on the half's mbarrier).  The next row's halves are issued as soon as the current
// row's k-steps over that half are done (every warp past the barrier), so that the fill of one
// half overlaps the products over the other, and a row's matrix is read from HBM / L2 once per CTA.
struct DFPStream {
    double *buf[2];               // shared halves (DF_WMAX / 2 + 4 rows of DF_WMAX doubles each)
    unsigned long long *mb;       // [2] mbarriers
    unsigned par;                 // bits: parity of each half's next fill
};
constexpr int DFP_HALF = (DF_WMAX / 2 + 4) * DF_WMAX;  // doubles per shared half (+ slack: offsets, rounding)
__device__ __forceinline__ int dfp_ksplit(int W) { return 4 * ((((W + 3) / 4) + 1) / 2); }
// (a half whose first element is not 16-byte aligned -- odd W -- is copied from the aligned
// address below it and read one double further in: dfp_half_off)
__device__ __forceinline__ int dfp_half_off(const double *MT, int W, int h) {
    const int k0 = h ? dfp_ksplit(W) : 0;
    return (int)((reinterpret_cast<uintptr_t>(MT + (long long)k0 * W) & 15) >> 3);
}
__device__ __forceinline__ void dfp_issue_half(DFPStream &st, const double *MT, int W, int h) {
    // one thread: copy rows [k0, k1) of MT (W doubles each) into half h
    const int ks = dfp_ksplit(W), k0 = h ? ks : 0, k1 = h ? W : min(ks, W);
    if (k1 <= k0) {
        mbar_arrive_expect(st.mb + h, 0);
        return;
    }
    const int off = dfp_half_off(MT, W, h);
    const unsigned bytes = (unsigned)((((size_t)(k1 - k0) * W + off) * sizeof(double) + 15) & ~(size_t)15);
    PRS_CHECK(bytes <= DFP_HALF * sizeof(double), "full-tensor matrix half larger than its shared buffer");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_arrive_expect(st.mb + h, bytes);
    const char *src = reinterpret_cast<const char *>(MT + (long long)k0 * W - off);
    for (unsigned off = 0; off < bytes; off += 32768u) {  // pieces of <= 32 KB
        const unsigned len = min(32768u, bytes - off);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         smem_u32(reinterpret_cast<char *>(st.buf[h]) + off)),
                     "l"(src + off), "r"(len), "r"(smem_u32(st.mb + h))
                     : "memory");
    }
}
__device__ __forceinline__ void dfp_issue(DFPStream &st, const double *MT, int W) {
    if (threadIdx.x == 0) {
        dfp_issue_half(st, MT, W, 0);
        dfp_issue_half(st, MT, W, 1);
    }
}
// D = R + sgn M Y with M's halves in st (issued before); `next` (or null): the matrix of the next
// row step, issued half by half as the halves free up
__device__ __forceinline__ void dfp_rowstep_s(DFPStream &st, const double *cur, const double *next, int W, const double *Y,
                                              double *D, double sgn, bool zero_r = false) {
    // (zero_r: R = 0, D is only written)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane >> 2, fk = lane & 3;
    const int r0 = 8 * warp + fr, r1 = r0 + 72;
    double acc[2][2][2], rv[2][2][2];  // M Y (from zero), R
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
        const int col = 8 * nt + 2 * fk;
        rv[0][nt][0] = (!zero_r && r0 < W) ? D[r0 * DFP_SP + col] : 0.0;
        rv[0][nt][1] = (!zero_r && r0 < W) ? D[r0 * DFP_SP + col + 1] : 0.0;
        rv[1][nt][0] = (!zero_r && r1 < W) ? D[r1 * DFP_SP + col] : 0.0;
        rv[1][nt][1] = (!zero_r && r1 < W) ? D[r1 * DFP_SP + col + 1] : 0.0;
        acc[0][nt][0] = acc[0][nt][1] = acc[1][nt][0] = acc[1][nt][1] = 0.0;
    }
    const int ks = dfp_ksplit(W), nks = (W + 3) / 4;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
        mbar_wait(st.mb + h, (st.par >> h) & 1u);
        st.par ^= 1u << h;
        const double *Ms = st.buf[h] + dfp_half_off(cur, W, h);
        const int q0 = h ? ks / 4 : 0, q1 = h ? nks : min(ks / 4, nks), kb = h ? ks : 0;
#pragma unroll 4
        for (int q = q0; q < q1; ++q) {
            const int k = 4 * q + fk;
            const bool kin = k < W;
            const double *mr = Ms + (long long)(k - kb) * W;
            const double a0 = (kin && r0 < W) ? mr[r0] : 0.0, a1 = (kin && r1 < W) ? mr[r1] : 0.0;
            const double b0 = kin ? Y[k * DFP_SP + fr] : 0.0, b1 = kin ? Y[k * DFP_SP + 8 + fr] : 0.0;
            dmma_f64(acc[0][0][0], acc[0][0][1], a0, b0);
            dmma_f64(acc[0][1][0], acc[0][1][1], a0, b1);
            dmma_f64(acc[1][0][0], acc[1][0][1], a1, b0);
            dmma_f64(acc[1][1][0], acc[1][1][1], a1, b1);
        }
        __syncthreads();  // half h consumed (h = 1: every read of R / Y done as well)
        if (next && threadIdx.x == 0) dfp_issue_half(st, next, W, h);
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
        const int col = 8 * nt + 2 * fk;
        if (r0 < W) {
            D[r0 * DFP_SP + col] = fma(sgn, acc[0][nt][0], rv[0][nt][0]);
            D[r0 * DFP_SP + col + 1] = fma(sgn, acc[0][nt][1], rv[0][nt][1]);
        }
        if (r1 < W) {
            D[r1 * DFP_SP + col] = fma(sgn, acc[1][nt][0], rv[1][nt][0]);
            D[r1 * DFP_SP + col + 1] = fma(sgn, acc[1][nt][1], rv[1][nt][1]);
        }
    }
    __syncthreads();
}
__device__ __forceinline__ DFPStream dfp_stream_init(double *smem_halves, unsigned long long *mb) {
    DFPStream st;
    st.buf[0] = smem_halves;
    st.buf[1] = smem_halves + DFP_HALF;
    st.mb = mb;
    st.par = 0;
    if (threadIdx.x == 0) {
        mbar_init(mb, 1);
        mbar_init(mb + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    return st;
}

// global W x DFP_S tile <-> shared tile
__device__ __forceinline__ void dfp_tile_load(double *T, const double *G, int W) {
    for (int e = threadIdx.x; e < W * DFP_S; e += blockDim.x) T[(e / DFP_S) * DFP_SP + e % DFP_S] = G[e];
}
__device__ __forceinline__ void dfp_tile_store(double *G, const double *T, int W) {
    for (int e = threadIdx.x; e < W * DFP_S; e += blockDim.x) G[e] = T[(e / DFP_S) * DFP_SP + e % DFP_S];
}
__device__ __forceinline__ void dfp_tile_zero(double *T, int W) {
    for (int e = threadIdx.x; e < W * DFP_SP; e += blockDim.x) T[e] = 0.0;
}

// one task: block blk, state group grp, partition p (CTA index = (blk * ngrp + grp) * P + p)
struct DFPTask {
    int blk, grp, p, W, i0, a, m;  // rows a .. a + m - 1
    long long bg;                  // blk * ngrp + grp
    __device__ __forceinline__ DFPTask(const DFPArgs &x, long long cta) {
        p = (int)(cta % x.P);
        bg = cta / x.P;
        grp = (int)(bg % x.ngrp);
        blk = (int)(bg / x.ngrp);
        W = x.bW[blk];
        i0 = x.bi0[blk];
        a = p * x.M;
        m = min(x.M, x.n - a);
        PRS_CHECK(blk < x.nblk && W <= DF_WMAX && m > 0 && i0 >= 0 && i0 + W <= x.n, "full-tensor task");
    }
};

// w = tau A_ot U at (gi, l) of state b (DR stage 0: the other colour's explicit term, ddfull.cuh)
__device__ __forceinline__ double dfp_wterm(const DFPArgs &x, const double *Ub, int gi, int l) {
    double cf[3][3];
    x.op_ot.stencil(gi, l, cf);
    double s = 0.0;
#pragma unroll
    for (int dl = -1; dl <= 1; ++dl) {
        const int ll = l + dl;
        if (ll < 0 || ll >= x.n) continue;
#pragma unroll
        for (int di = -1; di <= 1; ++di) {
            const int ii = gi + di;
            if (ii < 0 || ii >= x.n) continue;
            s = fma(cf[di + 1][dl + 1], Ub[(long long)ll * x.n + ii], s);
        }
    }
    return x.tau * s;
}

// the stage right-hand side of row l into the shared tile R (the stage logic
// of df_stage_kernel): stage 1 takes V on the columns already final after stage 0
// (consecutive threads take consecutive columns of one state: coalesced; ampt[s] = the source
// amplitude of state s of the group at its time, precomputed per CTA)
template <int DR, int SRC>
__device__ __forceinline__ void dfp_rhs(const DFPArgs &x, const DFPTask &t, int l, double *R, const double *ampt) {
    for (int e = threadIdx.x; e < t.W * DFP_S; e += blockDim.x) {
        const int s = e / t.W, i = e - s * t.W;
        const long long b = (long long)t.grp * DFP_S + s;
        double r = 0.0;
        if (b < x.B) {
            const int gi = t.i0 + i;
            const long long g = (long long)l * x.n + gi;
            const double *Ub = x.U + b * x.vol;
            if (x.stage == 1 && x.op_ot.rhon[gi] > 0.0) {
                r = x.V[b * x.vol + g];
            } else {
                r = Ub[g];
                if (SRC) r = fma(x.tau * ampt[s] * __ldg(x.sinpi + l), __ldg(x.sinpi + gi), r);
                if (DR && x.stage == 0) r += dfp_wterm(x, Ub, gi, l);
            }
        }
        R[i * DFP_SP + s] = r;
    }
}
// the same in two halves, for the rows whose right-hand side needs no stencil (not DR stage 0):
// dfp_rhs_load issues the thread's loads of row l into registers (ahead of the row step that
// precedes their use), dfp_rhs_put completes them into the tile
constexpr int DFP_RPT = (DF_WMAX * DFP_S + DFP_T - 1) / DFP_T;  // elements per thread (8)
// the thread's elements e = tid + j DFP_T of a W x DFP_S tile in state-major order: s = e / W,
// i = e % W, packed (s << 16 | i), -1 past the tile (computed once per CTA: no divisions per row)
struct DFPElems {
    int si[DFP_RPT];
    __device__ __forceinline__ DFPElems(int W) {
#pragma unroll
        for (int j = 0; j < DFP_RPT; ++j) {
            const int e = threadIdx.x + j * DFP_T, s = e / W;
            si[j] = (e < W * DFP_S) ? ((s << 16) | (e - s * W)) : -1;
        }
    }
};
template <int SRC>
__device__ __forceinline__ void dfp_rhs_load(const DFPArgs &x, const DFPTask &t, const DFPElems &el, int l,
                                             double (&r)[DFP_RPT]) {
#pragma unroll
    for (int j = 0; j < DFP_RPT; ++j) {
        r[j] = 0.0;
        if (el.si[j] >= 0 && l < x.n) {
            const int s = el.si[j] >> 16, i = el.si[j] & 0xffff;
            const long long b = (long long)t.grp * DFP_S + s;
            if (b < x.B) {
                const int gi = t.i0 + i;
                const long long g = (long long)l * x.n + gi;
                r[j] = (x.stage == 1 && x.op_ot.rhon[gi] > 0.0) ? x.V[b * x.vol + g] : x.U[b * x.vol + g];
            }
        }
    }
}
template <int SRC>
__device__ __forceinline__ void dfp_rhs_put(const DFPArgs &x, const DFPTask &t, const DFPElems &el, int l,
                                            const double (&r)[DFP_RPT], double *R, const double *ampt) {
#pragma unroll
    for (int j = 0; j < DFP_RPT; ++j) {
        if (el.si[j] >= 0) {
            const int s = el.si[j] >> 16, i = el.si[j] & 0xffff;
            const int gi = t.i0 + i;
            double v = r[j];
            if (SRC && !(x.stage == 1 && x.op_ot.rhon[gi] > 0.0) && (long long)t.grp * DFP_S + s < x.B)
                v = fma(x.tau * ampt[s] * __ldg(x.sinpi + l), __ldg(x.sinpi + gi), v);
            R[i * DFP_SP + s] = v;
        }
    }
}
__device__ __forceinline__ void dfp_ampt(const DFPArgs &x, int grp, double *ampt) {
    for (int s = threadIdx.x; s < DFP_S; s += blockDim.x)
        ampt[s] = x.src_amp * src_tf(x.ta, (long long)grp * DFP_S + s);
}

// ------------------------------------------------------------------ forward sweeps ------
// MODE 0: y_in = 0, the partition's last y -> tl;  MODE 1: y_in = bnd_y, every y -> ys;
// MODE 2 (setup): zero right-hand sides, y_in = unit columns 16 grp .. (A_p^T -> setup_out)
template <int DR, int SRC, int MODE>
__global__ void __launch_bounds__(DFP_T, 1) dfp_fwd_kernel(DFPArgs x) {
    extern __shared__ __align__(16) double sm[];  // matrix halves, 2 tiles
    __shared__ __align__(8) unsigned long long mb[2];
    __shared__ double ampt[DFP_S];
    DFPStream st = dfp_stream_init(sm, mb);
    double *Yc = sm + 2 * DFP_HALF, *Yn = Yc + DFP_TILE;
    const DFPTask t(x, blockIdx.x);
    const int W = t.W;
    const long long tix = t.bg * x.P + t.p;
    const double *ET = x.ET[t.blk];
    const long long WW = (long long)W * W;
    const int lfirst = max(t.a, 1);  // the first row with an E term
    if (lfirst < t.a + t.m) dfp_issue(st, ET + lfirst * WW, W);
    if (SRC && MODE != 2) dfp_ampt(x, t.grp, ampt);
    if (MODE == 1) {
        dfp_tile_load(Yc, x.bnd_y + tix * DF_WMAX * DFP_S, W);
    } else {
        dfp_tile_zero(Yc, W);
        if (MODE == 2) {
            __syncthreads();
            for (int s = threadIdx.x; s < DFP_S; s += blockDim.x)
                if (DFP_S * t.grp + s < W) Yc[(DFP_S * t.grp + s) * DFP_SP + s] = 1.0;
        }
    }
    __syncthreads();
    const bool pre = MODE != 2 && !(DR && x.stage == 0);  // right-hand sides loaded a row ahead
    const DFPElems el(W);
    double rr[DFP_RPT];
    if (pre) dfp_rhs_load<SRC>(x, t, el, t.a, rr);
    for (int rl = 0; rl < t.m; ++rl) {
        const int l = t.a + rl;
        if (MODE == 2) dfp_tile_zero(Yn, W);
        else if (pre) dfp_rhs_put<SRC>(x, t, el, l, rr, Yn, ampt);
        else dfp_rhs<DR, SRC>(x, t, l, Yn, ampt);
        __syncthreads();
        if (pre && rl + 1 < t.m) dfp_rhs_load<SRC>(x, t, el, l + 1, rr);
        if (l > 0)  // y_l = r_l - E_l y_{l-1}
            dfp_rowstep_s(st, ET + l * WW, rl + 1 < t.m ? ET + (l + 1) * WW : nullptr, W, Yc, Yn, -1.0);
        if (MODE == 1) dfp_tile_store(x.ys + (t.bg * x.n + l) * DF_WMAX * DFP_S, Yn, W);
        double *tmp = Yc;
        Yc = Yn;
        Yn = tmp;
        __syncthreads();
    }
    if (MODE == 0) dfp_tile_store(x.tl + tix * DF_WMAX * DFP_S, Yc, W);
    if (MODE == 2) {  // A_p^T [k][i] = A_p[i][k]: unit column k = 16 grp + s of the output
        double *AT = x.setup_out[t.blk] + (long long)t.p * WW;
        for (int e = threadIdx.x; e < W * DFP_S; e += blockDim.x) {
            const int i = e / DFP_S, s = e % DFP_S, k = DFP_S * t.grp + s;
            if (k < W) AT[(long long)k * W + i] = Yc[i * DFP_SP + s];
        }
    }
}

// ----------------------------------------------------------------- backward sweeps ------
// T_l = y_l - C_l x_{l+1} (C_l tridiagonal, ddfull.cuh DFOp::up), x_l = P_l^{-1} T_l.
// MODE 0: x_in = 0, the partition's first x -> tl;  MODE 1: x_in = bnd_x, every x through the
// stage epilogue;  MODE 2 (setup): y = 0, x_in = unit columns (Pp_p^T -> setup_out)
template <int DR, int MODE>
__global__ void __launch_bounds__(DFP_T, 1) dfp_bwd_kernel(DFPArgs x) {
    extern __shared__ __align__(16) double sm[];  // matrix halves, 2 tiles
    __shared__ __align__(8) unsigned long long mb[2];
    DFPStream st = dfp_stream_init(sm, mb);
    double *Xc = sm + 2 * DFP_HALF, *Tt = Xc + DFP_TILE;
    const DFPTask t(x, blockIdx.x);
    const int W = t.W, n = x.n;
    const long long tix = t.bg * x.P + t.p;
    const double *PI = x.PI[t.blk];
    const long long WW = (long long)W * W;
    dfp_issue(st, PI + (t.a + t.m - 1) * WW, W);
    if (MODE == 1) {
        dfp_tile_load(Xc, x.bnd_x + tix * DF_WMAX * DFP_S, W);
    } else {
        dfp_tile_zero(Xc, W);
        if (MODE == 2) {
            __syncthreads();
            for (int s = threadIdx.x; s < DFP_S; s += blockDim.x)
                if (DFP_S * t.grp + s < W) Xc[(DFP_S * t.grp + s) * DFP_SP + s] = 1.0;
        }
    }
    __syncthreads();
    double dmax = 0.0;
    unsigned long long bad = 0;
    const DFPElems el(W);
    double yr[DFP_RPT];  // y of the row, loaded a row ahead
    auto ldy = [&](int l) {
#pragma unroll
        for (int j = 0; j < DFP_RPT; ++j) {
            const int e = threadIdx.x + j * DFP_T;
            yr[j] = (MODE != 2 && e < W * DFP_S && l >= 0) ? x.ys[(t.bg * n + l) * DF_WMAX * DFP_S + e] : 0.0;
        }
    };
    // the y-face coefficient d(x_i, y_{l+3/2}) of C_l's diagonal, a row ahead like y (an L2 load
    // per element and row: on the critical path it was the kernel's top stall)
    double dyr[DFP_RPT];
    auto ldd = [&](int l) {
#pragma unroll
        for (int j = 0; j < DFP_RPT; ++j) {
            const int e = threadIdx.x + j * DFP_T;
            dyr[j] = (e < W * DFP_S && l >= 0 && l < n - 1) ? x.op_me.dyf[(long long)(l + 1) * n + t.i0 + e / DFP_S] : 0.0;
        }
    };
    ldy(t.a + t.m - 1);
    ldd(t.a + t.m - 1);
    for (int rl = t.m - 1; rl >= 0; --rl) {
        const int l = t.a + rl;
        // T = y_l - C_l x_{l+1}  (C = -tau (coefficients of row l + 1), DFOp::up)
#pragma unroll
        for (int j = 0; j < DFP_RPT; ++j) {
            const int e = threadIdx.x + j * DFP_T;
            if (e >= W * DFP_S) continue;
            const int i = e / DFP_S, s = e % DFP_S;
            double v = yr[j];
            if (l < n - 1) {
                const int gi = t.i0 + i;
                const double rxm = x.op_me.rhof[gi], rxp = x.op_me.rhof[gi + 1], rn = x.op_me.rhon[gi];
                const double h2i = x.op_me.h2inv;
                const double c0 = rn * dyr[j] * h2i, cp = rxp * 0.125 * h2i, cm = -rxm * 0.125 * h2i;
                double sx = c0 * Xc[i * DFP_SP + s];
                if (i > 0) sx = fma(cm, Xc[(i - 1) * DFP_SP + s], sx);
                if (i + 1 < W) sx = fma(cp, Xc[(i + 1) * DFP_SP + s], sx);
                v = fma(x.tau, sx, v);
            }
            Tt[i * DFP_SP + s] = v;
        }
        __syncthreads();
        if (rl > 0) {
            ldy(l - 1);
            ldd(l - 1);
        }
        // x_l = P_l^{-1} T_l into Xc (x_{l+1} is dead)
        dfp_rowstep_s(st, PI + l * WW, rl > 0 ? PI + (l - 1) * WW : nullptr, W, Tt, Xc, 1.0, true);
        if (MODE == 1) {
            // the stage epilogue (df_stage_kernel): DR stage 0 subtracts w; final columns take the
            // parareal epilogue, the others are stored for the next stage
#pragma unroll
            for (int j = 0; j < DFP_RPT; ++j) {
                if (el.si[j] < 0) continue;
                const int s = el.si[j] >> 16, i = el.si[j] & 0xffff;  // consecutive threads: consecutive columns
                const long long b = (long long)t.grp * DFP_S + s;
                if (b >= x.B) continue;
                const int gi = t.i0 + i;
                const long long g = (long long)l * n + gi;
                double xv = Xc[i * DFP_SP + s];
                if (DR && x.stage == 0) xv -= dfp_wterm(x, x.U + b * x.vol, gi, l);
                const bool final_here = x.stage == 1 || !(x.op_ot.rhon[gi] > 0.0);
                const int ep = final_here ? x.epi : EPI_STORE;
                const long long gb = b * x.vol + g;
                if (ep == EPI_STORE) {
                    x.V[gb] = xv;
                } else if (ep == EPI_DELTA) {
                    x.V[gb] = xv - x.e_gc[gb];
                } else if (ep == EPI_CORRECT) {
                    const double nv = xv + x.e_delta[g];
                    const double ov = x.e_traj[g];
                    x.e_gcache[g] = xv;
                    x.e_traj[g] = nv;
                    dmax = fmax(dmax, fabs(nv - ov));
                    if (!isfinite(nv)) bad = 1;
                } else {  // INIT
                    x.e_gcache[g] = xv;
                    x.e_traj[g] = xv;
                }
            }
        }
        __syncthreads();
    }
    if (MODE == 0) dfp_tile_store(x.tl + tix * DF_WMAX * DFP_S, Xc, W);
    if (MODE == 2) {
        double *PT = x.setup_out[t.blk] + (long long)t.p * WW;
        for (int e = threadIdx.x; e < W * DFP_S; e += blockDim.x) {
            const int i = e / DFP_S, s = e % DFP_S, k = DFP_S * t.grp + s;
            if (k < W) PT[(long long)k * W + i] = Xc[i * DFP_SP + s];
        }
    }
    if (MODE == 1 && x.epi == EPI_CORRECT) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
            bad |= __shfl_xor_sync(0xffffffffu, bad, off);
        }
        if (lane == 0) {
            atomicMax(x.e_red, (unsigned long long)__double_as_longlong(dmax));
            if (bad) atomicOr(x.e_red + 1, 1ull);
        }
    }
}

// ------------------------------------------------------------ scans over partitions ------
// one CTA per (block, group): FWD: y_in(0) = 0, y_in(p+1) = A_p y_in(p) + y_b(p) (tl);
// BWD: x_in(P-1) = 0, x_in(p-1) = Pp_p x_in(p) + x_a(p) (tl)
template <int FWD>
__global__ void __launch_bounds__(DFP_T, 1) dfp_scan_kernel(DFPArgs x) {
    extern __shared__ __align__(16) double sm[];  // matrix halves, 2 tiles
    __shared__ __align__(8) unsigned long long mb[2];
    DFPStream st = dfp_stream_init(sm, mb);
    double *Yc = sm + 2 * DFP_HALF, *Yn = Yc + DFP_TILE;
    const long long bg = blockIdx.x;
    const int blk = (int)(bg / x.ngrp), W = x.bW[blk];
    const long long WW = (long long)W * W;
    const double *M = FWD ? x.AT[blk] : x.PpT[blk];
    double *bnd = FWD ? x.bnd_y : x.bnd_x;
    auto part = [&](int q) { return FWD ? q : x.P - 1 - q; };
    if (x.P > 1) dfp_issue(st, M + part(0) * WW, W);
    dfp_tile_zero(Yc, W);
    __syncthreads();
    for (int q = 0; q < x.P; ++q) {
        const int p = part(q);
        const long long tix = bg * x.P + p;
        dfp_tile_store(bnd + tix * DF_WMAX * DFP_S, Yc, W);
        if (q + 1 == x.P) break;
        dfp_tile_load(Yn, x.tl + tix * DF_WMAX * DFP_S, W);
        __syncthreads();
        dfp_rowstep_s(st, M + p * WW, q + 2 < x.P ? M + part(q + 1) * WW : nullptr, W, Yc, Yn, 1.0);
        double *tmp = Yc;
        Yc = Yn;
        Yn = tmp;
    }
}

}  // namespace prs
