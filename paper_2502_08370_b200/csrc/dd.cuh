// dd.cuh -- domain-decomposition (DD) splitting stage solves.
//
// Colour j's stage matrix I - tau A_j is block diagonal with one block per connected strip of
// its support (rho_j > 0) and identity rows elsewhere.  With
// kappa = 1 and rho = rho(x) a block (W columns x n rows, U as a W x n matrix) reads
//     (I - tau A_j) U = S U - tau R U Y,   S = I - tau X + tau c R,   R = diag(rho_j(x_i)),
// X the rho_j-face-weighted 1-D operator in x and Y the 1-D Dirichlet second difference in y.
// With the generalised eigenpairs S q_a = theta_a R q_a, Q^T R Q = I (precomputed once per
// block and tau from the symmetric tridiagonal C = R^{-1/2} S R^{-1/2} by Jacobi rotations),
// the block solve is exactly (up to rounding)
//     G = Q^T F  ->  (theta_a I - tau Y) v_a = g_a  (n-long tridiagonal, one per mode a)
//     ->  U = Q V.
// A block of one state is cut into CL row pieces of R <= 64 rows, one per CTA (two CTAs per SM,
// so one piece's transforms overlap another's loads, waits and walks), each held in
// shared memory: two dense W x W transforms on the fp64 FMA pipes (register-tiled, Q streamed
// through shared memory), and the n-long tridiagonal solves with the chunk-parallel Thomas of
// common.cuh across the pieces.  The pieces exchange their scan totals through L2 (default: a
// persistent grid taking pieces in order, every SM busy) or through distributed shared memory
// within a cluster of CL CTAs (PRS_DDCL=1; 8-CTA clusters pack two per GPC, leaving SMs idle).
// This is the fp64-ALU-bound kernel of the path (~4W flops per support point
// per stage).
//
// FIE step = stage 0 (colour 0) then stage 1 (colour 1), both in place in
// the output buffer V:
//   stage 0: r = U + tau F [DR: + w, w = tau A_1 U (colour-1 operator)], solve colour-0
//            blocks, V = x [DR: - w]; points with rho_1 = 0 are final after this stage.
//   stage 1: r = V where rho_0 > 0, else U + tau F (the identity rows of stage 0, where for
//            DR the w terms cancel), solve colour-1 blocks, V = x.
// The parareal epilogues (Delta, correction, initial guess) are fused into the stores of
// the final values of each stage.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/prs.h"
#include "common.cuh"
#include "ddfull.cuh"
#include "lpass.cuh"
#include "xpass3.cuh"

struct prs_ctx;
int prs_internal_prof_begin(prs_ctx *ctx);
int prs_internal_prof_end(prs_ctx *ctx, int kind, double bytes);

namespace prs {

constexpr int DD_RMAX = 64;    // rows per CTA (row piece)
constexpr int DD_WMAX = 144;   // widest block (2 x 72 output columns in the GEMMs)
constexpr int DD_WPAD = 148;   // shared row stride of a tile (>= DD_WMAX, == 4 mod 16)
constexpr int DD_KC = 8;       // Q rows staged per k-chunk
constexpr int DD_THREADS = 256;  // 8 warps: DD_RMAX / 16 row groups x 2 column halves (GEMM)
constexpr int DD_NCH = DD_RMAX / 16;  // 16-row chunks of a piece (y solve)
constexpr int DD_FTHREADS = 512;      // factorisation kernel

// ------------------------------------------------------------- partition of unity --
// rho_0 at a 1-based position xpos (integer = node, half-integer = face), index-space
// geometry of DESIGN.md R6: S strips of w = n/S nodes, interface m at w m + 1/2, ramp of
// width beta = ov centred on it; colour 0 = even strips.  rho_1 = 1 - rho_0.
__device__ inline double dd_ramp_down(double xpos, double xl, int ov, int cosine) {
    const double u = (xpos - xl) / (double)ov;
    if (u <= 0.0) return 1.0;
    if (u >= 1.0) return 0.0;
    if (cosine) return 0.5 * (1.0 + cos(3.14159265358979323846 * u));
    return 1.0 - u;
}
__device__ inline double dd_rho0(double xpos, int n, int S, int ov, int cosine) {
    const int w = n / S;
    int k = (int)floor((xpos - 0.5) / (double)w);
    k = max(0, min(S - 1, k));
    const double half = 0.5 * (double)ov;
    if (k + 1 <= S - 1) {
        const double xi = (double)(w * (k + 1)) + 0.5;
        if (xpos > xi - half) {
            const double d = dd_ramp_down(xpos, xi - half, ov, cosine);
            return (k % 2 == 0) ? d : 1.0 - d;
        }
    }
    if (k >= 1) {
        const double xi = (double)(w * k) + 0.5;
        if (xpos < xi + half) {
            const double d = dd_ramp_down(xpos, xi - half, ov, cosine);
            return ((k - 1) % 2 == 0) ? d : 1.0 - d;
        }
    }
    return (k % 2 == 0) ? 1.0 : 0.0;
}
// rhon[j*n + i] = rho_j(node i+1), rhof[j*(n+1) + f] = rho_j(face f + 1/2)
__global__ void dd_rho_tables(int n, int S, int ov, int cosine, double *rhon, double *rhof) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const double r = dd_rho0((double)(i + 1), n, S, ov, cosine);
        rhon[i] = r;
        rhon[n + i] = 1.0 - r;
    }
    if (i <= n) {
        const double r = dd_rho0((double)i + 0.5, n, S, ov, cosine);
        rhof[i] = r;
        rhof[n + 1 + i] = 1.0 - r;
    }
}

// -------------------------------------------------------- per-block factorisation --
// Symmetric tridiagonal C = R^{-1/2} S R^{-1/2} of block (colour j, columns i0..i0+W-1):
//   S_ii = 1 + tau h^-2 (rho(i-1/2) + rho(i+1/2)) + tau c rho(i),  S_i,i+1 = -tau h^-2 rho(i+1/2)
// then cyclic Jacobi (parallel round-robin pairs) on C in shared memory, eigenvectors in
// global memory; Q = R^{-1/2} Z, QT = Q^T, theta, and the pivots of theta_a I - tau Y.
struct DDBlock {
    int colour, i0, W;
    double *Q = nullptr, *QT = nullptr, *theta = nullptr, *idy = nullptr;  // per tau slot
};

__global__ void __launch_bounds__(DD_FTHREADS) dd_factor_kernel(int n, int i0, int W, const double *rhon,
                                                               const double *rhof, double tau, double h2inv,
                                                               double c, double *Z, double *Q, double *QT,
                                                               double *theta, double *idy, int sweeps) {
    extern __shared__ double sh[];
    double *C = sh;                 // W x W (row stride W)
    double *cs = sh + W * W;        // rotation cos per pair
    double *sn = cs + DD_WMAX / 2 + 1;
    int *pp = reinterpret_cast<int *>(sn + DD_WMAX / 2 + 1);
    int *qq = pp + DD_WMAX / 2 + 1;
    const int tid = threadIdx.x;
    // assemble C and Z = I
    for (int e = tid; e < W * W; e += blockDim.x) {
        const int r = e / W, k = e % W;
        const int gi = i0 + r;  // 0-based node index
        const double rr = rhon[gi];
        double v = 0.0;
        if (r == k) {
            v = (1.0 + tau * h2inv * (rhof[gi] + rhof[gi + 1]) + tau * c * rr) / rr;
        } else if (k == r + 1) {
            v = -tau * h2inv * rhof[gi + 1] / sqrt(rr * rhon[gi + 1]);
        } else if (r == k + 1) {
            v = -tau * h2inv * rhof[gi] / sqrt(rr * rhon[gi - 1]);
        }
        C[e] = v;
        Z[e] = (r == k) ? 1.0 : 0.0;
    }
    __syncthreads();
    // round-robin pairing over Wp = W rounded up to even (a dummy index when W is odd)
    const int Wp = W + (W & 1);
    const int npair = Wp / 2;
    for (int sw = 0; sw < sweeps; ++sw) {
        for (int round = 0; round < Wp - 1; ++round) {
            if (tid < npair) {
                // circle method: pair k of round r is (r+k, r-k) mod (Wp-1), pair 0 is (r, Wp-1);
                // every index appears once per round and every pair once per sweep
                const int k = tid;
                const int a = (round + k) % (Wp - 1);
                const int b = (k == 0) ? (Wp - 1) : (round - k + Wp - 1) % (Wp - 1);
                int p = min(a, b), q = max(a, b);
                double cc = 1.0, ss = 0.0;
                if (q < W && p != q) {
                    const double apq = C[p * W + q];
                    if (apq != 0.0) {
                        const double app = C[p * W + p], aqq = C[q * W + q];
                        const double th = (aqq - app) / (2.0 * apq);
                        const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                        cc = 1.0 / sqrt(t * t + 1.0);
                        ss = t * cc;
                    }
                } else {
                    p = q = -1;
                }
                pp[tid] = p;
                qq[tid] = q;
                cs[tid] = cc;
                sn[tid] = ss;
            }
            __syncthreads();
            // rows: C <- J^T C  (each pair mixes rows p, q)
            for (int e = tid; e < npair * W; e += blockDim.x) {
                const int k = e / W, col = e % W;
                const int p = pp[k], q = qq[k];
                if (p < 0) continue;
                const double cc = cs[k], ss = sn[k];
                const double xp = C[p * W + col], xq = C[q * W + col];
                C[p * W + col] = cc * xp - ss * xq;
                C[q * W + col] = ss * xp + cc * xq;
            }
            __syncthreads();
            // columns: C <- C J, Z <- Z J
            for (int e = tid; e < npair * W; e += blockDim.x) {
                const int k = e / W, row = e % W;
                const int p = pp[k], q = qq[k];
                if (p < 0) continue;
                const double cc = cs[k], ss = sn[k];
                const double xp = C[row * W + p], xq = C[row * W + q];
                C[row * W + p] = cc * xp - ss * xq;
                C[row * W + q] = ss * xp + cc * xq;
                const double zp = Z[row * W + p], zq = Z[row * W + q];
                Z[row * W + p] = cc * zp - ss * zq;
                Z[row * W + q] = ss * zp + cc * zq;
            }
            __syncthreads();
        }
    }
    // eigenvalues on the diagonal; Q = R^{-1/2} Z; pivots of theta_a + 2 s, off -s (s = tau/h^2)
    const double s = tau * h2inv;
    for (int a = tid; a < W; a += blockDim.x) {
        const double th = C[a * W + a];
        theta[a] = th;
        const double bd = th + 2.0 * s;
        double d = bd;
        for (int l = 0; l < n; ++l) {
            if (l > 0) d = bd - s * s / d;
            idy[(long long)l * W + a] = 1.0 / d;
        }
    }
    for (int e = tid; e < W * W; e += blockDim.x) {
        const int r = e / W, k = e % W;
        const double q = Z[e] / sqrt(rhon[i0 + r]);
        Q[e] = q;             // Q[i][a]
        QT[k * W + r] = q;    // QT[a][i]
    }
}

// ------------------------------------------------------------------ stage kernel ---
struct DDStageArgs {
    const double *U;     // step input (batch)
    double *V;           // step output (batch), stage 1 reads it too
    long long vol;
    int n, B;
    int stage;           // 0 or 1 (colour)
    int CL, R;           // cluster size, rows per CTA
    int nblk;            // blocks of this colour
    const int *bi0, *bW; // block column start / width
    const double *const *Q, *const *QT, *const *idy;  // per block
    double tau, h2inv, c;
    const double *rhon, *rhof;  // rho tables (colour 0 then colour 1)
    double src_amp;
    const double *sinpi;
    TimeArgs ta;
    int epi;
    const double *e_gc;
    double *e_gcache;
    const double *e_delta;
    double *e_traj;
    unsigned long long *e_red;
    // global exchange (GX): task counter, per-task flags [2 * ntasks] (forward, backward), per
    // task scan totals [ntasks][2][DD_WMAX]; zeroed before each launch
    unsigned *gctr;
    int *gflag;
    double2 *gtot;
    int ntasks;
};

#ifdef PRS_DD_TIMING
// diagnostic build only (-DPRS_DD_TIMING): per task, ns spent waiting for the forward / the
// backward scan totals of the other row pieces, the task's duration, and the task count
__device__ unsigned long long g_dd_timing[4];
__device__ __forceinline__ unsigned long long dd_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// L2-scope flag hand-off between CTAs (GX): release after the CTA's total is written, acquire
// before reading the totals of other row pieces.  A wait that outlives any legitimate one (a
// task lasts ~0.1 ms) traps instead of hanging the device.
__device__ __forceinline__ void dd_flag_release(int *f) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(f), "r"(1) : "memory");
}
__device__ __forceinline__ void dd_flag_wait(const int *f) {
    int v;
    for (long long it = 0;; ++it) {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
        if (v) return;
        if (it > (1ll << 24)) __trap();
        __nanosleep(32);
    }
}

// GEMM on the shared tile: T[l][:] <- T[l][:] . M  (M is W x W, row-major, global), in place,
// on the fp64 tensor cores (dd_tile_gemm below).  M streams through two shared k-chunks of
// DD_KC rows with cp.async (next chunk in flight while the current one is consumed).  Columns
// >= W of T and staged rows >= W are zero, so the inner loops need no predicates; rows >= nrow
// and columns >= W of the product are computed and discarded.  (The register-tiled DFMA form reached ~55 % of the fp64
// pipe: 13 shared loads and 49 issue slots per 36 FMAs; DMMA and DFMA peak alike on B200,
// profiles/r01_fp64_peak_probe.txt.)
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void dd_stage_mchunk(const double *M, int W, int k0, double *dst) {
    const int kc = min(DD_KC, W - k0);
    if ((W & 1) == 0) {  // 16-byte pieces (rows of M are 16-byte aligned), DD_WMAX / 2 slots per row
        constexpr int PR = DD_WMAX / 2;
        for (int e = threadIdx.x; e < kc * PR; e += blockDim.x) {
            const int r = e / PR, h = e - r * PR;
            if (2 * h < W) cp_async16(dst + r * DD_WPAD + 2 * h, M + (long long)(k0 + r) * W + 2 * h);
        }
    } else {
        for (int e = threadIdx.x; e < kc * DD_WMAX; e += blockDim.x) {
            const int r = e / DD_WMAX, c = e - r * DD_WMAX;
            if (c < W) cp_async8(dst + r * DD_WPAD + c, M + (long long)(k0 + r) * W + c);
        }
    }
}
// one contiguous global -> shared copy on the async (TMA) engine, completing on an mbarrier
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(mb))
                 : "memory");
}

__device__ __forceinline__ void dmma_f64(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}
__device__ __forceinline__ void dd_tile_gemm(double *T, const double *M, int W, int nrow, double *Ms) {
    // fp64 tensor-core MMA (m8n8k4): warp w owns rows 16 (w % NCH) .. +15 and columns
    // 72 (w / NCH) .. +71 of the output, i.e. 2 x 9 tiles of 8 x 8, accumulators in registers.
    // Per 4-wide k step: 2 A fragments (A[r][k], r = lane / 4, k = lane % 4) from the tile and 9
    // B fragments (B[k][c], k = lane % 4, c = lane / 4) from the staged chunk, all bank-conflict
    // free with the 148-double row stride; 18 MMAs of 256 FMAs each.
    static_assert(DD_THREADS / 32 == 2 * DD_NCH && DD_WMAX == 144 && DD_KC % 4 == 0, "dmma tiling");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rb = 16 * (warp % DD_NCH), cb = 72 * (warp / DD_NCH);
    const int fr = lane >> 2, fk = lane & 3;
    double acc[2][9][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < 9; ++j) acc[h][j][0] = acc[h][j][1] = 0.0;
    const int nk = (W + DD_KC - 1) / DD_KC;
    __syncthreads();  // Ms aliases the y-solve scratch: all of its readers are done
    // the rows a partial last chunk leaves unwritten meet the zero columns >= W of T and must be
    // zero (stale scratch need not be finite); staged columns >= W only reach discarded outputs
    {
        const int kl = W - (nk - 1) * DD_KC;  // rows of the last chunk
        double *last = Ms + ((nk - 1) & 1) * DD_KC * DD_WPAD;
        for (int e = tid; e < (DD_KC - kl) * DD_WMAX; e += blockDim.x) {
            const int r = e / DD_WMAX;
            last[(kl + r) * DD_WPAD + (e - r * DD_WMAX)] = 0.0;
        }
    }
    // chunks of M: even W -> one bulk copy per row (W * 8 bytes, 16-byte aligned) by thread 0,
    // completing on the buffer's mbarrier; odd W -> 8-byte cp.async by all threads
    __shared__ __align__(8) unsigned long long mbq[2];
    const bool bulk = (W & 1) == 0;
    if (bulk && tid == 0) {
        mbar_init(&mbq[0], 1);
        mbar_init(&mbq[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto stage = [&](int kb) {
        double *dst = Ms + (kb & 1) * DD_KC * DD_WPAD;
        if (bulk) {
            if (tid == 0) {
                const int k0 = kb * DD_KC, kc = min(DD_KC, W - k0);
                // the buffer was last touched by generic loads / stores (previous chunk, y-solve
                // scratch): order them before the async-proxy writes
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                mbar_arrive_expect(&mbq[kb & 1], (unsigned)(kc * W * sizeof(double)));
                for (int r = 0; r < kc; ++r)
                    bulk_g2s(dst + r * DD_WPAD, M + (long long)(k0 + r) * W, (unsigned)(W * sizeof(double)),
                             &mbq[kb & 1]);
            }
        } else {
            dd_stage_mchunk(M, W, kb * DD_KC, dst);
        }
        cp_async_commit();
    };
    stage(0);
    const double *ta0 = T + cpad(rb + fr) * DD_WPAD + fk;
    const double *ta1 = T + cpad(rb + 8 + fr) * DD_WPAD + fk;
    for (int kb = 0; kb < nk; ++kb) {
        double *cur = Ms + (kb & 1) * DD_KC * DD_WPAD;
        if (kb + 1 < nk) stage(kb + 1);
        else cp_async_commit();
        if (bulk) {
            mbar_wait(&mbq[kb & 1], (unsigned)((kb >> 1) & 1));  // this chunk's bytes have landed
        } else {
            cp_async_wait<1>();
            __syncthreads();
        }
        const int k0 = kb * DD_KC;
        const double *tb = cur + fk * DD_WPAD + cb + fr;
#pragma unroll
        for (int kq = 0; kq < DD_KC; kq += 4) {
            const double a0 = ta0[k0 + kq], a1 = ta1[k0 + kq];
#pragma unroll
            for (int j = 0; j < 9; ++j) {
                if (j == 8 && cb + 64 >= W) break;  // (warp-uniform) a tile of padding columns only
                const double bv = tb[kq * DD_WPAD + 8 * j];
                dmma_f64(acc[0][j][0], acc[0][j][1], a0, bv);
                dmma_f64(acc[1][j][0], acc[1][j][1], a1, bv);
            }
        }
        __syncthreads();  // chunk consumed before it is refilled
    }
    // all reads of T are done (last barrier above): write in place
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int l = rb + 8 * h + fr;
        if (l < nrow) {
#pragma unroll
            for (int j = 0; j < 9; ++j) {
                const int col = cb + 8 * j + 2 * fk;
                if (col < W) T[cpad(l) * DD_WPAD + col] = acc[h][j][0];
                if (col + 1 < W) T[cpad(l) * DD_WPAD + col + 1] = acc[h][j][1];
            }
        }
    }
    __syncthreads();
}

// One task: row piece `crank` (of CL) of block `blk` of state `b` (task = b * nblk + blk).
// GX = 0: the CL pieces are the CTAs of one cluster and exchange their scan totals through
// distributed shared memory; GX = 1: the pieces are independent tasks of a persistent grid and
// exchange them through L2 (per-task flags), see dd_stage_kernel.
template <int DR, int SRC, int GX>
__device__ __forceinline__ void dd_stage_task(const DDStageArgs &a, double *sh, long long task, int crank) {
    double *T = sh;                                          // (cpad(R-1)+1) x DD_WPAD
    double *Ms = sh + (size_t)(cpad(DD_RMAX - 1) + 1) * DD_WPAD;  // 2 x DD_KC x DD_WPAD (GEMM)
    double2 *sc = reinterpret_cast<double2 *>(Ms);           // 8 x DD_WMAX chunk maps (y solve)
    double2 *ctf = reinterpret_cast<double2 *>(Ms + 2 * DD_KC * DD_WPAD);  // cluster totals fwd
    double2 *ctb = ctf + DD_WMAX;                             // cluster totals bwd
    const long long tk = task * a.CL + crank;                 // GX slot
    double2 *gtf = a.gtot + tk * 2 * DD_WMAX, *gtb = gtf + DD_WMAX;

    const int tid = threadIdx.x;
    const int blk = (int)(task % a.nblk);
    const long long b = task / a.nblk;
    const int i0 = a.bi0[blk], W = a.bW[blk];
    const int n = a.n;
    const int r0 = crank * a.R;
    const int nrow = max(0, min(a.R, n - r0));
    const double *Ub = a.U + b * a.vol;
    double *Vb = a.V + b * a.vol;
    const int me = a.stage, other = 1 - a.stage;
    const double *rn_ot = a.rhon + other * n, *rf_ot = a.rhof + other * (n + 1);
    double ampt = 0.0;
    if (SRC) ampt = a.src_amp * exp(-src_time(a.ta, b));

    // ---- load the right-hand side tile: one row per warp, columns across lanes; every
    // global load of a row is issued before the first use (several rows' worth in flight) ----
    constexpr int NCW = (DD_WMAX + 31) / 32;  // column slots per lane
    // per-lane column constants, loaded once: the source profile and, for stage 1, which
    // columns are already final after stage 0 (rho_0 > 0)
    // finm: columns whose value is final after this stage (stage 1: all; stage 0: rho_1 = 0)
    unsigned done0m = 0, finm = 0;
    double spk[NCW];
#pragma unroll
    for (int k = 0; k < NCW; ++k) {
        const int ci = (tid & 31) + 32 * k;
        spk[k] = (SRC && ci < W) ? __ldg(a.sinpi + i0 + ci) : 0.0;
        const bool pos = ci < W && rn_ot[i0 + ci] > 0.0;
        if (me == 1 && pos) done0m |= 1u << k;
        if (ci < W && (me == 1 || !pos)) finm |= 1u << k;
    }
    {
        const int wp = tid >> 5, ln = tid & 31;
        // the source profile of the warp's rows wp + 16 q, one per lane (q = lane), shuffled out
        static_assert(DD_RMAX / (DD_THREADS / 32) <= 32, "rows per warp");
        double slq = 0.0;
        if (SRC && wp + (DD_THREADS / 32) * ln < nrow) slq = a.tau * ampt * __ldg(a.sinpi + r0 + wp + (DD_THREADS / 32) * ln);
#pragma unroll 2
        for (int rl = wp; rl < nrow; rl += DD_THREADS / 32) {
            const int l = r0 + rl;
            const long long g0 = (long long)l * n + i0;
            double r[NCW], u[NCW];
#pragma unroll
            for (int k = 0; k < NCW; ++k) {
                const int ci = ln + 32 * k;
                const bool in = ci < W;
                const long long g = g0 + ci;
                if (me == 0) {
                    u[k] = in ? Ub[g] : 0.0;
                    r[k] = 0.0;
                } else {
                    const bool done0 = (done0m >> k) & 1u;  // final after stage 0
                    r[k] = done0 ? Vb[g] : 0.0;
                    u[k] = (in && !done0) ? Ub[g] : 0.0;
                }
            }
            double wv[NCW];
            if (DR && me == 0) {  // w = tau A_1 U (colour-1 operator)
#pragma unroll
                for (int k = 0; k < NCW; ++k) {
                    const int ci = ln + 32 * k, i = i0 + ci;
                    wv[k] = 0.0;
                    if (ci < W) {
                        const long long g = g0 + ci;
                        const double um = (i > 0) ? Ub[g - 1] : 0.0, up = (i < n - 1) ? Ub[g + 1] : 0.0;
                        const double vm = (l > 0) ? Ub[g - n] : 0.0, vp = (l < n - 1) ? Ub[g + n] : 0.0;
                        const double uu = u[k], rnode = rn_ot[i];
                        wv[k] = a.tau * ((rf_ot[i + 1] * (up - uu) - rf_ot[i] * (uu - um) +
                                          rnode * (vp - 2.0 * uu + vm)) * a.h2inv - rnode * a.c * uu);
                    }
                }
            }
            const double sl = SRC ? __shfl_sync(0xffffffffu, slq, (rl - wp) / (DD_THREADS / 32)) : 0.0;
#pragma unroll
            for (int k = 0; k < NCW; ++k) {
                const int ci = ln + 32 * k, i = i0 + ci;
                double v = 0.0;  // columns W..DD_WMAX-1 are zero for the unpredicated GEMM
                if (ci < W) {
                    if (me == 0) {
                        v = u[k];
                        if (SRC) v += sl * spk[k];
                        if (DR) v += wv[k];
                    } else if ((done0m >> k) & 1u) {
                        v = r[k];
                    } else {
                        v = u[k];
                        if (SRC) v += sl * spk[k];
                    }
                }
                if (ci < DD_WMAX) T[cpad(rl) * DD_WPAD + ci] = v;
            }
        }
    }
    // ---- G = F Q ----
    dd_tile_gemm(T, a.Q[blk], W, nrow, Ms);

    // ---- (theta_a I - tau Y) v_a = g_a along y: warp = chunk t (of 16 rows) x mode half,
    // lanes = modes: half 0 walks mode rounds 0..2 (modes 0..95), half 1 rounds 3..4 ----
    const int t = (tid >> 5) % DD_NCH, lane = tid & 31, mh = (tid >> 5) / DD_NCH;
    const int e0 = t * LCH;
    const int cnt = max(0, min(LCH, nrow - e0));
    const double ms = -a.tau * a.h2inv;  // off-diagonal of theta I - tau Y
    const double *idy = a.idy[blk];
    constexpr int NMR = 3;  // mode rounds per thread
    const int rr0 = 3 * mh;  // first mode round of this half (round rr covers modes 32 rr .. 32 rr + 31)
    double Ain[NMR], Bin[NMR];
    // The walks below come in a predicated form (partial last chunk) and an unpredicated one
    // for full chunks (every chunk of c4); the line's first and last rows (m = 0 / cc = 0)
    // are the only boundary cases and are tested once per walk.
    const int lb = r0 + e0;  // global row of the chunk's first element
    const bool full = (cnt == LCH);
    // multiplier of element i (row lb + i): m = -tau/h^2 * id(row - 1); 0 on the line's first row
    auto mrow = [&](const double *ip, int i) {
        return (i == 0 && lb == 0) ? 0.0 : ms * __ldg(ip + (long long)(i - 1) * W);
    };
    auto f1 = [&](auto FT, int am, double &A, double &B) {
        constexpr bool FULL = decltype(FT)::value;
        const double *ip = idy + (long long)lb * W + am;
        A = 1.0;
        B = 0.0;
#pragma unroll
        for (int i = 0; i < LCH; ++i)
            if (FULL || i < cnt) {
                const double m = mrow(ip, i);
                B = fma(-m, B, T[cpad(e0 + i) * DD_WPAD + am]);
                A = -m * A;
            }
    };
#pragma unroll
    for (int rr = 0; rr < NMR; ++rr) {
        const int am = lane + 32 * (rr0 + rr);
        double A = 1.0, B = 0.0;
        if (am < W) {
            if (full) f1(std::true_type{}, am, A, B);
            else f1(std::false_type{}, am, A, B);
            sc[t * DD_WMAX + am] = make_double2(A, B);
        }
        Ain[rr] = A;
        Bin[rr] = B;
    }
    __syncthreads();
    const int nch = (nrow + LCH - 1) / LCH;
    double yin[NMR];
#pragma unroll
    for (int rr = 0; rr < NMR; ++rr) {
        const int am = lane + 32 * (rr0 + rr);
        double EA = 1.0, EB = 0.0, TA = 1.0, TB = 0.0;  // exclusive prefix, CTA total
        if (am < W) {
            for (int q = 0; q < nch; ++q) {
                const double2 v = sc[q * DD_WMAX + am];
                if (q == t) {
                    EA = TA;
                    EB = TB;
                }
                TB = fma(v.x, TB, v.y);
                TA = v.x * TA;
            }
            if (t >= nch) {
                EA = TA;
                EB = TB;
            }
            if (t == 0) {
                if (GX) {
                    gtf[am] = make_double2(TA, TB);
                    __threadfence();
                } else {
                    ctf[am] = make_double2(TA, TB);
                }
            }
        }
        Ain[rr] = EA;
        Bin[rr] = EB;
    }
    double Ycta[NMR];
#pragma unroll
    for (int rr = 0; rr < NMR; ++rr) Ycta[rr] = 0.0;
    if (GX && a.CL > 1) {
        __syncthreads();  // every total of this piece written (and fenced)
        if (tid == 0) {
            dd_flag_release(a.gflag + 2 * tk);
#ifdef PRS_DD_TIMING
            const unsigned long long tw0 = dd_gtimer();
#endif
            for (int r = 0; r < crank; ++r) dd_flag_wait(a.gflag + 2 * (task * a.CL + r));
#ifdef PRS_DD_TIMING
            atomicAdd(&g_dd_timing[0], dd_gtimer() - tw0);
#endif
        }
        __syncthreads();
#pragma unroll
        for (int rr = 0; rr < NMR; ++rr) {
            const int am = lane + 32 * (rr0 + rr);
            if (am < W)
                for (int r = 0; r < crank; ++r) {
                    const double2 v = __ldcg(a.gtot + (task * a.CL + r) * 2 * DD_WMAX + am);
                    Ycta[rr] = fma(v.x, Ycta[rr], v.y);
                }
        }
    } else if (!GX && a.CL > 1) {
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();
#pragma unroll
        for (int rr = 0; rr < NMR; ++rr) {
            const int am = lane + 32 * (rr0 + rr);
            if (am < W)
                for (int r = 0; r < crank; ++r) {
                    const double2 v = cl.map_shared_rank(ctf, r)[am];
                    Ycta[rr] = fma(v.x, Ycta[rr], v.y);
                }
        }
    }
#pragma unroll
    for (int rr = 0; rr < NMR; ++rr) yin[rr] = fma(Ain[rr], Ycta[rr], Bin[rr]);
    __syncthreads();
    // F3 + backward composition
    auto f3 = [&](auto FT, int am, double y, double &Pb, double &Qb) {
        constexpr bool FULL = decltype(FT)::value;
        const double *ip = idy + (long long)lb * W + am;
        Pb = 1.0;
        Qb = 0.0;
#pragma unroll
        for (int i = 0; i < LCH; ++i)
            if (FULL || i < cnt) {
                const double m = mrow(ip, i);
                const double id = __ldg(ip + (long long)i * W);
                const double ccv = (lb + i == n - 1) ? 0.0 : ms * id;
                double *p = T + cpad(e0 + i) * DD_WPAD + am;
                y = fma(-m, y, *p);
                *p = y;
                Qb = fma(Pb * id, y, Qb);
                Pb *= -ccv;
            }
    };
#pragma unroll
    for (int rr = 0; rr < NMR; ++rr) {
        const int am = lane + 32 * (rr0 + rr);
        if (am < W) {
            double Pb, Qb;
            if (full) f3(std::true_type{}, am, yin[rr], Pb, Qb);
            else f3(std::false_type{}, am, yin[rr], Pb, Qb);
            sc[t * DD_WMAX + am] = make_double2(Pb, Qb);
        }
    }
    __syncthreads();
    double xin[NMR];
#pragma unroll
    for (int rr = 0; rr < NMR; ++rr) {
        const int am = lane + 32 * (rr0 + rr);
        double EP = 1.0, EQ = 0.0, TP = 1.0, TQ = 0.0;
        if (am < W) {
            for (int q = nch - 1; q >= 0; --q) {
                const double2 v = sc[q * DD_WMAX + am];
                if (q == t) {
                    EP = TP;
                    EQ = TQ;
                }
                TQ = fma(v.x, TQ, v.y);
                TP = v.x * TP;
            }
            if (t >= nch) {
                EP = 1.0;
                EQ = 0.0;
            }
            if (t == 0) {
                if (GX) {
                    gtb[am] = make_double2(TP, TQ);
                    __threadfence();
                } else {
                    ctb[am] = make_double2(TP, TQ);
                }
            }
        }
        Ain[rr] = EP;
        Bin[rr] = EQ;
    }
    double Xcta[NMR];
#pragma unroll
    for (int rr = 0; rr < NMR; ++rr) Xcta[rr] = 0.0;
    if (GX && a.CL > 1) {
        __syncthreads();
        if (tid == 0) {
            dd_flag_release(a.gflag + 2 * tk + 1);
#ifdef PRS_DD_TIMING
            const unsigned long long tw1 = dd_gtimer();
#endif
            for (int r = a.CL - 1; r > crank; --r) dd_flag_wait(a.gflag + 2 * (task * a.CL + r) + 1);
#ifdef PRS_DD_TIMING
            atomicAdd(&g_dd_timing[1], dd_gtimer() - tw1);
#endif
        }
        __syncthreads();
#pragma unroll
        for (int rr = 0; rr < NMR; ++rr) {
            const int am = lane + 32 * (rr0 + rr);
            if (am < W)
                for (int r = a.CL - 1; r > crank; --r) {
                    const double2 v = __ldcg(a.gtot + (task * a.CL + r) * 2 * DD_WMAX + DD_WMAX + am);
                    Xcta[rr] = fma(v.x, Xcta[rr], v.y);
                }
        }
    } else if (!GX && a.CL > 1) {
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();
#pragma unroll
        for (int rr = 0; rr < NMR; ++rr) {
            const int am = lane + 32 * (rr0 + rr);
            if (am < W)
                for (int r = a.CL - 1; r > crank; --r) {
                    const double2 v = cl.map_shared_rank(ctb, r)[am];
                    Xcta[rr] = fma(v.x, Xcta[rr], v.y);
                }
        }
        cl.sync();
    }
#pragma unroll
    for (int rr = 0; rr < NMR; ++rr) xin[rr] = fma(Ain[rr], Xcta[rr], Bin[rr]);
    // B3
    auto b3 = [&](auto FT, int am, double x) {
        constexpr bool FULL = decltype(FT)::value;
        const double *ip = idy + (long long)lb * W + am;
#pragma unroll
        for (int i = LCH - 1; i >= 0; --i)
            if (FULL || i < cnt) {
                const double id = __ldg(ip + (long long)i * W);
                const double ccv = (lb + i == n - 1) ? 0.0 : ms * id;
                double *p = T + cpad(e0 + i) * DD_WPAD + am;
                x = fma(id, *p, -ccv * x);
                *p = x;
            }
    };
#pragma unroll
    for (int rr = 0; rr < NMR; ++rr) {
        const int am = lane + 32 * (rr0 + rr);
        if (am < W) {
            if (full) b3(std::true_type{}, am, xin[rr]);
            else b3(std::false_type{}, am, xin[rr]);
        }
    }
    // ---- U = V Q^T ----
    dd_tile_gemm(T, a.QT[blk], W, nrow, Ms);

    // ---- store (+ fused parareal epilogue for final values): one row per warp ----
    double dmax = 0.0;
    unsigned long long bad = 0;
    {
        const int wp = tid >> 5;
        for (int rl = wp; rl < nrow; rl += DD_THREADS / 32) {
            const int l = r0 + rl;
            const long long g0 = (long long)l * n + i0;
#pragma unroll
            for (int k = 0; k < NCW; ++k) {
                const int ci = lane + 32 * k, i = i0 + ci;
                if (ci >= W) continue;
                const long long g = g0 + ci;
                double x = T[cpad(rl) * DD_WPAD + ci];
                if (DR && me == 0) {  // V = x - w
                    const double u = Ub[g];
                    const double um = (i > 0) ? Ub[g - 1] : 0.0, up = (i < n - 1) ? Ub[g + 1] : 0.0;
                    const double vm = (l > 0) ? Ub[g - n] : 0.0, vp = (l < n - 1) ? Ub[g + n] : 0.0;
                    const double rnode = rn_ot[i];
                    x -= a.tau * ((rf_ot[i + 1] * (up - u) - rf_ot[i] * (u - um) + rnode * (vp - 2.0 * u + vm)) *
                                      a.h2inv -
                                  rnode * a.c * u);
                }
                const bool final_here = (finm >> k) & 1u;
                const int ep = final_here ? a.epi : EPI_STORE;
                const long long gb = b * a.vol + g;
                if (ep == EPI_STORE) {
                    Vb[g] = x;
                } else if (ep == EPI_DELTA) {
                    Vb[g] = x - a.e_gc[gb];
                } else if (ep == EPI_CORRECT) {
                    const double nv = x + a.e_delta[g];
                    const double ov = a.e_traj[g];
                    a.e_gcache[g] = x;
                    a.e_traj[g] = nv;
                    dmax = fmax(dmax, fabs(nv - ov));
                    if (!isfinite(nv)) bad = 1;
                } else {  // INIT
                    a.e_gcache[g] = x;
                    a.e_traj[g] = x;
                }
            }
        }
    }
    if (a.epi == EPI_CORRECT) {
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

// GX = 0: one CTA per task piece, clusters of CL CTAs.  GX = 1: a persistent grid (one CTA per
// SM) whose CTAs take task pieces in order from a global counter; pieces of one block need not
// be co-resident: a piece waits only on pieces taken before it (forward) or on later pieces of
// the same block, which the earliest unfinished block always has CTAs free to take, so the
// in-order hand-out cannot deadlock.  No SM idles for want of a whole free cluster.
template <int DR, int SRC, int GX>
__global__ void __launch_bounds__(DD_THREADS, 2) dd_stage_kernel(DDStageArgs a) {
    extern __shared__ double sh[];
    if (GX) {
        __shared__ int s_task;
        for (;;) {
            __syncthreads();  // the previous task's last reads of shared memory are done
            if (threadIdx.x == 0) s_task = (int)atomicAdd(a.gctr, 1u);
            __syncthreads();
            const int tk = s_task;
            if (tk >= a.ntasks) break;
#ifdef PRS_DD_TIMING
            const unsigned long long tt0 = dd_gtimer();
#endif
            dd_stage_task<DR, SRC, 1>(a, sh, tk / a.CL, tk % a.CL);
#ifdef PRS_DD_TIMING
            if (threadIdx.x == 0) {
                atomicAdd(&g_dd_timing[2], dd_gtimer() - tt0);
                atomicAdd(&g_dd_timing[3], 1ull);
            }
#endif
        }
    } else {
        const int crank = (a.CL > 1) ? (int)cg::this_cluster().block_rank() : 0;
        dd_stage_task<DR, SRC, 0>(a, sh, blockIdx.x / a.CL, crank);
    }
}

inline size_t dd_stage_smem_bytes() {
    // tile + two staged M chunks (the y-solve chunk maps alias them) + cluster totals
    static_assert(2 * DD_KC * DD_WPAD * sizeof(double) >= DD_NCH * DD_WMAX * sizeof(double2), "sc alias");
    return sizeof(double) * ((size_t)(cpad(DD_RMAX - 1) + 1) * DD_WPAD + 2 * DD_KC * DD_WPAD) +
           sizeof(double2) * (2 * DD_WMAX);
}

// ------------------------------------------------------------------ host side ------
struct DDData {
    const double *sinpi = nullptr;
    int n = 0, S = 0, ov = 0, ramp = 0, dim = 2;
    double c = 0, h2inv = 0;
    double *rhon = nullptr, *rhof = nullptr, *Z = nullptr;
    std::vector<int> bi0[2], bW[2];
    int *d_bi0[2] = {nullptr, nullptr}, *d_bW[2] = {nullptr, nullptr};
    // per tau slot (3) and colour (2): device arrays of per-block pointers + the storage
    double tau[3] = {-1.0, -1.0, -1.0};
    std::vector<double *> store[3];
    const double **d_Q[3][2] = {}, **d_QT[3][2] = {}, **d_idy[3][2] = {};
    // global-exchange stage launch (default; PRS_DDCL=1: clusters)
    bool gx = true;
    int num_sms = 148;
    int *gbuf = nullptr;        // [1 + 2 * gcap]: task counter, flags
    double2 *gtot = nullptr;    // [gcap][2][DD_WMAX]
    int gen = 0;                // bumped when gbuf / gtot are reallocated (captured graphs hold them)
    long long gcap = 0;
    // full diffusion tensor (coef_kind 2, ddfull.cuh): d tables and per (slot, colour) the
    // block-Thomas factors E_l^T, P_l^{-1} of every block
    bool full = false;
    double h = 0;
    double *dxf = nullptr, *dyf = nullptr;
    double **d_ET[3][2] = {}, **d_PI[3][2] = {};
};

inline DFOp df_op(const DDData &d, int colour) {
    DFOp o;
    o.n = d.n;
    o.h2inv = d.h2inv;
    o.c = d.c;
    o.rhon = d.rhon + colour * d.n;
    o.rhof = d.rhof + colour * (d.n + 1);
    o.dxf = d.dxf;
    o.dyf = d.dyf;
    return o;
}

// block extents from the index-space geometry (host; integers only, R6)
inline void dd_blocks(int n, int S, int ov, int colour, std::vector<int> &i0, std::vector<int> &W) {
    const int w = n / S, half = ov / 2;
    i0.clear();
    W.clear();
    for (int k = colour; k < S; k += 2) {
        // nodes (0-based) with rho > 0: strip k interior plus the ramps (half nodes each side)
        int lo = k * w - (k > 0 ? half : 0);
        int hi = (k + 1) * w - 1 + (k < S - 1 ? half : 0);
        i0.push_back(lo);
        W.push_back(hi - lo + 1);
    }
}

inline int dd_init(DDData &d, const prs_problem &p, double h, double h2inv, cudaStream_t st, std::string &err) {
    if (p.coef_kind != 0 && p.coef_kind != 2) {
        err = "DD splitting on the GPU path: kappa = 1 or the full tensor of section 5.2";
        return PRS_EUNSUPPORTED;
    }
    d.full = p.coef_kind == 2;
    d.h = h;
    d.n = p.n;
    d.S = p.dd_strips;
    d.ov = p.dd_overlap;
    d.ramp = p.dd_ramp;
    d.c = p.c;
    d.h2inv = h2inv;
    if (d.S < 2 || d.ov < 2) {
        err = "DD GPU path needs at least 2 strips and an overlap of at least 2 cells";
        return PRS_EUNSUPPORTED;
    }
    if ((d.n + DD_RMAX - 1) / DD_RMAX > 16) {
        err = "DD GPU path supports n <= 1024";
        return PRS_EUNSUPPORTED;
    }
    for (int col = 0; col < 2; ++col) {
        dd_blocks(d.n, d.S, d.ov, col, d.bi0[col], d.bW[col]);
        for (int w : d.bW[col])
            if (w > (d.full ? DF_WMAX : DD_WMAX)) {
                err = "DD block wider than " + std::to_string(d.full ? DF_WMAX : DD_WMAX) + " columns";
                return PRS_EUNSUPPORTED;
            }
    }
    if (cudaMalloc(&d.rhon, sizeof(double) * 2 * d.n) != cudaSuccess ||
        cudaMalloc(&d.rhof, sizeof(double) * 2 * (d.n + 1)) != cudaSuccess ||
        cudaMalloc(&d.Z, sizeof(double) * DD_WMAX * DD_WMAX) != cudaSuccess) {
        err = "cudaMalloc (DD tables) failed";
        return PRS_ECUDA;
    }
    dd_rho_tables<<<(d.n + 1 + 255) / 256, 256, 0, st>>>(d.n, d.S, d.ov, d.ramp, d.rhon, d.rhof);
    if (d.full) {
        const long long tot = (long long)d.n * (d.n + 1);
        if (cudaMalloc(&d.dxf, sizeof(double) * tot) != cudaSuccess ||
            cudaMalloc(&d.dyf, sizeof(double) * tot) != cudaSuccess) {
            err = "cudaMalloc (full-tensor tables) failed";
            return PRS_ECUDA;
        }
        df_tables<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(d.n, h, d.dxf, d.dyf);
    }
    for (int col = 0; col < 2; ++col) {
        const size_t nb = d.bi0[col].size();
        if (cudaMalloc(&d.d_bi0[col], sizeof(int) * nb) != cudaSuccess ||
            cudaMalloc(&d.d_bW[col], sizeof(int) * nb) != cudaSuccess) {
            err = "cudaMalloc (DD blocks) failed";
            return PRS_ECUDA;
        }
        cudaMemcpyAsync(d.d_bi0[col], d.bi0[col].data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d.d_bW[col], d.bW[col].data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st);
    }
    const char *clv = getenv("PRS_DDCL");
    d.gx = !(clv && clv[0] == '1');
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStreamSynchronize(st);
    if (cudaGetLastError() != cudaSuccess) {
        err = "DD table setup failed";
        return PRS_ECUDA;
    }
    return PRS_OK;
}

// full tensor: block-Thomas factors of every block of both colours (one CTA per block)
inline int df_factors(DDData &d, int slot, double tau, cudaStream_t st, std::string &err) {
    for (int col = 0; col < 2; ++col) {
        const size_t nb = d.bi0[col].size();
        std::vector<double *> hE(nb), hP(nb);
        int wmax = 0;
        for (size_t k = 0; k < nb; ++k) {
            const int W = d.bW[col][k];
            wmax = std::max(wmax, W);
            const size_t bytes = sizeof(double) * (size_t)d.n * W * W;
            if (cudaMalloc(&hE[k], bytes) != cudaSuccess || cudaMalloc(&hP[k], bytes) != cudaSuccess) {
                err = "cudaMalloc (full-tensor factors) failed";
                return PRS_ECUDA;
            }
            d.store[slot].insert(d.store[slot].end(), {hE[k], hP[k]});
        }
        double **dE, **dP;
        if (cudaMalloc(&dE, sizeof(double *) * nb) != cudaSuccess || cudaMalloc(&dP, sizeof(double *) * nb) != cudaSuccess) {
            err = "cudaMalloc (full-tensor pointer tables) failed";
            return PRS_ECUDA;
        }
        d.store[slot].insert(d.store[slot].end(), {(double *)dE, (double *)dP});
        cudaMemcpyAsync(dE, hE.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dP, hP.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
        d.d_ET[slot][col] = dE;
        d.d_PI[slot][col] = dP;
        const size_t fsm = df_factor_smem_bytes(wmax);
        if (cudaFuncSetAttribute(df_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm) !=
            cudaSuccess) {
            err = "cudaFuncSetAttribute(df_factor_kernel) failed";
            return PRS_ECUDA;
        }
        df_factor_kernel<<<(unsigned)nb, DF_FTHREADS, fsm, st>>>(df_op(d, col), d.d_bi0[col], d.d_bW[col], tau, dE,
                                                               dP);
    }
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        err = "full-tensor factorisation failed";
        return PRS_ECUDA;
    }
    return PRS_OK;
}

inline int dd_factors(DDData &d, int slot, double tau, cudaStream_t st, std::string &err) {
    if (d.tau[slot] == tau) return PRS_OK;
    for (double *p : d.store[slot]) cudaFree(p);
    d.store[slot].clear();
    d.tau[slot] = tau;
    if (d.full) return df_factors(d, slot, tau, st, err);
    const size_t fsm = sizeof(double) * ((size_t)DD_WMAX * DD_WMAX + 2 * (DD_WMAX / 2 + 1)) +
                       sizeof(int) * 2 * (DD_WMAX / 2 + 1);
    if (cudaFuncSetAttribute(dd_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm) !=
        cudaSuccess) {
        err = "cudaFuncSetAttribute(dd_factor_kernel) failed";
        return PRS_ECUDA;
    }
    for (int col = 0; col < 2; ++col) {
        const size_t nb = d.bi0[col].size();
        std::vector<const double *> hQ(nb), hQT(nb), hI(nb);
        for (size_t k = 0; k < nb; ++k) {
            const int W = d.bW[col][k];
            double *Q, *QT, *th, *idy;
            if (cudaMalloc(&Q, sizeof(double) * W * W) != cudaSuccess ||
                cudaMalloc(&QT, sizeof(double) * W * W) != cudaSuccess ||
                cudaMalloc(&th, sizeof(double) * W) != cudaSuccess ||
                cudaMalloc(&idy, sizeof(double) * (size_t)W * d.n) != cudaSuccess) {
                err = "cudaMalloc (DD factors) failed";
                return PRS_ECUDA;
            }
            d.store[slot].insert(d.store[slot].end(), {Q, QT, th, idy});
            dd_factor_kernel<<<1, DD_FTHREADS, fsm, st>>>(d.n, d.bi0[col][k], W, d.rhon + col * d.n,
                                                         d.rhof + col * (d.n + 1), tau, d.h2inv, d.c, d.Z, Q, QT,
                                                         th, idy, 14);
            hQ[k] = Q;
            hQT[k] = QT;
            hI[k] = idy;
        }
        const double **dq, **dqt, **di;
        if (cudaMalloc(&dq, sizeof(double *) * nb) != cudaSuccess ||
            cudaMalloc(&dqt, sizeof(double *) * nb) != cudaSuccess ||
            cudaMalloc(&di, sizeof(double *) * nb) != cudaSuccess) {
            err = "cudaMalloc (DD pointer tables) failed";
            return PRS_ECUDA;
        }
        d.store[slot].insert(d.store[slot].end(), {(double *)dq, (double *)dqt, (double *)di});
        cudaMemcpyAsync(dq, hQ.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dqt, hQT.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(di, hI.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
        d.d_Q[slot][col] = dq;
        d.d_QT[slot][col] = dqt;
        d.d_idy[slot][col] = di;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        err = "DD factorisation failed";
        return PRS_ECUDA;
    }
    return PRS_OK;
}

inline void dd_free(DDData &d) {
    for (auto &v : d.store) {
        for (double *p : v) cudaFree(p);
        v.clear();
    }
    if (d.gbuf) cudaFree(d.gbuf);
    if (d.gtot) cudaFree(d.gtot);
    double *bufs[] = {d.rhon, d.rhof, d.Z, d.dxf, d.dyf};
    for (double *p : bufs)
        if (p) cudaFree(p);
    for (int c = 0; c < 2; ++c) {
        if (d.d_bi0[c]) cudaFree(d.d_bi0[c]);
        if (d.d_bW[c]) cudaFree(d.d_bW[c]);
    }
}

// one DD step (two colour stages) on B states: in -> out
inline int dd_step(DDData &d, int scheme, int slot, const double *in, double *out, long long B, const TimeArgs &ta,
                   int epi, const double *gc, double *gcache, const double *delta, double *traj,
                   unsigned long long *red, cudaStream_t st, prs_ctx *prof, std::string &err, long long &launches,
                   double src_amp, int src) {
    const int n = d.n;
    if (d.full) {
        for (int stage = 0; stage < 2; ++stage) {
            DFStageArgs a{};
            a.U = in;
            a.V = out;
            a.vol = (long long)n * n;
            a.n = n;
            a.B = (int)B;
            a.stage = stage;
            a.nblk = (int)d.bi0[stage].size();
            a.bi0 = d.d_bi0[stage];
            a.bW = d.d_bW[stage];
            a.ET = d.d_ET[slot][stage];
            a.PI = d.d_PI[slot][stage];
            a.tau = d.tau[slot];
            a.c = d.c;
            a.op_me = df_op(d, stage);
            a.op_ot = df_op(d, 1 - stage);
            a.src_amp = src_amp;
            a.sinpi = d.sinpi;
            a.ta = ta;
            a.epi = epi;
            a.e_gc = gc;
            a.e_gcache = gcache;
            a.e_delta = delta;
            a.e_traj = traj;
            a.e_red = red;
            void (*kern)(DFStageArgs) = nullptr;
            const int dr = scheme == PRS_DR;
#define DK(D, S_) if (dr == D && src == S_) kern = df_stage_kernel<D, S_>;
            DK(0, 0) DK(0, 1) DK(1, 0) DK(1, 1)
#undef DK
            if (prof && prs_internal_prof_begin(prof) != PRS_OK) return PRS_ECUDA;
            kern<<<(unsigned)(B * a.nblk), DF_THREADS, 0, st>>>(a);
            launches++;
            const cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) {
                err = std::string("df_stage_kernel: ") + cudaGetErrorString(e);
                return PRS_ECUDA;
            }
            if (prof) {
                // algorithmic fp64 flops: two dense W x W mat-vecs per block row and state
                double flops = 0.0;
                for (int w : d.bW[stage]) flops += (double)n * (4.0 * w * w + 20.0 * w);
                if (prs_internal_prof_end(prof, PRS_K_DD, (double)B * flops) != PRS_OK) return PRS_ECUDA;
            }
        }
        return PRS_OK;
    }
    const int CL = (n + DD_RMAX - 1) / DD_RMAX;
    const size_t shm = dd_stage_smem_bytes();
    for (int stage = 0; stage < 2; ++stage) {
        DDStageArgs a{};
        a.U = in;
        a.V = out;
        a.vol = (long long)n * n;
        a.n = n;
        a.B = (int)B;
        a.stage = stage;
        a.CL = CL;
        a.R = (n + CL - 1) / CL;
        a.nblk = (int)d.bi0[stage].size();
        a.bi0 = d.d_bi0[stage];
        a.bW = d.d_bW[stage];
        a.Q = d.d_Q[slot][stage];
        a.QT = d.d_QT[slot][stage];
        a.idy = d.d_idy[slot][stage];
        a.tau = d.tau[slot];
        a.h2inv = d.h2inv;
        a.c = d.c;
        a.rhon = d.rhon;
        a.rhof = d.rhof;
        a.src_amp = src_amp;
        a.sinpi = d.sinpi;
        a.ta = ta;
        a.epi = epi;
        a.e_gc = gc;
        a.e_gcache = gcache;
        a.e_delta = delta;
        a.e_traj = traj;
        a.e_red = red;
        const long long ntasks = B * a.nblk * CL;
        if (d.gx && ntasks > d.gcap) {
            if (d.gbuf) cudaFree(d.gbuf);
            if (d.gtot) cudaFree(d.gtot);
            d.gbuf = nullptr;
            d.gtot = nullptr;
            d.gcap = 0;
            if (cudaMalloc(&d.gbuf, sizeof(int) * (1 + 2 * ntasks)) != cudaSuccess ||
                cudaMalloc(&d.gtot, sizeof(double2) * 2 * DD_WMAX * ntasks) != cudaSuccess) {
                err = "cudaMalloc (DD exchange) failed";
                return PRS_ECUDA;
            }
            d.gcap = ntasks;
            ++d.gen;
        }
        a.gctr = reinterpret_cast<unsigned *>(d.gbuf);
        a.gflag = d.gbuf + 1;
        a.gtot = d.gtot;
        a.ntasks = (int)ntasks;
        void (*kern)(DDStageArgs) = nullptr;
        const int dr = scheme == PRS_DR;
#define DK(D, S_, X) if (dr == D && src == S_ && (int)d.gx == X) kern = dd_stage_kernel<D, S_, X>;
        DK(0, 0, 0) DK(0, 1, 0) DK(1, 0, 0) DK(1, 1, 0) DK(0, 0, 1) DK(0, 1, 1) DK(1, 0, 1) DK(1, 1, 1)
#undef DK
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm) != cudaSuccess) {
            err = "cudaFuncSetAttribute(dd_stage_kernel) failed";
            return PRS_ECUDA;
        }
        cudaLaunchConfig_t cfg{};
        int per_sm = 1;  // persistent grid: every co-resident CTA slot
        if (d.gx && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, DD_THREADS, shm) != cudaSuccess)
            per_sm = 1;
        per_sm = std::max(per_sm, 1);
        cfg.gridDim = dim3((unsigned)(d.gx ? std::min<long long>(ntasks, (long long)per_sm * d.num_sms) : ntasks));
        cfg.blockDim = dim3(DD_THREADS);
        cfg.dynamicSmemBytes = shm;
        cfg.stream = st;
        if (!d.gx && CL > 8) {
            err = "DD cluster exchange (PRS_DDCL=1): at most 8 row pieces per block";
            return PRS_EUNSUPPORTED;
        }
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = d.gx ? 0 : 1;
        if (d.gx && cudaMemsetAsync(d.gbuf, 0, sizeof(int) * (1 + 2 * ntasks), st) != cudaSuccess) {
            err = "cudaMemsetAsync (DD exchange flags) failed";
            return PRS_ECUDA;
        }
        if (prof && prs_internal_prof_begin(prof) != PRS_OK) return PRS_ECUDA;
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
        launches++;
        if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) {
            err = std::string("dd_stage_kernel: ") + cudaGetErrorString(e);
            return PRS_ECUDA;
        }
        if (prof) {
            // algorithmic fp64 flops: per support point of a W-wide block, two W x W
            // transforms (2 W each) and the tridiagonal solve along y (~10)
            double flops = 0.0;
            for (int w : d.bW[stage]) flops += (double)w * n * (4.0 * w + 10.0);
            if (prs_internal_prof_end(prof, PRS_K_DD, (double)B * flops) != PRS_OK) return PRS_ECUDA;
        }
    }
    return PRS_OK;
}

}  // namespace prs
