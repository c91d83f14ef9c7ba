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
#include "dfpart.cuh"
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

// double-double arithmetic (setup only): a value hi + lo with |lo| <= ulp(hi) / 2
struct DDd {
    double hi, lo;
};
__device__ __forceinline__ DDd ddd_two_sum(double a, double b) {
    const double s = a + b, bb = s - a;
    return DDd{s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ DDd ddd_norm(double hi, double lo) {
    const double s = hi + lo;
    return DDd{s, lo - (s - hi)};
}
__device__ __forceinline__ DDd ddd_add(DDd a, DDd b) {
    const DDd s = ddd_two_sum(a.hi, b.hi);
    return ddd_norm(s.hi, s.lo + a.lo + b.lo);
}
__device__ __forceinline__ DDd ddd_mul_d(DDd a, double b) {
    const double p = a.hi * b;
    return ddd_norm(p, fma(a.hi, b, -p) + a.lo * b);
}
__device__ __forceinline__ DDd ddd_div(DDd a, DDd b) {
    const double q1 = a.hi / b.hi;
    const DDd r = ddd_add(a, ddd_mul_d(b, -q1));
    const double q2 = r.hi / b.hi;
    const DDd q = ddd_norm(q1, q2);
    const DDd r2 = ddd_add(r, ddd_mul_d(b, -q2));
    return ddd_norm(q.hi, q.lo + r2.hi / b.hi);
}
// s += a b (a, b doubles)
__device__ __forceinline__ void dd_acc(DDd &s, double a, double b) {
    const double p = a * b, pe = fma(a, b, -p);
    const DDd t = ddd_two_sum(s.hi, p);
    s = ddd_norm(t.hi, t.lo + s.lo + pe);
}

// theta_a and the pivots of mode a's y system theta_a I - tau Y (diagonal theta_a + 2 s, off -s,
// s = tau / h^2): id_l = 1 / d_l, and in theta[W + a] the row from which they are constant.
// The recurrence d_l = theta_a + 2 s - s^2 / d_{l-1} runs in double-double and only id_l is
// rounded: in fp64, theta_a + 2 s alone rounds by eps s -- at c4's coarse step (s = 3.3e4) a
// COHERENT shift of every low mode's theta_a (~16) by ~1e-12 of itself, which the smooth part of
// the solution takes over whole (GPU 4e-12 off the extended-precision step, the oracle, whose
// band-matrix entries are exact here, 2e-13).  Rounding id_l alone perturbs the implied
// matrix by independent +-eps dipoles per row, which smooth solutions do not feel.
__device__ inline void dd_mode_pivots(int n, int W, int a, DDd th, double s, double *theta, double *idy) {
    theta[a] = th.hi;
    const DDd bd = ddd_add(th, DDd{2.0 * s, 0.0});
    const DDd s2 = ddd_norm(s * s, fma(s, s, -s * s));
    DDd d = bd;
    double prev = 0.0;
    int lc = 0;  // last row whose pivot differs from the row before: rows >= lc share one value
    for (int l = 0; l < n; ++l) {
        if (l > 0) {
            const DDd q = ddd_div(s2, d);
            d = ddd_add(bd, DDd{-q.hi, -q.lo});
        }
        const DDd idd = ddd_div(DDd{1.0, 0.0}, d);
        const double id = idd.hi + idd.lo;
        if (l > 0 && id != prev) lc = l;
        prev = id;
        idy[(long long)l * W + a] = id;
    }
    theta[W + a] = (double)lc;  // (the recurrence reaches its fixed point in a few hundred rows)
}

// The m x m generalised problem S x = theta R x of one factorisation (a whole block, m = W, or
// one half of a folded block, m = W / 2): S tridiagonal (diagonal sd, off-diagonal se), R =
// diag(sr), assembled by dd_assemble_kernel.
//   fold 0: the block rows of I - tau A_j:  S_ii = 1 + tau h^-2 (rho(i-1/2) + rho(i+1/2)) +
//           tau c rho(i),  S_i,i+1 = -tau h^-2 rho(i+1/2),  R = rho(i);
//   fold 1 / 2 (symmetric / antisymmetric vectors q = [u; +-J u] of a mirror-symmetric block):
//           the upper W/2 rows of S with the coupling across the centre folded onto the last
//           diagonal entry (+ / -), everything times 2, so that u^T (2 R) u = q^T R q = 1.
__global__ void dd_assemble_kernel(int i0, int W, int fold, const double *rhon, const double *rhof, double tau,
                                   double h2inv, double c, double *sd, double *se, double *sr) {
    const int m = fold ? W / 2 : W;
    const double s = tau * h2inv, f = fold ? 2.0 : 1.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int gi = i0 + i;
        double dv = 1.0 + s * (rhof[gi] + rhof[gi + 1]) + tau * c * rhon[gi];
        const double ev = -s * rhof[gi + 1];
        if (fold && i == m - 1) dv += (fold == 1) ? ev : -ev;
        sd[i] = f * dv;
        se[i] = f * ev;
        sr[i] = f * rhon[gi];
    }
}

// Jacobi on C = R^{-1/2} S R^{-1/2} (symmetric tridiagonal) in shared memory; X = R^{-1/2} Z
// (m x m, [i][a]) and, without refinement, theta and the mode pivots of modes moff + a.
__global__ void __launch_bounds__(DD_FTHREADS) dd_factor_kernel(int n, int m, const double *sd, const double *se,
                                                               const double *sr, double s, int W, int moff,
                                                               double *Z, double *X, double *theta, double *idy,
                                                               int sweeps, int pivots) {
    extern __shared__ double sh[];
    const int Wf = W;
    W = m;  // the Jacobi below runs on the m x m problem
    double *C = sh;                 // W x W (row stride W)
    double *cs = sh + W * W;        // rotation cos per pair
    double *sn = cs + DD_WMAX / 2 + 1;
    int *pp = reinterpret_cast<int *>(sn + DD_WMAX / 2 + 1);
    int *qq = pp + DD_WMAX / 2 + 1;
    const int tid = threadIdx.x;
    // assemble C and Z = I
    for (int e = tid; e < W * W; e += blockDim.x) {
        const int r = e / W, k = e % W;
        double v = 0.0;
        if (r == k) v = sd[r] / sr[r];
        else if (k == r + 1) v = se[r] / sqrt(sr[r] * sr[k]);
        else if (r == k + 1) v = se[k] / sqrt(sr[r] * sr[k]);
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
    // eigenvalues on the diagonal; X = R^{-1/2} Z; pivots of theta_a + 2 s, off -s (s = tau/h^2)
    if (pivots)
        for (int a = tid; a < W; a += blockDim.x) dd_mode_pivots(n, Wf, moff + a, DDd{C[a * W + a], 0.0}, s, theta, idy);
    else
        for (int a = tid; a < W; a += blockDim.x) Z[W * W + a] = C[a * W + a];  // theta for the refinement
    for (int e = tid; e < W * W; e += blockDim.x) X[e] = Z[e] / sqrt(sr[e / W]);
}

// ------------------------------------------------ refinement of the eigenbasis ---
// Jacobi in fp64 leaves each eigenvector of C off by ~eps ||C|| / gap: at c4's coarse step
// (tau / h^2 = 3.3e4, ||C|| ~ 2e6, low-mode gaps ~ 50) that is ~1e-11, and the block solve
// inherits it (one coarse step 7e-12 of |U| off the extended-precision value, against the
// oracle's band elimination at 2e-13).  One Newton step on the generalised problem (the
// Ogita-Aishima refinement with R in place of I) restores full accuracy: with X = Q from Jacobi,
//     Ms = X^T S X,  Mr = X^T R X   (products exact to double-double: the off-diagonal terms
//                                     sought are ~eps ||C|| residues of sums of size ||C||),
//     theta_a = Ms_aa / Mr_aa,  E_aa = (1 - Mr_aa) / 2,
//     E_ab = (Ms_ab - theta_b Mr_ab) / (theta_b - theta_a)   (a != b; E_ab = -Mr_ab / 2 for a
//            relative gap below 1e-6, where the coupling left behind is below eps theta),
//     Q' = X (I + E),
// after which Q'^T R Q' = I and Q'^T S Q' = Theta up to (eps ||C|| / gap)^2 and the rounding
// of Q' itself.  One CTA per block, once per tau (setup).
__global__ void __launch_bounds__(DD_FTHREADS) dd_refine_kernel(int n, int m, const double *sd, const double *se,
                                                               const double *sr, double s, int Wf, int moff,
                                                               double *scr, double *X, double *theta,
                                                               double *idy) {
    const int tid = threadIdx.x;
    const int W = m;  // the m x m problem (dd_assemble_kernel)
    const int WW = W * W;
    double *Q = X;
    double *Thi = scr, *Tlo = scr + WW, *Ms = scr + 2 * WW, *Mr = scr + 3 * WW;
    __shared__ double th[DD_WMAX], thl[DD_WMAX], dr[DD_WMAX];
    // T = S X (S tridiagonal) in double-double
    for (int e = tid; e < WW; e += blockDim.x) {
        const int i = e / W;
        DDd t{0.0, 0.0};
        dd_acc(t, sd[i], Q[e]);
        if (i > 0) dd_acc(t, se[i - 1], Q[e - W]);
        if (i + 1 < W) dd_acc(t, se[i], Q[e + W]);
        Thi[e] = t.hi;
        Tlo[e] = t.lo;
    }
    __syncthreads();
    // Ms = X^T T, Mr = X^T R X (a <= b), double-double
    for (int e = tid; e < WW; e += blockDim.x) {
        const int a = e / W, b = e % W;
        if (b < a) continue;
        DDd ms{0.0, 0.0}, mr{0.0, 0.0};
        for (int i = 0; i < W; ++i) {
            const double xa = Q[i * W + a], xb = Q[i * W + b];
            dd_acc(ms, xa, Thi[i * W + b]);
            ms.lo = fma(xa, Tlo[i * W + b], ms.lo);
            const double r = sr[i];
            const double pr = xa * r, pre = fma(xa, r, -pr);  // xa r exactly = pr + pre
            dd_acc(mr, pr, xb);
            mr.lo = fma(pre, xb, mr.lo);
        }
        if (a == b) {
            const DDd q = ddd_div(ms, mr);  // the Rayleigh quotient, double-double
            th[a] = q.hi;
            thl[a] = q.lo;
            dr[a] = 0.5 * ((1.0 - mr.hi) - mr.lo);
        } else {
            Ms[a * W + b] = Ms[b * W + a] = ms.hi + ms.lo;
            Mr[a * W + b] = Mr[b * W + a] = mr.hi + mr.lo;
        }
    }
    __syncthreads();
    // E (into Ms): E_ab = (Ms_ab - theta_b Mr_ab) / (theta_b - theta_a)
    for (int e = tid; e < WW; e += blockDim.x) {
        const int a = e / W, b = e % W;
        double v;
        if (a == b) {
            v = dr[a];
        } else {
            const double gap = th[b] - th[a];
            v = (fabs(gap) > 1e-6 * fmax(fabs(th[a]), fabs(th[b]))) ? (Ms[e] - th[b] * Mr[e]) / gap : -0.5 * Mr[e];
        }
        Thi[e] = v;  // (T is dead)
    }
    __syncthreads();
    // X' = X + X E (the correction is ~1e-11 of X: fp64 suffices), into Tlo, then X
    for (int e = tid; e < WW; e += blockDim.x) {
        const int i = e / W, k = e % W;
        double corr = 0.0;
        for (int a = 0; a < W; ++a) corr = fma(Q[i * W + a], Thi[a * W + k], corr);
        Tlo[e] = Q[e] + corr;
    }
    __syncthreads();
    for (int e = tid; e < WW; e += blockDim.x) Q[e] = Tlo[e];
    for (int a = tid; a < W; a += blockDim.x) dd_mode_pivots(n, Wf, moff + a, DDd{th[a], thl[a]}, s, theta, idy);
}

// Q (W x W, [i][a]) and QT = Q^T of a block from the m x m X of one factorisation: fold 0: Q = X;
// fold 1 (modes 0 .. m-1): Q[k][a] = X[k][a]; fold 2 (modes m .. W-1): Q[W-1-j][m+a] = X[j][a].
// Positions k < W/2 of a folded tile hold F_k + F_{W-1-k}, positions W-1-j hold F_j - F_{W-1-j}
// (dd_fold_tile), so G = T Q is [F_s U_s | F_a U_a]; the other entries stay zero (block
// diagonal: the GEMM reads each n-tile's own block only).
__global__ void dd_place_kernel(int W, int m, int fold, const double *X, double *Q, double *QT) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += gridDim.x * blockDim.x) {
        const int j = e / m, a = e % m;
        const int row = (fold == 2) ? W - 1 - j : j, col = (fold == 2) ? m + a : a;
        Q[row * W + col] = X[e];
        QT[col * W + row] = X[e];
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
    const int *bWs;      // split stage: symmetric-half width of a folded block (dd_fold_tile), else W
    const double *const *Q, *const *QT, *const *idy;  // per block
    const double *const *conv;  // per block [W]: pivots of mode a are equal from this row on
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
    // split stage (dd_p1 / dd_scan / dd_p2): per task the transformed tile G [R][DD_WMAX], the
    // piece's transfer tuple [5][DD_WMAX] and its boundary values y_in, x_in [2][DD_WMAX]
    double *gs, *tup, *bnd;
    long long gs_end, tup_end, bnd_end;  // PRS_CHECKS: element counts of gs / tup / bnd from their pointers
    int abl;  // diagnostic build (-DPRS_DD_TIMING) only: PRS_DD_ABL bit 0 skips the GEMMs, bit 1 the walks
};

#ifdef PRS_DD_TIMING
// diagnostic build only (-DPRS_DD_TIMING): per task, ns spent waiting for the forward / the
// backward scan totals of the other row pieces, the task's duration, and the task count
__device__ unsigned long long g_dd_timing[4];
// split stage: per task (thread 0) ns in p1 load / GEMM / G store + walk, p2 load / walk / GEMM /
// store, and the task counts of p1, p2
__device__ unsigned long long g_dd2_timing[9];
#define DD2T(i)                                                   \
    do {                                                          \
        if (threadIdx.x == 0) {                                   \
            const unsigned long long t_ = dd_gtimer();            \
            atomicAdd(&g_dd2_timing[i], t_ - tt_);                \
            tt_ = t_;                                             \
        }                                                         \
    } while (0)
#define DD2T0 unsigned long long tt_ = dd_gtimer()
__device__ __forceinline__ unsigned long long dd_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#else
#define DD2T(i) \
    do {        \
    } while (0)
#define DD2T0 \
    do {      \
    } while (0)
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
// Barrier of the threads working on one tile (the whole CTA).
struct CtaSync {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

// Per-lane column masks of a tile (lane owns columns lane + 32 k): done0m -- already final
// after stage 0 (stage 1 takes them from V); finm -- final after this stage (epilogue applies).
struct DDCols {
    unsigned done0m, finm;
};

// Load the right-hand side tile of rows r0 .. r0 + nrow - 1 of block blk of state b into the
// chunk-padded shared tile T (columns >= W zero): one row per warp, columns across lanes.
template <int DR, int SRC, int NT = DD_THREADS, class SY = CtaSync>
__device__ __forceinline__ DDCols dd_load_tile(const DDStageArgs &a, double *T, long long b, int blk, int r0,
                                               int nrow, int tid = threadIdx.x, SY sync = SY{}) {
    const int i0 = a.bi0[blk], W = a.bW[blk];
    const int n = a.n;
    const double *Ub = a.U + b * a.vol;
    const double *Vb = a.V + b * a.vol;
    const int me = a.stage, other = 1 - a.stage;
    const double *rn_ot = a.rhon + other * n, *rf_ot = a.rhof + other * (n + 1);
    double ampt = 0.0;
    if (SRC) ampt = a.src_amp * src_tf(a.ta, b);
    // every global load of a row is issued before the first use (several rows' worth in flight)
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
    if (!(DR && me == 0)) {
        // no stencil: asynchronous 8-byte copies of the raw rows (stage 1: V on the columns that
        // are final after stage 0, U elsewhere), every one of the tile in flight at once; the
        // source term is added in shared memory after they land
        const int wp = tid >> 5, ln = tid & 31;
        if (((n | i0 | W) & 1) == 0) {
            // 16-byte copies of column pairs (both columns from the same source: V where rho_0 > 0,
            // which holds pairwise here -- else two 8-byte copies)
            const double *rn0 = a.rhon;  // colour 0
            for (int rl = wp; rl < nrow; rl += (NT / 32)) {
                const long long g0 = (long long)(r0 + rl) * n + i0;
                double *trow = T + cpad(rl) * DD_WPAD;
#pragma unroll
                for (int k = 0; k < (DD_WMAX / 2 + 31) / 32; ++k) {
                    const int ci = 2 * (ln + 32 * k);
                    if (ci < W) {
                        const bool v0 = me == 1 && rn0[i0 + ci] > 0.0, v1 = me == 1 && rn0[i0 + ci + 1] > 0.0;
                        if (v0 == v1) {
                            cp_async16(trow + ci, (v0 ? Vb : Ub) + g0 + ci);
                        } else {
                            cp_async8(trow + ci, (v0 ? Vb : Ub) + g0 + ci);
                            cp_async8(trow + ci + 1, (v1 ? Vb : Ub) + g0 + ci + 1);
                        }
                    } else if (ci < DD_WMAX) {
                        trow[ci] = 0.0;
                        trow[ci + 1] = 0.0;
                    }
                }
            }
        } else {
            for (int rl = wp; rl < nrow; rl += (NT / 32)) {
                const long long g0 = (long long)(r0 + rl) * n + i0;
                double *trow = T + cpad(rl) * DD_WPAD;
#pragma unroll
                for (int k = 0; k < NCW; ++k) {
                    const int ci = ln + 32 * k;
                    if (ci < W) cp_async8(trow + ci, (((done0m >> k) & 1u) ? Vb : Ub) + g0 + ci);
                    else if (ci < DD_WMAX) trow[ci] = 0.0;
                }
            }
        }
        cp_async_commit();
        cp_async_wait<0>();
        sync();
        if (SRC) {
            for (int rl = wp; rl < nrow; rl += (NT / 32)) {
                const double sl = a.tau * ampt * __ldg(a.sinpi + r0 + rl);
                double *trow = T + cpad(rl) * DD_WPAD;
#pragma unroll
                for (int k = 0; k < NCW; ++k) {
                    const int ci = ln + 32 * k;
                    if (ci < W && !((done0m >> k) & 1u)) trow[ci] += sl * spk[k];
                }
            }
        }
        return DDCols{done0m, finm};
    }
    {
        const int wp = tid >> 5, ln = tid & 31;
        // the source profile of the warp's rows wp + 16 q, one per lane (q = lane), shuffled out
        static_assert(DD_RMAX / ((NT / 32)) <= 32, "rows per warp");
        double slq = 0.0;
        if (SRC && wp + ((NT / 32)) * ln < nrow) slq = a.tau * ampt * __ldg(a.sinpi + r0 + wp + ((NT / 32)) * ln);
#pragma unroll 2
        for (int rl = wp; rl < nrow; rl += (NT / 32)) {
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
            const double sl = SRC ? __shfl_sync(0xffffffffu, slq, (rl - wp) / ((NT / 32))) : 0.0;
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
    return DDCols{done0m, finm};
}

// Store the solved tile (V = x [DR stage 0: - w]) with the fused parareal epilogue on the values
// that are final after this stage: one row per warp.
template <int DR, int NT = DD_THREADS>
__device__ __forceinline__ void dd_store_tile(const DDStageArgs &a, const double *T, long long b, int blk, int r0,
                                              int nrow, unsigned finm, int tid = threadIdx.x) {
    const int lane = tid & 31;
    const int i0 = a.bi0[blk], W = a.bW[blk];
    const int n = a.n;
    const double *Ub = a.U + b * a.vol;
    double *Vb = a.V + b * a.vol;
    const int me = a.stage, other = 1 - a.stage;
    const double *rn_ot = a.rhon + other * n, *rf_ot = a.rhof + other * (n + 1);
    constexpr int NCW = (DD_WMAX + 31) / 32;
    double dmax = 0.0;
    unsigned long long bad = 0;
    {
        const int wp = tid >> 5;
        for (int rl = wp; rl < nrow; rl += (NT / 32)) {
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

    const DDCols cols = dd_load_tile<DR, SRC>(a, T, b, blk, r0, nrow);

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
                x = fma(-ccv, x, id * *p);
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

    dd_store_tile<DR>(a, T, b, blk, r0, nrow, cols.finm);
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

// GEMM of the split stage: T[l][:] <- T[l][:] . M for every row of the tile, in place, on DMMA
// (m8n8k4 f64), without shared staging of M or barriers inside the k loop.  Warp w owns output
// columns 16 w .. 16 w + 15 for all DD_RMAX rows (8 x 2 tiles of 8 x 8, accumulators in
// registers): its B fragments (M[k][c], k = lane % 4, c = lane / 4) are read straight from
// global memory (L2-resident; no other warp of the CTA needs them) DD2_PF k-steps ahead of use,
// its A fragments (T[r][k], r = lane / 4) from the shared tile.  Rows >= nrow compute and
// discard; columns >= W of T are zero and B is zero outside the W x W matrix.
constexpr int DD2_THREADS = 32 * (DD_WMAX / 16);  // 9 warps
constexpr int DD_SUB = DD_RMAX / 2;                // rows of a walk sub-piece (two per tile)
static_assert(DD2_THREADS >= 2 * DD_WMAX, "two walking threads per mode");
constexpr int DD2_PF = 3;
template <class SY>
__device__ __forceinline__ void dd_tile_gemm2(double *T, const double *__restrict__ M, int W, int Ws, int tid,
                                              SY sync) {
    static_assert(DD_RMAX == 64 && DD_WMAX % 16 == 0, "dmma tiling of the split stage");
    const int lane = tid & 31, warp = tid >> 5;
    const int fr = lane >> 2, fk = lane & 3;
    // the warp's two 8-column n-tiles: 2 warp and 2 warp + 1, except on a folded block whose
    // halves meet inside an n-tile (Ws % 8 != 0, e.g. c4's W = 136): that n-tile needs both
    // halves' k ranges (twice the k-steps), so it stays alone in its warp and its partner moves
    // to the last warp's free slot (an odd n-tile count), which keeps the warps balanced
    const int ntiles = (W + 7) >> 3;
    int nt0 = 2 * warp, nt1 = 2 * warp + 1;
    {
        const int ns = (Ws < W && (Ws & 7)) ? (Ws >> 3) : -1, wl = (ntiles - 1) >> 1;
        if (ns >= 0 && (ntiles & 1) && (ns >> 1) != wl) {
            if (warp == (ns >> 1)) {
                nt0 = ns;
                nt1 = -1;
            } else if (warp == wl) {
                nt1 = ns ^ 1;
            }
        }
    }
    if (nt0 >= ntiles) nt0 = -1;
    if (nt1 >= ntiles) nt1 = -1;
    const bool active = nt0 >= 0;  // warp-uniform
    double acc[8][2][2];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) acc[r][c][0] = acc[r][c][1] = 0.0;
    sync();  // the tile is complete
    if (active) {
        const int c0 = 8 * nt0 + fr, c1 = 8 * nt1 + fr;
        const bool v0 = c0 < W, v1 = nt1 >= 0 && c1 < W;
        // k range of each n-tile (warp-uniform): Ws < W (a folded block, see dd_fold_tile): M is
        // block diagonal -- output columns c < Ws take k < Ws only, columns >= Ws take k >= Ws
        auto kr = [&](int nt, int &kb, int &ke) {
            const int cs = 8 * nt;
            if (nt < 0) { kb = ke = 0; }
            else if (cs + 8 <= Ws) { kb = 0; ke = Ws; }
            else if (cs >= Ws) { kb = Ws; ke = W; }
            else { kb = 0; ke = W; }
        };
        int kb0, ke0, kb1, ke1;
        kr(nt0, kb0, ke0);
        kr(nt1, kb1, ke1);
        // mask bit j: n-tile j accumulates in this run
        auto run = [&](int kb, int ke, int mask) {
            const int ks0 = kb >> 2, ks1 = (ke + 3) >> 2;
            double b0[DD2_PF], b1[DD2_PF];
            auto ldb = [&](int ks, double &x0, double &x1) {
                const int k = 4 * ks + fk;
                const bool kin = k < ke && k >= kb;
                x0 = (kin && v0 && (mask & 1)) ? __ldg(M + (long long)k * W + c0) : 0.0;
                x1 = (kin && v1 && (mask & 2)) ? __ldg(M + (long long)k * W + c1) : 0.0;
            };
#pragma unroll
            for (int q = 0; q < DD2_PF; ++q) ldb(ks0 + q, b0[q], b1[q]);
            const double *ta = T + fk;
            for (int ksb = ks0; ksb < ks1; ksb += DD2_PF) {
#pragma unroll
                for (int q = 0; q < DD2_PF; ++q) {
                    const int ks = ksb + q;
                    if (ks < ks1) {
                        const double bb0 = b0[q], bb1 = b1[q];
                        ldb(ks + DD2_PF, b0[q], b1[q]);
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            const double av = ta[cpad(8 * r + fr) * DD_WPAD + 4 * ks];
                            if (mask & 1) dmma_f64(acc[r][0][0], acc[r][0][1], av, bb0);
                            if (mask & 2) dmma_f64(acc[r][1][0], acc[r][1][1], av, bb1);
                        }
                    }
                }
            }
        };
        if (nt1 < 0) {
            run(kb0, ke0, 1);
        } else if (kb0 == kb1 && ke0 == ke1) {
            run(kb0, ke0, 3);
        } else {
            run(kb0, ke0, 1);
            run(kb1, ke1, 2);
        }
    }
    sync();  // every read of the tile is done: write in place
    if (active) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int nt = c ? nt1 : nt0;
                if (nt < 0) continue;
                const int col = 8 * nt + 2 * fk;
                double *p = T + cpad(8 * r + fr) * DD_WPAD + col;
                if (col < W) p[0] = acc[r][c][0];
                if (col + 1 < W) p[1] = acc[r][c][1];
            }
    }
    sync();
}

// Folded blocks (Ws = W / 2 < W: W even and rho bitwise mirror-symmetric over the block, so
// S and R are centrosymmetric and every generalised eigenvector is symmetric or antisymmetric,
// q = [u; +-J u]).  Then F Q = [F_s U_s | F_a U_a] with F_s,k = F_k + F_{W-1-k}, F_a,k =
// F_k - F_{W-1-k} (k < W/2) and U_s / U_a the upper halves of the symmetric / antisymmetric
// eigenvectors, and Q V^T unfolds the same way: half the GEMM flops.  In place, pairwise:
// position k < W/2 takes the sum, position W-1-k the difference (the folded factors are laid
// out to match, dd_place_kernel); the same pairwise map unfolds.
__device__ __forceinline__ void dd_fold_tile(double *T, int W, int nrow, int tid, int nthreads) {
    const int h = W >> 1;
    for (int e = tid; e < nrow * h; e += nthreads) {
        const int rl = e / h, k = e - rl * h;
        double *row = T + cpad(rl) * DD_WPAD;
        const double x = row[k], y = row[W - 1 - k];
        row[k] = x + y;
        row[W - 1 - k] = x - y;
    }
}

// ------------------------------------------------------- split stage (default path) ----
// The same stage as two passes over every block's row pieces with a scan between them, so that
// no piece waits on another (in dd_stage_task the scan-total exchange and the barriers behind it
// cost ~30 % of the stall samples, profiles/r02_ncu_dd_fine_summary.txt):
//   dd_p1_kernel: load + G = F Q (DMMA); store G; per mode a, over the piece's rows, the transfer
//     tuple of the y recurrences from the piece's boundary values
//        y_l     = alpha_l y_in + beta_l        (y_in: y at the row before the piece)
//        x_first = P x_in + Q1 y_in + Q0        (x_in: x at the row after the piece)
//     i.e. (A, B) = (alpha, beta) at the piece's last row, P the product of -cc, Q0 / Q1 the
//     backward maps' weights applied to beta / alpha;
//   dd_scan_kernel: per (state, block, mode) the y_in of every half piece (the walks run on
//     half pieces, two threads per mode) in order, then x_in in reverse order;
//   dd_p2_kernel: reload G, the exact forward recurrence from y_in and the backward one from
//     x_in (the arithmetic of the F3 / B3 walks), U = V Q^T (DMMA), store with the epilogue.
// Pieces are independent CTAs (two per SM): one piece's loads and walks overlap another's GEMM.

// the walk's row coefficients: m_l = -tau/h^2 id_{l-1} (0 on the line's first row),
// cc_l = -tau/h^2 id_l (0 on its last row), id_l = 1 / pivot (precomputed per mode, dd_factor_kernel)
// The walking thread's scalars, loaded ahead of the walk (before the GEMM in pass 1, before the
// wait for G in pass 2) so that their latency hides behind other work: the row from which the
// mode's pivots are constant, that pivot, and (pass 2) the sub-piece's boundary values.
struct DDWalkPre {
    int lc;
    double ids, yb, xb;
};
template <int P1>
__device__ __forceinline__ DDWalkPre dd_walk_prefetch(const DDStageArgs &a, int blk, long long tk, int tid) {
    DDWalkPre w{0, 0.0, 0.0, 0.0};
    const int W = a.bW[blk], h = tid / DD_WMAX, am = tid - h * DD_WMAX;
    if (am >= W || h > 1) return w;
    w.lc = (int)__ldg(a.conv[blk] + am);
    w.ids = __ldg(a.idy[blk] + am + (long long)(a.n - 1) * W);
    if (!P1) {
        const long long t2 = 2 * tk + h;
        w.yb = a.bnd[t2 * 2 * DD_WMAX + am];
        w.xb = a.bnd[(t2 * 2 + 1) * DD_WMAX + am];
    }
    return w;
}

template <int P1>
__device__ __forceinline__ void dd_piece_walks(const DDStageArgs &a, double *T, int blk, int r0, int nrow,
                                               long long tk, int tid, const DDWalkPre &wp) {
    // Two threads per mode: thread (h, am) walks half h of the piece (sub-piece 2 tk + h, DD_SUB
    // rows; the scan runs over sub-pieces), in batches of U rows: the batch's tile values are
    // read into registers before the recurrence runs over them (no shared-memory latency inside
    // the chain) and the next batch's pivots are in flight meanwhile.
    const int W = a.bW[blk], n = a.n, h = tid / DD_WMAX, am = tid - h * DD_WMAX;
    if (am >= W || h > 1) return;
#ifdef PRS_DD_TIMING
    if (a.abl & 2) return;
#endif
    const int rb = DD_SUB * h;  // first tile row of the sub-piece
    r0 += rb;
    nrow = max(0, min(DD_SUB, nrow - rb));
    tk = 2 * tk + h;
    const double ms = -a.tau * a.h2inv;
    const double *idc = a.idy[blk] + am;
    constexpr int U = 8;
    // rows >= lc (most pieces of a long block) share the converged pivot: no loads there
    const int lc = wp.lc;
    const double ids = wp.ids;
    auto ldid = [&](int rl) {
        return (rl >= 0 && rl < nrow) ? (r0 + rl >= lc ? ids : __ldg(idc + (long long)(r0 + rl) * W)) : 0.0;
    };
    auto trow = [&](int rl) { return T + cpad(rb + rl) * DD_WPAD + am; };
    double idn[U];
    if (P1) {
        double al = 1.0, be = 0.0, pr = 1.0, q0 = 0.0, q1 = 0.0;
        double idp = (r0 > 0) ? (r0 - 1 >= lc ? ids : __ldg(idc + (long long)(r0 - 1) * W)) : 0.0;
#pragma unroll
        for (int i = 0; i < U; ++i) idn[i] = ldid(i);
        for (int c0 = 0; c0 < nrow; c0 += U) {
            double id[U], t[U];
#pragma unroll
            for (int i = 0; i < U; ++i) {
                id[i] = idn[i];
                idn[i] = ldid(c0 + U + i);
                t[i] = (c0 + i < nrow) ? *trow(c0 + i) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < U; ++i)
                if (c0 + i < nrow) {
                    const int l = r0 + c0 + i;
                    const double m = (l == 0) ? 0.0 : ms * idp;
                    const double cc = (l == n - 1) ? 0.0 : ms * id[i];
                    be = fma(-m, be, t[i]);
                    al = -m * al;
                    const double wv = pr * id[i];
                    q0 = fma(wv, be, q0);
                    q1 = fma(wv, al, q1);
                    pr *= -cc;
                    idp = id[i];
                }
        }
        PRS_CHECK((tk + 1) * 5 * DD_WMAX <= a.tup_end, "DD tuple outside the scratch");
        double *tp = a.tup + tk * 5 * DD_WMAX + am;
        tp[0] = al;
        tp[DD_WMAX] = be;
        tp[2 * DD_WMAX] = pr;
        tp[3 * DD_WMAX] = q0;
        tp[4 * DD_WMAX] = q1;
    } else {
        double y = wp.yb;
        double idp = (r0 > 0) ? (r0 - 1 >= lc ? ids : __ldg(idc + (long long)(r0 - 1) * W)) : 0.0;
#pragma unroll
        for (int i = 0; i < U; ++i) idn[i] = ldid(i);
        for (int c0 = 0; c0 < nrow; c0 += U) {
            double id[U], t[U];
#pragma unroll
            for (int i = 0; i < U; ++i) {
                id[i] = idn[i];
                idn[i] = ldid(c0 + U + i);
                t[i] = (c0 + i < nrow) ? *trow(c0 + i) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < U; ++i) {
                const int l = r0 + c0 + i;
                const double m = (l == 0) ? 0.0 : ms * idp;
                y = fma(-m, y, t[i]);
                t[i] = y;
                idp = id[i];
            }
#pragma unroll
            for (int i = 0; i < U; ++i)
                if (c0 + i < nrow) *trow(c0 + i) = t[i];
        }
        // backward, from the piece's last row (the batches in reverse)
        double x = wp.xb;
#pragma unroll
        for (int i = 0; i < U; ++i) idn[i] = ldid(nrow - 1 - i);
        for (int c1 = nrow - 1; c1 >= 0; c1 -= U) {
            double id[U], t[U];
#pragma unroll
            for (int i = 0; i < U; ++i) {
                id[i] = idn[i];
                idn[i] = ldid(c1 - U - i);
                t[i] = (c1 - i >= 0) ? *trow(c1 - i) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < U; ++i) {
                const int l = r0 + c1 - i;
                const double ccv = (l == n - 1) ? 0.0 : ms * id[i];
                x = fma(-ccv, x, id[i] * t[i]);
                t[i] = x;
            }
#pragma unroll
            for (int i = 0; i < U; ++i)
                if (c1 - i >= 0) *trow(c1 - i) = t[i];
        }
    }
}

// A task of the split stage: row piece crank of block blk of state b (tk = (b nblk + blk) CL + crank).
struct DDTask {
    long long tk, task, b;
    int crank, blk, W, r0, nrow;
    __device__ __forceinline__ DDTask(const DDStageArgs &a, long long t) : tk(t), task(t / a.CL) {
        crank = (int)(t % a.CL);
        blk = (int)(task % a.nblk);
        b = task / a.nblk;
        W = a.bW[blk];
        r0 = crank * a.R;
        nrow = max(0, min(a.R, a.n - r0));
    }
};

// pass 1 before its GEMM: the right-hand side tile
template <int DR, int SRC, class SY>
__device__ __forceinline__ void dd_p1_pre(const DDStageArgs &a, double *T, const DDTask &t, int tid, SY sync) {
    dd_load_tile<DR, SRC, DD2_THREADS>(a, T, t.b, t.blk, t.r0, t.nrow, tid, sync);
    if (a.bWs[t.blk] < t.W) {
        sync();
        dd_fold_tile(T, t.W, t.nrow, tid, DD2_THREADS);
    }
}
// pass 1 after its GEMM: G to global (bulk copies by one thread while the walks read the tile),
// the piece's transfer tuples; the tile is free again when this returns
template <class SY>
__device__ __forceinline__ void dd_p1_post(const DDStageArgs &a, double *T, const DDTask &t, int tid, SY sync,
                                           const DDWalkPre &wp) {
    double *G = a.gs + (t.task * a.n + t.r0) * (long long)DD_WMAX;
    PRS_CHECK((t.task * a.n + t.r0 + t.nrow) * (long long)DD_WMAX <= a.gs_end, "DD G tile outside the scratch");
    const bool bulk = (t.W & 1) == 0;  // rows of W doubles are 16-byte multiples
    if (bulk) {
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            for (int rl = 0; rl < t.nrow; ++rl)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                                 G + (long long)rl * DD_WMAX),
                             "r"(smem_u32(T + cpad(rl) * DD_WPAD)), "r"((unsigned)(t.W * sizeof(double)))
                             : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
    } else {
        const int lane = tid & 31;
        for (int rl = tid >> 5; rl < t.nrow; rl += DD2_THREADS / 32)
#pragma unroll
            for (int k = 0; k < (DD_WMAX + 31) / 32; ++k) {
                const int ci = lane + 32 * k;
                if (ci < t.W) G[(long long)rl * DD_WMAX + ci] = T[cpad(rl) * DD_WPAD + ci];
            }
    }
    dd_piece_walks<1>(a, T, t.blk, t.r0, t.nrow, t.tk, tid, wp);
    if (bulk && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    sync();
}
// pass 2 before its GEMM: G back (bulk copies completing on the group's mbarrier, phase `par`),
// the exact recurrences of the piece from its boundary values
template <class SY>
__device__ __forceinline__ void dd_p2_pre(const DDStageArgs &a, double *T, const DDTask &t, int tid, SY sync,
                                          unsigned long long *mbg, unsigned par) {
    const DDWalkPre wp = dd_walk_prefetch<0>(a, t.blk, t.tk, tid);  // in flight with the G copies
    const double *G = a.gs + (t.task * a.n + t.r0) * (long long)DD_WMAX;
    PRS_CHECK((t.task * a.n + t.r0 + t.nrow) * (long long)DD_WMAX <= a.gs_end, "DD G tile outside the scratch");
    PRS_CHECK(t.nrow <= DD_RMAX && t.W <= DD_WMAX, "DD tile shape");
    const bool bulk = (t.W & 1) == 0;
    const int lane = tid & 31;
    if (bulk && tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive_expect(mbg, (unsigned)(t.nrow * t.W * sizeof(double)));
        for (int rl = 0; rl < t.nrow; ++rl)
            bulk_g2s(T + cpad(rl) * DD_WPAD, G + (long long)rl * DD_WMAX, (unsigned)(t.W * sizeof(double)), mbg);
    }
    for (int rl = tid >> 5; rl < t.nrow; rl += DD2_THREADS / 32)
#pragma unroll
        for (int k = 0; k < (DD_WMAX + 31) / 32; ++k) {
            const int ci = lane + 32 * k;
            if (ci >= t.W && ci < DD_WMAX) T[cpad(rl) * DD_WPAD + ci] = 0.0;
            else if (!bulk && ci < t.W) T[cpad(rl) * DD_WPAD + ci] = G[(long long)rl * DD_WMAX + ci];
        }
    if (bulk) mbar_wait(mbg, par);
    sync();
    dd_piece_walks<0>(a, T, t.blk, t.r0, t.nrow, t.tk, tid, wp);
}
// pass 2 after its GEMM: store with the fused epilogue; the tile is free again when this returns
template <int DR, class SY>
__device__ __forceinline__ void dd_p2_post(const DDStageArgs &a, double *T, const DDTask &t, int tid, SY sync) {
    unsigned finm = 0;  // columns final after this stage (stage 1: all; stage 0: rho_1 = 0)
    {
        const double *rn_ot = a.rhon + (1 - a.stage) * a.n;
        const int i0 = a.bi0[t.blk], lane = tid & 31;
#pragma unroll
        for (int k = 0; k < (DD_WMAX + 31) / 32; ++k) {
            const int ci = lane + 32 * k;
            if (ci < t.W && (a.stage == 1 || !(rn_ot[i0 + ci] > 0.0))) finm |= 1u << k;
        }
    }
    if (a.bWs[t.blk] < t.W) {  // the GEMM's sync published the tile
        dd_fold_tile(T, t.W, t.nrow, tid, DD2_THREADS);
        sync();
    }
    dd_store_tile<DR, DD2_THREADS>(a, T, t.b, t.blk, t.r0, t.nrow, finm, tid);
    sync();
}

// One tile per CTA, two CTAs per SM: one CTA's loads, walks and stores overlap the other's GEMM.
template <int DR, int SRC, int PASS>
__global__ void __launch_bounds__(DD2_THREADS, 2) dd_pass_kernel(DDStageArgs a) {
    extern __shared__ double sh[];
    double *T = sh;
    __shared__ __align__(8) unsigned long long mbg;
    const int tid = threadIdx.x;
    const CtaSync sy{};
    if (PASS == 2 && tid == 0) {
        mbar_init(&mbg, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const DDTask t(a, blockIdx.x);
    DD2T0;
    if (PASS == 1) dd_p1_pre<DR, SRC>(a, T, t, tid, sy);
    else dd_p2_pre(a, T, t, tid, sy, &mbg, 0);
    DD2T(PASS == 1 ? 0 : 3);
    const DDWalkPre wp = PASS == 1 ? dd_walk_prefetch<1>(a, t.blk, t.tk, tid) : DDWalkPre{};
#ifdef PRS_DD_TIMING
    if (!(a.abl & 1))
#endif
    dd_tile_gemm2(T, (PASS == 1 ? a.Q : a.QT)[t.blk], t.W, a.bWs[t.blk], tid, sy);
    DD2T(PASS == 1 ? 1 : 4);
    if (PASS == 1) dd_p1_post(a, T, t, tid, sy, wp);
    else dd_p2_post<DR>(a, T, t, tid, sy);
    DD2T(PASS == 1 ? 2 : 5);
#ifdef PRS_DD_TIMING
    if (tid == 0) atomicAdd(&g_dd2_timing[PASS == 1 ? 7 : 8], 1ull);
#endif
}

// per (state, block, mode): y_in of every sub-piece forward, then x_in backward
__global__ void dd_scan_kernel(DDStageArgs a) {
    const long long task = blockIdx.x;
    const int am = threadIdx.x, W = a.bW[(int)(task % a.nblk)];
    if (am >= W) return;
    const int NS = 2 * a.CL;  // sub-pieces of the block
    const long long s0 = task * NS;
    constexpr int PB = 8;  // sub-pieces per batch: every load of a batch in flight together
    double y = 0.0;
    for (int p0 = 0; p0 < NS; p0 += PB) {
        double tA[PB], tB[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q)
            if (p0 + q < NS) {
                const double *t = a.tup + (s0 + p0 + q) * 5 * DD_WMAX + am;
                tA[q] = t[0];
                tB[q] = t[DD_WMAX];
            }
#pragma unroll
        for (int q = 0; q < PB; ++q)
            if (p0 + q < NS) {
                a.bnd[(s0 + p0 + q) * 2 * DD_WMAX + am] = y;
                y = fma(tA[q], y, tB[q]);
            }
    }
    double x = 0.0;
    for (int p1 = NS - 1; p1 >= 0; p1 -= PB) {
        double tP[PB], t0[PB], t1[PB], yi[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q)
            if (p1 - q >= 0) {
                const double *t = a.tup + (s0 + p1 - q) * 5 * DD_WMAX + am;
                tP[q] = t[2 * DD_WMAX];
                t0[q] = t[3 * DD_WMAX];
                t1[q] = t[4 * DD_WMAX];
                yi[q] = a.bnd[(s0 + p1 - q) * 2 * DD_WMAX + am];
            }
#pragma unroll
        for (int q = 0; q < PB; ++q)
            if (p1 - q >= 0) {
                a.bnd[((s0 + p1 - q) * 2 + 1) * DD_WMAX + am] = x;
                x = fma(tP[q], x, fma(t1[q], yi[q], t0[q]));
            }
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
    double *rhon = nullptr, *rhof = nullptr, *Z = nullptr;  // Z: Jacobi eigenvectors + refinement scratch
    bool refine = true;  // Newton refinement of the eigenbasis (PRS_DDREFINE=0: Jacobi only)
    std::vector<int> bi0[2], bW[2], bWs[2];  // bWs: W / 2 for a folded block (dd_fold_tile), else W
    int *d_bi0[2] = {nullptr, nullptr}, *d_bW[2] = {nullptr, nullptr}, *d_bWs[2] = {nullptr, nullptr};
    bool fold = true;  // split stage: mirror-symmetric even blocks folded (PRS_DDFOLD=0: never)
    // per tau slot (3) and colour (2): device arrays of per-block pointers + the storage
    double tau[3] = {-1.0, -1.0, -1.0};
    std::vector<double *> store[3];
    const double **d_Q[3][2] = {}, **d_QT[3][2] = {}, **d_idy[3][2] = {}, **d_conv[3][2] = {};
    // global-exchange stage launch (default; PRS_DDCL=1: clusters)
    bool gx = true;
    int num_sms = 148;
    int *gbuf = nullptr;        // [1 + 2 * gcap]: task counter, flags
    double2 *gtot = nullptr;    // [gcap][2][DD_WMAX]
    int gen = 0;                // bumped when exchange / split scratch is reallocated (captured graphs hold it)
    long long gcap = 0;
    // split stage (default; PRS_DDSPLIT=0: the single-kernel stage with the L2 exchange)
    bool split = true;
    bool two = true;            // split stage: the batch's two halves on two streams (PRS_DD2S=0: one)
    cudaStream_t st2 = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    double *gs = nullptr, *tup = nullptr, *bnd = nullptr;
    long long scap = 0;         // block-states (B x blocks) the split scratch holds
    // full diffusion tensor (coef_kind 2, ddfull.cuh): d tables and per (slot, colour) the
    // block-Thomas factors E_l^T, P_l^{-1} of every block
    bool full = false;
    double h = 0;
    double *dxf = nullptr, *dyf = nullptr;
    double **d_ET[3][2] = {}, **d_PI[3][2] = {};
    // partitioned application (dfpart.cuh, default; PRS_DFPART=0: df_stage_kernel): per (slot,
    // colour) A_p^T, Pp_p^T of every block; scratch tiles sized for dcap block-groups
    bool dfpart = true;
    double **d_AT[3][2] = {}, **d_PpT[3][2] = {};
    double *dfp_tl = nullptr, *dfp_by = nullptr, *dfp_bx = nullptr, *dfp_ys = nullptr;
    long long dcap = 0;
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
        cudaMalloc(&d.Z, sizeof(double) * (7 * DD_WMAX * DD_WMAX + 3 * DD_WMAX)) != cudaSuccess) {
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
    const char *spv = getenv("PRS_DDSPLIT");
    d.split = d.gx && !(spv && spv[0] == '0');
    const char *d2v = getenv("PRS_DD2S");
    d.two = !(d2v && d2v[0] == '0');
    const char *dpv = getenv("PRS_DFPART");
    d.dfpart = !(dpv && dpv[0] == '0');
    const char *rfv = getenv("PRS_DDREFINE");
    d.refine = !(rfv && rfv[0] == '0');
    const char *fdv = getenv("PRS_DDFOLD");
    d.fold = d.split && !d.full && !(fdv && fdv[0] == '0');
    {
        // folded blocks: W even, rho_j bitwise mirror-symmetric over the block's nodes and faces
        std::vector<double> hn(2 * d.n), hf(2 * (d.n + 1));
        cudaMemcpyAsync(hn.data(), d.rhon, sizeof(double) * hn.size(), cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(hf.data(), d.rhof, sizeof(double) * hf.size(), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        for (int col = 0; col < 2; ++col) {
            const size_t nb = d.bi0[col].size();
            d.bWs[col].assign(nb, 0);
            for (size_t k = 0; k < nb; ++k) {
                const int i0 = d.bi0[col][k], W = d.bW[col][k];
                bool sym = d.fold && (W % 2 == 0);
                for (int q = 0; sym && q < W; ++q) sym = hn[col * d.n + i0 + q] == hn[col * d.n + i0 + W - 1 - q];
                for (int q = 0; sym && q <= W; ++q)
                    sym = hf[col * (d.n + 1) + i0 + q] == hf[col * (d.n + 1) + i0 + W - q];
                d.bWs[col][k] = sym ? W / 2 : W;
            }
            if (cudaMalloc(&d.d_bWs[col], sizeof(int) * nb) != cudaSuccess) {
                err = "cudaMalloc (DD blocks) failed";
                return PRS_ECUDA;
            }
            cudaMemcpyAsync(d.d_bWs[col], d.bWs[col].data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st);
        }
    }
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
// Rows per partition of the partitioned full-tensor sweeps: DFP_M, shortened (not below 48) when
// that lets two state groups of a colour's blocks fill the SMs in one wave -- c5: 4 blocks x 2
// groups x 16 partitions of 64 rows = 128 CTAs on 148 SMs becomes 18 partitions of 57 = 144.
inline int dfp_rows(const DDData &d) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    const int nbmax = (int)std::max(d.bi0[0].size(), d.bi0[1].size());
    const int P0 = (d.n + DFP_M - 1) / DFP_M, P1 = nbmax > 0 ? sms / (2 * nbmax) : 0;
    if (P1 > P0) {
        const int M = (d.n + P1 - 1) / P1;
        if (M >= 48) return M;
    }
    return DFP_M;
}

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
        if (d.dfpart) {
            // the partition products A_p^T, Pp_p^T: the sweeps of dfpart.cuh on unit columns
            const int Mr = dfp_rows(d), P = (d.n + Mr - 1) / Mr;
            std::vector<double *> hA(nb), hPp(nb);
            for (size_t k = 0; k < nb; ++k) {
                const size_t bytes = sizeof(double) * (size_t)P * d.bW[col][k] * d.bW[col][k];
                if (cudaMalloc(&hA[k], bytes) != cudaSuccess || cudaMalloc(&hPp[k], bytes) != cudaSuccess) {
                    err = "cudaMalloc (full-tensor partition products) failed";
                    return PRS_ECUDA;
                }
                d.store[slot].insert(d.store[slot].end(), {hA[k], hPp[k]});
            }
            double **dA, **dPp;
            if (cudaMalloc(&dA, sizeof(double *) * nb) != cudaSuccess ||
                cudaMalloc(&dPp, sizeof(double *) * nb) != cudaSuccess) {
                err = "cudaMalloc (full-tensor pointer tables) failed";
                return PRS_ECUDA;
            }
            d.store[slot].insert(d.store[slot].end(), {(double *)dA, (double *)dPp});
            cudaMemcpyAsync(dA, hA.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
            cudaMemcpyAsync(dPp, hPp.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
            d.d_AT[slot][col] = dA;
            d.d_PpT[slot][col] = dPp;
            DFPArgs x{};
            x.n = d.n;
            x.nblk = (int)nb;
            x.ngrp = (DF_WMAX + DFP_S - 1) / DFP_S;  // unit columns in groups of DFP_S
            x.P = P;
            x.M = Mr;
            x.bi0 = d.d_bi0[col];
            x.bW = d.d_bW[col];
            x.ET = dE;
            x.PI = dP;
            x.tau = tau;
            x.op_me = df_op(d, col);
            x.op_ot = df_op(d, 1 - col);
            x.setup = 1;
            const unsigned grid = (unsigned)(nb * x.ngrp * P);
            const size_t s2 = sizeof(double) * (2 * DFP_HALF + 2 * DFP_TILE);  // matrix halves + 2 tiles
            cudaFuncSetAttribute(dfp_fwd_kernel<0, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
            cudaFuncSetAttribute(dfp_bwd_kernel<0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
            x.setup_out = dA;
            dfp_fwd_kernel<0, 0, 2><<<grid, DFP_T, s2, st>>>(x);
            x.setup_out = dPp;
            dfp_bwd_kernel<0, 2><<<grid, DFP_T, s2, st>>>(x);
        }
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
        std::vector<const double *> hQ(nb), hQT(nb), hI(nb), hC(nb);
        for (size_t k = 0; k < nb; ++k) {
            const int W = d.bW[col][k];
            double *Q, *QT, *th, *idy;
            if (cudaMalloc(&Q, sizeof(double) * W * W) != cudaSuccess ||
                cudaMalloc(&QT, sizeof(double) * W * W) != cudaSuccess ||
                cudaMalloc(&th, sizeof(double) * 2 * W) != cudaSuccess ||
                cudaMalloc(&idy, sizeof(double) * (size_t)W * d.n) != cudaSuccess) {
                err = "cudaMalloc (DD factors) failed";
                return PRS_ECUDA;
            }
            d.store[slot].insert(d.store[slot].end(), {Q, QT, th, idy});
            // one factorisation per block, or two (symmetric / antisymmetric half) per folded block
            const bool fold = d.bWs[col][k] < W;
            if (fold) {
                cudaMemsetAsync(Q, 0, sizeof(double) * W * W, st);
                cudaMemsetAsync(QT, 0, sizeof(double) * W * W, st);
            }
            constexpr size_t WW2 = (size_t)DD_WMAX * DD_WMAX;
            double *Zb = d.Z, *Xb = d.Z + 2 * WW2, *scr = d.Z + 3 * WW2;
            double *sd = d.Z + 7 * WW2, *se = sd + DD_WMAX, *sr = se + DD_WMAX;
            for (int f = fold ? 1 : 0; f <= (fold ? 2 : 0); ++f) {
                const int m = f ? W / 2 : W, moff = (f == 2) ? m : 0;
                dd_assemble_kernel<<<1, 256, 0, st>>>(d.bi0[col][k], W, f, d.rhon + col * d.n,
                                                      d.rhof + col * (d.n + 1), tau, d.h2inv, d.c, sd, se, sr);
                dd_factor_kernel<<<1, DD_FTHREADS, fsm, st>>>(d.n, m, sd, se, sr, tau * d.h2inv, W, moff, Zb, Xb, th,
                                                             idy, 14, d.refine ? 0 : 1);
                if (d.refine)
                    dd_refine_kernel<<<1, DD_FTHREADS, 0, st>>>(d.n, m, sd, se, sr, tau * d.h2inv, W, moff, scr, Xb,
                                                                th, idy);
                dd_place_kernel<<<64, 256, 0, st>>>(W, m, f, Xb, Q, QT);
            }
            hQ[k] = Q;
            hQT[k] = QT;
            hI[k] = idy;
            hC[k] = th + W;
        }
        const double **dq, **dqt, **di, **dc;
        if (cudaMalloc(&dq, sizeof(double *) * nb) != cudaSuccess ||
            cudaMalloc(&dqt, sizeof(double *) * nb) != cudaSuccess ||
            cudaMalloc(&di, sizeof(double *) * nb) != cudaSuccess ||
            cudaMalloc(&dc, sizeof(double *) * nb) != cudaSuccess) {
            err = "cudaMalloc (DD pointer tables) failed";
            return PRS_ECUDA;
        }
        d.store[slot].insert(d.store[slot].end(), {(double *)dq, (double *)dqt, (double *)di, (double *)dc});
        cudaMemcpyAsync(dq, hQ.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dqt, hQT.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(di, hI.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dc, hC.data(), sizeof(double *) * nb, cudaMemcpyHostToDevice, st);
        d.d_Q[slot][col] = dq;
        d.d_QT[slot][col] = dqt;
        d.d_idy[slot][col] = di;
        d.d_conv[slot][col] = dc;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        err = "DD factorisation failed";
        return PRS_ECUDA;
    }
    return PRS_OK;
}

inline void dd_free(DDData &d) {
    if (d.st2) cudaStreamDestroy(d.st2);
    for (auto e : d.ev)
        if (e) cudaEventDestroy(e);
    for (auto &v : d.store) {
        for (double *p : v) cudaFree(p);
        v.clear();
    }
    if (d.gbuf) cudaFree(d.gbuf);
    if (d.gtot) cudaFree(d.gtot);
    double *bufs[] = {d.rhon, d.rhof, d.Z, d.dxf, d.dyf, d.gs, d.tup, d.bnd, d.dfp_tl, d.dfp_by, d.dfp_bx, d.dfp_ys};
    for (double *p : bufs)
        if (p) cudaFree(p);
    for (int c = 0; c < 2; ++c) {
        if (d.d_bi0[c]) cudaFree(d.d_bi0[c]);
        if (d.d_bW[c]) cudaFree(d.d_bW[c]);
        if (d.d_bWs[c]) cudaFree(d.d_bWs[c]);
    }
}

// one DD step (two colour stages) on B states: in -> out
// algorithmic fp64 flops of one split-stage colour per state: per support point of a W-wide
// block two W x W transforms (2 W each) and the tridiagonal solve along y (~10); a folded block
// (dd_fold_tile) does two W/2 x W/2 transforms per half (2 W in all) plus the fold / unfold (2)
inline double dd_split_flops(const DDData &d, int stage) {
    double flops = 0.0;
    for (size_t k = 0; k < d.bW[stage].size(); ++k) {
        const double w = d.bW[stage][k];
        flops += w * d.n * ((d.bWs[stage][k] < d.bW[stage][k]) ? (2.0 * w + 12.0) : (4.0 * w + 10.0));
    }
    return flops;
}

inline int dd_step_impl(DDData &d, int scheme, int slot, const double *in, double *out, long long B,
                        const TimeArgs &ta, int epi, const double *gc, double *gcache, const double *delta,
                        double *traj, unsigned long long *red, cudaStream_t st, prs_ctx *prof, std::string &err,
                        long long &launches, double src_amp, int src, long long soff = 0, long long Btot = -1);

// one DD step (two colour stages) on B states: in -> out.  Split DD stage with a batch of at least
// two DD_HALFB groups: the two halves of the batch run on two streams (fork / join), so that the
// passes of one half (e.g. its GEMMs) meet the other half's loads and walks on the SMs instead
// of every CTA of a launch moving through the same phase at the same time
constexpr int DD_HALFB = 8;
inline int dd_step(DDData &d, int scheme, int slot, const double *in, double *out, long long B, const TimeArgs &ta,
                   int epi, const double *gc, double *gcache, const double *delta, double *traj,
                   unsigned long long *red, cudaStream_t st, prs_ctx *prof, std::string &err, long long &launches,
                   double src_amp, int src) {
    if (!(d.two && d.split && !d.full && B >= 2 * DD_HALFB))
        return dd_step_impl(d, scheme, slot, in, out, B, ta, epi, gc, gcache, delta, traj, red, st, prof, err,
                            launches, src_amp, src);
    if (!d.st2) {
        if (cudaStreamCreateWithFlags(&d.st2, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&d.ev[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&d.ev[1], cudaEventDisableTiming) != cudaSuccess) {
            err = "DD second stream";
            return PRS_ECUDA;
        }
    }
    const long long B1 = B / 2, B2 = B - B1;
    if (prof && prs_internal_prof_begin(prof) != PRS_OK) return PRS_ECUDA;
    if (cudaEventRecord(d.ev[0], st) != cudaSuccess || cudaStreamWaitEvent(d.st2, d.ev[0], 0) != cudaSuccess) {
        err = "DD fork";
        return PRS_ECUDA;
    }
    TimeArgs ta2 = ta;
    ta2.slice0 = ta.slice0 + B1 * ta.sstride;
    const long long vol = (long long)d.n * d.n;
    int rc = dd_step_impl(d, scheme, slot, in, out, B1, ta, epi, gc, gcache, delta, traj, red, st, nullptr, err,
                          launches, src_amp, src, 0, B);
    if (rc != PRS_OK) return rc;
    rc = dd_step_impl(d, scheme, slot, in + B1 * vol, out + B1 * vol, B2, ta2, epi, gc ? gc + B1 * vol : nullptr,
                      gcache, delta, traj, red, d.st2, nullptr, err, launches, src_amp, src, B1, B);
    if (rc != PRS_OK) return rc;
    if (cudaEventRecord(d.ev[1], d.st2) != cudaSuccess || cudaStreamWaitEvent(st, d.ev[1], 0) != cudaSuccess) {
        err = "DD join";
        return PRS_ECUDA;
    }
    if (prof) {
        const double flops = dd_split_flops(d, 0) + dd_split_flops(d, 1);
        // both colour stages of the step in one interval: accounted as two stage launches
        if (prs_internal_prof_end(prof, PRS_K_DD, (double)B * flops) != PRS_OK) return PRS_ECUDA;
    }
    return PRS_OK;
}

inline int dd_step_impl(DDData &d, int scheme, int slot, const double *in, double *out, long long B,
                        const TimeArgs &ta, int epi, const double *gc, double *gcache, const double *delta,
                        double *traj, unsigned long long *red, cudaStream_t st, prs_ctx *prof, std::string &err,
                        long long &launches, double src_amp, int src, long long soff, long long Btot) {
    const int n = d.n;
    if (Btot < 0) Btot = B;
    if (d.full && d.dfpart) {
        const int Mr = dfp_rows(d), P = (n + Mr - 1) / Mr, ngrp = (int)((B + DFP_S - 1) / DFP_S);
        const int nbmax = (int)std::max(d.bi0[0].size(), d.bi0[1].size());
        const long long bgs = (long long)nbmax * ngrp;
        if (bgs > d.dcap) {
            double *bufs[] = {d.dfp_tl, d.dfp_by, d.dfp_bx, d.dfp_ys};
            for (double *q : bufs)
                if (q) cudaFree(q);
            d.dfp_tl = d.dfp_by = d.dfp_bx = d.dfp_ys = nullptr;
            d.dcap = 0;
            const size_t tile = sizeof(double) * DF_WMAX * DFP_S;
            if (cudaMalloc(&d.dfp_tl, tile * bgs * P) != cudaSuccess ||
                cudaMalloc(&d.dfp_by, tile * bgs * P) != cudaSuccess ||
                cudaMalloc(&d.dfp_bx, tile * bgs * P) != cudaSuccess ||
                cudaMalloc(&d.dfp_ys, tile * bgs * n) != cudaSuccess) {
                err = "cudaMalloc (full-tensor partition scratch) failed";
                return PRS_ECUDA;
            }
            d.dcap = bgs;
            ++d.gen;
        }
        const size_t s2 = sizeof(double) * (2 * DFP_HALF + 2 * DFP_TILE), s3 = s2;  // matrix halves + 2 tiles
        for (int stage = 0; stage < 2; ++stage) {
            DFPArgs x{};
            x.U = in;
            x.V = out;
            x.vol = (long long)n * n;
            x.n = n;
            x.B = (int)B;
            x.stage = stage;
            x.nblk = (int)d.bi0[stage].size();
            x.ngrp = ngrp;
            x.P = P;
            x.M = Mr;
            x.bi0 = d.d_bi0[stage];
            x.bW = d.d_bW[stage];
            x.ET = d.d_ET[slot][stage];
            x.PI = d.d_PI[slot][stage];
            x.AT = d.d_AT[slot][stage];
            x.PpT = d.d_PpT[slot][stage];
            x.tau = d.tau[slot];
            x.c = d.c;
            x.op_me = df_op(d, stage);
            x.op_ot = df_op(d, 1 - stage);
            x.src_amp = src_amp;
            x.sinpi = d.sinpi;
            x.ta = ta;
            x.epi = epi;
            x.e_gc = gc;
            x.e_gcache = gcache;
            x.e_delta = delta;
            x.e_traj = traj;
            x.e_red = red;
            x.tl = d.dfp_tl;
            x.bnd_y = d.dfp_by;
            x.bnd_x = d.dfp_bx;
            x.ys = d.dfp_ys;
            void (*f0)(DFPArgs) = nullptr, (*f1)(DFPArgs) = nullptr, (*b0)(DFPArgs) = nullptr, (*b1)(DFPArgs) = nullptr;
            const int dr = scheme == PRS_DR;
#define DK(D, S_)                              \
    if (dr == D && src == S_) {                \
        f0 = dfp_fwd_kernel<D, S_, 0>;         \
        f1 = dfp_fwd_kernel<D, S_, 1>;         \
        b0 = dfp_bwd_kernel<D, 0>;             \
        b1 = dfp_bwd_kernel<D, 1>;             \
    }
            DK(0, 0) DK(0, 1) DK(1, 0) DK(1, 1)
#undef DK
            void (*fs[4])(DFPArgs) = {f0, f1, dfp_scan_kernel<1>, dfp_scan_kernel<0>};
            for (auto fk : fs) cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
            cudaFuncSetAttribute(b0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s3);
            cudaFuncSetAttribute(b1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s3);
            const unsigned grid = (unsigned)(x.nblk * ngrp * P), sgrid = (unsigned)(x.nblk * ngrp);
            if (prof && prs_internal_prof_begin(prof) != PRS_OK) return PRS_ECUDA;
            f0<<<grid, DFP_T, s2, st>>>(x);
            dfp_scan_kernel<1><<<sgrid, DFP_T, s2, st>>>(x);
            f1<<<grid, DFP_T, s2, st>>>(x);
            b0<<<grid, DFP_T, s3, st>>>(x);
            dfp_scan_kernel<0><<<sgrid, DFP_T, s2, st>>>(x);
            b1<<<grid, DFP_T, s3, st>>>(x);
            launches += 6;
            const cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) {
                err = std::string("full-tensor partitioned stage: ") + cudaGetErrorString(e);
                return PRS_ECUDA;
            }
            if (prof) {
                // algorithmic fp64 flops: the sequential block Thomas (two dense W x W mat-vecs per
                // block row and state); the partitioned form does twice this plus the scans
                double flops = 0.0;
                for (int w : d.bW[stage]) flops += (double)n * (4.0 * w * w + 20.0 * w);
                if (prs_internal_prof_end(prof, PRS_K_DD, (double)B * flops) != PRS_OK) return PRS_ECUDA;
            }
        }
        return PRS_OK;
    }
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
        a.bWs = d.d_bWs[stage];
        a.Q = d.d_Q[slot][stage];
        a.QT = d.d_QT[slot][stage];
        a.idy = d.d_idy[slot][stage];
        a.conv = d.d_conv[slot][stage];
#ifdef PRS_DD_TIMING
        a.abl = getenv("PRS_DD_ABL") ? atoi(getenv("PRS_DD_ABL")) : 0;
#endif
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
        if (d.split) {
            const long long ntot = Btot * a.nblk * CL;  // the whole batch's tasks (two-stream halves share)
            if (Btot * a.nblk > d.scap) {
                double *bufs[] = {d.gs, d.tup, d.bnd};
                for (double *p : bufs)
                    if (p) cudaFree(p);
                d.gs = d.tup = d.bnd = nullptr;
                d.scap = 0;
                if (cudaMalloc(&d.gs, sizeof(double) * DD_WMAX * (size_t)n * Btot * a.nblk) != cudaSuccess ||
                    cudaMalloc(&d.tup, sizeof(double) * 5 * DD_WMAX * 2 * ntot) != cudaSuccess ||
                    cudaMalloc(&d.bnd, sizeof(double) * 2 * DD_WMAX * 2 * ntot) != cudaSuccess) {
                    err = "cudaMalloc (DD split scratch) failed";
                    return PRS_ECUDA;
                }
                d.scap = Btot * a.nblk;
                ++d.gen;
            }
            // (a second half of the batch takes the scratch after the first half's)
            const long long toff = soff * a.nblk * CL;
            a.gs = d.gs + (size_t)DD_WMAX * n * soff * a.nblk;
            a.tup = d.tup + (size_t)5 * DD_WMAX * 2 * toff;
            a.bnd = d.bnd + (size_t)2 * DD_WMAX * 2 * toff;
            a.gs_end = (long long)DD_WMAX * n * (d.scap - soff * a.nblk);
            a.tup_end = (long long)5 * DD_WMAX * 2 * (d.scap * CL - toff);
            a.bnd_end = (long long)2 * DD_WMAX * 2 * (d.scap * CL - toff);
            a.ntasks = (int)ntasks;
            void (*k1)(DDStageArgs) = nullptr, (*k2)(DDStageArgs) = nullptr;
            const int dr = scheme == PRS_DR;
#define DK(D, S_)                     \
    if (dr == D && src == S_) {       \
        k1 = dd_pass_kernel<D, S_, 1>; \
        k2 = dd_pass_kernel<D, S_, 2>; \
    }
            DK(0, 0) DK(0, 1) DK(1, 0) DK(1, 1)
#undef DK
            const size_t shm2 = sizeof(double) * (size_t)(cpad(DD_RMAX - 1) + 1) * DD_WPAD;  // the tile only
            if (cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm2) != cudaSuccess ||
                cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm2) != cudaSuccess) {
                err = "cudaFuncSetAttribute(dd split passes) failed";
                return PRS_ECUDA;
            }
            const unsigned nthr = DD2_THREADS, grid = (unsigned)ntasks;
            if (prof && prs_internal_prof_begin(prof) != PRS_OK) return PRS_ECUDA;
            void (*ks[3])(DDStageArgs) = {k1, dd_scan_kernel, k2};
            for (int q = 0; q < 3; ++q) {
                if (q == 1) dd_scan_kernel<<<(unsigned)(B * a.nblk), DD_WMAX, 0, st>>>(a);
                else ks[q]<<<grid, nthr, shm2, st>>>(a);
                launches++;
                const cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) {
                    cudaFuncAttributes fa{};
                    cudaFuncGetAttributes(&fa, ks[q]);
                    err = std::string("dd split stage, launch ") + std::to_string(q) + ": " + cudaGetErrorString(e) +
                          " (regs " + std::to_string(fa.numRegs) + ", max threads " +
                          std::to_string(fa.maxThreadsPerBlock) + ", static smem " + std::to_string(fa.sharedSizeBytes) +
                          ", dynamic " + std::to_string(q == 1 ? 0 : shm2) + ", threads " +
                          std::to_string(q == 1 ? DD_WMAX : (int)nthr) + ")";
                    return PRS_ECUDA;
                }
            }
            if (prof && prs_internal_prof_end(prof, PRS_K_DD, (double)B * dd_split_flops(d, stage)) != PRS_OK)
                return PRS_ECUDA;
            continue;
        }
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
