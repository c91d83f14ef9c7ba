// ddfull.cuh -- DD stage solves for the FULL diffusion tensor of PAPER.md:520-546 (section 5.2,
// SURVEY.md 8(f) NEXT-3):  d11 = d22 = 1 / (2 + cos(3 pi x) cos(2 pi y)), d12 = 1/4.
//
// Operator (R21, R22; PAPER.md:133 L_j u = div(rho_j D grad u) - rho_j c u): conservative
// face fluxes on the 3 x 3 stencil -- x faces d11 (u_{i+1} - u_i)/h weighted by rho_j(face),
// y faces d22 (u_{l+1} - u_l)/h weighted by rho_j(node), the mixed parts as means over the
// face's two corners of d12 times the corner difference, each corner weighted by rho_j at its
// x.  Collected per node (0-based i, l; rxm, rxp = rho_j at the left / right x face, rn at the node):
//     cf[+-1][0]  = r_x+- d11(x face, y_l) / h^2,   cf[0][+-1] = rn d22(x_i, y face) / h^2,
//     cf[+1][+1] = -cf[+1][-1] = rxp d12 / (2 h^2),   cf[-1][-1] = -cf[-1][+1] = rxm d12 / (2 h^2),
//     cf[0][0]   = -(sum of the four face coefficients) - rn c     (the mixed parts cancel there).
// Colour j's stage matrix I - tau A_j is block diagonal: one block per strip of its support,
// identity elsewhere (the corner and face weights vanish together at a block's edge, R22), as
// in the kappa = 1 case (dd.cuh).  A block (W columns x n rows) is block tridiagonal over rows,
//     D_l u_l + B_l u_{l-1} + C_l u_{l+1} = r_l,   D, B, C tridiagonal W x W,
// and symmetric positive definite (B_l = C_{l-1}^T), so block Thomas without pivoting is stable:
//     P_0 = D_0,  E_l = B_l P_{l-1}^{-1},  P_l = D_l - E_l C_{l-1}            (setup, per tau)
//     y_0 = r_0,  y_l = r_l - E_l y_{l-1};   x_{n-1} = P_{n-1}^{-1} y_{n-1},
//     x_l = P_l^{-1} (y_l - C_l x_{l+1})                                       (per right-hand side)
// The setup stores E_l (transposed) and P_l^{-1} (symmetric) per row: 2 n W^2 doubles per block
// and tau.  The solve runs one CTA per (block, state): per row two dense W x W mat-vecs whose
// matrices stream from L2 (the CTAs of one block read the same rows at about the same time),
// 576 threads = 4 partial sums per output for loads in flight.  Stage logic and the fused
// parareal epilogues are those of dd.cuh.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "lpass.cuh"

namespace prs {

constexpr int DF_WMAX = 144;
constexpr int DF_KQ = 4;                    // partial sums per output of a mat-vec
constexpr int DF_THREADS = DF_WMAX * DF_KQ; // 576
constexpr int DF_FTHREADS = 512;

// d11 = d22 of section 5.2 at a physical point
__device__ __forceinline__ double df_diag(double x, double y) {
    return 1.0 / (2.0 + cos(3.0 * 3.14159265358979323846 * x) * cos(2.0 * 3.14159265358979323846 * y));
}
// dxf[l * (n+1) + f] = d(x = (f + 1/2) h, y = (l + 1) h)   (x faces, f = 0..n)
// dyf[f * n + i]     = d(x = (i + 1) h, y = (f + 1/2) h)   (y faces, f = 0..n)
__global__ void df_tables(int n, double h, double *dxf, double *dyf) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long tot = (long long)n * (n + 1);
    if (e >= tot) return;
    {
        const int l = (int)(e / (n + 1)), f = (int)(e % (n + 1));
        dxf[e] = df_diag(((double)f + 0.5) * h, (double)(l + 1) * h);
    }
    {
        const int f = (int)(e / n), i = (int)(e % n);
        dyf[e] = df_diag((double)(i + 1) * h, ((double)f + 0.5) * h);
    }
}

struct DFOp {
    int n;
    double h2inv, c;
    const double *rhon, *rhof;  // rho_j at nodes (n), faces (n + 1)
    const double *dxf, *dyf;
    // the nine coefficients of A_j at node (i, l): cf[di + 1][dl + 1]
    __device__ __forceinline__ void stencil(int i, int l, double cf[3][3]) const {
        const double rxm = rhof[i], rxp = rhof[i + 1], rn = rhon[i];
        const double axm = rxm * dxf[(long long)l * (n + 1) + i] * h2inv;
        const double axp = rxp * dxf[(long long)l * (n + 1) + i + 1] * h2inv;
        const double aym = rn * dyf[(long long)l * n + i] * h2inv;
        const double ayp = rn * dyf[(long long)(l + 1) * n + i] * h2inv;
        const double gp = rxp * 0.125 * h2inv, gm = rxm * 0.125 * h2inv;  // rho d12 / (2 h^2)
        cf[0][1] = axm;
        cf[2][1] = axp;
        cf[1][0] = aym;
        cf[1][2] = ayp;
        cf[2][2] = gp;
        cf[2][0] = -gp;
        cf[0][0] = gm;
        cf[0][2] = -gm;
        cf[1][1] = -(axm + axp + aym + ayp) - rn * c;
    }
    // only the row-(l+1) coefficients (the C_l block): di = -1, 0, +1
    __device__ __forceinline__ void up(int i, int l, double &cm, double &c0, double &cp) const {
        const double rxm = rhof[i], rxp = rhof[i + 1], rn = rhon[i];
        c0 = rn * dyf[(long long)(l + 1) * n + i] * h2inv;
        cp = rxp * 0.125 * h2inv;
        cm = -rxm * 0.125 * h2inv;
    }
};

// ------------------------------------------------------------ setup (one CTA per block)
// Sequential over rows: E_l = B_l P_{l-1}^{-1} (to global, transposed), P_l = D_l - E_l C_{l-1}
// in shared memory, inverted in place by Gauss-Jordan without pivoting (SPD), P_l^{-1} to global.
__global__ void __launch_bounds__(DF_FTHREADS) df_factor_kernel(DFOp op, const int *bi0, const int *bW, double tau,
                                                                double *const *ETs, double *const *PIs) {
    extern __shared__ double S[];        // W x W
    const int i0 = bi0[blockIdx.x], W = bW[blockIdx.x];
    double *ET = ETs[blockIdx.x], *PI = PIs[blockIdx.x];
    double *rk = S + W * W, *ck = rk + DF_WMAX;
    const int tid = threadIdx.x, n = op.n;
    const long long WW = (long long)W * W;
    for (int l = 0; l < n; ++l) {
        if (l > 0) {
            // E_l[i][k] = sum_di B_l[i][i+di] Pinv_{l-1}[i+di][k], B_l[i][i+di] = -tau cf_{i,l}[di][-1]
            double *E = ET + (long long)l * WW;  // stored transposed: E[k * W + i]
            for (int e = tid; e < W * W; e += blockDim.x) {
                const int i = e / W, k = e % W;
                double cf[3][3];
                op.stencil(i0 + i, l, cf);
                double s = 0.0;
#pragma unroll
                for (int di = -1; di <= 1; ++di) {
                    const int ii = i + di;
                    if (ii < 0 || ii >= W) continue;
                    s = fma(-tau * cf[di + 1][0], S[ii * W + k], s);
                }
                E[(long long)k * W + i] = s;
            }
            __syncthreads();  // E_l written (visible to the block), S free
            // P_l = D_l - E_l C_{l-1},  C_{l-1}[k'][k] = -tau cf_{k',l-1}[k - k'][+1]
            for (int e = tid; e < W * W; e += blockDim.x) {
                const int i = e / W, k = e % W;
                double s = 0.0;
#pragma unroll
                for (int dk = -1; dk <= 1; ++dk) {
                    const int kk = k + dk;  // row of C_{l-1} (column of E_l)
                    if (kk < 0 || kk >= W) continue;
                    double cm, c0, cp;
                    op.up(i0 + kk, l - 1, cm, c0, cp);
                    const double cv = (dk == 0) ? c0 : (dk == 1 ? cm : cp);  // C[kk][k], k = kk - dk
                    s = fma(E[(long long)kk * W + i], -tau * cv, s);
                }
                double d = 0.0;
                if (k >= i - 1 && k <= i + 1) {
                    double cf[3][3];
                    op.stencil(i0 + i, l, cf);
                    d = (k == i ? 1.0 : 0.0) - tau * cf[k - i + 1][1];
                }
                S[e] = d - s;
            }
        } else {
            for (int e = tid; e < W * W; e += blockDim.x) {
                const int i = e / W, k = e % W;
                double d = 0.0;
                if (k >= i - 1 && k <= i + 1) {
                    double cf[3][3];
                    op.stencil(i0 + i, 0, cf);
                    d = (k == i ? 1.0 : 0.0) - tau * cf[k - i + 1][1];
                }
                S[e] = d;
            }
        }
        __syncthreads();
        // in-place Gauss-Jordan inversion (no pivoting: P_l is SPD)
        for (int k = 0; k < W; ++k) {
            const double piv = S[k * W + k];
            for (int j = tid; j < W; j += blockDim.x) {
                rk[j] = S[k * W + j] / piv;
                ck[j] = S[j * W + k];
            }
            __syncthreads();
            for (int e = tid; e < W * W; e += blockDim.x) {
                const int i = e / W, j = e % W;
                if (i == k && j == k) S[e] = 1.0 / piv;
                else if (i == k) S[e] = rk[j];
                else if (j == k) S[e] = -ck[i] / piv;
                else S[e] = fma(-ck[i], rk[j], S[e]);
            }
            __syncthreads();
        }
        double *P = PI + (long long)l * WW;
        for (int e = tid; e < W * W; e += blockDim.x) P[e] = S[e];
        __syncthreads();
    }
}

inline size_t df_factor_smem_bytes(int W) { return sizeof(double) * ((size_t)W * W + 2 * DF_WMAX); }

// ------------------------------------------------------------ stage (one CTA per block x state)
struct DFStageArgs {
    const double *U;
    double *V;
    long long vol;
    int n, B, stage, nblk;
    const int *bi0, *bW;
    const double *const *ET, *const *PI;  // per block of this colour
    double tau, c;
    DFOp op_me, op_ot;                    // this colour's operator, the other colour's (DR w)
    double src_amp;
    const double *sinpi;
    TimeArgs ta;
    int epi;
    const double *e_gc;
    double *e_gcache;
    const double *e_delta;
    double *e_traj;
    unsigned long long *e_red;
};

// y[i] (i < W) = base[i] - sign * sum_k M[k * W + i] x[k]; 576 threads = 4 partial sums per i
__device__ __forceinline__ void df_matvec(const double *__restrict__ M, const double *x, int W, double *part) {
    const int t = threadIdx.x, i = t % DF_WMAX, q = t / DF_WMAX;
    double s = 0.0;
    if (i < W) {
        const int kq = (W + DF_KQ - 1) / DF_KQ, k0 = q * kq, k1 = min(W, k0 + kq);
        int k = k0;
        for (; k + 8 <= k1; k += 8) {
            double m[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) m[u] = __ldg(M + (long long)(k + u) * W + i);
#pragma unroll
            for (int u = 0; u < 8; ++u) s = fma(m[u], x[k + u], s);
        }
        for (; k < k1; ++k) s = fma(__ldg(M + (long long)k * W + i), x[k], s);
    }
    part[q * DF_WMAX + i] = s;
}

template <int DR, int SRC>
__global__ void __launch_bounds__(DF_THREADS, 1) df_stage_kernel(DFStageArgs a) {
    __shared__ double xs[2][DF_WMAX];     // y_{l-1} / x_{l+1}
    __shared__ double part[DF_KQ * DF_WMAX];
    __shared__ double ts[DF_WMAX];
    const int tid = threadIdx.x;
    const int blk = (int)(blockIdx.x % a.nblk);
    const long long b = blockIdx.x / a.nblk;
    const int i0 = a.bi0[blk], W = a.bW[blk], n = a.n;
    const double *ET = a.ET[blk], *PI = a.PI[blk];
    const double *Ub = a.U + b * a.vol;
    double *Vb = a.V + b * a.vol;
    const int me = a.stage;
    const long long WW = (long long)W * W;
    double ampt = 0.0;
    if (SRC) ampt = a.src_amp * src_tf(a.ta, b);
    // column constants of thread i (< W): is the column final after stage 0 (rho_other = 0)?
    const int ci = tid;  // owner of column ci for the scalar work (tid < W)
    const bool col = ci < W;
    const int gi = i0 + (col ? ci : 0);
    const bool pos_ot = col && a.op_ot.rhon[gi] > 0.0;       // other colour present here
    const bool done0 = (me == 1) && pos_ot;                  // stage 1: final after stage 0
    const bool final_here = col && (me == 1 || !pos_ot);
    // w = tau A_ot U at (gi, l) (DR stage 0: the other colour's explicit term)
    auto wterm = [&](int l) {
        double cf[3][3];
        a.op_ot.stencil(gi, l, cf);
        double s = 0.0;
#pragma unroll
        for (int dl = -1; dl <= 1; ++dl) {
            const int ll = l + dl;
            if (ll < 0 || ll >= n) continue;
#pragma unroll
            for (int di = -1; di <= 1; ++di) {
                const int ii = gi + di;
                if (ii < 0 || ii >= n) continue;
                s = fma(cf[di + 1][dl + 1], Ub[(long long)ll * n + ii], s);
            }
        }
        return a.tau * s;
    };
    // ---- forward: y_l = r_l - E_l y_{l-1}, y_l stored in V ----
    for (int l = 0; l < n; ++l) {
        double r = 0.0;
        if (col) {
            const long long g = (long long)l * n + gi;
            if (done0) {
                r = Vb[g];
            } else {
                r = Ub[g];
                if (SRC) r = fma(a.tau * ampt * __ldg(a.sinpi + l), __ldg(a.sinpi + gi), r);
                if (DR && me == 0) r += wterm(l);
            }
        }
        if (l > 0) {
            df_matvec(ET + (long long)l * WW, xs[(l - 1) & 1], W, part);
            __syncthreads();
        }
        if (col) {
            double s = r;
            if (l > 0)
#pragma unroll
                for (int q = 0; q < DF_KQ; ++q) s -= part[q * DF_WMAX + ci];
            xs[l & 1][ci] = s;
            Vb[(long long)l * n + gi] = s;
        }
        __syncthreads();
    }
    // ---- backward: x_l = P_l^{-1} (y_l - C_l x_{l+1}) ----
    double dmax = 0.0;
    unsigned long long bad = 0;
    for (int l = n - 1; l >= 0; --l) {
        const double *xn = xs[(l + 1) & 1];  // x_{l+1} (unused at l = n - 1)
        if (col) {
            const long long g = (long long)l * n + gi;
            double t = Vb[g];
            if (l < n - 1) {
                double cm, c0, cp;
                a.op_me.up(gi, l, cm, c0, cp);
                double s = c0 * xn[ci];
                if (ci > 0) s = fma(cm, xn[ci - 1], s);
                if (ci + 1 < W) s = fma(cp, xn[ci + 1], s);
                t = fma(a.tau, s, t);  // y - C x with C = -tau (coefficients)
            }
            ts[ci] = t;
        }
        __syncthreads();
        df_matvec(PI + (long long)l * WW, ts, W, part);
        __syncthreads();
        if (col) {
            double x = 0.0;
#pragma unroll
            for (int q = 0; q < DF_KQ; ++q) x += part[q * DF_WMAX + ci];
            xs[l & 1][ci] = x;
            const long long g = (long long)l * n + gi;
            if (DR && me == 0) x -= wterm(l);
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
        __syncthreads();
    }
    if (a.epi == EPI_CORRECT) {
        const int lane = tid & 31;
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

}  // namespace prs
