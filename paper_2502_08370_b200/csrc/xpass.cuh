// xpass.cuh -- line solves along the contiguous axis x, with the stage-1 right-hand side fused
// into the load:
//   FIE  r = U_n + tau F(t_{n+1})
//   DR   w = tau A_2 U_n,  r = U_n + w + tau F(t_{n+1}),
//        output U_{n,1} - w  (the right-hand side of stage 2)   (M = 2)
// One CTA holds lpb lines (P threads each, LCH elements per thread) in shared memory; the
// state is read and written once with 16-byte vectors, the DR stencil's neighbour rows come
// from L2, and w stays in registers between the load and the store (same thread <-> element
// mapping in both phases).
#pragma once
#include "common.cuh"

namespace prs {

struct XArgs {
    const double *in;
    double *out;
    long long vol;        // points per state
    int n;                // line length
    int lines_per_state;  // n^(dim-1)
    long long nlines;     // batch * lines_per_state
    int P;                // threads per line (power of two, P * LCH >= n)
    int S;                // shared-memory stride per line (odd)
    int St;               // shared-memory stride per coefficient table (odd)
    int dim;
    double tau, h2inv, creact;  // creact = c / M
    double src_amp;             // (dim pi^2 + c - 1)
    const double *sinpi;        // sin(pi x_i)
    TimeArgs ta;
    CoefTab tab;                     // COEF == 0
    const double *invd, *s2n, *s2f;  // COEF == 1 (2-D)
};

inline size_t xpass_smem_doubles(int lpb, int S, int St, int coef, int threads) {
    const size_t body = (size_t)(1 + coef) * lpb * S + (coef ? (size_t)St : 3 * (size_t)St);
    return even_up(body) + 2 * (size_t)(threads / 32 + 1);
}

template <int COEF, int DR, int SRC>
__global__ void __launch_bounds__(256) xpass_kernel(XArgs a) {
    extern __shared__ double smem[];
    const int P = a.P, n = a.n;
    const int lpb = blockDim.x / P;
    const int lb = threadIdx.x / P, t = threadIdx.x - lb * P;
    const long long line = (long long)blockIdx.x * lpb + lb;
    const bool active = line < a.nlines;
    double *sr = smem + (size_t)lb * a.S;
    double *sd = smem + (size_t)(lpb + lb) * a.S;
    double *tabs = smem + (size_t)(1 + COEF) * lpb * a.S;
    double2 *scr = reinterpret_cast<double2 *>(
        smem + even_up((size_t)(1 + COEF) * lpb * a.S + (COEF ? (size_t)a.St : 3 * (size_t)a.St)));
    if (COEF) {
        stage_table(tabs, a.s2f, n + 1);
    } else {
        stage_table(tabs, a.tab.m, n);
        stage_table(tabs + a.St, a.tab.id, n);
        stage_table(tabs + 2 * a.St, a.tab.cc, n);
    }

    long long b = 0;
    int j = 0;
    if (active) {
        b = line / a.lines_per_state;
        j = (int)(line - b * a.lines_per_state);
    }
    const double *uin = a.in + b * a.vol + (long long)j * n;
    const int jy = (a.dim == 2) ? j : (j % n);  // y index of this x-line

    // ---- load + fused stage-1 right-hand side ----
    double ampt = 0.0, sj = 0.0;
    if (SRC && active) {
        ampt = a.src_amp * src_tf(a.ta, b);
        sj = (a.dim == 2) ? a.sinpi[j] : a.sinpi[j % n] * a.sinpi[j / n];
    }
    const bool has_m = j > 0, has_p = j < n - 1;
    const double *dinv = COEF ? a.invd + (long long)jy * n : nullptr;
    double kfm = 0.0, kfp = 0.0;  // y-face sines of this row (DR stencil, variable kappa)
    if (DR && COEF && active) {
        kfm = __ldg(a.s2f + j);
        kfp = __ldg(a.s2f + j + 1);
    }
    double Wr[LCH];
#pragma unroll
    for (int i = 0; i < LCH; ++i) Wr[i] = 0.0;
    auto emit = [&](int e, double u, double um, double up, double dv) -> double {
        double rhs = u, w = 0.0;
        if (DR) {  // 2-D only: w = tau A_y U_n (y-term of the dimensional split, c/2 share)
            double km = 1.0, kp = 1.0;
            if (COEF) {
                const double sx = __ldg(a.s2n + e);
                km = 1.0 + 0.5 * sx * kfm;
                kp = 1.0 + 0.5 * sx * kfp;
            }
            w = a.tau * ((kp * (up - u) - km * (u - um)) * a.h2inv - a.creact * u);
            rhs += w;
        }
        if (SRC) rhs += a.tau * (ampt * __ldg(a.sinpi + e) * sj);
        sr[cpad(e)] = rhs;
        if (COEF) sd[cpad(e)] = dv;
        return w;
    };
    const bool vec = (n & 1) == 0;
    if (active) {
        if (vec) {  // 16-byte vectors: pairs k = t + q P
#pragma unroll
            for (int g = 0; g < LCH / 2; g += QG) {
                double2 U[QG], UM[QG], UP[QG], D[QG];
#pragma unroll
                for (int q = 0; q < QG; ++q) {
                    const int k = t + (g + q) * P;
                    if (2 * k < n) {
                        U[q] = ld2(uin + 2 * k);
                        if (DR) {
                            UM[q] = has_m ? ld2(uin - n + 2 * k) : make_double2(0.0, 0.0);
                            UP[q] = has_p ? ld2(uin + n + 2 * k) : make_double2(0.0, 0.0);
                        }
                        if (COEF) D[q] = ld2(dinv + 2 * k);
                    }
                }
#pragma unroll
                for (int q = 0; q < QG; ++q) {
                    const int k = t + (g + q) * P;
                    if (2 * k < n) {
                        Wr[2 * (g + q)] = emit(2 * k, U[q].x, DR ? UM[q].x : 0.0, DR ? UP[q].x : 0.0,
                                               COEF ? D[q].x : 0.0);
                        Wr[2 * (g + q) + 1] = emit(2 * k + 1, U[q].y, DR ? UM[q].y : 0.0,
                                                   DR ? UP[q].y : 0.0, COEF ? D[q].y : 0.0);
                    }
                }
            }
        } else {
#pragma unroll
            for (int g = 0; g < LCH; g += 2 * QG) {
                double U[2 * QG], UM[2 * QG], UP[2 * QG], D[2 * QG];
#pragma unroll
                for (int q = 0; q < 2 * QG; ++q) {
                    const int e = t + (g + q) * P;
                    if (e < n) {
                        U[q] = uin[e];
                        if (DR) {
                            UM[q] = has_m ? uin[e - n] : 0.0;
                            UP[q] = has_p ? uin[e + n] : 0.0;
                        }
                        if (COEF) D[q] = dinv[e];
                    }
                }
#pragma unroll
                for (int q = 0; q < 2 * QG; ++q) {
                    const int e = t + (g + q) * P;
                    if (e < n) Wr[g + q] = emit(e, U[q], DR ? UM[q] : 0.0, DR ? UP[q] : 0.0, COEF ? D[q] : 0.0);
                }
            }
        }
    }
    __syncthreads();

    // ---- chunk-parallel Thomas ----
    const int e0 = t * LCH;
    const int cnt = active ? max(0, min(LCH, n - e0)) : 0;
    const bool full = n == P * LCH;  // kernel-uniform: every chunk of every line is complete
    const int lane = threadIdx.x & 31;
    const int Wd = P < 32 ? P : 32;
    const int tl = lane & (Wd - 1);
    double *sp = sr + t * LCP;
    const int co = t * LCP;
    ConstView cv0{tabs + co, tabs + a.St + co, tabs + 2 * a.St + co};
    VarView cv1{sd + co, tabs + co, 0.5 * ((COEF && active) ? __ldg(a.s2n + jy) : 0.0), -a.tau * a.h2inv,
                (COEF && t > 0) ? sd[co - 2] : 0.0};

    double A, B, EA, EB;
    if (COEF) walk_f1_any(full, sp, cnt, cv1, A, B);
    else walk_f1_any(full, sp, cnt, cv0, A, B);
    seg_scan_fwd(A, B, Wd, tl, EA, EB);
    double Yw = 0.0;
    if (P > 32) {
        const int warp = threadIdx.x >> 5, wib = t >> 5, wl0 = warp - wib;
        if (lane == 31) scr[warp] = make_double2(A, B);
        __syncthreads();
        for (int q = 0; q < wib; ++q) {
            const double2 v = scr[wl0 + q];
            Yw = v.x * Yw + v.y;
        }
        __syncthreads();
    }
    double Pb, Qb, EP, EQ;
    if (COEF) walk_f3_any(full, sp, cnt, cv1, fma(EA, Yw, EB), Pb, Qb);
    else walk_f3_any(full, sp, cnt, cv0, fma(EA, Yw, EB), Pb, Qb);
    seg_scan_bwd(Pb, Qb, Wd, tl, EP, EQ);
    double Xw = 0.0;
    if (P > 32) {
        const int warp = threadIdx.x >> 5, wib = t >> 5, wl0 = warp - wib, nwl = P >> 5;
        if (lane == 0) scr[warp] = make_double2(Pb, Qb);
        __syncthreads();
        for (int q = nwl - 1; q > wib; --q) {
            const double2 v = scr[wl0 + q];
            Xw = v.x * Xw + v.y;
        }
    }
    if (COEF) walk_b3_any(full, sp, cnt, cv1, fma(EP, Xw, EQ));
    else walk_b3_any(full, sp, cnt, cv0, fma(EP, Xw, EQ));
    __syncthreads();

    // ---- store (DR: subtract w kept in registers) ----
    if (active) {
        double *uout = a.out + b * a.vol + (long long)j * n;
        if (vec) {
#pragma unroll
            for (int q = 0; q < LCH / 2; ++q) {
                const int k = t + q * P;
                if (2 * k < n) st2(uout + 2 * k, sr[cpad(2 * k)] - Wr[2 * q], sr[cpad(2 * k + 1)] - Wr[2 * q + 1]);
            }
        } else {
#pragma unroll
            for (int q = 0; q < LCH; ++q) {
                const int e = t + q * P;
                if (e < n) uout[e] = sr[cpad(e)] - Wr[q];
            }
        }
    }
}

}  // namespace prs
