// lpass.cuh -- line solves along a strided axis (y, or z in 3-D).  A CTA holds PW adjacent
// columns (coalesced PW*8-byte row segments) of R rows in shared memory; lines longer than
// 32*LCH rows are split over a thread-block cluster whose CTAs exchange their per-column
// affine compositions through distributed shared memory (2 cluster barriers).  The epilogue
// fuses the parareal bookkeeping:
//   EPI_DELTA   Delta_n = F^s(U^k_n) - G(U^k_n)                   (last fine step)
//   EPI_CORRECT U^{k+1}_{n+1} = G(U^{k+1}_n) + Delta_n, G cache <- G(U^{k+1}_n),
//               max |U^{k+1}_{n+1} - U^k_{n+1}| and a non-finite flag (coarse chain)
//   EPI_INIT    U^0_{n+1} = G(U^0_n), G cache <- U^0_{n+1}           (initial guess)
#pragma once
#include "common.cuh"

namespace prs {

enum Epi { EPI_STORE = 0, EPI_DELTA = 1, EPI_CORRECT = 2, EPI_INIT = 3 };

struct LArgs {
    const double *in;
    double *out;
    long long vol;
    int n;
    long long Sl;        // element stride along the line
    int nq;              // planes per state (2-D: 1; 3-D: n)
    long long Sq;        // stride between planes
    int nwb;             // column blocks per plane, ceil(n / PW)
    long long npanels;   // batch * nq * nwb
    int CL;              // CTAs per panel (cluster size)
    int R;               // rows per CTA (multiple of LCH unless CL == 1)
    int CP;              // chunks per column (power of two <= 32), CP * LCH >= R
    int S;               // shared-memory stride per column (odd)
    int St;              // shared-memory stride per coefficient table (odd)
    double tau, h2inv;
    CoefTab tab;
    const double *invd, *s2n, *s2f;  // COEF == 1 (2-D y-lines)
    // epilogue operands (single-state for CORRECT / INIT; batch for DELTA)
    const double *e_gc;     // DELTA: G cache (batch)
    double *e_gcache;       // CORRECT/INIT: G cache slot of this slice
    const double *e_delta;  // CORRECT: Delta_n
    double *e_traj;         // CORRECT/INIT: U_{n+1}
    unsigned long long *e_red;  // CORRECT: [0] max |update| bits, [1] non-finite flag
};

inline size_t lpass_smem_doubles(int PWc, int S, int St, int coef) {
    const size_t body = (size_t)(1 + coef) * PWc * S + (coef ? (size_t)St : 3 * (size_t)St);
    return even_up(body) + 2 * 2 * (size_t)PWc;
}

template <int PW, int COEF, int EPI>
__global__ void __launch_bounds__(512) lpass_kernel(LArgs a) {
    extern __shared__ double smem[];
    constexpr int PH = PW / 2;  // 16-byte pairs per row segment
    const int CP = a.CP, n = a.n;
    const int crank = (a.CL > 1) ? (int)cg::this_cluster().block_rank() : 0;
    const long long panel = blockIdx.x / a.CL;
    const int wb = (int)(panel % a.nwb);
    const long long rest = panel / a.nwb;
    const int q = (int)(rest % a.nq);
    const long long b = rest / a.nq;
    const long long base = b * a.vol + (long long)q * a.Sq + (long long)wb * PW;
    const int ncol = min(PW, n - wb * PW);
    const int r0 = crank * a.R;
    const int nrow = max(0, min(a.R, n - r0));
    const bool vec = ((n & 1) == 0);

    double *sm = smem;                     // PW columns x S
    double *sd = smem + (size_t)PW * a.S;  // COEF: inverse pivots
    double *tabs = smem + (size_t)(1 + COEF) * PW * a.S;
    double2 *ctot = reinterpret_cast<double2 *>(
        smem + even_up((size_t)(1 + COEF) * PW * a.S + (COEF ? (size_t)a.St : 3 * (size_t)a.St)));
    if (COEF) {
        stage_table(tabs, a.s2f + r0, min(a.R + 1, n + 1 - r0));
    } else {
        stage_table(tabs, a.tab.m + r0, nrow);
        stage_table(tabs + a.St, a.tab.id + r0, nrow);
        stage_table(tabs + 2 * a.St, a.tab.cc + r0, nrow);
    }

    // ---- coalesced load (rows of PW doubles) ----
    if (vec) {
#pragma unroll
        for (int g = 0; g < 8; g += QG) {
            double2 U[QG], D[QG];
#pragma unroll
            for (int qq = 0; qq < QG; ++qq) {
                const int k = threadIdx.x + (g + qq) * blockDim.x;
                const int rl = k / PH, c2 = (k % PH) * 2;
                if (rl < nrow && c2 < ncol) {
                    U[qq] = ld2(a.in + base + (long long)(r0 + rl) * a.Sl + c2);
                    if (COEF) D[qq] = ld2(a.invd + (long long)(r0 + rl) * n + wb * PW + c2);
                }
            }
#pragma unroll
            for (int qq = 0; qq < QG; ++qq) {
                const int k = threadIdx.x + (g + qq) * blockDim.x;
                const int rl = k / PH, c2 = (k % PH) * 2;
                if (rl < nrow && c2 < ncol) {
                    sm[c2 * a.S + cpad(rl)] = U[qq].x;
                    sm[(c2 + 1) * a.S + cpad(rl)] = U[qq].y;
                    if (COEF) {
                        sd[c2 * a.S + cpad(rl)] = D[qq].x;
                        sd[(c2 + 1) * a.S + cpad(rl)] = D[qq].y;
                    }
                }
            }
        }
    } else {
#pragma unroll
        for (int g = 0; g < 16; g += 2 * QG) {
            double U[2 * QG], D[2 * QG];
#pragma unroll
            for (int qq = 0; qq < 2 * QG; ++qq) {
                const int k = threadIdx.x + (g + qq) * blockDim.x;
                const int rl = k / PW, w = k % PW;
                if (rl < nrow && w < ncol) {
                    U[qq] = a.in[base + (long long)(r0 + rl) * a.Sl + w];
                    if (COEF) D[qq] = a.invd[(long long)(r0 + rl) * n + wb * PW + w];
                }
            }
#pragma unroll
            for (int qq = 0; qq < 2 * QG; ++qq) {
                const int k = threadIdx.x + (g + qq) * blockDim.x;
                const int rl = k / PW, w = k % PW;
                if (rl < nrow && w < ncol) {
                    sm[w * a.S + cpad(rl)] = U[qq];
                    if (COEF) sd[w * a.S + cpad(rl)] = D[qq];
                }
            }
        }
    }
    __syncthreads();

    const int w = threadIdx.x / CP, t = threadIdx.x - w * CP;
    const int col = wb * PW + w;
    const bool colok = w < ncol;
    const int e0 = t * LCH;
    const int cnt = colok ? max(0, min(LCH, nrow - e0)) : 0;
    const bool full = nrow == CP * LCH;  // CTA-uniform: every chunk of every column is complete
    const int co = t * LCP;
    double *sp = sm + w * a.S + co;
    ConstView cv0{tabs + co, tabs + a.St + co, tabs + 2 * a.St + co};
    VarView cv1{sd + w * a.S + co, tabs + co, 0.0, -a.tau * a.h2inv, 0.0};
    if (COEF && colok) {
        cv1.hsx = 0.5 * __ldg(a.s2n + col);
        cv1.idm1 = (t > 0) ? sd[w * a.S + co - 2] : ((r0 > 0) ? a.invd[(long long)(r0 - 1) * n + col] : 0.0);
    }

    // F1 + F2 (segment = CP lanes of one column)
    double A, B, EA, EB;
    if (COEF) walk_f1_any(full, sp, cnt, cv1, A, B);
    else walk_f1_any(full, sp, cnt, cv0, A, B);
    seg_scan_fwd(A, B, CP, t, EA, EB);
    double Ycta = 0.0;
    if (a.CL > 1) {
        cg::cluster_group cl = cg::this_cluster();
        if (t == CP - 1) ctot[w] = make_double2(A, B);
        cl.sync();
        if (t == 0) {
            for (int r = 0; r < crank; ++r) {
                const double2 *rem = cl.map_shared_rank(ctot, r);
                const double2 v = rem[w];
                Ycta = v.x * Ycta + v.y;
            }
        }
        Ycta = __shfl_sync(0xffffffffu, Ycta, 0, CP);
    }
    // F3 + B2
    double Pb, Qb, EP, EQ;
    if (COEF) walk_f3_any(full, sp, cnt, cv1, fma(EA, Ycta, EB), Pb, Qb);
    else walk_f3_any(full, sp, cnt, cv0, fma(EA, Ycta, EB), Pb, Qb);
    seg_scan_bwd(Pb, Qb, CP, t, EP, EQ);
    double Xcta = 0.0;
    if (a.CL > 1) {
        cg::cluster_group cl = cg::this_cluster();
        double2 *ctb = ctot + PW;
        if (t == 0) ctb[w] = make_double2(Pb, Qb);
        cl.sync();
        if (t == 0) {
            for (int r = a.CL - 1; r > crank; --r) {
                const double2 *rem = cl.map_shared_rank(ctb, r);
                const double2 v = rem[w];
                Xcta = v.x * Xcta + v.y;
            }
        }
        Xcta = __shfl_sync(0xffffffffu, Xcta, 0, CP);
        cl.sync();  // no CTA leaves while its shared memory may still be read
    }
    // B3
    if (COEF) walk_b3_any(full, sp, cnt, cv1, fma(EP, Xcta, EQ));
    else walk_b3_any(full, sp, cnt, cv0, fma(EP, Xcta, EQ));
    __syncthreads();

    // ---- store + fused epilogue ----
    double dmax = 0.0;
    unsigned long long bad = 0;
    auto epi = [&](long long gi, double x0, double x1, bool two) {
        if (EPI == EPI_STORE) {
            if (two) st2(a.out + gi, x0, x1);
            else a.out[gi] = x0;
        } else if (EPI == EPI_DELTA) {
            if (two) {
                const double2 g = ld2(a.e_gc + gi);
                st2(a.out + gi, x0 - g.x, x1 - g.y);
            } else {
                a.out[gi] = x0 - a.e_gc[gi];
            }
        } else if (EPI == EPI_CORRECT) {
            double d0, d1 = 0.0, o0, o1 = 0.0;
            if (two) {
                const double2 dd = ld2(a.e_delta + gi), oo = ld2(a.e_traj + gi);
                d0 = dd.x;
                d1 = dd.y;
                o0 = oo.x;
                o1 = oo.y;
            } else {
                d0 = a.e_delta[gi];
                o0 = a.e_traj[gi];
            }
            const double n0 = x0 + d0, n1 = x1 + d1;
            if (two) {
                st2(a.e_gcache + gi, x0, x1);
                st2(a.e_traj + gi, n0, n1);
            } else {
                a.e_gcache[gi] = x0;
                a.e_traj[gi] = n0;
            }
            dmax = fmax(dmax, fabs(n0 - o0));
            if (!isfinite(n0)) bad = 1;
            if (two) {
                dmax = fmax(dmax, fabs(n1 - o1));
                if (!isfinite(n1)) bad = 1;
            }
        } else {  // EPI_INIT
            if (two) {
                st2(a.e_gcache + gi, x0, x1);
                st2(a.e_traj + gi, x0, x1);
            } else {
                a.e_gcache[gi] = x0;
                a.e_traj[gi] = x0;
            }
        }
    };
    if (vec) {
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
            const int k = threadIdx.x + qq * blockDim.x;
            const int rl = k / PH, c2 = (k % PH) * 2;
            if (rl < nrow && c2 < ncol)
                epi(base + (long long)(r0 + rl) * a.Sl + c2, sm[c2 * a.S + cpad(rl)], sm[(c2 + 1) * a.S + cpad(rl)],
                    true);
        }
    } else {
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) {
            const int k = threadIdx.x + qq * blockDim.x;
            const int rl = k / PW, ww = k % PW;
            if (rl < nrow && ww < ncol) epi(base + (long long)(r0 + rl) * a.Sl + ww, sm[ww * a.S + cpad(rl)], 0.0, false);
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
