// lpass3.cuh -- persistent, software-pipelined strided-axis line pass (y, or z in 3-D) for
// n = 16 * 2^k, 64 <= n <= 4096.  Same arithmetic as lpass.cuh, organised for streaming:
//  * 256 threads per CTA = PW columns x CP chunks of 16 rows (PW = 256/CP); a cluster of CL
//    CTAs covers one panel of PW columns x n rows (R = n/CL rows per CTA); clusters loop over
//    panels (persistent), so every thread keeps the row-dependent coefficient data of its 16
//    rows (face sines, or the constant-coefficient pivot tables) in registers;
//  * panels stream into shared memory with cp.async 16-byte copies two panels ahead (ring of
//    3 value buffers and, for variable kappa, 3 per-point pivot buffers), in a chunk-padded
//    row layout ((r + r/16) * PW) that makes the column walks bank-conflict free;
//  * each thread moves its 16 values (and pivots) into registers, walks in registers, and
//    stores the results straight from registers (PW-wide coalesced row segments) through the
//    fused parareal epilogue of lpass.cuh.
#pragma once
#include "common.cuh"
#include "lpass.cuh"
#include "xpass3.cuh"

namespace prs {

constexpr int L3T = 256;

struct L3Args {
    const double *in;
    double *out;
    long long vol;
    int n;
    long long Sl;        // element stride along the line
    int nq;              // planes per state
    long long Sq;        // plane stride
    int PW, CP, CL, R;   // columns per panel, chunks per CTA, cluster size, rows per CTA
    int nwb;             // panels per plane = n / PW
    long long npanels;   // batch * nq * nwb
    double tau, h2inv;
    CoefTab tab;
    const double *invd, *s2n, *s2f;
    const double *e_gc;
    double *e_gcache;
    const double *e_delta;
    double *e_traj;
    unsigned long long *e_red;
    int noex;  // experiment switch: skip the cluster exchange (wrong results; timing only)
};

inline int lpass3_rows_stride(int R) { return R + R / LCH; }
inline size_t lpass3_smem_bytes(int PW, int R, int CL, int coef) {
    const size_t buf = (size_t)lpass3_rows_stride(R) * PW;
    return sizeof(double) * (3 * buf * (coef ? 2 : 1)) + sizeof(double2) * (L3T + 4 * (size_t)CL * PW) +
           sizeof(double) * PW;
}

template <int PW, int COEF, int EPI>
__global__ void __launch_bounds__(L3T, 1) lpass3_kernel(L3Args a) {
    extern __shared__ __align__(16) double smem[];
    constexpr int CP = L3T / PW;  // chunks per column per CTA (R = 16 CP)
    constexpr int PH = PW / 2;    // 16-byte pieces per row segment
    constexpr int RSTEP = L3T / PH;  // rows covered by one pass of the 256 threads
    const int n = a.n;
    const int buf = (a.R + a.R / LCH) * PW;
    double *vb = smem;                        // 3 value buffers
    double *db = smem + 3 * buf;              // COEF: 3 pivot buffers
    double2 *sc = reinterpret_cast<double2 *>(smem + 3 * buf * (COEF ? 2 : 1));  // L3T maps
    double2 *ctf = sc + L3T;                  // cluster totals [parity][rank][column], fwd
    double2 *ctb = ctf + 2 * a.CL * PW;       // bwd
    double *ycta = reinterpret_cast<double *>(ctb + 2 * a.CL * PW);
    __shared__ __align__(8) unsigned long long mbf[2], mbb[2];  // [parity] fwd / bwd arrivals

    const int tid = threadIdx.x;
    const int w = tid % PW, t = tid / PW;     // column, chunk
    const int crank = (a.CL > 1) ? (int)cg::this_cluster().block_rank() : 0;
    const int r0 = crank * a.R;
    const int GT = PW < 32 ? 32 / PW : 1;     // chunks of one column inside a warp
    const int tg = t / GT, tl = t - tg * GT;  // chunk group (warp), position in the group
    const int lane = tid & 31;

    // ---- per-thread row data (rows r0 + 16t .. +15), loaded once ----
    const int gr0 = r0 + t * LCH;
    double sf[LCH + 1], tm[LCH], ti[LCH], tc[LCH];
#pragma unroll
    for (int i = 0; i <= LCH; ++i) sf[i] = COEF ? __ldg(a.s2f + gr0 + i) : 0.0;
#pragma unroll
    for (int i = 0; i < LCH; ++i) {
        tm[i] = COEF ? 0.0 : __ldg(a.tab.m + gr0 + i);
        ti[i] = COEF ? 0.0 : __ldg(a.tab.id + gr0 + i);
        tc[i] = COEF ? 0.0 : __ldg(a.tab.cc + gr0 + i);
    }
    const double tauh = a.tau * a.h2inv;

    const int cid = blockIdx.x / a.CL, ncl = gridDim.x / a.CL;
    if (a.CL > 1) {
        if (tid == 0) {
            mbar_init(&mbf[0], 1);
            mbar_init(&mbf[1], 1);
            mbar_init(&mbb[0], 1);
            mbar_init(&mbb[1], 1);
            mbar_fence_init();
        }
        cg::this_cluster().sync();  // barriers initialised before any remote complete_tx
    }
    const bool ex = a.CL > 1 && !a.noex;
    const unsigned bytes_f = 16u * PW * crank, bytes_b = 16u * PW * (a.CL - 1 - crank);
    // panel p -> (state b, plane q, column block wb); nwb and nq are powers of two
    const int nwb_sh = __ffs(a.nwb) - 1, nq_sh = __ffs(a.nq) - 1;
    auto panel_base = [&](int p) {
        const int wb = p & (a.nwb - 1);
        const int rest = p >> nwb_sh;
        const int q = rest & (a.nq - 1);
        const int b = rest >> nq_sh;
        return (long long)b * a.vol + (long long)q * a.Sq + (long long)wb * PW;
    };
    // issue the 16-byte copies of this CTA's R rows of panel p (values, and pivots):
    // exactly R*PW/2 = 8 * 256 pieces, 8 per thread, rows rr + q*RSTEP
    const int rr = tid / PH, hh = tid % PH;
    const long long roff0 = (long long)(r0 + rr) * a.Sl + 2 * hh;
    const long long doff0 = (long long)(r0 + rr) * n + 2 * hh;
    auto issue = [&](int p, int slot) {
        const long long base = panel_base(p);
        const int wcol = (p & (a.nwb - 1)) * PW;
        double *dv = vb + slot * buf;
        double *dd = db + slot * buf;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int r = rr + q * RSTEP;
            const int so = (r + r / LCH) * PW + 2 * hh;
            cp_async16(dv + so, a.in + base + roff0 + (long long)(q * RSTEP) * a.Sl);
            if (COEF) cp_async16(dd + so, a.invd + doff0 + (long long)(q * RSTEP) * n + wcol);
        }
    };
    int p = cid;
    if (p < a.npanels) issue(p, 0);
    cp_async_commit();
    if (p + ncl < a.npanels) issue(p + ncl, 1);
    cp_async_commit();
    double dmax = 0.0;
    unsigned long long bad = 0;
    int slot = 0, iter = 0;
    // column sine and the pivot above the first row of the CTA (another CTA's row) for panel
    // p are loaded one panel ahead, off the critical path
    auto col_of = [&](int pp) { return (pp & (a.nwb - 1)) * PW + w; };
    double nx_sx = 0.0, nx_halo = 0.0;
    if (COEF && p < a.npanels) {
        nx_sx = __ldg(a.s2n + col_of(p));
        if (t == 0 && r0 > 0) nx_halo = __ldg(a.invd + (long long)(r0 - 1) * n + col_of(p));
    }
    for (; p < a.npanels; p += ncl) {
        const double cur_sx = nx_sx, cur_halo = nx_halo;
        if (COEF && p + ncl < a.npanels) {
            nx_sx = __ldg(a.s2n + col_of(p + ncl));
            if (t == 0 && r0 > 0) nx_halo = __ldg(a.invd + (long long)(r0 - 1) * n + col_of(p + ncl));
        }
        if (p + 2 * (long long)ncl < a.npanels) issue(p + 2 * ncl, (slot + 2) % 3);
        cp_async_commit();
        cp_async_wait<2>();
        __syncthreads();
        const int it = iter;  // panel counter of this cluster
        const int par = (int)(it & 1);         // cluster totals double-buffered by parity
        const unsigned wpar = (unsigned)((it >> 1) & 1);
        if (ex && tid == 0) {
            if (crank > 0) mbar_arrive_expect(&mbf[par], bytes_f);
            if (crank < a.CL - 1) mbar_arrive_expect(&mbb[par], bytes_b);
        }
        const long long base = panel_base(p);
        // registers: values and pivots of this chunk
        const int so = (t * LCH + t) * PW + w;  // chunk-padded row (16t) * PW + w
        const double *sv = vb + slot * buf + so;
        double v[LCH], id[LCH], idm1 = 0.0;
#pragma unroll
        for (int i = 0; i < LCH; ++i) v[i] = sv[i * PW];
        if (COEF) {
            const double *sd = db + slot * buf + so;
#pragma unroll
            for (int i = 0; i < LCH; ++i) id[i] = sd[i * PW];
            if (t > 0) idm1 = sd[-2 * PW];  // row 16t-1 sits at chunk-padded index 17t-2
            else idm1 = cur_halo;
        }
        const double hsx = 0.5 * cur_sx;
        auto af = [&](int i) { return -tauh * fma(hsx, sf[i], 1.0); };
        auto cm = [&](int i) { return COEF ? af(i) * (i == 0 ? idm1 : id[i - 1]) : tm[i]; };
        auto ci = [&](int i) { return COEF ? id[i] : ti[i]; };
        auto cc = [&](int i) { return COEF ? af(i + 1) * id[i] : tc[i]; };

        // F1
        double A = 1.0, B = 0.0;
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            const double m = cm(i);
            B = fma(-m, B, v[i]);
            A = -m * A;
        }
        // F2: within the warp (lanes w + PW * tl), then across chunk groups, then across CTAs
        for (int off = 1; off < GT; off <<= 1) {
            const double A2 = __shfl_up_sync(0xffffffffu, A, off * PW);
            const double B2 = __shfl_up_sync(0xffffffffu, B, off * PW);
            if (tl >= off) {
                B = fma(A, B2, B);
                A = A * A2;
            }
        }
        double EA = __shfl_up_sync(0xffffffffu, A, PW < 32 ? PW : 0);
        double EB = __shfl_up_sync(0xffffffffu, B, PW < 32 ? PW : 0);
        if (tl == 0) {
            EA = 1.0;
            EB = 0.0;
        }
        sc[t * PW + w] = make_double2(A, B);
        __syncthreads();
        double YA = 1.0, YB = 0.0;  // composition of the previous chunk groups
        for (int g = 0; g < tg; ++g) {
            const double2 s = sc[((g + 1) * GT - 1) * PW + w];
            YB = fma(s.x, YB, s.y);
            YA = s.x * YA;
        }
        if (ex) {
            if (t == CP - 1) {  // push the CTA total of column w to every later CTA of the cluster
                const double2 tot = make_double2(A * YA, fma(A, YB, B));
                for (int q = crank + 1; q < a.CL; ++q)
                    st_async_remote(ctf + (par * a.CL + crank) * PW + w, &mbf[par], (unsigned)q, tot);
            }
            if (t == 0) {
                if (crank > 0) mbar_wait(&mbf[par], wpar);
                double Y = 0.0;
                for (int r = 0; r < crank; ++r) {
                    const double2 s = ctf[(par * a.CL + r) * PW + w];
                    Y = fma(s.x, Y, s.y);
                }
                ycta[w] = Y;
            }
            __syncthreads();
        }
        const double Yc = (a.CL > 1) ? ycta[w] : 0.0;
        const double yin = fma(EA, fma(YA, Yc, YB), EB);
        // F3
        double y = yin, Pb = 1.0, Qb = 0.0;
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            y = fma(-cm(i), y, v[i]);
            v[i] = y;
            Qb = fma(Pb * ci(i), y, Qb);
            Pb *= -cc(i);
        }
        // B2
        for (int off = 1; off < GT; off <<= 1) {
            const double P2 = __shfl_down_sync(0xffffffffu, Pb, off * PW);
            const double Q2 = __shfl_down_sync(0xffffffffu, Qb, off * PW);
            if (tl + off < GT) {
                Qb = fma(Pb, Q2, Qb);
                Pb = Pb * P2;
            }
        }
        double EP = __shfl_down_sync(0xffffffffu, Pb, PW < 32 ? PW : 0);
        double EQ = __shfl_down_sync(0xffffffffu, Qb, PW < 32 ? PW : 0);
        if (tl == GT - 1) {
            EP = 1.0;
            EQ = 0.0;
        }
        __syncthreads();  // forward maps consumed
        sc[t * PW + w] = make_double2(Pb, Qb);
        __syncthreads();
        double XP = 1.0, XQ = 0.0;  // composition of the following chunk groups
        const int ngr = CP / GT;
        for (int g = ngr - 1; g > tg; --g) {
            const double2 s = sc[(g * GT) * PW + w];
            XQ = fma(s.x, XQ, s.y);
            XP = s.x * XP;
        }
        if (ex) {
            if (t == 0) {  // push the backward total to every earlier CTA
                const double2 tot = make_double2(Pb * XP, fma(Pb, XQ, Qb));
                for (int q = 0; q < crank; ++q)
                    st_async_remote(ctb + (par * a.CL + crank) * PW + w, &mbb[par], (unsigned)q, tot);
                if (crank < a.CL - 1) mbar_wait(&mbb[par], wpar);
                double X = 0.0;
                for (int r = a.CL - 1; r > crank; --r) {
                    const double2 s = ctb[(par * a.CL + r) * PW + w];
                    X = fma(s.x, X, s.y);
                }
                ycta[w] = X;
            }
            __syncthreads();
        }
        const double Xc = (a.CL > 1) ? ycta[w] : 0.0;
        double x = fma(EP, fma(XP, Xc, XQ), EQ);
        // B3
#pragma unroll
        for (int i = LCH - 1; i >= 0; --i) {
            x = fma(-cc(i), x, ci(i) * v[i]);
            v[i] = x;
        }
        // ---- store from registers + fused epilogue ----
        const long long g0 = base + (long long)gr0 * a.Sl + w;
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            const long long gi = g0 + (long long)i * a.Sl;
            const double xv = v[i];
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
        // (cluster totals are double-buffered by panel parity: a CTA writes parity P again only
        // after passing the next panel's first cluster barrier, which every reader of parity P
        // reaches only after its reads)
        __syncthreads();  // slot free before it is refilled
        slot = (slot == 2) ? 0 : slot + 1;
        ++iter;
    }
    cp_async_wait<0>();
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

}  // namespace prs
