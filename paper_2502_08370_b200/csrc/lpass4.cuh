// lpass4.cuh -- strided-axis line pass for lines split over a cluster (n = 1024..4096).
//
// lpass3 needs two dependent cluster exchanges per panel (forward y, then backward x), and
// its 2-8 CTAs wait for each other twice per panel.  Here every chunk first runs ONE local
// walk with y_in = 0 that yields a 5-tuple T = (A, B, P, Q, R):
//     y_last  = A * Y + B                      (forward affine map of the chunk)
//     x_first = P * X + Q + R * Y              (backward map, with its dependence on Y)
// for the incoming Y (y before the chunk) and X (x after it).  Tuples compose associatively
//     (T1 then T2):  A = A2 A1,  B = A2 B1 + B2,  P = P1 P2,
//                    Q = Q1 + P1 (Q2 + R2 B1),  R = R1 + P1 R2 A1,
// so one exchange of the CTA totals gives every chunk both Y (prefix) and X (suffix).  The
// exchange of panel i (st.async + mbarrier, cluster-wide) is then hidden: while its totals
// travel the CTA finishes panel i-1 (whose totals arrived during the previous iteration):
// exact forward and backward recurrences from Y and X, fused epilogue, stores.
// Values of the previous panel stay in registers; per-point pivots stay in a shared ring.
#pragma once
#include "common.cuh"
#include "lpass.cuh"
#include "lpass3.cuh"

namespace prs {

struct Tup {
    double A, B, P, Q, R;
};
__device__ __forceinline__ Tup tup_id() { return Tup{1.0, 0.0, 1.0, 0.0, 0.0}; }
// t1 then t2
__device__ __forceinline__ Tup tup_cat(const Tup &t1, const Tup &t2) {
    Tup r;
    r.A = t2.A * t1.A;
    r.B = fma(t2.A, t1.B, t2.B);
    r.P = t1.P * t2.P;
    r.Q = fma(t1.P, fma(t2.R, t1.B, t2.Q), t1.Q);
    r.R = fma(t1.P * t2.R, t1.A, t1.R);
    return r;
}
__device__ __forceinline__ Tup tup_shfl_up(const Tup &t, int d) {
    return Tup{__shfl_up_sync(0xffffffffu, t.A, d), __shfl_up_sync(0xffffffffu, t.B, d),
               __shfl_up_sync(0xffffffffu, t.P, d), __shfl_up_sync(0xffffffffu, t.Q, d),
               __shfl_up_sync(0xffffffffu, t.R, d)};
}
__device__ __forceinline__ Tup tup_shfl_down(const Tup &t, int d) {
    return Tup{__shfl_down_sync(0xffffffffu, t.A, d), __shfl_down_sync(0xffffffffu, t.B, d),
               __shfl_down_sync(0xffffffffu, t.P, d), __shfl_down_sync(0xffffffffu, t.Q, d),
               __shfl_down_sync(0xffffffffu, t.R, d)};
}

inline size_t lpass4_smem_bytes(int PW, int R, int CL, int coef) {
    const size_t buf = (size_t)lpass3_rows_stride(R) * PW;
    // 2 value buffers, 3 pivot buffers, per-chunk tuples (fwd-inclusive + bwd-inclusive),
    // cluster totals [parity][rank][column] (6 doubles each)
    return sizeof(double) * (2 * buf + (coef ? 3 * buf : 0) + 2 * 5 * (size_t)L3T + 2 * (size_t)CL * PW * 6);
}

template <int PW, int COEF, int EPI>
__global__ void __launch_bounds__(L3T, 1) lpass4_kernel(L3Args a) {
    extern __shared__ __align__(16) double smem[];
    constexpr int CP = L3T / PW;
    constexpr int PH = PW / 2;
    constexpr int RSTEP = L3T / PH;
    constexpr int GT = PW < 32 ? 32 / PW : 1;  // chunks of one column inside a warp
    constexpr int NG = CP / GT;                // chunk groups (warps) per column
    const int n = a.n, CL = a.CL;
    const int buf = (a.R + a.R / LCH) * PW;
    double *vbuf = smem;                            // 2 value buffers
    double *pbuf = smem + 2 * buf;                  // COEF: 3 pivot buffers
    double *sfw = pbuf + (COEF ? 3 * buf : 0);      // [5][L3T] forward-inclusive tuples
    double *sbw = sfw + 5 * L3T;                    // [5][L3T] backward-inclusive tuples
    double2 *ctot = reinterpret_cast<double2 *>(sbw + 5 * L3T);  // [par][rank][w][3] double2
    __shared__ __align__(8) unsigned long long mbx[2];

    const int tid = threadIdx.x;
    const int w = tid % PW, t = tid / PW;
    const int crank = (int)cg::this_cluster().block_rank();
    const int r0 = crank * a.R;
    const int tg = t / GT, tl = t - tg * GT;
    const int lane = tid & 31;
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

    const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
    if (tid == 0) {
        mbar_init(&mbx[0], 1);
        mbar_init(&mbx[1], 1);
        mbar_fence_init();
    }
    cg::this_cluster().sync();
    const unsigned bytes_x = 48u * PW * (CL - 1);

    const int nwb_sh = __ffs(a.nwb) - 1, nq_sh = __ffs(a.nq) - 1;
    auto panel_base = [&](int p) {
        const int wb = p & (a.nwb - 1);
        const int rest = p >> nwb_sh;
        const int q = rest & (a.nq - 1);
        const int b = rest >> nq_sh;
        return (long long)b * a.vol + (long long)q * a.Sq + (long long)wb * PW;
    };
    const int rr = tid / PH, hh = tid % PH;
    const long long roff0 = (long long)(r0 + rr) * a.Sl + 2 * hh;
    const long long doff0 = (long long)(r0 + rr) * n + 2 * hh;
    auto issue = [&](int p, int vslot, int pslot) {
        const long long base = panel_base(p);
        const int wcol = (p & (a.nwb - 1)) * PW;
        double *dv = vbuf + vslot * buf;
        double *dd = pbuf + pslot * buf;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int r = rr + q * RSTEP;
            const int so = (r + r / LCH) * PW + 2 * hh;
            cp_async16(dv + so, a.in + base + roff0 + (long long)(q * RSTEP) * a.Sl);
            if (COEF) cp_async16(dd + so, a.invd + doff0 + (long long)(q * RSTEP) * n + wcol);
        }
    };
    auto col_of = [&](int pp) { return (pp & (a.nwb - 1)) * PW + w; };
    const int so = (t * LCH + t) * PW + w;  // this thread's chunk in a buffer

    // coefficient accessors for a panel whose pivots sit in pivot slot ps
    struct Coef {
        const double *pd;
        double hsx, idm1;
    };
    auto make_coef = [&](int ps, double sx, double halo) {
        Coef c;
        c.pd = pbuf + ps * buf + so;
        c.hsx = 0.5 * sx;
        c.idm1 = (t > 0) ? (COEF ? c.pd[-2 * PW] : 0.0) : halo;
        return c;
    };
    auto af = [&](const Coef &c, int i) { return -tauh * fma(c.hsx, sf[i], 1.0); };
    auto cm = [&](const Coef &c, int i) {
        return COEF ? af(c, i) * (i == 0 ? c.idm1 : c.pd[(i - 1) * PW]) : tm[i];
    };
    auto ci = [&](const Coef &c, int i) { return COEF ? c.pd[i * PW] : ti[i]; };
    auto cc = [&](const Coef &c, int i) { return COEF ? af(c, i + 1) * c.pd[i * PW] : tc[i]; };

    // state carried from panel i to its completion in iteration i+1
    double vprev[LCH];
    double Ypre = 0.0;      // y before this chunk from chunks of this CTA only (own-CTA prefix)
    double preA = 1.0;      // own-CTA prefix forward map A (to apply the cluster prefix)
    Tup own = tup_id();     // this chunk's tuple
    Tup suf = tup_id();     // composition of the following chunks of this CTA
    int prev_p = -1, prev_ps = 0, prev_par = 0;
    double prev_sx = 0.0, prev_halo = 0.0;
    double dmax = 0.0;
    unsigned long long bad = 0;

    // finish panel p (tuples exchanged): Y, X of this chunk, exact recurrences, store
    auto finish = [&](int p, int pit, int ps, int par, double sx, double halo) {
        if (CL > 1) mbar_wait(&mbx[par], (unsigned)((pit >> 1) & 1));
        // cluster prefix (forward) and suffix (tuple) for column w
        double Yc = 0.0;
        for (int r = 0; r < crank; ++r) {
            const double2 *s = ctot + ((par * CL + r) * PW + w) * 3;
            const double2 ab = s[0];
            Yc = fma(ab.x, Yc, ab.y);
        }
        Tup cs = tup_id();
        for (int r = CL - 1; r > crank; --r) {
            const double2 *s = ctot + ((par * CL + r) * PW + w) * 3;
            const double2 ab = s[0], pq = s[1], rx = s[2];
            cs = tup_cat(Tup{ab.x, ab.y, pq.x, pq.y, rx.x}, cs);
        }
        const double Y = fma(preA, Yc, Ypre);        // y before this chunk
        const double Ylast = fma(own.A, Y, own.B);   // y at this chunk's last row
        const Tup after = tup_cat(suf, cs);          // everything after this chunk
        const double X = fma(after.R, Ylast, after.Q);  // x after this chunk (x_end = 0)
        const Coef c = make_coef(ps, sx, halo);
        double v[LCH];
#pragma unroll
        for (int i = 0; i < LCH; ++i) v[i] = vprev[i];
        double y = Y;
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            y = fma(-cm(c, i), y, v[i]);
            v[i] = y;
        }
        double x = X;
#pragma unroll
        for (int i = LCH - 1; i >= 0; --i) {
            x = fma(-cc(c, i), x, ci(c, i) * v[i]);
            v[i] = x;
        }
        const long long g0 = panel_base(p) + (long long)gr0 * a.Sl + w;
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
    };

    int p = cid, it = 0;
    if (p < a.npanels) issue(p, 0, 0);
    cp_async_commit();
    double nx_sx = 0.0, nx_halo = 0.0;
    if (COEF && p < a.npanels) {
        nx_sx = __ldg(a.s2n + col_of(p));
        if (t == 0 && r0 > 0) nx_halo = __ldg(a.invd + (long long)(r0 - 1) * n + col_of(p));
    }
    for (; p < a.npanels; p += ncl, ++it) {
        const int vs = it & 1, ps = it % 3, par = it & 1;
        const double cur_sx = nx_sx, cur_halo = nx_halo;
        // prefetch the next panel (values slot vs^1, pivots slot (it+1)%3: both are free --
        // the value slot was moved to registers last iteration, the pivot slot belonged to
        // the panel finished last iteration)
        if (p + ncl < a.npanels) {
            issue(p + ncl, vs ^ 1, (it + 1) % 3);
            if (COEF) {
                nx_sx = __ldg(a.s2n + col_of(p + ncl));
                if (t == 0 && r0 > 0) nx_halo = __ldg(a.invd + (long long)(r0 - 1) * n + col_of(p + ncl));
            }
        }
        cp_async_commit();
        cp_async_wait<1>();
        if (tid == 0) mbar_arrive_expect(&mbx[par], bytes_x);
        __syncthreads();

        // ---- walk 1 on panel p (y_in = 0): chunk tuple ----
        double vcur[LCH];
        {
            const double *sv = vbuf + vs * buf + so;
#pragma unroll
            for (int i = 0; i < LCH; ++i) vcur[i] = sv[i * PW];
        }
        const Coef c = make_coef(ps, cur_sx, cur_halo);
        Tup T;
        {
            double y0 = 0.0, g = 1.0, cprod = 1.0, Q = 0.0, R = 0.0;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                const double m = cm(c, i);
                y0 = fma(-m, y0, vcur[i]);
                g = -m * g;
                const double cid_ = cprod * ci(c, i);
                Q = fma(cid_, y0, Q);
                R = fma(cid_, g, R);
                cprod *= -cc(c, i);
            }
            T = Tup{g, y0, cprod, Q, R};
        }
        // ---- scans inside the CTA: forward-inclusive and backward-inclusive per warp ----
        Tup fi = T, bi = T;
#pragma unroll
        for (int off = 1; off < GT; off <<= 1) {
            const Tup u = tup_shfl_up(fi, off * PW);
            if (tl >= off) fi = tup_cat(u, fi);
            const Tup d = tup_shfl_down(bi, off * PW);
            if (tl + off < GT) bi = tup_cat(bi, d);
        }
        // exclusive within the warp
        Tup fex = tup_shfl_up(fi, GT > 1 ? PW : 0);
        if (tl == 0) fex = tup_id();
        Tup bex = tup_shfl_down(bi, GT > 1 ? PW : 0);
        if (tl == GT - 1) bex = tup_id();
        {
            const int q = t * PW + w;
            sfw[0 * L3T + q] = fi.A;
            sfw[1 * L3T + q] = fi.B;
            sbw[0 * L3T + q] = bi.A;
            sbw[1 * L3T + q] = bi.B;
            sbw[2 * L3T + q] = bi.P;
            sbw[3 * L3T + q] = bi.Q;
            sbw[4 * L3T + q] = bi.R;
        }
        // finish the previous panel while this panel's tables land (its totals were pushed
        // one iteration ago)
        if (prev_p >= 0) finish(prev_p, it - 1, prev_ps, prev_par, prev_sx, prev_halo);
        __syncthreads();
        // prefix of earlier warps (forward part) and suffix of later warps (tuples)
        double gA = 1.0, gB = 0.0;
        for (int gq = 0; gq < tg; ++gq) {
            const int q = ((gq + 1) * GT - 1) * PW + w;
            const double A2 = sfw[q], B2 = sfw[L3T + q];
            gB = fma(A2, gB, B2);
            gA = A2 * gA;
        }
        Tup gsuf = tup_id();
        for (int gq = NG - 1; gq > tg; --gq) {
            const int q = (gq * GT) * PW + w;
            gsuf = tup_cat(Tup{sbw[q], sbw[L3T + q], sbw[2 * L3T + q], sbw[3 * L3T + q], sbw[4 * L3T + q]}, gsuf);
        }
        // own-CTA prefix before this chunk: (earlier warps) then (earlier lanes of this warp)
        Ypre = fma(fex.A, gB, fex.B);
        preA = fex.A * gA;
        own = T;
        suf = tup_cat(bex, gsuf);
        // CTA total of column w (thread t == 0 holds the backward-inclusive of warp 0 and
        // composes the later warps) -> push to every other CTA of the cluster
        if (t == 0) {
            const Tup tot = tup_cat(bi, gsuf);
            for (int q = 0; q < CL; ++q) {
                if (q == crank) continue;
                double2 *d = ctot + ((par * CL + crank) * PW + w) * 3;
                st_async_remote(d + 0, &mbx[par], (unsigned)q, make_double2(tot.A, tot.B));
                st_async_remote(d + 1, &mbx[par], (unsigned)q, make_double2(tot.P, tot.Q));
                st_async_remote(d + 2, &mbx[par], (unsigned)q, make_double2(tot.R, 0.0));
            }
        }
#pragma unroll
        for (int i = 0; i < LCH; ++i) vprev[i] = vcur[i];
        prev_p = p;
        prev_ps = ps;
        prev_par = par;
        prev_sx = cur_sx;
        prev_halo = cur_halo;
        __syncthreads();  // tuple scratch and the value slot free for the next iteration
    }
    if (prev_p >= 0) finish(prev_p, it - 1, prev_ps, prev_par, prev_sx, prev_halo);
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
