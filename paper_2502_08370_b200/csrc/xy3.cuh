// xy3.cuh -- the x and y stages of a 3-D FIE step fused per z-plane (kappa = 1, n = 128; c2).
//
// FIE with the dimensional split A = A_x + A_y + A_z (M = 3) solves
// (I - tau A_x) V_1 = U + tau F, (I - tau A_y) V_2 = V_1, (I - tau A_z) U' = V_2.  The first
// two stages only couple points of the same z-plane, so a plane (128 x 128 doubles) is read
// once, solved along x and then y on chip, and written once: 32 B per update over the step
// instead of 48 with one pass per stage.  The z stage stays the strided pass (lpass3).
//
// One plane per cluster of 2 CTAs, 64 rows each (70 KB of shared memory per CTA, 2 CTAs per
// SM from different clusters, so one plane's load or store overlaps another's solves):
//  * x lines are CTA-local: 8 chunks of 16 per row, 4 rows per warp, chunk-parallel Thomas
//    with 8-wide segmented warp scans (common.cuh), values in registers, the pivot tables in
//    shared memory (chunk-padded: the 8 chunks of a half-warp read 8 different banks);
//  * y lines cross the two CTAs: each thread walks a 16-row chunk of a column, the 4 chunk
//    tuples of a CTA are composed through shared memory (lpass4.cuh's 5-tuples), and one
//    exchange gives CTA 1 the y entering its half and CTA 0 the x leaving its half: each CTA
//    pushes its column totals into the partner's shared memory with st.async, completing on
//    the partner's mbarrier (no cluster-wide barrier per plane; the only one, split around the
//    plane load, publishes the mbarrier initialisation);
//  * the tile uses the chunk-padded row layout (x at x + x/16, row stride 136): the x walks
//    (rows r, r+1 x 8 chunks per half-warp) and the y walks (consecutive columns) are both
//    bank-conflict free;
//  * the walks read only the inverse pivots id from shared memory and form the multipliers
//    m_i = o id_{i-1} and cc_i = o id_i (o = -tau/h^2, constant off-diagonals for kappa = 1) --
//    the very products setup_const_tab stores, so the results are bitwise those of the full
//    tables, with half the shared-memory traffic of the walks (the pass is bound by it).
#pragma once
#include "common.cuh"
#include "lpass4.cuh"

namespace prs {

constexpr int XY_N = 128;               // plane edge (n)
constexpr int XY_R = 64;                // rows per CTA
constexpr int XY_S = XY_N + XY_N / LCH; // padded row stride (136)
constexpr int XY_T = 256;

struct XYArgs {
    const double *in;
    double *out;
    long long vol;      // slice stride
    long long nplanes;  // batch * n
    double tau;
    double src_amp;
    const double *sinpi;
    TimeArgs ta;
    CoefTab tab;        // kappa = 1 pivots (m, id, cc), the same for x and y
    double offd;        // the off-diagonal -tau / h^2: m_i = offd id_{i-1}, cc_i = offd id_i
};

inline size_t xy3_smem_bytes() {
    return sizeof(double) * ((size_t)XY_R * XY_S + 5 * 4 * XY_N + 3 * XY_N + 3 * XY_S);
}

template <int SRC>
__global__ void __launch_bounds__(XY_T, 2) xy3_kernel(XYArgs a) {
    extern __shared__ __align__(16) double sm[];
    double *tile = sm;                             // 64 x 136
    double *st = tile + XY_R * XY_S;               // [5][4][128] chunk tuples (y)
    double *ex = st + 5 * 4 * XY_N;                // [3][128]: B of CTA 0's column totals (first row)
    double *ty = ex + 3 * XY_N;                    // [3][136] pivots m, id, cc, chunk-padded (x and y)
    __shared__ __align__(16) double2 xin[XY_N];  // the partner's column totals
    __shared__ __align__(8) unsigned long long mbx;
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        mbar_init(&mbx, 1);
        mbar_fence_init();
        mbar_arrive_expect(&mbx, XY_N * sizeof(double2));
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    const long long plane = blockIdx.x / 2;
    const long long b = plane / XY_N;
    const int z = (int)(plane - b * XY_N);
    const int n = XY_N;
    const long long base = b * a.vol + (long long)z * n * n + (long long)crank * XY_R * n;
    const int rg0 = crank * XY_R;  // first global row (y) of this CTA

    // ---- load the half plane (+ tau F, FIE stage-1 RHS) ----
    {
        constexpr int NLD = XY_R * XY_N / 2 / XY_T;  // 16 pieces per thread, all in flight
        double2 v[NLD];
#pragma unroll
        for (int k = 0; k < NLD; ++k) {
            const int e = tid + k * XY_T, r = e >> 6, x2 = (e & 63) * 2;
            v[k] = __ldg(reinterpret_cast<const double2 *>(a.in + base + (long long)r * n + x2));
        }
        for (int e = tid; e < XY_N; e += XY_T) {  // pivot tables (while the plane is in flight)
            ty[cpad(e)] = __ldg(a.tab.m + e);
            ty[XY_S + cpad(e)] = __ldg(a.tab.id + e);
            ty[2 * XY_S + cpad(e)] = __ldg(a.tab.cc + e);
        }
        double sz = 0.0;
        if (SRC) sz = a.tau * a.src_amp * src_tf(a.ta, b) * __ldg(a.sinpi + z);
#pragma unroll
        for (int k = 0; k < NLD; ++k) {
            const int e = tid + k * XY_T, r = e >> 6, x2 = (e & 63) * 2;
            if (SRC) {
                const double f = sz * __ldg(a.sinpi + rg0 + r);
                v[k].x = fma(f, __ldg(a.sinpi + x2), v[k].x);
                v[k].y = fma(f, __ldg(a.sinpi + x2 + 1), v[k].y);
            }
            double *d = tile + r * XY_S + cpad(x2);
            d[0] = v[k].x;
            d[1] = v[k].y;
        }
    }
    __syncthreads();

    // ---- x stage: rows of this CTA, 8 chunks per row, 4 rows per warp ----
    {
        const int c = lane & 7;  // chunk along x
        // pivots of the chunk from the padded table: the 8 chunks of a half-warp hit 8 banks
        const double *ti = ty + XY_S + c * LCP;
        const double o = a.offd, m0 = ty[c * LCP];  // m of the chunk's first point (0 on the row's first)
        auto tmv = [&](int i) { return i == 0 ? m0 : o * ti[i - 1]; };
        auto tcv = [&](int i) { return (c == 7 && i == LCH - 1) ? 0.0 : o * ti[i]; };
        for (int k = 0; k < 2; ++k) {
            const int q = tid + k * XY_T;
            const int r = (q >> 5) * 4 + (lane >> 3);
            double *p = tile + r * XY_S + c * LCP;
            double v[LCH];
#pragma unroll
            for (int i = 0; i < LCH; ++i) v[i] = p[i];
            double A = 1.0, B = 0.0;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                const double m = tmv(i);
                B = fma(-m, B, v[i]);
                A = -m * A;
            }
            double EA, EB;
            seg_scan_fwd(A, B, 8, c, EA, EB);
            double y = EB, Pb = 1.0, Qb = 0.0;  // y entering the chunk (y_in of the row = 0)
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                y = fma(-tmv(i), y, v[i]);
                v[i] = y;
                Qb = fma(Pb * ti[i], y, Qb);
                Pb *= -tcv(i);
            }
            double EP, EQ;
            seg_scan_bwd(Pb, Qb, 8, c, EP, EQ);
            double x = EQ;  // x leaving the chunk (x after the row's end = 0)
#pragma unroll
            for (int i = LCH - 1; i >= 0; --i) {
                x = fma(-tcv(i), x, ti[i] * v[i]);
                v[i] = x;
            }
#pragma unroll
            for (int i = 0; i < LCH; ++i) p[i] = v[i];
        }
    }
    __syncthreads();

    // ---- y stage: columns, 4 chunks of 16 rows per CTA, 2 tasks per thread ----
    const int w = tid & (XY_N - 1), t0 = tid >> 7;  // column, first chunk (t0, t0 + 2)
    double v0[LCH], v1[LCH];
    Tup u0, u1;
    auto yi = [&](int t, int i) { return ty[XY_S + cpad(rg0 + t * LCH) + i]; };
    auto ym = [&](int t, int i) { return i == 0 ? ty[cpad(rg0 + t * LCH)] : a.offd * yi(t, i - 1); };
    auto yc = [&](int t, int i) { return (rg0 + t * LCH + i == XY_N - 1) ? 0.0 : a.offd * yi(t, i); };
    auto walk1 = [&](int t, const double (&v)[LCH]) {
        double y0 = 0.0, g = 1.0, cp = 1.0, Q = 0.0, R = 0.0;
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            const double m = ym(t, i);
            y0 = fma(-m, y0, v[i]);
            g = -m * g;
            const double cid = cp * yi(t, i);
            Q = fma(cid, y0, Q);
            R = fma(cid, g, R);
            cp *= -yc(t, i);
        }
        return Tup{g, y0, cp, Q, R};
    };
    {
        const double *p0 = tile + (t0 * LCH) * XY_S + cpad(w);
        const double *p1 = tile + ((t0 + 2) * LCH) * XY_S + cpad(w);
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            v0[i] = p0[i * XY_S];
            v1[i] = p1[i * XY_S];
        }
        u0 = walk1(t0, v0);
        u1 = walk1(t0 + 2, v1);
        auto put = [&](int t, const Tup &u) {
            st[(0 * 4 + t) * XY_N + w] = u.A;
            st[(1 * 4 + t) * XY_N + w] = u.B;
            st[(2 * 4 + t) * XY_N + w] = u.P;
            st[(3 * 4 + t) * XY_N + w] = u.Q;
            st[(4 * 4 + t) * XY_N + w] = u.R;
        };
        put(t0, u0);
        put(t0 + 2, u1);
    }
    __syncthreads();
    auto get = [&](int t) {
        return Tup{st[(0 * 4 + t) * XY_N + w], st[(1 * 4 + t) * XY_N + w], st[(2 * 4 + t) * XY_N + w],
                   st[(3 * 4 + t) * XY_N + w], st[(4 * 4 + t) * XY_N + w]};
    };
    // CTA totals of the column -> the partner (one thread per column)
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");  // partner's mbarrier initialised
    if (tid < XY_N) {
        Tup tot = tup_id();
#pragma unroll
        for (int q = 0; q < 4; ++q) tot = tup_cat(tot, get(q));
        if (crank == 0) {
            ex[w] = tot.B;  // y at this half's last row, from y_in = 0
            st_async_remote(&xin[w], &mbx, 1, make_double2(tot.B, 0.0));
        } else {
            st_async_remote(&xin[w], &mbx, 0, make_double2(tot.Q, tot.R));
        }
    }
    __syncthreads();  // ex[] (CTA 0's own totals) visible to the column's second thread
    mbar_wait(&mbx, 0);
    double Yin = 0.0, Xout = 0.0;
    if (crank == 0) {
        const double2 qr = xin[w];
        Xout = fma(qr.y, ex[w], qr.x);  // x at row 64: Q1 + R1 y(63)
    } else {
        Yin = xin[w].x;
    }
    auto finish = [&](int t, double (&v)[LCH], const Tup &u) {
        double Y = Yin;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < t) {
                const Tup g = get(q);
                Y = fma(g.A, Y, g.B);
            }
        const double Ylast = fma(u.A, Y, u.B);
        Tup s = tup_id();
#pragma unroll
        for (int q = 3; q >= 0; --q)
            if (q > t) s = tup_cat(get(q), s);
        const double X = fma(s.P, Xout, fma(s.R, Ylast, s.Q));
        double y = Y;
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            y = fma(-ym(t, i), y, v[i]);
            v[i] = y;
        }
        double x = X;
#pragma unroll
        for (int i = LCH - 1; i >= 0; --i) {
            x = fma(-yc(t, i), x, yi(t, i) * v[i]);
            v[i] = x;
        }
        double *p = tile + (t * LCH) * XY_S + cpad(w);
#pragma unroll
        for (int i = 0; i < LCH; ++i) p[i * XY_S] = v[i];
    };
    finish(t0, v0, u0);
    finish(t0 + 2, v1, u1);
    __syncthreads();
    // ---- store the half plane (coalesced) ----
    for (int e = tid; e < XY_R * XY_N / 2; e += XY_T) {
        const int r = e >> 6, x2 = (e & 63) * 2;
        const double *s = tile + r * XY_S + cpad(x2);
        *reinterpret_cast<double2 *>(a.out + base + (long long)r * n + x2) = make_double2(s[0], s[1]);
    }
}

}  // namespace prs
