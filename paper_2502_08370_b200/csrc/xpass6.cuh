// xpass6.cuh -- 2-D x-line pass with the y-line block tuples fused into its epilogue, for
// long lines (n = 8 NT in {1024, 2048, 4096}; c3 is n = 4096).
//
// One FIE / DR step under dimensional splitting is two line-solve stages (PAPER.md:153-157,
// 167-171): (I - tau A_x) along every x-line, then (I - tau A_y) along every y-line.  A long
// y-line (4096 rows, 32 KB apart) cannot sit in one CTA, so the y-stage is solved with block
// tuples (lpass4.cuh): for every block of 64 rows and every column, the forward map
// y_last = A Y + B and the backward map x_first = P X + Q + R Y of the block.  A, P and R
// depend on the pivots only (a per-tau table, setup_ytuple_tab); B and Q depend on the
// right-hand side of the y-stage, which is exactly what this pass produces row by row.  So
// this pass also walks its output rows down each column, accumulating B and Q of the block
// in registers (8 columns per thread), and writes them when the block ends: the y-stage
// then needs one read of the state (lp5_finish) instead of two (lp5_tuples + lp5_finish).
//
// Organisation (B200, HBM-bound):
//  * 8 elements per thread, NT = n / 8 threads per CTA, one x-line (row) per iteration;
//  * work units are (64 ub)-row blocks of one state, ordered slice-fastest, taken round-robin
//    by persistent CTAs: at any moment all CTAs work on the same few row blocks of different
//    slices, so the per-point pivot rows (shared by every slice) are served by L2;
//  * state rows stream through a 6-slot shared-memory ring with cp.async 16-byte copies, four
//    rows ahead of the compute (~96 KB in flight per SM at n = 4096); 16-byte units are XOR
//    swizzled so both the coalesced copies and the per-thread chunk reads are conflict free;
//  * the DR stencil (w = tau A_y U) reads rows j-1 / j+1 from the ring (a unit adds one halo
//    row on each side); pivots of the x- and y-stage are read straight into registers (L2);
//  * the chunk-parallel Thomas solve is the one of common.cuh (walks, warp scans, a second
//    16-lane scan of the warp totals), the result is staged through the freed ring slot for
//    coalesced 16-byte stores.
#pragma once
#include "common.cuh"
#include "xpass3.cuh"

namespace prs {

constexpr int X6C = 8;      // elements per thread
constexpr int X6RB = 64;    // rows per y tuple block (= L5RB)
constexpr int X6SLOTS = 5;  // state ring depth
constexpr int X6AHEAD = 3;  // rows in flight ahead of the computed row

struct X6Args {
    const double *in;
    double *out;
    long long vol;
    int n;
    int B;                // states in the batch
    int nrb;              // tuple blocks per line, n / 64
    int ub;               // tuple blocks per work unit
    int nunits;           // B * nrb / ub
    double tau, h2inv, creact, src_amp;
    const double *sinpi;
    TimeArgs ta;
    CoefTab tab;          // kappa = 1 pivots (the same for both axes)
    const double *invdx, *s2n, *s2f;  // invdx: thread-interleaved copy (x6_perm)
    const double *ymt, *ycid;  // y-walk tables: m_y and cp * id_y per point (kappa = 1: per row)
    double *ttB, *ttQ;    // [B][nrb][n]: data parts of the y block tuples
};

// ring, x-face sine table (n + 1), y-face coefficient slope table (n), scan scratch
inline size_t xpass6_smem_bytes(int n) {
    return sizeof(double) * ((size_t)X6SLOTS * n + 2 * (size_t)n + 2) + sizeof(double2) * 32;
}
// conflict-free layout of per-thread 8-element runs read with 8-byte loads
__device__ __forceinline__ int x6_swz(int e) { return (e & ~7) | ((e & 7) ^ ((e >> 4) & 7)); }

// Factor tables read per row by xpass6 (x pivots, y-walk m and cp id) are stored
// thread-interleaved: element e = 8 k + 2 u + h of a row sits at (u NT + k) 2 + h, so thread k's
// four 16-byte loads are, warp-wide, four fully coalesced 512-byte reads.
__host__ __device__ inline long long x6_perm(int n, int e) {
    const int NT = n / X6C, k = e / X6C, i = e % X6C;
    return (long long)((i >> 1) * NT + k) * 2 + (i & 1);
}
__global__ void x6_permute_rows(const double *__restrict__ src, double *__restrict__ dst, int n) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)n * n) return;
    const long long j = idx / n;
    const int e = (int)(idx - j * n);
    dst[j * n + x6_perm(n, e)] = src[idx];
}

// position in the per-CTA sequence of ring entries (unit m, entry e; a unit is its rows plus
// one halo row before and after for DR)
struct X6Cursor {
    int m, b, e, jb;
};

template <int NT, int COEF, int DR, int SRC, int TUP>
__global__ void __launch_bounds__(NT, 512 / NT) xpass6_kernel(X6Args a) {
    constexpr int C = X6C;
    constexpr int NW = NT / 32;
    constexpr int n = NT * C;
    extern __shared__ __align__(16) double smem[];
    double *tsf = smem + X6SLOTS * n;  // sin(2 pi x) at x faces, swizzled (+ face n at [n])
    double *tnx = tsf + n + 2;         // -tau/h^2 * 0.5 sin(2 pi x_i), swizzled
    double2 *scr = reinterpret_cast<double2 *>(tnx + n);  // [0,16) fwd, [16,32) bwd
    const int k = threadIdx.x, lane = k & 31, warp = k >> 5;
    const int e0 = k * C;
    const int swz = (k >> 1) & 3;
    const unsigned FULL = 0xffffffffu;

    // ---- per-thread x-dependent data (registers for the whole launch) ----
    const double tauh = a.tau * a.h2inv, taucr = a.tau * a.creact;
    double spi[C], tm[C], ti[C], tc[C];
    if (COEF) {
        for (int e = k; e < n; e += NT) {
            tsf[x6_swz(e)] = __ldg(a.s2f + e);
            tnx[x6_swz(e)] = -tauh * 0.5 * __ldg(a.s2n + e);
        }
        if (k == 0) tsf[n] = __ldg(a.s2f + n);
    }
    auto SF = [&](int i) { return tsf[(i == C) ? ((k == NT - 1) ? n : x6_swz(e0 + C)) : x6_swz(e0 + i)]; };
    auto NSX = [&](int i) { return tnx[x6_swz(e0 + i)]; };
#pragma unroll
    for (int i = 0; i < C; ++i) {
        spi[i] = SRC ? __ldg(a.sinpi + e0 + i) : 0.0;
        tm[i] = COEF ? 0.0 : __ldg(a.tab.m + e0 + i);
        ti[i] = COEF ? 0.0 : __ldg(a.tab.id + e0 + i);
        tc[i] = COEF ? 0.0 : __ldg(a.tab.cc + e0 + i);
    }

    // ---- this CTA's entries ----
    const int RU = a.ub * X6RB;      // rows per unit
    const int E = RU + 2 * DR;       // ring entries per unit
    const int Mu = (a.nunits > (int)blockIdx.x) ? (a.nunits - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int QE = Mu * E;
    auto set_unit = [&](X6Cursor &c) {
        const int u = (int)blockIdx.x + c.m * (int)gridDim.x;
        const int rbu = u / a.B;
        c.b = u - rbu * a.B;
        c.jb = rbu * RU - DR;
    };
    auto advance = [&](X6Cursor &c) {
        if (++c.e == E) {
            c.e = 0;
            ++c.m;
            if (c.m < Mu) set_unit(c);
        }
    };
    auto is_comp = [&](const X6Cursor &c) { return c.e >= DR && c.e < DR + RU; };
    auto row_of = [&](const X6Cursor &c) { return c.jb + c.e; };

    auto issue = [&](const X6Cursor &c, int slot) {
        const int j = row_of(c);
        if (j < 0 || j >= n) return;
        const double *src = a.in + (long long)c.b * a.vol + (long long)j * n;
        double *dst = smem + slot * n;
#pragma unroll
        for (int q = 0; q < C / 2; ++q) {
            const int p = k + q * NT;          // 16-byte unit of the row
            const int c4 = p >> 2, u = p & 3;  // chunk, unit within the chunk
            cp_async16(dst + 2 * (4 * c4 + (u ^ ((c4 >> 1) & 3))), src + 2 * p);
        }
    };
    auto load_chunk = [&](int slot, double (&v)[C]) {
        const double *s = smem + slot * n + 4 * 2 * k;
#pragma unroll
        for (int u = 0; u < C / 2; ++u) {
            const double2 x = *reinterpret_cast<const double2 *>(s + 2 * (u ^ swz));
            v[2 * u] = x.x;
            v[2 * u + 1] = x.y;
        }
    };

    // per-row data: x pivots (registers) and row scalars, loaded at the start of the row
    // (their L2 latency overlaps the DR stencil)
    double pidx[C], pidm1 = 0.0, ps2n = 0.0, psfm = 0.0, psfp = 0.0, psrc = 0.0, pym = 0.0, pyi = 0.0;
    auto row_loads = [&](const X6Cursor &c) {
        const int j = row_of(c);
        if (COEF) {
            const double *px = a.invdx + (long long)j * n;  // thread-interleaved (x6_perm)
#pragma unroll
            for (int u = 0; u < C / 2; ++u) {
                const double2 x = __ldg(reinterpret_cast<const double2 *>(px + 2 * (u * NT + k)));
                pidx[2 * u] = x.x;
                pidx[2 * u + 1] = x.y;
            }
            pidm1 = (k > 0) ? __ldg(px + 2 * (3 * NT + k - 1) + 1) : 0.0;
            ps2n = __ldg(a.s2n + j);
            psfm = __ldg(a.s2f + j);
            psfp = __ldg(a.s2f + j + 1);
        } else {
            pym = __ldg(a.ymt + j);
            pyi = __ldg(a.ycid + j);
        }
        if (SRC) psrc = a.tau * a.src_amp * exp(-src_time(a.ta, c.b)) * __ldg(a.sinpi + j);
    };

    // prologue: the first X6AHEAD entries in flight
    X6Cursor ci{0, 0, 0, 0}, cc{0, 0, 0, 0};
    if (Mu > 0) {
        set_unit(ci);
        set_unit(cc);
    }
#pragma unroll 1
    for (int p = 0; p < X6AHEAD; ++p) {
        if (p < QE) issue(ci, p % X6SLOTS);
        cp_async_commit();
        advance(ci);
    }
    if (QE > 0) {  // x pivots / scalars of the first compute row; later rows: loaded after the
                   // previous row's backward sweep, when these registers are free again
        X6Cursor c0 = cc;
        while (!is_comp(c0)) advance(c0);
        row_loads(c0);
    }
    // y-stage tuple accumulators of this thread's 8 columns
    double y0[C], Qa[C];
#pragma unroll
    for (int i = 0; i < C; ++i) {
        y0[i] = 0.0;
        Qa[i] = 0.0;
    }

    int slot = 0;  // = q % X6SLOTS
#pragma unroll 1
    for (int q = 0; q < QE; ++q) {
        const int slot_m = (slot == 0) ? X6SLOTS - 1 : slot - 1;
        const int slot_p = (slot == X6SLOTS - 1) ? 0 : slot + 1;
        {
            int s4 = slot + X6AHEAD;
            if (s4 >= X6SLOTS) s4 -= X6SLOTS;
            if (q + X6AHEAD < QE) issue(ci, s4);
            cp_async_commit();
            advance(ci);
        }
        cp_async_wait<X6AHEAD - 1>();
        __syncthreads();
        if (is_comp(cc)) {
            const int j = row_of(cc);
            const int b = cc.b;
            const double sfm = psfm, sfp = psfp;  // y-face sines of this row
            double v[C];
            load_chunk(slot, v);
            // DR: w is parked in this thread's own chunk of the slot of row q-1 (read just above;
            // no other thread touches that chunk) until the end of the x solve
            double *wpark = smem + slot_m * n + 4 * 2 * k;
            if (DR) {  // w = tau A_y U_n (M = 2 form, R1)
                double dm[C], dp[C];
                if (j > 0) load_chunk(slot_m, dm);
                else
#pragma unroll
                    for (int i = 0; i < C; ++i) dm[i] = 0.0;
                if (j < n - 1) load_chunk(slot_p, dp);
                else
#pragma unroll
                    for (int i = 0; i < C; ++i) dp[i] = 0.0;
#pragma unroll
                for (int i = 0; i < C; ++i) {
                    // -tau/h^2 kappa at the faces (x_i, y_{j -+ 1/2})
                    const double nsx = COEF ? NSX(i) : 0.0;
                    const double aym = COEF ? fma(nsx, sfm, -tauh) : -tauh;
                    const double ayp = COEF ? fma(nsx, sfp, -tauh) : -tauh;
                    const double uu = v[i];
                    dm[i] = fma(-ayp, dp[i] - uu, fma(aym, uu - dm[i], -taucr * uu));
                    v[i] = uu + dm[i];
                }
#pragma unroll
                for (int u = 0; u < C / 2; ++u)
                    *reinterpret_cast<double2 *>(wpark + 2 * (u ^ swz)) = make_double2(dm[2 * u], dm[2 * u + 1]);
            }
            if (SRC) {
#pragma unroll
                for (int i = 0; i < C; ++i) v[i] = fma(psrc, spi[i], v[i]);
            }
            // x-stage coefficients of this chunk
            double cm[C], cid[C], ccx[C];
            {
                const double nh = -tauh * 0.5 * ps2n;
#pragma unroll
                for (int i = 0; i < C; ++i) {
                    if (COEF) {
                        const double af = fma(nh, SF(i), -tauh);       // off-diagonal at face i - 1/2
                        const double afp = fma(nh, SF(i + 1), -tauh);  // face i + 1/2
                        cm[i] = af * (i == 0 ? pidm1 : pidx[i - 1]);
                        cid[i] = pidx[i];
                        ccx[i] = afp * pidx[i];
                    } else {
                        cm[i] = tm[i];
                        cid[i] = ti[i];
                        ccx[i] = tc[i];
                    }
                }
            }
            // F1: forward map of the chunk
            double A = 1.0, Bv = 0.0;
#pragma unroll
            for (int i = 0; i < C; ++i) {
                Bv = fma(-cm[i], Bv, v[i]);
                A = -cm[i] * A;
            }
            double EA, EB;
            seg_scan_fwd(A, Bv, 32, lane, EA, EB);
            double Yw = 0.0;
            if (NW > 1) {
                if (lane == 31) scr[warp] = make_double2(A, Bv);
                __syncthreads();
                const double2 s = (lane < NW) ? scr[lane] : make_double2(1.0, 0.0);
                double sA = s.x, sB = s.y, dA, dB;
                seg_scan_fwd(sA, sB, NW, lane & (NW - 1), dA, dB);
                const double yprev = __shfl_sync(FULL, sB, (warp > 0 ? warp - 1 : 0));
                Yw = (warp > 0) ? yprev : 0.0;
            }
            // F3: exact forward recurrence, backward map of the chunk
            double y = fma(EA, Yw, EB), Pb = 1.0, Qb = 0.0;
#pragma unroll
            for (int i = 0; i < C; ++i) {
                y = fma(-cm[i], y, v[i]);
                v[i] = y;
                Qb = fma(Pb * cid[i], y, Qb);
                Pb *= -ccx[i];
            }
            double EP, EQ;
            seg_scan_bwd(Pb, Qb, 32, lane, EP, EQ);
            double Xw = 0.0;
            if (NW > 1) {
                if (lane == 0) scr[16 + warp] = make_double2(Pb, Qb);
                __syncthreads();
                const double2 s = (lane < NW) ? scr[16 + lane] : make_double2(1.0, 0.0);
                double sP = s.x, sQ = s.y, dP, dQ;
                seg_scan_bwd(sP, sQ, NW, lane & (NW - 1), dP, dQ);
                const double xnext = __shfl_sync(FULL, sQ, (warp < NW - 1 ? warp + 1 : 0));
                Xw = (warp < NW - 1) ? xnext : 0.0;
            }
            // B3: exact backward recurrence; result of the x-stage (DR: minus w, the y-stage RHS)
            double x = fma(EP, Xw, EQ);
#pragma unroll
            for (int i = C - 1; i >= 0; --i) {
                x = fma(cid[i], v[i], -ccx[i] * x);
                v[i] = x;
            }
            if (DR) {
#pragma unroll
                for (int u = 0; u < C / 2; ++u) {
                    const double2 wv = *reinterpret_cast<const double2 *>(wpark + 2 * (u ^ swz));
                    v[2 * u] -= wv.x;
                    v[2 * u + 1] -= wv.y;
                }
            }
            // next compute row's x pivots and scalars (this row's are dead from here on)
            const double ym = pym, yi = pyi;
            {
                X6Cursor cn = cc;
                advance(cn);
                while (cn.m < Mu && !is_comp(cn)) advance(cn);
                if (cn.m < Mu) row_loads(cn);
            }
            // y-walk coefficients of this row (used after the store below)
            double tmy[C], tcid[C];
            if (COEF && TUP) {
                const double *p1 = a.ymt + (long long)j * n, *p2 = a.ycid + (long long)j * n;
#pragma unroll
                for (int u = 0; u < C / 2; ++u) {
                    const double2 x1 = __ldg(reinterpret_cast<const double2 *>(p1 + 2 * (u * NT + k)));
                    const double2 x2 = __ldg(reinterpret_cast<const double2 *>(p2 + 2 * (u * NT + k)));
                    tmy[2 * u] = x1.x;
                    tmy[2 * u + 1] = x1.y;
                    tcid[2 * u] = x2.x;
                    tcid[2 * u + 1] = x2.y;
                }
            }
            // stage through the slot of row q-1 (its last reader, the DR stencil, is behind the
            // scan barriers) and store coalesced
            if (NW == 1) __syncthreads();
            {
                double *s = smem + slot_m * n + 4 * 2 * k;
#pragma unroll
                for (int u = 0; u < C / 2; ++u)
                    *reinterpret_cast<double2 *>(s + 2 * (u ^ swz)) = make_double2(v[2 * u], v[2 * u + 1]);
            }
            __syncthreads();
            {
                const double *s = smem + slot_m * n;
                double *o = a.out + (long long)b * a.vol + (long long)j * n;
#pragma unroll
                for (int qq = 0; qq < C / 2; ++qq) {
                    const int p = k + qq * NT;
                    const int c4 = p >> 2, u = p & 3;
                    const double2 xx = *reinterpret_cast<const double2 *>(s + 2 * (4 * c4 + (u ^ ((c4 >> 1) & 3))));
                    *reinterpret_cast<double2 *>(o + 2 * p) = xx;
                }
            }
            // y-stage block tuple: this row's step of the walk down each of the 8 columns
            // (y0 = forward elimination from y_in = 0, Q = sum of cp id_y y0: lpass4.cuh)
            if (TUP) {
#pragma unroll
            for (int i = 0; i < C; ++i) {
                const double my = COEF ? tmy[i] : ym, cdy = COEF ? tcid[i] : yi;
                y0[i] = fma(-my, y0[i], v[i]);
                Qa[i] = fma(cdy, y0[i], Qa[i]);
            }
            if ((j & (X6RB - 1)) == X6RB - 1) {
                const long long o = ((long long)b * a.nrb + (j >> 6)) * n + e0;
#pragma unroll
                for (int u = 0; u < C / 2; ++u) {
                    *reinterpret_cast<double2 *>(a.ttB + o + 2 * u) = make_double2(y0[2 * u], y0[2 * u + 1]);
                    *reinterpret_cast<double2 *>(a.ttQ + o + 2 * u) = make_double2(Qa[2 * u], Qa[2 * u + 1]);
                }
#pragma unroll
                for (int i = 0; i < C; ++i) {
                    y0[i] = 0.0;
                    Qa[i] = 0.0;
                }
            }
            }
            __syncthreads();  // staging slot free before the next prefetch lands in it
        }
        advance(cc);
        slot = slot_p;
    }
    cp_async_wait<0>();
}

// y-stage walk tables of (I - tau A_y) for the fused pass: per block of 64 rows and column,
// the walk of lpass4.cuh's 5-tuple (y0 = r - m y0, Q += cp id y0, cp *= -cc) splits into the
// data parts (y0, Q: xpass6) and pivot-only parts, tabulated here once per tau:
//   ymt[j][i] = m_y (the multiplier of row j),  ycid[j][i] = cp * id_y (cp over the block rows
//   before j),  apr = [3][nrb][n] the block's A = prod(-m), P = prod(-cc), R = sum cp id A_part.
// kappa = 1: the coefficients do not depend on the column, ymt / ycid are length-n vectors.
__global__ void setup_ytuple_tab(int n, int coef, double tau, double h2inv, CoefTab tab, const double *invdy,
                                 const double *s2n, const double *s2f, double *apr, double *ymt, double *ycid) {
    const int nrb = n / X6RB;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)nrb * n) return;
    const int rb = (int)(idx / n), col = (int)(idx - (long long)rb * n);
    const double tauh = tau * h2inv;
    const double sxh = coef ? 0.5 * s2n[col] : 0.0;
    double g = 1.0, cp = 1.0, R = 0.0;
    for (int r = 0; r < X6RB; ++r) {
        const int j = rb * X6RB + r;
        double m, ci, cc;
        if (coef) {
            ci = invdy[(long long)j * n + col];
            m = (-tauh * fma(sxh, s2f[j], 1.0)) * (j > 0 ? invdy[(long long)(j - 1) * n + col] : 0.0);
            cc = (-tauh * fma(sxh, s2f[j + 1], 1.0)) * ci;
        } else {
            m = tab.m[j];
            ci = tab.id[j];
            cc = tab.cc[j];
        }
        const double cid = cp * ci;
        if (coef) {
            ymt[(long long)j * n + x6_perm(n, col)] = m;
            ycid[(long long)j * n + x6_perm(n, col)] = cid;
        } else if (col == 0) {
            ymt[j] = m;
            ycid[j] = cid;
        }
        g = -m * g;
        R = fma(cid, g, R);
        cp *= -cc;
    }
    const long long plane = (long long)nrb * n;
    apr[idx] = g;
    apr[plane + idx] = cp;
    apr[2 * plane + idx] = R;
}

}  // namespace prs
