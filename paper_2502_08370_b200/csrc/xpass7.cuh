// xpass7.cuh -- the x-line pass for 4096-point rows (2-D, c3) with each row split over a
// cluster of 2 CTAs of 128 threads, so that two rows' dependency chains are in flight per SM.
//
// Same arithmetic as xpass3.cuh (stage-1 RHS, DR stencil, chunk-parallel Thomas, PAPER.md:153,
// 167): xpass3 walks one row per CTA with 256 threads and 254 registers per thread, so an SM
// holds one row at a time and the row's chain (walk, warp scan, barrier, cross-warp scan,
// walk, reverse scans, walk, staged store) bounds the pass (profiles/r01_fused_notes.md).
// Here CTA r of the pair owns chunks [128 r, 128 r + 128) of every row (a half row, 16 KB,
// in a ring of half-row slots: 110 KB per CTA, so two CTAs fit per SM).  The chunk-parallel
// recurrences cross the pair through two point-to-point messages per row (st.async into the
// partner's shared memory, completing on its mbarrier):
//   forward : CTA 0's composition of its forward maps from y_in = 0, i.e. the y entering
//             CTA 1's half, right after CTA 0's first walk and scan;
//   backward: CTA 1's x at its first point (its backward maps composed from x = 0 at the row
//             end, after its exact forward recurrence), to CTA 0 before CTA 0's last walk.
//
// TMA = 1 (default): the ring slots are filled by TMA tensor copies (one 2-D copy of 128 rows of
// 128 bytes per half row, issued by one thread, completing on the slot's mbarrier) and the
// output half row leaves by one TMA tensor store from a staging slot; the tensor maps' 128-byte
// swizzle puts 16-byte unit u of chunk k at unit u ^ (k & 7), so the per-thread chunk accesses
// stay bank-conflict free without padding.  No per-thread copy instructions remain for the
// 48 KB a row moves through shared memory (TMA = 0: 16-byte cp.async fills, staged coalesced
// stores; the load/store issue ahead of each row cost ~1k cycles of its chain,
// profiles/r02_notes.md).
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "xpass3.cuh"

namespace prs {

#ifdef PRS_X7_TIMING
// diagnostic build only (-DPRS_X7_TIMING): clock64 cycles of thread 0 of every CTA per phase of
// a row, summed over rows, per cluster rank: [rank][phase], phase 8 = rows
__device__ unsigned long long g_x7_timing[2][10];
#define X7T_MARK(ph)                                                      \
    do {                                                                  \
        if (k == 0) {                                                     \
            const long long t_ = clock64();                               \
            tacc[ph] += (unsigned long long)(t_ - tlast);                 \
            tlast = t_;                                                   \
        }                                                                 \
    } while (0)
#else
#define X7T_MARK(ph) \
    do {             \
    } while (0)
#endif

constexpr int X7T = 128;           // threads = chunks per half row
constexpr int X7G = X7T * X3C;     // doubles per half-row slot (padded chunk layout)
constexpr int X7N = 2 * X7T * LCH; // row length (4096)

struct X7Args {
    CUtensorMap tm_in, tm_out, tm_piv;  // TMA: the batch in / out and the x pivots as rows of 16 doubles
    const double *in;
    double *out;
    long long vol;        // slice stride (= n^2)
    long long nrows;      // rows in the batch (B * 4096)
    int nstates;          // B
    int nranges;          // > 0: state-fastest row ranges (as xpass3); 0: contiguous
    double tau, h2inv, creact, src_amp;
    const double *sinpi;
    TimeArgs ta;
    CoefTab tab;
    const double *invd, *s2n, *s2f;
};

constexpr int X7S = X7T * LCH;      // doubles per half-row slot (TMA: unpadded, swizzled)
inline size_t xpass7_smem_bytes(int coef, int tma) {
    if (tma) return sizeof(double) * ((size_t)6 * X7S) + 1024 + 8 * 16;
    return sizeof(double) * ((size_t)(4 + (coef ? 2 : 1)) * X7G) + 8 * 16;
}

template <int COEF, int DR, int SRC, int TMA>
__global__ void __launch_bounds__(X7T, 2) xpass7_kernel(const __grid_constant__ X7Args a) {
    extern __shared__ __align__(16) double smem_raw[];
    // TMA: slots 1024-byte aligned (the 128-byte swizzle atom)
    double *smem = TMA ? reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023)
                       : smem_raw;
    constexpr int SLOT = TMA ? X7S : X7G;  // doubles per slot
    double *ubuf = smem;                     // 4 half-row state slots
    double *ibuf = smem + 4 * SLOT;          // 2 pivot slots (COEF; the output staging after the walks),
                                             // else 1 staging slot (TMA: 2)
    double2 *scr = reinterpret_cast<double2 *>(smem + (4 + ((COEF || TMA) ? 2 : 1)) * SLOT);  // [4] fwd, [4] bwd
    __shared__ __align__(8) unsigned long long mbu[4], mbp[2];  // TMA: one per ring slot
    __shared__ __align__(16) double2 xin;    // message from the partner CTA
    __shared__ __align__(8) unsigned long long mbx;
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank();
    const int k = threadIdx.x, lane = k & 31, warp = k >> 5;
    constexpr int NW = X7T / 32;
    const int e0 = (crank * X7T + k) * LCH;  // x-range of this thread's chunk
    const int n = X7N;

    if (k == 0) {
        mbar_init(&mbx, 1);
        if (TMA) {
            for (int i = 0; i < 4; ++i) mbar_init(mbu + i, 1);
            for (int i = 0; i < 2; ++i) mbar_init(mbp + i, 1);
        }
        mbar_fence_init();
    }
    // ---- per-thread x-dependent data ----
    double sf[LCH + 1], sxn[LCH], spi[LCH], tm[LCH], tid_[LCH], tcc[LCH];
#pragma unroll
    for (int i = 0; i <= LCH; ++i) sf[i] = COEF ? __ldg(a.s2f + e0 + i) : 0.0;
#pragma unroll
    for (int i = 0; i < LCH; ++i) {
        sxn[i] = (COEF && DR) ? __ldg(a.s2n + e0 + i) : 0.0;
        spi[i] = SRC ? __ldg(a.sinpi + e0 + i) : 0.0;
        tm[i] = COEF ? 0.0 : __ldg(a.tab.m + e0 + i);
        tid_[i] = COEF ? 0.0 : __ldg(a.tab.id + e0 + i);
        tcc[i] = COEF ? 0.0 : __ldg(a.tab.cc + e0 + i);
    }
    cl.sync();  // both mbarriers initialised before any message

    const long long G = a.nrows;
    const long long ncl = gridDim.x / 2, clid = blockIdx.x / 2;
    const long long ntasks = a.nranges ? (long long)a.nranges * a.nstates : ncl;
    const double tauh = a.tau * a.h2inv;
    const long long hoff = (long long)crank * (X7T * LCH);  // this CTA's half of a row
    unsigned rowpar = 0;  // parity of the incoming message of the current row
#ifdef PRS_X7_TIMING
    unsigned long long tacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tlast = clock64();
#endif

    // offset (doubles) of 16-byte unit u of chunk c within a slot
    auto uoff = [&](int c, int u) { return TMA ? c * LCH + ((u ^ (c & 7)) << 1) : c * X3C + 2 * u; };
    auto issue_group = [&](const double *rowp, double *dst) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int p = k + q * X7T;        // 16-byte pair within the half row, 0..1023
            const int c = p >> 3, u = p & 7;  // chunk, 16-byte unit
            cp_async16(dst + c * X3C + 2 * u, rowp + hoff + 2 * p);
        }
    };
    auto ub = [&](long long g) { return ubuf + (int)(g & 3) * SLOT; };
    auto ib = [&](long long g) { return ibuf + ((COEF || TMA) ? (int)(g & 1) : 0) * SLOT; };
    // TMA: tensor row (128-byte row = chunk) of this CTA's half of batch row g / pivot row j
    auto trow_state = [&](long long g) { return (g >> 12) * (a.vol / LCH) + (g & 4095) * (X7N / LCH) + crank * X7T; };
    auto tma_load = [&](const CUtensorMap *tm, long long tr, double *dst, unsigned long long *mb) {
        PRS_CHECK(dst >= smem && dst + X7S <= smem + 6 * X7S && ((reinterpret_cast<uintptr_t>(dst) & 1023) == 0),
                  "xpass7 TMA destination outside the 1024-aligned slots");
        PRS_CHECK(tr >= 0 && tr + X7T <= a.nrows * (X7N / LCH), "xpass7 TMA row");
        mbar_arrive_expect(mb, (unsigned)(X7S * sizeof(double)));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
                "r"(smem_u32(dst)),
            "l"(reinterpret_cast<uint64_t>(tm)), "r"(0), "r"((int)tr), "r"(smem_u32(mb))
            : "memory");
    };
    auto issue_state = [&](long long g) {
        if (TMA) {
            if (k == 0) tma_load(&a.tm_in, trow_state(g), ub(g), mbu + (g & 3));
        } else {
            issue_group(a.in + (g >> 12) * a.vol + (g & 4095) * (long long)n, ub(g));
        }
    };
    auto issue_piv = [&](long long g) {
        if (TMA) {
            if (k == 0) tma_load(&a.tm_piv, (g & 4095) * (X7N / LCH) + crank * X7T, ib(g), mbp + (g & 1));
        } else {
            issue_group(a.invd + (g & 4095) * (long long)n, ib(g));
        }
    };
    // TMA: every thread waits once on every fill, in issue order; bits = parity of each slot's next fill
    unsigned upar = 0, ppar = 0;
    long long wr = 0, wlast = -1;  // next state row to wait for, last row issued in this task
    auto wait_rows = [&](long long upto) {
        for (; wr <= upto && wr <= wlast; ++wr) {
            const int sl = (int)(wr & 3);
            mbar_wait(mbu + sl, (upar >> sl) & 1u);
            upar ^= 1u << sl;
        }
    };

    struct LineScalars {
        double kfm, kfp, hsx, srcf, idm1;
    };
    auto line_scalars = [&](long long gg) {
        LineScalars s{1.0, 1.0, 0.0, 0.0, 0.0};
        if (gg >= G) return s;
        const int jj = (int)(gg & 4095);
        if (DR && COEF) {
            s.kfm = __ldg(a.s2f + jj);
            s.kfp = __ldg(a.s2f + jj + 1);
        }
        if (COEF) {
            s.hsx = __ldg(a.s2n + jj);
            // the pivot before this CTA's first point (the partner's last one) for chunk 0
            if (crank == 1 && k == 0) s.idm1 = __ldg(a.invd + (long long)jj * n + hoff - 1);
        }
        if (SRC) s.srcf = a.tau * a.src_amp * src_tf(a.ta, gg >> 12) * __ldg(a.sinpi + jj);
        return s;
    };

    for (long long task = clid; task < ntasks; task += ncl) {
        long long g0, g1;
        if (a.nranges) {
            const long long Gs = G / a.nstates;
            const long long b = task % a.nstates, r = task / a.nstates;
            g0 = b * Gs + (r * Gs) / a.nranges;
            g1 = b * Gs + ((r + 1) * Gs) / a.nranges;
        } else {
            const long long per = G / ncl, rem = G % ncl;
            g0 = task * per + min(task, rem);
            g1 = g0 + per + (task < rem ? 1 : 0);
        }
        __syncthreads();
        if (TMA && k == 0) {
            // the slots were last read by generic loads (and the staging slots by TMA stores)
            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        }
        if (g0 < g1) {
            wr = (DR && g0 > 0) ? g0 - 1 : g0;
            wlast = min(G - 1, g1 - 1 + (DR ? 1 : 0));
            if (DR && g0 > 0) issue_state(g0 - 1);
            issue_state(g0);
            if (COEF) issue_piv(g0);
            cp_async_commit();
            if (g0 + 1 <= wlast) issue_state(g0 + 1);
            cp_async_commit();
        }
        LineScalars nxt = line_scalars(g0);
        for (long long g = g0; g < g1; ++g) {
            const LineScalars cur = nxt;
            nxt = line_scalars(g + 1);
            // every generic access of the slots refilled below is behind the last barrier
            if (TMA && k == 0 && g > g0) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            if (g + 2 < G && g + 2 < g1 + (DR ? 1 : 0)) issue_state(g + 2);
            // (TMA: the pivots of row g + 1 go into the staging slot of row g - 1, after its store
            // has read it out -- issued after this row's first walk, below)
            if (!TMA && COEF && g + 1 < g1) issue_piv(g + 1);
            if (!TMA) cp_async_commit();
            X7T_MARK(8);  // scalars + issue
            if (TMA) {
                wait_rows(g + (DR ? 1 : 0));
                if (COEF) {
                    mbar_wait(mbp + (g & 1), (ppar >> (g & 1)) & 1u);
                    ppar ^= 1u << (g & 1);
                }
            } else {
                cp_async_wait<1>();
            }
            if (k == 0) mbar_arrive_expect(&mbx, 16);  // this row's incoming message
            X7T_MARK(0);  // wait for this row's copies
            if (!TMA) __syncthreads();
            X7T_MARK(1);  // barrier (cp.async: every thread's copies visible)

            const int j = (int)(g & 4095);
            const double *U = ub(g);
            double v[LCH], w[LCH];
            {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double2 x = *reinterpret_cast<const double2 *>(U + uoff(k, u));
                    v[2 * u] = x.x;
                    v[2 * u + 1] = x.y;
                }
            }
            if (DR) {  // w = tau A_y U (rows j -+ 1 of the same half, from the ring)
                const bool hm = j > 0, hp = j < n - 1;
                const double *um = ub(g - 1), *up = ub(g + 1);
                const double kfm = 0.5 * cur.kfm, kfp = 0.5 * cur.kfp;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double2 xm = hm ? *reinterpret_cast<const double2 *>(um + uoff(k, u)) : make_double2(0.0, 0.0);
                    const double2 xp = hp ? *reinterpret_cast<const double2 *>(up + uoff(k, u)) : make_double2(0.0, 0.0);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int i = 2 * u + h;
                        const double uu = v[i];
                        const double dm = h ? xm.y : xm.x, dp = h ? xp.y : xp.x;
                        const double km = COEF ? fma(sxn[i], kfm, 1.0) : 1.0;
                        const double kp = COEF ? fma(sxn[i], kfp, 1.0) : 1.0;
                        w[i] = a.tau * ((kp * (dp - uu) - km * (uu - dm)) * a.h2inv - a.creact * uu);
                        v[i] = uu + w[i];
                    }
                }
            }
            if (SRC) {
#pragma unroll
                for (int i = 0; i < LCH; ++i) v[i] = fma(cur.srcf, spi[i], v[i]);
            }
            double idr[LCH], idm1 = 0.0, hsx = 0.0;
            if (COEF) {
                const double *I = ib(g);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double2 x = *reinterpret_cast<const double2 *>(I + uoff(k, u));
                    idr[2 * u] = x.x;
                    idr[2 * u + 1] = x.y;
                }
                idm1 = (k > 0) ? I[uoff(k - 1, 7) + 1] : cur.idm1;
                hsx = 0.5 * cur.hsx;
            }
            X7T_MARK(2);  // loads + DR stencil
            auto af = [&](int i) { return -tauh * fma(hsx, sf[i], 1.0); };
            auto cm = [&](int i) { return COEF ? af(i) * (i == 0 ? idm1 : idr[i - 1]) : tm[i]; };
            auto cid = [&](int i) { return COEF ? idr[i] : tid_[i]; };
            auto ccc = [&](int i) { return COEF ? af(i + 1) * idr[i] : tcc[i]; };
            // F1 + forward scans: the CTA's composition, and (CTA 0) the y entering CTA 1
            double A = 1.0, B = 0.0;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                const double m = cm(i);
                B = fma(-m, B, v[i]);
                A = -m * A;
            }
            double EA, EB;
            seg_scan_fwd(A, B, 32, lane, EA, EB);
            if (lane == 31) scr[warp] = make_double2(A, B);
            __syncthreads();
            X7T_MARK(3);  // F1 + forward warp scan + barrier
            if (TMA && k == 0) {
                // the staging slot of row g - 1 (its store has read it out by now) takes the
                // pivots of row g + 1 (COEF), or row g + 1's output (barriers before it is written)
                asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                if (COEF && g + 1 < g1) {
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    issue_piv(g + 1);
                }
            }
            double Yc = 0.0;  // y entering this CTA's half
            if (crank == 0) {
                if (k == 0) {  // y at the end of the half from y = 0 at the row start -> CTA 1
                    double Yt = 0.0, At = 1.0;
#pragma unroll
                    for (int q = 0; q < NW; ++q) {
                        const double2 s = scr[q];
                        Yt = fma(s.x, Yt, s.y);
                        At *= s.x;
                    }
                    st_async_remote(&xin, &mbx, 1, make_double2(At, Yt));
                }
            } else {
                mbar_wait(&mbx, rowpar);
                Yc = xin.y;
            }
            X7T_MARK(4);  // forward message (send / wait)
            double Yw = Yc;
            for (int q = 0; q < warp; ++q) {
                const double2 s = scr[q];
                Yw = fma(s.x, Yw, s.y);
            }
            // F3
            double y = fma(EA, Yw, EB), Pb = 1.0, Qb = 0.0;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                y = fma(-cm(i), y, v[i]);
                v[i] = y;
                Qb = fma(Pb * cid(i), y, Qb);
                Pb *= -ccc(i);
            }
            double EP, EQ;
            seg_scan_bwd(Pb, Qb, 32, lane, EP, EQ);
            if (lane == 0) scr[NW + warp] = make_double2(Pb, Qb);
            __syncthreads();
            X7T_MARK(5);  // F3 + backward warp scan + barrier
            double Xc = 0.0;  // x after this CTA's half
            if (crank == 1) {
                if (k == 0) {  // x at this half's first point from x = 0 at the row end -> CTA 0
                    double Xt = 0.0, Pt = 1.0;
#pragma unroll
                    for (int q = NW - 1; q >= 0; --q) {
                        const double2 s = scr[NW + q];
                        Xt = fma(s.x, Xt, s.y);
                        Pt *= s.x;
                    }
                    st_async_remote(&xin, &mbx, 0, make_double2(Pt, Xt));
                }
            } else {
                mbar_wait(&mbx, rowpar);
                Xc = xin.y;
            }
            rowpar ^= 1u;
            X7T_MARK(6);  // backward message (send / wait)
            double Xw = Xc;
            for (int q = NW - 1; q > warp; --q) {
                const double2 s = scr[NW + q];
                Xw = fma(s.x, Xw, s.y);
            }
            // B3
            double x = fma(EP, Xw, EQ);
#pragma unroll
            for (int i = LCH - 1; i >= 0; --i) {
                x = fma(-ccc(i), x, cid(i) * v[i]);  // one fma on the chain (cid v off it)
                v[i] = DR ? x - w[i] : x;
            }
#ifdef PRS_X7_DIRECT
            {  // experiment: each thread stores its chunk (one 128-byte line) straight from registers
                double *o = a.out + (g >> 12) * a.vol + (long long)j * n + hoff + (long long)k * LCH;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    *reinterpret_cast<double2 *>(o + 2 * u) = make_double2(v[2 * u], v[2 * u + 1]);
            }
            __syncthreads();  // every read of ib(g), scr and xin is done before the slots are refilled
#else
            if (TMA) {
                // no barrier before the staging writes: the staging slot ib(g) held row g's pivots,
                // read into registers before this row's first barrier; the scratch totals of the
                // next row are written only after the barrier below, which every warp reaches past
                // its reads of this row's totals
                double *dst = ib(g);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    *reinterpret_cast<double2 *>(dst + uoff(k, u)) = make_double2(v[2 * u], v[2 * u + 1]);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> TMA reads
                __syncthreads();
                if (k == 0) {
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                                     reinterpret_cast<uint64_t>(&a.tm_out)),
                                 "r"(0), "r"((int)trow_state(g)), "r"(smem_u32(dst))
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                }
            } else {
            __syncthreads();  // every read of ib(g), scr and xin is done
            {
                double *dst = ib(g) + k * X3C;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    *reinterpret_cast<double2 *>(dst + 2 * u) = make_double2(v[2 * u], v[2 * u + 1]);
            }
            __syncthreads();
            {
                const double *src = ib(g);
                double *o = a.out + (g >> 12) * a.vol + (long long)j * n + hoff;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int p = k + q * X7T;
                    const int c = p >> 3, u = p & 7;
                    const double2 xx = *reinterpret_cast<const double2 *>(src + c * X3C + 2 * u);
                    *reinterpret_cast<double2 *>(o + 2 * p) = xx;
                }
            }
            __syncthreads();  // staging slot free before the next prefetch lands in it
            }
#endif
            X7T_MARK(7);  // B3 + staging + store
#ifdef PRS_X7_TIMING
            if (k == 0) tacc[9] += 1;
#endif
        }
        if (!TMA) cp_async_wait<0>();
    }
    if (TMA && k == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // stores done
#ifdef PRS_X7_TIMING
    if (k == 0)
        for (int p = 0; p < 10; ++p) atomicAdd(&g_x7_timing[crank][p], tacc[p]);
#endif
    cl.sync();  // neither CTA leaves while its partner may still address its shared memory
}

}  // namespace prs
