// sweep2.cuh -- the whole fine sweep F^s of a small 2-D slice on chip (kappa = 1,
// n = 32 CL with CL = 1, 2, 4, 8 CTAs per cluster; c0: n = 32, c1 / c1p: n = 256).
//
// F^s is s FIE or DR steps of delta t.  For small states the per-step kernels
// are latency-bound (c1: 36 us per step for 32 slices of 512 KB, L2-resident).  Here one cluster
// of CL CTAs holds one slice for all s steps: each CTA keeps 32 rows in shared memory, so the
// state is read once at the start and Delta_n = F^s(U) - G(U) written once at the end.
// Per step (PAPER.md:153-157 FIE, 167-171 DR in the M = 2 form of DESIGN.md R1):
//  * x stage: rows are CTA-local; r_1 = U (+ tau A_y U for DR: rows j +- 1 of the neighbour
//    CTAs arrive as st.async messages into a parity slot, completing on this CTA's mbarrier)
//    (+ tau F); chunk-parallel Thomas with segmented warp scans over the CH = n/16 chunks of a
//    row; r_2 = V_1 (- w) in place;
//  * y stage: columns cross the cluster: each thread walks 16-row chunks (lpass4.cuh 5-tuples),
//    the CTA totals per column (double-buffered by step parity) are read through distributed
//    shared memory after the step's one cluster barrier (every CTA composes the totals of the
//    CTAs before and after it), then the exact recurrences.
// Pivot tables (kappa = 1: the same for x and y) sit chunk-padded in shared memory.
// CHAIN = 1 reuses the step for the coarse chain of the parareal correction:
// one cluster advances U_i -> G(U_i) slice after slice with the state on chip, applying the
// fused correction (G cache, U_{i+1} = G(U_i) + Delta_i, update max, non-finite flag) after
// every step; the initial guess (EPI_INIT) likewise.
#pragma once
#include "common.cuh"
#include "lpass.cuh"
#include "lpass4.cuh"

namespace prs {

constexpr int SW_R = 32;   // rows per CTA
constexpr int SW_T = 256;  // threads per CTA

struct SWArgs {
    const double *in;     // fine sweep: U^k_n of the batch (slice stride vol); chain: U_{i0}
    double *out;          // Delta_n (EPI_DELTA) or F^s(U) (EPI_STORE)
    const double *gc;     // G cache (EPI_DELTA)
    // coarse chain (CHAIN = 1): one cluster runs the s G steps of slices i0 .. i0+s-1 in turn,
    // U_{i+1} <- G(U_i) (+ Delta_i, EPI_CORRECT), the G cache of slice i <- G(U_i)
    double *traj;         // U_i of local slice i at traj + i vol
    const double *trajold;  // U^k_i for the update norm when it is not in traj (pipelined
                            // parareal: the previous iterate lives in the other parity buffer)
    double *gcache;
    const double *delta;
    unsigned long long *red;  // [0] max |update| bits, [1] non-finite flag (EPI_CORRECT)
    long long vol;
    int s;                // fine steps
    double tau, h2inv, creact, src_amp;
    const double *sinpi;
    long long slice0;     // global slice index of batch state 0
    long long sstride;    // global slice stride between batch states (1; P under cyclic ownership)
    double dt;
    CoefTab tab;          // kappa = 1 pivots of (I - tau A_d), length n
};

// n = 256: each thread owns both 16-row chunks of its column, so the chunk tuples and the
// per-column boundary values stay in registers (no chk / yxb buffers: 2 CTAs per SM fit)
template <int N>
constexpr bool sweep2_own_column() { return N == SW_T; }
template <int N>
constexpr size_t sweep2_smem_doubles() {
    return (size_t)SW_R * (N + N / LCH) + 3 * (N + N / LCH) + (sweep2_own_column<N>() ? 0 : 5 * 2 * N + 2 * N) +
           2 * 5 * N + 2 * 2 * (N + N / LCH);
}

template <int N, int DR, int SRC, int EPI, int CHAIN = 0>
__global__ void __launch_bounds__(SW_T, 2) sweep2_kernel(SWArgs a) {
    constexpr int CL = N / SW_R;      // CTAs per slice
    constexpr int S = N + N / LCH;    // padded row stride
    constexpr int CH = N / LCH;       // chunks per row
    constexpr int XT = SW_R * CH;     // x tasks (row, chunk)
    constexpr int YT = 2 * N;         // y tasks (column, chunk of 16 rows)
    extern __shared__ __align__(16) double sm[];
    double *tile = sm;                          // 32 x S
    double *tb = tile + SW_R * S;               // [3][S] m, id, cc (chunk-padded)
    constexpr bool OWN = sweep2_own_column<N>();
    double *ctot0 = tb + 3 * S;                 // [parity][5][N] this CTA's column totals (read remotely)
    double *ein = ctot0 + 2 * 5 * N;            // [parity][2][S] the neighbours' edge rows (DR halo): [0] the
                                                // row above this CTA's first, [1] the row below its last
    double *chk = ein + 2 * 2 * S;              // (!OWN) [5][2][N] chunk tuples (y)
    double *yxb = chk + 5 * 2 * N;              // (!OWN) [2][N] y entering / x leaving this CTA
    __shared__ __align__(8) unsigned long long mbe;  // edge rows received (DR)
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31;
    const long long b = blockIdx.x / CL;
    const int r0 = crank * SW_R;  // first global row of this CTA
    const long long base = b * a.vol + (long long)r0 * N;
    constexpr bool HALO = DR && CL > 1;
    const unsigned ebytes = (unsigned)(((crank > 0) + (crank < CL - 1)) * N * sizeof(double));
    if (HALO && tid == 0) {
        mbar_init(&mbe, 1);
        mbar_fence_init();
        mbar_arrive_expect(&mbe, ebytes);  // step 0's halo rows
    }
    if (HALO) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");

    for (int e = tid; e < N; e += SW_T) {
        tb[cpad(e)] = __ldg(a.tab.m + e);
        tb[S + cpad(e)] = __ldg(a.tab.id + e);
        tb[2 * S + cpad(e)] = __ldg(a.tab.cc + e);
    }
    for (int e = tid; e < SW_R * N / 2; e += SW_T) {
        const int r = e / (N / 2), x2 = (e % (N / 2)) * 2;
        const double2 v = __ldg(reinterpret_cast<const double2 *>(a.in + base + (long long)r * N + x2));
        double *d = tile + r * S + cpad(x2);
        d[0] = v.x;
        d[1] = v.y;
    }
    // DR halo: this CTA's first row goes to the CTA above (its "row below"), its last row to
    // the CTA below (its "row above"), pushed with st.async into the receiver's parity slot and
    // completing on the receiver's mbarrier; a CTA waits only for its two neighbours
    auto send_edges = [&](int par) {
        for (int e = tid; e < N; e += SW_T) {  // (chunk-padded offsets: 8-byte messages)
            const int x = cpad(e);
            if (crank > 0) st_async_remote_f64(ein + par * 2 * S + S + x, &mbe, crank - 1, tile[x]);
            if (crank < CL - 1) st_async_remote_f64(ein + par * 2 * S + x, &mbe, crank + 1, tile[(SW_R - 1) * S + x]);
        }
    };
    __syncthreads();  // the whole tile is loaded
    if (HALO) {
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");  // neighbours' mbarriers initialised
        send_edges(0);
    }
    const double tauh = a.tau * a.h2inv, taucr = a.tau * a.creact;
    constexpr int NXT = (XT + SW_T - 1) / SW_T, NYT = (YT + SW_T - 1) / SW_T;
    double cdmax = 0.0;         // CHAIN, EPI_CORRECT: max |U^{k+1} - U^k| of this thread's points
    unsigned long long cbad = 0;

    for (int j = 0; j < a.s; ++j) {
        // (no cluster barrier here: the column totals are double-buffered by step parity, and
        // the halo rows arrive as messages)
        const int par = j & 1;
        double *ctot = ctot0 + par * 5 * N;
        if (HALO) {
            mbar_wait(&mbe, (unsigned)par);  // this step's halo rows have landed
            if (tid == 0 && j + 1 < a.s) mbar_arrive_expect(&mbe, ebytes);  // arm the next step's
        }
        // ---------------- x stage ----------------
        // (a) w = tau A_y U of every task (reads rows r-1, r+1, the neighbour CTAs' edge rows)
        double w[NXT][LCH];
#pragma unroll
        for (int k = 0; k < NXT; ++k) {
            const int q = tid + k * SW_T;
            if (!DR || q >= XT) break;
            const int r = q / CH, c = q % CH;
            const double *p = tile + r * S + c * LCP;
            // the neighbours' edge rows are local copies (parity of this step), so the in-place
            // solve below needs no cluster barrier before it
            const double *pm = (r > 0) ? p - S : (crank > 0 ? ein + par * 2 * S + c * LCP : nullptr);
            const double *pp = (r < SW_R - 1) ? p + S : (crank < CL - 1 ? ein + par * 2 * S + S + c * LCP : nullptr);
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                const double uu = p[i];
                const double dm = pm ? pm[i] : 0.0, dp = pp ? pp[i] : 0.0;
                w[k][i] = fma(tauh, (dp - uu) - (uu - dm), -taucr * uu);
            }
        }
        if (DR) __syncthreads();  // every read of other tasks' rows of this tile is done
        // (b) r_1 = U (+ w) (+ tau F) from the task's own region (untouched so far), solve, r_2 back
#pragma unroll
        for (int k = 0; k < NXT; ++k) {
            const int q = tid + k * SW_T;
            if (q >= XT) break;  // (uniform per warp: XT is a multiple of 32)
            const int r = q / CH, c = q % CH, tl = lane % CH;
            double *p = tile + r * S + c * LCP;
            double v[LCH];
#pragma unroll
            for (int i = 0; i < LCH; ++i) v[i] = DR ? p[i] + w[k][i] : p[i];
            if (SRC) {
                const double t = CHAIN ? (double)(a.slice0 + j + 1) * a.dt
                                       : (double)((a.slice0 + b * a.sstride) * a.s + j + 1) * a.dt;
                const double f = a.tau * a.src_amp * exp(-t) * __ldg(a.sinpi + r0 + r);
#pragma unroll
                for (int i = 0; i < LCH; ++i) v[i] = fma(f, __ldg(a.sinpi + c * LCH + i), v[i]);
            }
            const double *tm = tb + c * LCP, *ti = tb + S + c * LCP, *tc = tb + 2 * S + c * LCP;
            double A = 1.0, B = 0.0;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                B = fma(-tm[i], B, v[i]);
                A = -tm[i] * A;
            }
            double EA, EB;
            seg_scan_fwd(A, B, CH, tl, EA, EB);
            double y = EB, Pb = 1.0, Qb = 0.0;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                y = fma(-tm[i], y, v[i]);
                v[i] = y;
                Qb = fma(Pb * ti[i], y, Qb);
                Pb *= -tc[i];
            }
            double EP, EQ;
            seg_scan_bwd(Pb, Qb, CH, tl, EP, EQ);
            double x = EQ;
#pragma unroll
            for (int i = LCH - 1; i >= 0; --i) {
                x = fma(-tc[i], x, ti[i] * v[i]);
                p[i] = DR ? x - w[k][i] : x;
            }
        }
        __syncthreads();
        // ---------------- y stage ----------------
        Tup tu[NYT];
        auto ym = [&](int t, int i) { return tb[cpad(r0 + t * LCH) + i]; };
        auto yi = [&](int t, int i) { return tb[S + cpad(r0 + t * LCH) + i]; };
        auto yc = [&](int t, int i) { return tb[2 * S + cpad(r0 + t * LCH) + i]; };
#pragma unroll
        for (int k = 0; k < NYT; ++k) {
            const int q = tid + k * SW_T;
            if (q >= YT) break;
            const int col = q % N, t = q / N;
            const double *p = tile + (t * LCH) * S + cpad(col);
            double y0 = 0.0, g = 1.0, cp = 1.0, Q = 0.0, R = 0.0;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                const double m = ym(t, i);
                y0 = fma(-m, y0, p[i * S]);
                g = -m * g;
                const double cid = cp * yi(t, i);
                Q = fma(cid, y0, Q);
                R = fma(cid, g, R);
                cp *= -yc(t, i);
            }
            tu[k] = Tup{g, y0, cp, Q, R};
            if (!OWN) {
                chk[(0 * 2 + t) * N + col] = g;
                chk[(1 * 2 + t) * N + col] = y0;
                chk[(2 * 2 + t) * N + col] = cp;
                chk[(3 * 2 + t) * N + col] = Q;
                chk[(4 * 2 + t) * N + col] = R;
            }
        }
        if (!OWN) __syncthreads();
        auto getc = [&](int t, int col) {
            return Tup{chk[(0 * 2 + t) * N + col], chk[(1 * 2 + t) * N + col], chk[(2 * 2 + t) * N + col],
                       chk[(3 * 2 + t) * N + col], chk[(4 * 2 + t) * N + col]};
        };
        for (int col = tid; col < N; col += SW_T) {
            const Tup tot = OWN ? tup_cat(tu[0], tu[1]) : tup_cat(getc(0, col), getc(1, col));
            ctot[col] = tot.A;
            ctot[N + col] = tot.B;
            ctot[2 * N + col] = tot.P;
            ctot[3 * N + col] = tot.Q;
            ctot[4 * N + col] = tot.R;
        }
        cl.sync();  // every CTA's column totals visible
        double Yown = 0.0, Xown = 0.0;  // (OWN) y entering / x leaving this CTA for column tid
        for (int col = tid; col < N; col += SW_T) {
            // y entering each CTA (compile-time indices only: the array stays in registers)
            double yin[CL];
            double Y = 0.0, Ymine = 0.0;
#pragma unroll
            for (int q = 0; q < CL; ++q) {
                yin[q] = Y;
                if (q == crank) Ymine = Y;
                const double *ct = cl.map_shared_rank(ctot, q);
                Y = fma(ct[col], Y, ct[N + col]);
            }
            double X = 0.0;
#pragma unroll
            for (int q = CL - 1; q >= 1; --q) {
                if (q > crank) {
                    const double *ct = cl.map_shared_rank(ctot, q);
                    X = fma(ct[2 * N + col], X, fma(ct[4 * N + col], yin[q], ct[3 * N + col]));
                }
            }
            if (OWN) {
                Yown = Ymine;
                Xown = X;
            } else {
                yxb[col] = Ymine;
                yxb[N + col] = X;
            }
        }
        if (!OWN) __syncthreads();
#pragma unroll
        for (int k = 0; k < NYT; ++k) {
            const int q = tid + k * SW_T;
            if (q >= YT) break;
            const int col = q % N, t = q / N;
            double Y = OWN ? Yown : yxb[col];
            if (t == 1) {
                const Tup g0 = OWN ? tu[0] : getc(0, col);
                Y = fma(g0.A, Y, g0.B);
            }
            const double Ylast = fma(tu[k].A, Y, tu[k].B);
            double X = OWN ? Xown : yxb[N + col];
            if (t == 0) {
                const Tup g1 = OWN ? tu[NYT - 1] : getc(1, col);
                X = fma(g1.P, X, fma(g1.R, Ylast, g1.Q));
            }
            // (the task's own column chunk is still r_2: re-read it, walk forward in place,
            // then backward)
            double *p = tile + (t * LCH) * S + cpad(col);
            double y = Y;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                y = fma(-ym(t, i), y, p[i * S]);
                p[i * S] = y;
            }
            double x = X;
#pragma unroll
            for (int i = LCH - 1; i >= 0; --i) {
                x = fma(-yc(t, i), x, yi(t, i) * p[i * S]);
                p[i * S] = x;
            }
        }
        __syncthreads();
        if (CHAIN) {
            // the correction of slice j: g = G(U_j) in the tile; the G cache,
            // U_{j+1} = g + Delta_j (EPI_CORRECT) or g (EPI_INIT); the tile carries U_{j+1} on
            for (int e = tid; e < SW_R * N / 2; e += SW_T) {
                const int r = e / (N / 2), x2 = (e % (N / 2)) * 2;
                double *d = tile + r * S + cpad(x2);
                const long long off = (long long)r0 * N + (long long)r * N + x2;
                const double2 gv = make_double2(d[0], d[1]);
                *reinterpret_cast<double2 *>(a.gcache + (long long)j * a.vol + off) = gv;
                double2 nv = gv;
                if (EPI == EPI_CORRECT) {
                    const double2 dv = *reinterpret_cast<const double2 *>(a.delta + (long long)j * a.vol + off);
                    const double2 ov = *reinterpret_cast<const double2 *>((a.trajold ? a.trajold : a.traj) +
                                                                         (long long)(j + 1) * a.vol + off);
                    nv.x += dv.x;
                    nv.y += dv.y;
                    cdmax = fmax(cdmax, fmax(fabs(nv.x - ov.x), fabs(nv.y - ov.y)));
                    if (!isfinite(nv.x) || !isfinite(nv.y)) cbad = 1;
                    d[0] = nv.x;
                    d[1] = nv.y;
                }
                *reinterpret_cast<double2 *>(a.traj + (long long)(j + 1) * a.vol + off) = nv;
            }
            __syncthreads();
        }
        // this step's edge rows into the neighbours' other parity slot (read in step j + 1; the
        // slot read in step j is not touched)
        if (HALO && j + 1 < a.s) send_edges(par ^ 1);
    }
    cl.sync();  // no CTA leaves while a neighbour may still read its shared memory
    if (CHAIN) {
        if (EPI == EPI_CORRECT) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                cdmax = fmax(cdmax, __shfl_xor_sync(0xffffffffu, cdmax, off));
                cbad |= __shfl_xor_sync(0xffffffffu, cbad, off);
            }
            if (lane == 0) {
                atomicMax(a.red, (unsigned long long)__double_as_longlong(cdmax));
                if (cbad) atomicOr(a.red + 1, 1ull);
            }
        }
        return;
    }
    // ---- F^s(U) (or Delta_n = F^s(U) - G(U)) ----
    for (int e = tid; e < SW_R * N / 2; e += SW_T) {
        const int r = e / (N / 2), x2 = (e % (N / 2)) * 2;
        const double *d = tile + r * S + cpad(x2);
        const long long g = base + (long long)r * N + x2;
        double2 o = make_double2(d[0], d[1]);
        if (EPI == EPI_DELTA) {
            const double2 gcv = __ldg(reinterpret_cast<const double2 *>(a.gc + g));
            o.x -= gcv.x;
            o.y -= gcv.y;
        }
        *reinterpret_cast<double2 *>(a.out + g) = o;
    }
}

}  // namespace prs
