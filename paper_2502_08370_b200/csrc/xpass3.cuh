// xpass3.cuh -- persistent, software-pipelined x-line pass (contiguous axis) for n = 16 P,
// P a power of two <= 256 (c0-c3).  Same arithmetic as xpass.cuh (stage-1 RHS fused,
// chunk-parallel Thomas), organised for HBM streaming on B200:
//  * one CTA of 256 threads per SM, looping over groups of 256 chunks (= 4096 elements =
//    256/P consecutive lines); thread k always owns chunk k of the group, so its x-range,
//    and with it the x-dependent coefficient data (face sines, node sines, source sines),
//    stays in registers for the whole launch;
//  * group data (state rows, DR neighbour rows, per-point pivots) stream into shared memory
//    with cp.async 16-byte copies two groups ahead of the compute (ring of 4 state groups,
//    2 pivot groups), so HBM always has the next groups' bytes in flight;
//  * each thread moves its chunk into registers once (conflict-free LDS.128 thanks to a
//    stride-18 chunk layout), runs the three walks entirely in registers, and writes the
//    result back through shared memory for coalesced 16-byte stores.
// DR's neighbour rows come from the same ring (row j-1 / j+1 of the previous / next group),
// so every state row is read from HBM once per pass.
#pragma once
#include "common.cuh"

namespace prs {

constexpr int X3T = 256;        // threads per CTA = chunks per group
constexpr int X3C = 18;         // shared stride of a chunk (16 + 2 pad, 16-byte aligned pairs)
constexpr int X3G = X3T * X3C;  // doubles per group buffer

struct X3Args {
    const double *in;
    double *out;
    long long vol;        // points per state
    int n;                // line length = 16 P
    int P;                // chunks per line
    int lines_per_state;  // n^(dim-1)
    long long ngroups;    // batch * lines_per_state / (256 / P)
    int nstates;          // batch size B
    int nranges;          // > 0: each state's groups split into nranges contiguous ranges, tasks
                          // (range, state) taken round-robin with the state fastest, so CTAs
                          // running at the same time hold the same rows of different states and
                          // the per-point pivot rows they share hit L2; 0: one contiguous range
                          // of the whole batch per CTA
    int dim;
    int row0;             // 2-D: global row of the state's first line (a band of a state, SURVEY
                          // 8(e) space-parallel G); 0 for whole states
    double tau, h2inv, creact;
    double src_amp;
    const double *sinpi;
    TimeArgs ta;
    CoefTab tab;
    const double *invd, *s2n, *s2f;
};

inline size_t xpass3_smem_bytes(int coef) {
    return sizeof(double) * ((size_t)(4 + (coef ? 2 : 1)) * X3G) + sizeof(double2) * 16;
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Group copies: 8 16-byte cp.async per thread per group into the padded (stride-18) chunk
// layout.  (A TMA tensor-copy ring was measured ~3 % slower on c3: the pass is bound by its
// row latency chain, not by the copy issue.)
template <int COEF, int DR, int SRC>
__global__ void __launch_bounds__(X3T, 1) xpass3_kernel(const __grid_constant__ X3Args a) {
    extern __shared__ __align__(16) double smem[];
    constexpr int SLOT = X3G;  // doubles per ring slot
    // offset (doubles) of 16-byte unit u of chunk (row) r within a slot
    auto uoff = [&](int r, int u) { return r * X3C + 2 * u; };
    double *ubuf = smem;                          // 4 slots: ring of state groups
    double *ibuf = smem + 4 * SLOT;               // COEF: 2 pivot slots; else 1 out staging slot
    double2 *scr = reinterpret_cast<double2 *>(smem + (4 + (COEF ? 2 : 1)) * SLOT);
    const int k = threadIdx.x;
    const int P = a.P, n = a.n;
    const int lpg = X3T / P;  // lines per group
    const int l = k / P, t = k - l * P;
    const int lane = k & 31;
    const int Wd = P < 32 ? P : 32;
    const int tl = lane & (Wd - 1);
    const int e0 = t * LCH;  // x-range of this thread's chunk

    // ---- per-thread x-dependent data, loaded once ----
    double sf[LCH + 1], sxn[LCH], spi[LCH];
#pragma unroll
    for (int i = 0; i <= LCH; ++i) sf[i] = COEF ? __ldg(a.s2f + e0 + i) : 0.0;
#pragma unroll
    for (int i = 0; i < LCH; ++i) {
        sxn[i] = (COEF && DR) ? __ldg(a.s2n + e0 + i) : 0.0;
        spi[i] = SRC ? __ldg(a.sinpi + e0 + i) : 0.0;
    }
    double tm[LCH], tid_[LCH], tcc[LCH];  // constant-coefficient pivots of this chunk
#pragma unroll
    for (int i = 0; i < LCH; ++i) {
        tm[i] = COEF ? 0.0 : __ldg(a.tab.m + e0 + i);
        tid_[i] = COEF ? 0.0 : __ldg(a.tab.id + e0 + i);
        tcc[i] = COEF ? 0.0 : __ldg(a.tab.cc + e0 + i);
    }

    // ---- this CTA's ranges of groups ----
    const long long G = a.ngroups;
    const int lps_sh = __ffs(a.lines_per_state) - 1;  // lines per state is a power of two
    const long long group_elems = (long long)X3T * LCH;  // 4096 doubles per group (contiguous)
    const long long ntasks = a.nranges ? (long long)a.nranges * a.nstates : gridDim.x;
    for (long long task = blockIdx.x; task < ntasks; task += gridDim.x) {
    long long g0, g1;
    if (a.nranges) {
        const long long Gs = G / a.nstates;  // groups per state
        const long long b = task % a.nstates, r = task / a.nstates;
        g0 = b * Gs + (r * Gs) / a.nranges;
        g1 = b * Gs + ((r + 1) * Gs) / a.nranges;
    } else {
        const long long per = G / gridDim.x, rem = G % gridDim.x;
        g0 = task * per + min(task, rem);
        g1 = g0 + per + (task < rem ? 1 : 0);
    }
    __syncthreads();  // the previous range's buffers are free

    // issue the copies of group g into a slot (all threads)
    auto issue_group = [&](const double *src, long long g, double *dst) {
        const double *s = src + g * group_elems;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int p = k + q * X3T;    // pair index within the group, 0..2047
            const int c = p >> 3, u = p & 7;  // chunk, 16-byte unit within the chunk
            cp_async16(dst + c * X3C + 2 * u, s + 2 * p);
        }
    };
    // state groups are contiguous in memory across the whole batch: group g = elements
    // [g*4096, (g+1)*4096) of the batch buffer; a group never splits a line (n | 4096).
    const double *pin = a.in;
    auto ub = [&](long long g) { return ubuf + (int)(g & 3) * SLOT; };
    auto ib = [&](long long g) { return ibuf + (COEF ? (int)(g & 1) : 0) * SLOT; };
    auto issue_state = [&](long long g) { issue_group(pin, g, ub(g)); };
    // pivot rows repeat every state: the group of pivots for global group g starts at
    // row (g * lpg) mod lines_per_state
    auto issue_piv = [&](long long g) {
        const long long row0 = ((g * lpg) & (a.lines_per_state - 1)) + a.row0;
        issue_group(a.invd + row0 * n, 0, ib(g));
    };

    // prologue: U(g0-1) (DR halo), U(g0), U(g0+1), pivots(g0)
    if (g0 < g1) {
        if (DR && g0 > 0) issue_state(g0 - 1);
        issue_state(g0);
        if (COEF) issue_piv(g0);
        cp_async_commit();
        if (g0 + 1 < G) issue_state(g0 + 1);
        cp_async_commit();
    }

    const double tauh = a.tau * a.h2inv;
    // per-line scalars (y-face sines, the line's sine for kappa, the source factor) are
    // loaded / computed one group ahead so their latency is off the critical path
    struct LineScalars {
        double kfm, kfp, hsx, srcf;
    };
    // (raw loads only: the 0.5 factors are applied at the use, one group later, so no
    // instruction waits on these loads here)
    auto line_scalars = [&](long long gg) {
        LineScalars s{1.0, 1.0, 0.0, 0.0};
        if (gg >= G) return s;
        const long long gl = gg * lpg + l;
        const long long bs = gl >> lps_sh;
        const int jj = (int)(gl & (a.lines_per_state - 1)) + a.row0;
        if (DR && COEF) {
            s.kfm = __ldg(a.s2f + jj);
            s.kfp = __ldg(a.s2f + jj + 1);
        }
        if (COEF) s.hsx = __ldg(a.s2n + ((a.dim == 2) ? jj : jj % n));
        if (SRC) {
            const double ampt = a.src_amp * src_tf(a.ta, bs);
            const double sj =
                (a.dim == 2) ? __ldg(a.sinpi + jj) : __ldg(a.sinpi + jj % n) * __ldg(a.sinpi + jj / n);
            s.srcf = a.tau * ampt * sj;
        }
        return s;
    };
    LineScalars nxt = line_scalars(g0);
    for (long long g = g0; g < g1; ++g) {
        const LineScalars cur = nxt;
        nxt = line_scalars(g + 1);
        // prefetch two ahead (state) / one ahead (pivots)
        if (g + 2 < G && g + 2 < g1 + (DR ? 1 : 0)) issue_state(g + 2);
        if (COEF && g + 1 < g1) issue_piv(g + 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();

        // line of this thread: global line index, state, row
        const long long gl = g * lpg + l;
        const int j = (int)(gl & (a.lines_per_state - 1));
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
        if (DR) {  // w = tau A_y U with rows j-1, j+1 from the ring (2-D)
            const bool hm = j > 0, hp = j < n - 1;
            // rows (chunks) of the neighbour lines in this group's slot or the previous / next one
            const double *ums = (l > 0) ? U : ub(g - 1);
            const double *ups = (l < lpg - 1) ? U : ub(g + 1);
            const int rm = (l > 0) ? k - P : k - P + X3T, rp = (l < lpg - 1) ? k + P : k + P - X3T;
            const double kfm = 0.5 * cur.kfm, kfp = 0.5 * cur.kfp;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double2 xm = hm ? *reinterpret_cast<const double2 *>(ums + uoff(rm, u)) : make_double2(0.0, 0.0);
                const double2 xp = hp ? *reinterpret_cast<const double2 *>(ups + uoff(rp, u)) : make_double2(0.0, 0.0);
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
            const double f = cur.srcf;
#pragma unroll
            for (int i = 0; i < LCH; ++i) v[i] = fma(f, spi[i], v[i]);
        }
        // coefficients of this chunk: constant tables, or off-diagonals from the face sines
        // (registers) times the per-point inverse pivots of this group
        double idr[LCH], idm1 = 0.0, hsx = 0.0;
        if (COEF) {
            const double *I = ib(g);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double2 x = *reinterpret_cast<const double2 *>(I + uoff(k, u));
                idr[2 * u] = x.x;
                idr[2 * u + 1] = x.y;
            }
            idm1 = (t > 0) ? I[uoff(k - 1, 7) + 1] : 0.0;  // last element of the previous chunk
            hsx = 0.5 * cur.hsx;
        }
        auto af = [&](int i) { return -tauh * fma(hsx, sf[i], 1.0); };
        auto cm = [&](int i) { return COEF ? af(i) * (i == 0 ? idm1 : idr[i - 1]) : tm[i]; };
        auto cid = [&](int i) { return COEF ? idr[i] : tid_[i]; };
        auto ccc = [&](int i) { return COEF ? af(i + 1) * idr[i] : tcc[i]; };
        // F1
        double A = 1.0, B = 0.0;
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            const double m = cm(i);
            B = fma(-m, B, v[i]);
            A = -m * A;
        }
        double EA, EB;
        seg_scan_fwd(A, B, Wd, tl, EA, EB);
        double Yw = 0.0;
        if (P > 32) {
            const int warp = k >> 5, wib = t >> 5, wl0 = warp - wib;
            if (lane == 31) scr[warp] = make_double2(A, B);
            __syncthreads();
            for (int q = 0; q < wib; ++q) {
                const double2 s = scr[wl0 + q];
                Yw = fma(s.x, Yw, s.y);
            }
            __syncthreads();
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
        seg_scan_bwd(Pb, Qb, Wd, tl, EP, EQ);
        double Xw = 0.0;
        if (P > 32) {
            const int warp = k >> 5, wib = t >> 5, wl0 = warp - wib, nwl = P >> 5;
            if (lane == 0) scr[warp] = make_double2(Pb, Qb);
            __syncthreads();
            for (int q = nwl - 1; q > wib; --q) {
                const double2 s = scr[wl0 + q];
                Xw = fma(s.x, Xw, s.y);
            }
        }
        // B3
        double x = fma(EP, Xw, EQ);
#pragma unroll
        for (int i = LCH - 1; i >= 0; --i) {
            x = fma(-ccc(i), x, cid(i) * v[i]);
            v[i] = DR ? x - w[i] : x;
        }
        __syncthreads();  // every read of ib(g) / scr done
        {
            double *dst = ib(g);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                *reinterpret_cast<double2 *>(dst + uoff(k, u)) = make_double2(v[2 * u], v[2 * u + 1]);
        }
        __syncthreads();
        {
            const double *src = ib(g);
            double *o = a.out + g * group_elems;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int p = k + q * X3T;
                const int c = p >> 3, u = p & 7;
                const double2 xx = *reinterpret_cast<const double2 *>(src + uoff(c, u));
                *reinterpret_cast<double2 *>(o + 2 * p) = xx;
            }
        }
        __syncthreads();  // staging buffer free before the next prefetch lands in it
    }
    cp_async_wait<0>();
    }  // tasks
}

}  // namespace prs
