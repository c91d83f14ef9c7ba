// common.cuh -- building blocks of the chunk-parallel Thomas line solves (sm_100a).
//
// A stage of FIE / DR under dimensional splitting is a batch of independent tridiagonal
// systems (I - tau A_d) v = r along every grid line of axis d.  Each line is
// solved with precomputed pivots:
//   forward   y_i = r_i - m_i y_{i-1}                (m_i = a_i / d_{i-1})
//   backward  x_i = id_i y_i - cc_i x_{i+1}          (id_i = 1/d_i, cc_i = c_i / d_i)
// Both recurrences are affine maps, so a line is cut into chunks of LCH elements, one thread
// per chunk: (F1) each thread composes the maps of its chunk, (F2) an exclusive scan of the
// compositions over the chunks gives each chunk its incoming y, (F3) each thread runs the
// exact sequential forward recurrence over its chunk from that value while composing the
// backward maps, (B2) a reverse scan gives the incoming x, (B3) the exact sequential backward
// recurrence.  Lines and coefficient tables live in shared memory in a chunk-padded layout
// (element e at e + e/LCH, i.e. chunk t at [17t, 17t+16) with one pad slot; odd strides):
// the coalesced global<->shared copies and the per-thread chunk walks are then both
// bank-conflict free, and a walk addresses its chunk with compile-time offsets from one base
// pointer.  The boundary couplings (m at the line start, cc at the line end) only ever
// multiply y_{-1} = 0 or x_n = 0, so they need no special case, only to be finite.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

namespace prs {
namespace cg = cooperative_groups;

// Checked build (-DPRS_CHECKS, libprs_chk.so; compute-sanitizer is not available on the GPU
// pool): bounds of every shared-memory async-copy destination and scratch index of the async
// paths, and bounded waits on every mbarrier -- a violated check or a wait that outlives any
// legitimate one prints where and traps (the launch fails with an error instead of corrupting
// memory or hanging the device).  Production builds compile the checks away.
#ifdef PRS_CHECKS
#define PRS_CHECK(cond, what)                                                                       \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            printf("PRS_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,   \
                   (int)blockIdx.x, (int)threadIdx.x);                                              \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#else
#define PRS_CHECK(cond, what) \
    do {                      \
    } while (0)
#endif

constexpr int LCH = 16;  // elements per chunk (per thread per line)
constexpr int LCP = LCH + 1;  // padded chunk stride
constexpr int QG = 4;    // 16-byte loads issued per thread before first use

__host__ __device__ inline int cpad(int e) { return e + e / LCH; }
// odd shared-memory stride holding a chunk-padded line of `len` elements
inline int cpad_host(int len) {
    const int s = (len <= 0) ? 1 : (len - 1) + (len - 1) / LCH + 1;
    return s | 1;
}
__host__ __device__ inline size_t even_up(size_t x) { return (x + 1) & ~(size_t)1; }

__device__ __forceinline__ double2 ld2(const double *p) { return *reinterpret_cast<const double2 *>(p); }
__device__ __forceinline__ void st2(double *p, double x, double y) {
    *reinterpret_cast<double2 *>(p) = make_double2(x, y);
}

// Pivot tables of a constant-coefficient stage matrix along one axis (length n each, global).
struct CoefTab {
    const double *m, *id, *cc;
};

// Source time of state b of a launch: t = ((slice0 + b sstride) * tmul + toff) * tstep
// (fine step j of slice n: ((n s + j + 1) delta t), coarse: ((n + 1) Delta T); R2;
// sstride = P when a rank owns every P-th slice, cyclic ownership)
struct TimeArgs {
    long long slice0 = 0, tmul = 0, toff = 0;
    double tstep = 0.0;
    long long sstride = 1;
    int gk = 0;        // source time factor: 0 e^{-t} (source_kind 1), 1 the section-5.1 solution's
    double gc = 0.0;   // (source_kind 2): 2 pi cos(2 pi t) + gc sin(2 pi t), gc = 8 pi^2 + c
};
__device__ __forceinline__ double src_time(const TimeArgs &ta, long long b) {
    return (double)((ta.slice0 + b * ta.sstride) * ta.tmul + ta.toff) * ta.tstep;
}
// time factor of the source of state b (times src_amp and the spatial sine product):
// source_kind 1: f = (dim pi^2 + c - 1) e^{-t} prod sin(pi x_d)  (u = e^{-t} prod sin(pi x_d));
// source_kind 2: f = (2 pi cos 2 pi t + (8 pi^2 + c) sin 2 pi t) sin(2 pi x) sin(2 pi y), the
// solution u = sin(2 pi t) sin(2 pi x) sin(2 pi y) of PAPER.md:444-445 with D = I (src_amp = 1)
__device__ __forceinline__ double src_tf(const TimeArgs &ta, long long b) {
    const double t = src_time(ta, b);
    return ta.gk == 0 ? exp(-t) : fma(2.0 * M_PI, cospi(2.0 * t), ta.gc * sinpi(2.0 * t));
}

// Copy `len` doubles of a global table into chunk-padded shared memory (whole CTA).
__device__ __forceinline__ void stage_table(double *dst, const double *src, int len) {
    for (int i = threadIdx.x; i < len; i += blockDim.x) dst[cpad(i)] = __ldg(src + i);
}

// ------------------------------------------------ per-chunk coefficient views ------
// M(i): m of chunk element i; ID(i): id; CC(i): cc  (i is a compile-time offset 0..LCH-1).
struct ConstView {  // kappa = 1: chunk-padded shared tables, shared by every line of the axis
    const double *m, *id, *cc;  // already offset to the chunk
    __device__ __forceinline__ double M(int i) const { return m[i]; }
    __device__ __forceinline__ double ID(int i) const { return id[i]; }
    __device__ __forceinline__ double CC(int i) const { return cc[i]; }
};
// kappa = 1 + 0.5 sin(2 pi x) sin(2 pi y): off-diagonal a(face) = -tau/h^2 (1 + 0.5 sx sf(face))
// with sf the chunk-padded face sines (sf[i] = face left of element i; sf[17] = face right of
// element 15), sd the chunk-padded per-point inverse pivots, idm1 = id of the element before.
struct VarView {
    const double *sd, *sf;
    double hsx, ntauh, idm1;
    __device__ __forceinline__ double a(int i) const { return ntauh * fma(hsx, sf[i + (i >> 4)], 1.0); }
    __device__ __forceinline__ double M(int i) const { return a(i) * (i == 0 ? idm1 : sd[i - 1]); }
    __device__ __forceinline__ double ID(int i) const { return sd[i]; }
    __device__ __forceinline__ double CC(int i) const { return a(i + 1) * sd[i]; }
};

// ------------------------------------------------------------- chunk walks ---------
// FULL: every thread of the warp owns LCH elements (no predication); else cnt elements.
template <bool FULL, class V>
__device__ __forceinline__ void walk_f1(const double *sp, int cnt, const V &v, double &A, double &B) {
    A = 1.0;
    B = 0.0;
#pragma unroll
    for (int i = 0; i < LCH; ++i)
        if (FULL || i < cnt) {
            const double m = v.M(i);
            B = fma(-m, B, sp[i]);
            A = -m * A;
        }
}
template <bool FULL, class V>
__device__ __forceinline__ void walk_f3(double *sp, int cnt, const V &v, double yin, double &Pb, double &Qb) {
    double y = yin;
    Pb = 1.0;
    Qb = 0.0;
#pragma unroll
    for (int i = 0; i < LCH; ++i)
        if (FULL || i < cnt) {
            y = fma(-v.M(i), y, sp[i]);
            sp[i] = y;
            Qb = fma(Pb * v.ID(i), y, Qb);
            Pb *= -v.CC(i);
        }
}
template <bool FULL, class V>
__device__ __forceinline__ void walk_b3(double *sp, int cnt, const V &v, double xin) {
    double x = xin;
#pragma unroll
    for (int i = LCH - 1; i >= 0; --i)
        if (FULL || i < cnt) {
            x = fma(-v.CC(i), x, v.ID(i) * sp[i]);
            sp[i] = x;
        }
}

// Segmented (width W, power of two <= 32) inclusive scan of affine maps y -> A y + B composed
// in lane order; on return (A, B) is inclusive and (EA, EB) the exclusive prefix.
__device__ __forceinline__ void seg_scan_fwd(double &A, double &B, int W, int tl, double &EA, double &EB) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        if (off >= W) break;
        const double A2 = __shfl_up_sync(0xffffffffu, A, off, W);
        const double B2 = __shfl_up_sync(0xffffffffu, B, off, W);
        if (tl >= off) {
            B = fma(A, B2, B);
            A = A * A2;
        }
    }
    EA = __shfl_up_sync(0xffffffffu, A, 1, W);
    EB = __shfl_up_sync(0xffffffffu, B, 1, W);
    if (tl == 0) {
        EA = 1.0;
        EB = 0.0;
    }
}
// Same in reverse lane order (backward recurrence x_a = P x_next + Q).
__device__ __forceinline__ void seg_scan_bwd(double &Pm, double &Q, int W, int tl, double &EP, double &EQ) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        if (off >= W) break;
        const double P2 = __shfl_down_sync(0xffffffffu, Pm, off, W);
        const double Q2 = __shfl_down_sync(0xffffffffu, Q, off, W);
        if (tl + off < W) {
            Q = fma(Pm, Q2, Q);
            Pm = Pm * P2;
        }
    }
    EP = __shfl_down_sync(0xffffffffu, Pm, 1, W);
    EQ = __shfl_down_sync(0xffffffffu, Q, 1, W);
    if (tl == W - 1) {
        EP = 1.0;
        EQ = 0.0;
    }
}

// ---------------------------------------- cluster point-to-point (DSMEM + mbarrier) ---
// A producer CTA writes 16 bytes straight into a consumer CTA's shared memory with st.async,
// which signals the consumer's mbarrier (complete_tx) when the bytes land; the consumer arms
// the barrier with the byte count it expects and waits on the phase parity.  No cluster-wide
// barrier (and none of its release/acquire fences on outstanding global traffic) is needed.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *mb, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(unsigned long long *mb, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *mb, unsigned parity) {
    const unsigned a = smem_u32(mb);
#ifdef PRS_CHECKS
    for (long long it = 0;; ++it) {
        unsigned ok;
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) return;
        PRS_CHECK(it < (1ll << 22), "mbarrier wait outlived any legitimate one");
    }
#else
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
#endif
}
// st.async of a double2 into CTA `rank`'s copy of the local shared object `dst`, completing
// tx bytes on that CTA's mbarrier `mb` (local address of the same object)
__device__ __forceinline__ void st_async_remote(double2 *dst, unsigned long long *mb, unsigned rank, double2 v) {
    unsigned rd, rm;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rd) : "r"(smem_u32(dst)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rm) : "r"(smem_u32(mb)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(rd),
                 "d"(v.x), "d"(v.y), "r"(rm)
                 : "memory");
}

// the same for one double (8 bytes)
__device__ __forceinline__ void st_async_remote_f64(double *dst, unsigned long long *mb, unsigned rank, double v) {
    unsigned rd, rm;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rd) : "r"(smem_u32(dst)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rm) : "r"(smem_u32(mb)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(rd), "d"(v),
                 "r"(rm)
                 : "memory");
}

// fp64 tensor-core MMA (m8n8k4, row.col): D = A B + C on an 8 x 8 tile; per lane A[lane / 4][lane % 4],
// B[lane % 4][lane / 4], C / D [lane / 4][2 (lane % 4) + 0, 1]
__device__ __forceinline__ void dmma_f64(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

// Walk dispatch: `full` must be uniform over the CTA (every chunk of every line has LCH
// elements, or the predicated variant runs).
template <class V>
__device__ __forceinline__ void walk_f1_any(bool full, const double *sp, int cnt, const V &v, double &A, double &B) {
    if (full) walk_f1<true>(sp, cnt, v, A, B);
    else walk_f1<false>(sp, cnt, v, A, B);
}
template <class V>
__device__ __forceinline__ void walk_f3_any(bool full, double *sp, int cnt, const V &v, double yin, double &Pb,
                                            double &Qb) {
    if (full) walk_f3<true>(sp, cnt, v, yin, Pb, Qb);
    else walk_f3<false>(sp, cnt, v, yin, Pb, Qb);
}
template <class V>
__device__ __forceinline__ void walk_b3_any(bool full, double *sp, int cnt, const V &v, double xin) {
    if (full) walk_b3<true>(sp, cnt, v, xin);
    else walk_b3<false>(sp, cnt, v, xin);
}

}  // namespace prs
