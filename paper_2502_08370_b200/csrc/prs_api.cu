// prs_api.cu -- C ABI (include/prs.h) and the host-side propagator / parareal driver.
//
// Layers: L2 propagators = sequences of line-pass / DD-stage kernels on the
// context stream; L3 parareal driver = batched fine sweep over all local slices, sequential
// coarse chain with the fused correction epilogue, stop test, NCCL hand-off of slice end
// states between ranks (rank order = time order).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/prs.h"
#include "dd.cuh"
#include "lpass.cuh"
#include "setup.cuh"
#include "xpass.cuh"
#include "xpass3.cuh"
#include "lpass3.cuh"
#include "lpass4.cuh"
#include "lpass5.cuh"
#include "lpass8.cuh"
#include "xy3.cuh"
#include "gpar.cuh"
#include "sweep2.cuh"
#include "xpass7.cuh"
#include "transport.cuh"
#include "ie.cuh"

#include <algorithm>
#include <cstdlib>

using namespace prs;

namespace {

// ------------------------------------------------------------- NCCL (dlopen) -------
struct Nccl {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, ncclConfig_t *) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool load(std::string &err) {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return false;
        }
#define SYM(f, name)                                                \
    f = reinterpret_cast<decltype(f)>(dlsym(h, name));              \
    if (!f) {                                                       \
        err = std::string("missing NCCL symbol ") + name;           \
        return false;                                               \
    }
        SYM(GetUniqueId, "ncclGetUniqueId");
        SYM(CommInitRank, "ncclCommInitRank");
        SYM(CommDestroy, "ncclCommDestroy");
        SYM(Send, "ncclSend");
        SYM(Recv, "ncclRecv");
        SYM(AllReduce, "ncclAllReduce");
        SYM(AllGather, "ncclAllGather");
        SYM(GroupStart, "ncclGroupStart");
        SYM(GroupEnd, "ncclGroupEnd");
        SYM(CommSplit, "ncclCommSplit");
        SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
        return true;
    }
};
Nccl g_nccl;

// NCCL over NVLink / NVSwitch (transport.cuh): channel 0 = the data plane, channel 1 = a split
// communicator for the stop-test all-reduce (its own stream in the lagged stop test)
struct NcclTransport : Transport {
    ncclComm_t comm[2] = {nullptr, nullptr};
    ~NcclTransport() override {
        for (ncclComm_t c : comm)
            if (c && g_nccl.CommDestroy) g_nccl.CommDestroy(c);
    }
    int chk(ncclResult_t r, const char *what) {
        if (r == ncclSuccess) return 0;
        err = std::string(what) + ": " + g_nccl.GetErrorString(r);
        return PRS_ENCCL;
    }
    int init(const void *uid, int nranks, int rank) {
        if (!g_nccl.load(err)) return PRS_ENCCL;
        ncclUniqueId id;
        memcpy(&id, uid, sizeof(id));
        if (int rc = chk(g_nccl.CommInitRank(&comm[0], nranks, id, rank), "ncclCommInitRank")) return rc;
        return chk(g_nccl.CommSplit(comm[0], 0, rank, &comm[1], nullptr), "ncclCommSplit");
    }
    int group_start() override { return chk(g_nccl.GroupStart(), "ncclGroupStart"); }
    int group_end() override { return chk(g_nccl.GroupEnd(), "ncclGroupEnd"); }
    int send(const double *buf, size_t count, int peer, cudaStream_t st, int ch) override {
        return chk(g_nccl.Send(buf, count, ncclDouble, peer, comm[ch], st), "ncclSend");
    }
    int recv(double *buf, size_t count, int peer, cudaStream_t st, int ch) override {
        return chk(g_nccl.Recv(buf, count, ncclDouble, peer, comm[ch], st), "ncclRecv");
    }
    int allreduce_max_u64(unsigned long long *buf, size_t count, cudaStream_t st, int ch) override {
        return chk(g_nccl.AllReduce(buf, buf, count, ncclUint64, ncclMax, comm[ch], st), "ncclAllReduce");
    }
    // (in place: the send buffer is this rank's segment of recv)
    int allgather_inplace(double *recv, size_t count, cudaStream_t st, int ch) override {
        return chk(g_nccl.AllGather(recv + (size_t)my_rank * count, recv, count, ncclDouble, comm[ch], st),
                   "ncclAllGather");
    }
    int my_rank = 0;
};

}  // namespace

// per-tau pivot data
struct TauFactors {
    double tau = -1.0;
    double *tab = nullptr;               // 3 n (m, id, cc), kappa = 1
    double *invdx = nullptr, *invdy = nullptr;  // n^2 each, variable kappa
};

struct prs_ctx {
    double *cyc2 = nullptr;    // cyclic ownership, on-chip chain: two-state scratch (chain2_cyclic_one)
    bool x7_tma = true;        // c3 x pass: TMA tensor copies (PRS_X7TMA=0: cp.async + staged stores)
    // TMA tensor maps (rows of 16 doubles, 128-byte swizzle) by (address, rows)
    std::vector<std::pair<std::pair<const void *, long long>, CUtensorMap>> tmaps;
    prs_problem p{};
    int rank = 0, nranks = 1, first = 0, count = 0;
    // slice ownership (prs_set_ownership): 0 contiguous blocks (local slice i = global first + i;
    // traj[i] / traj[i+1] = its start / end state), 1 cyclic (local slice i = global rank + i P;
    // traj[i] = start, tend[i] = end state: consecutive slices live on consecutive ranks)
    int cyclic = 0;
    double *tend = nullptr;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int device = 0;
    long long vol = 0;
    long long ss = 0;  // slice stride (elements) of the batch buffers traj / fa / fb / gcache
    size_t sbytes = 0;
    int M = 2;
    double h = 0, h2inv = 0, creact = 0, dT = 0, dt = 0;
    double *traj = nullptr, *fa = nullptr, *fb = nullptr, *gcache = nullptr, *gtmp = nullptr;
    double *delta = nullptr;  // = fa or fb after a fine sweep
    double *u0 = nullptr;
    double *sinpi = nullptr, *s2n = nullptr, *s2f = nullptr;
    // source (R29): F = src_amp g(t) prod_d srcsin[i_d]; kind 1: dim pi^2 + c - 1, e^{-t},
    // sin(pi x); kind 2: 1, 2 pi cos 2 pi t + (8 pi^2 + c) sin 2 pi t, sin(2 pi x)
    double src_amp = 0.0;
    const double *srcsin = nullptr;
    TauFactors fac[3];  // 0 coarse, 1 fine, 2 custom (prs_step)
    DDData dd;
    unsigned long long *red = nullptr;  // [0] update bits, [1] flag, [2] scratch
    unsigned long long *red_host = nullptr;
    unsigned long long *red_base = nullptr;  // 8 words: [0,1] / [4,5] = (update bits, flag) of the
                                             // two iteration parities, [2] scratch; red points at
                                             // the current parity's pair
    cudaStream_t ctl = nullptr;              // lagged stop test (nranks > 1): the all-reduce stream
    cudaEvent_t ev_chain[2] = {nullptr, nullptr}, ev_red[2] = {nullptr, nullptr};
    double u0norm = 1.0;
    bool have_initial = false, have_coarse = false;
    long long launches = 0;
    // profiling
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, double>> ev_pending;  // (kind, bytes) per recorded pair
    size_t ev_used = 0;
    long long k_launch[4] = {0, 0, 0, 0};
    double k_ms[4] = {0, 0, 0, 0}, k_bytes[4] = {0, 0, 0, 0};
    // unsplit implicit Euler (ie.cuh, NEXT-4): DST-I matrix, sine eigenvalues, two scratch
    // batches of ie_cap states (grown on demand: scratch_gen++)
    double *ie_S = nullptr, *ie_mu = nullptr, *ie_w1 = nullptr, *ie_w2 = nullptr;
    long long ie_cap = 0;
    Transport *tr = nullptr;  // nranks > 1: NCCL (prs_create) or the in-process world (prs_create_local)
    int num_sms = 148;
    bool no_xy = false;        // PRS_XY=0: 3-D n = 128 takes separate x and y passes
    bool no_sweep2 = false;    // PRS_SWEEP2=0: small 2-D slices step through the per-step kernels
    // CUDA graphs of the per-iteration launch sequences (single rank, profiling off): the
    // fine sweep and the coarse correction chain are captured on their second call (the first
    // one allocates lazily-sized scratch) and replayed afterwards.  PRS_GRAPHS=0 disables.
    bool graphs = true;
    int fine_calls = 0, corr_calls = 0;
    cudaGraphExec_t fine_exec = nullptr, corr_exec = nullptr;
    long long fine_glaunch = 0, corr_glaunch = 0;  // kernels per replay
    // captured graphs hold pointers to lazily sized scratch (l5buf, the DD exchange buffers):
    // scratch_gen counts their reallocations; a graph captured under another generation is
    // destroyed and captured again
    int scratch_gen = 0;
    int fine_gen = -1, corr_gen = -1;
    // prs_iterate: slices n < kconv are converged (U^k_n exact and bitwise frozen for n <= k,
    // PAPER.md:214), so their fine propagation and coarse correction would reproduce the
    // previous iteration's Delta_n and U_{n+1}: they are skipped.  Enabled for states of
    // >= 2^18 points (PRS_SKIP=0/1 overrides); bare fine_sweep / correct calls never skip.
    bool skip_converged = false;
    int kconv = 0;
    bool lag = true;  // nranks > 1: prs_iterate reads the stop test one fine sweep late (PRS_LAG=0: off)
    // space-parallel G (gpar.cuh): P bands of gnb rows; one process runs all P (virtual bands)
    int gpar = 0, gP = 1, gnb = 0;
    double *gb_u = nullptr, *gb_d = nullptr, *gb_gc = nullptr;  // multi-rank: this rank's band of
                                                                 // U_0..U_N, Delta_0.., Gcache_0..
    bool gb_valid = false;     // multi-rank: gb_u holds this rank's bands of the current iterate
                               // U^k_1..U^k_N (the update norm of the chain's CORRECT epilogue reads
                               // them); false after anything that writes the trajectory outside
                               // the band chain (set_initial, coarse_sweep, a mode switch)
    double *gb_v = nullptr;    // x-stage output (a full state: P bands when virtual)
    double *gb_tt = nullptr;   // per band: block tuples [5] + scan [2] x (gnb/64) x n
    double *gb_tot = nullptr;  // band tuples [P][5][n]
    double *gb_yx = nullptr;   // per band: y entering / x leaving [P][2][n]
    double *l5buf = nullptr;  // lpass5 block tuples and block y/x
    size_t l5_bytes = 0;
    // pipelined parareal (prs_set_pipeline): the local slices in `pipe`
    // blocks; trajectory and G cache double-buffered by iteration parity (traj2, gcache2)
    int pipe = 0;
    double *traj2 = nullptr, *gcache2 = nullptr;
    cudaStream_t psC = nullptr;              // the coarse chain
    std::vector<cudaStream_t> psF;           // fine sweep of block b
    std::vector<cudaEvent_t> pevF, pevC;     // block b: fine sweep done / chain done
    cudaEvent_t pev0 = nullptr, pevRed[2] = {nullptr, nullptr};
    unsigned long long *pred = nullptr;      // [parity][2] update bits, non-finite flag
    unsigned long long *pred_host = nullptr; // pinned copy
    std::string err;
};

#define CK(call)                                                                 \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);       \
            return PRS_ECUDA;                                                    \
        }                                                                        \
    } while (0)

#define NK(call)                                                                 \
    do {                                                                         \
        int r_ = (call);                                                         \
        if (r_ != PRS_OK) {                                                      \
            ctx->err = ctx->tr->err;                                             \
            return r_;                                                           \
        }                                                                        \
    } while (0)

#define TRY(call)                 \
    do {                          \
        int rc_ = (call);         \
        if (rc_ != PRS_OK) return rc_; \
    } while (0)

static int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

static int last_launch(prs_ctx *ctx) {
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        ctx->err = std::string("kernel launch: ") + cudaGetErrorString(e);
        return PRS_ECUDA;
    }
    return PRS_OK;
}

// ---- profiling: events around fine-sweep launches ----
static int prof_begin(prs_ctx *ctx) {
    if (!ctx->prof) return PRS_OK;
    while (ctx->ev_pool.size() < ctx->ev_used + 2) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        ctx->ev_pool.push_back(e);
    }
    CK(cudaEventRecord(ctx->ev_pool[ctx->ev_used], ctx->stream));
    return PRS_OK;
}
static int prof_end(prs_ctx *ctx, int kind, double bytes) {
    if (!ctx->prof) return PRS_OK;
    CK(cudaEventRecord(ctx->ev_pool[ctx->ev_used + 1], ctx->stream));
    ctx->ev_pending.push_back({kind, bytes});
    ctx->ev_used += 2;
    return PRS_OK;
}
static int prof_flush(prs_ctx *ctx) {
    if (ctx->ev_used == 0) return PRS_OK;
    CK(cudaStreamSynchronize(ctx->stream));
    for (size_t i = 0; i < ctx->ev_pending.size(); ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev_pool[2 * i], ctx->ev_pool[2 * i + 1]));
        const int k = ctx->ev_pending[i].first;
        ctx->k_launch[k] += 1;
        ctx->k_ms[k] += ms;
        ctx->k_bytes[k] += ctx->ev_pending[i].second;
    }
    ctx->ev_pending.clear();
    ctx->ev_used = 0;
    return PRS_OK;
}

// ------------------------------------------------------------------ factors --------
static int ensure_factors(prs_ctx *ctx, int slot, double tau) {
    TauFactors &f = ctx->fac[slot];
    if (f.tau == tau) return PRS_OK;
    const int n = ctx->p.n;
    f.tau = tau;
    // an IE propagator solves in the sine basis (ie.cuh): no splitting factors for its slot
    if ((slot == 0 && ctx->p.G == PRS_IE) || (slot == 1 && ctx->p.F == PRS_IE)) return PRS_OK;
    if (ctx->p.split == 1) return dd_factors(ctx->dd, slot, tau, ctx->stream, ctx->err);
    if (ctx->p.coef_kind == 0) {
        if (!f.tab) CK(cudaMalloc(&f.tab, sizeof(double) * 3 * n));
        setup_const_tab<<<1, 1, 0, ctx->stream>>>(n, tau, ctx->h2inv, ctx->creact, f.tab, f.tab + n,
                                                  f.tab + 2 * n);
        TRY(last_launch(ctx));
    } else {
        const size_t bytes = sizeof(double) * (size_t)n * n;
        if (!f.invdx) CK(cudaMalloc(&f.invdx, bytes));
        if (!f.invdy) CK(cudaMalloc(&f.invdy, bytes));
        const int tpb = 128, nb = (n + tpb - 1) / tpb;
        setup_var_invd<<<nb, tpb, 0, ctx->stream>>>(n, 0, tau, ctx->h2inv, ctx->creact, ctx->s2n,
                                                    ctx->s2f, f.invdx);
        TRY(last_launch(ctx));
        setup_var_invd<<<nb, tpb, 0, ctx->stream>>>(n, 1, tau, ctx->h2inv, ctx->creact, ctx->s2n,
                                                    ctx->s2f, f.invdy);
        TRY(last_launch(ctx));
    }
    return PRS_OK;
}

// ----------------------------------------------------------- line-pass launchers ----
struct EpiArgs {
    int kind = EPI_STORE;
    const double *gc = nullptr;   // DELTA
    double *gcache = nullptr;     // CORRECT/INIT
    const double *delta = nullptr;
    double *traj = nullptr;
};

// persistent pipelined x-pass (xpass3.cuh) when the shape allows it
static bool xpass3_ok(const prs_ctx *ctx, long long B) {
    const int n = ctx->p.n;
    if (n < 16 || n > 4096 || (n & (n - 1)) != 0) return false;
    const long long lines = B * (ctx->p.dim == 2 ? (long long)n : (long long)n * n);
    const int lpg = 4096 / n;
    if (lines % lpg != 0) return false;
    if (ctx->p.coef_kind && n % lpg != 0) return false;
    return true;
}

static int launch_xpass3(prs_ctx *ctx, int scheme, const TauFactors &f, const double *in, double *out, long long B,
                         const TimeArgs &ta, bool prof) {
    const int n = ctx->p.n, dim = ctx->p.dim;
    X3Args a{};
    a.in = in;
    a.out = out;
    a.vol = ctx->vol;
    a.n = n;
    a.P = n / LCH;
    a.lines_per_state = (dim == 2) ? n : n * n;
    a.ngroups = B * ctx->vol / 4096;
    a.nstates = (int)B;
    // state-fastest ranges when every state has enough groups: the number of ranges makes
    // B * nranges a multiple of the grid (balanced), each range >= 64 groups
    a.nranges = 0;
    if (B > 1) {
        const long long grid = std::min<long long>(ctx->num_sms, a.ngroups);
        long long g = grid, bb = B;
        while (bb) { const long long t = g % bb; g = bb; bb = t; }  // gcd(grid, B)
        const long long R = grid / g;
        if ((a.ngroups / B) / R >= 64) a.nranges = (int)R;
    }
    a.dim = dim;
    a.tau = f.tau;
    a.h2inv = ctx->h2inv;
    a.creact = ctx->creact;
    a.src_amp = ctx->src_amp;
    a.sinpi = ctx->srcsin;
    a.ta = ta;
    a.tab = CoefTab{f.tab, f.tab ? f.tab + n : nullptr, f.tab ? f.tab + 2 * n : nullptr};
    a.invd = f.invdx;
    a.s2n = ctx->s2n;
    a.s2f = ctx->s2f;
    const int dr = (scheme == PRS_DR) ? 1 : 0;
    const int coef = ctx->p.coef_kind;
    const int src = ctx->p.source_kind != 0;
    const size_t shm = xpass3_smem_bytes(coef);
    void (*kern)(X3Args) = nullptr;
#define XK(C, D, S_) if (coef == C && dr == D && src == S_) kern = xpass3_kernel<C, D, S_>;
    XK(0, 0, 0) XK(0, 0, 1) XK(0, 1, 0) XK(0, 1, 1) XK(1, 0, 0) XK(1, 0, 1) XK(1, 1, 0) XK(1, 1, 1)
#undef XK
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    const long long grid = std::min<long long>(ctx->num_sms, a.ngroups);
    if (prof) TRY(prof_begin(ctx));
    kern<<<(unsigned)grid, X3T, shm, ctx->stream>>>(a);
    TRY(last_launch(ctx));
    if (prof) TRY(prof_end(ctx, PRS_K_XPASS, (double)B * (double)ctx->vol * (16.0 + (coef ? 8.0 : 0.0))));
    return PRS_OK;
}

// ---- TMA tensor maps: a buffer of `rows` x 16 doubles (128-byte rows), box 16 x 128 (a half
// row of xpass7), 128-byte swizzle; encoded through the driver entry point (no link-time libcuda
// dependency) and cached per (address, rows)
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static int get_tmap(prs_ctx *ctx, const void *ptr, long long rows, CUtensorMap *out) {
    for (auto &e : ctx->tmaps)
        if (e.first.first == ptr && e.first.second == rows) {
            *out = e.second;
            return PRS_OK;
        }
    static PFN_encodeTiled encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) {
            ctx->err = "cuTensorMapEncodeTiled unavailable";
            return PRS_ECUDA;
        }
        encode = reinterpret_cast<PFN_encodeTiled>(fn);
    }
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)LCH, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(LCH * sizeof(double))};
    const cuuint32_t box[2] = {(cuuint32_t)LCH, (cuuint32_t)X7T};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(ptr), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        ctx->err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
        return PRS_ECUDA;
    }
    if (ctx->tmaps.size() > 64) ctx->tmaps.clear();
    ctx->tmaps.push_back({{ptr, rows}, m});
    *out = m;
    return PRS_OK;
}

// 4096-point rows (c3): each row over a 2-CTA cluster (xpass7.cuh)
static int launch_xpass7(prs_ctx *ctx, int scheme, const TauFactors &f, const double *in, double *out, long long B,
                         const TimeArgs &ta, bool prof) {
    X7Args a{};
    a.in = in;
    a.out = out;
    a.vol = ctx->vol;
    a.nrows = B * (long long)X7N;
    a.nstates = (int)B;
    long long ncl = ctx->num_sms;  // one cluster per SM pair slot: 2 CTAs per SM
#ifdef PRS_X7_TIMING
    if (getenv("PRS_X7_NCL")) ncl = atoll(getenv("PRS_X7_NCL"));
#endif
    a.nranges = 0;
    if (B > 1) {
        long long g = ncl, bb = B;
        while (bb) { const long long t = g % bb; g = bb; bb = t; }
        const long long R = ncl / g;
        if (X7N / R >= 64) a.nranges = (int)R;
    }
    a.tau = f.tau;
    a.h2inv = ctx->h2inv;
    a.creact = ctx->creact;
    a.src_amp = ctx->src_amp;
    a.sinpi = ctx->srcsin;
    a.ta = ta;
    a.tab = CoefTab{f.tab, f.tab ? f.tab + X7N : nullptr, f.tab ? f.tab + 2 * X7N : nullptr};
    a.invd = f.invdx;
    a.s2n = ctx->s2n;
    a.s2f = ctx->s2f;
    const int dr = (scheme == PRS_DR) ? 1 : 0, coef = ctx->p.coef_kind, src = ctx->p.source_kind != 0;
    const int tma = ctx->x7_tma ? 1 : 0;
    if (tma) {
        TRY(get_tmap(ctx, in, B * ctx->vol / LCH, &a.tm_in));
        TRY(get_tmap(ctx, out, B * ctx->vol / LCH, &a.tm_out));
        if (coef) TRY(get_tmap(ctx, f.invdx, ctx->vol / LCH, &a.tm_piv));
    }
    void (*kern)(X7Args) = nullptr;
#define XK(C, D, S_)                                                  \
    if (coef == C && dr == D && src == S_)                            \
        kern = tma ? xpass7_kernel<C, D, S_, 1> : xpass7_kernel<C, D, S_, 0>;
    XK(0, 0, 0) XK(0, 0, 1) XK(0, 1, 0) XK(0, 1, 1) XK(1, 0, 0) XK(1, 0, 1) XK(1, 1, 0) XK(1, 1, 1)
#undef XK
    const size_t shm = xpass7_smem_bytes(coef, tma);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * std::min<long long>(ncl, a.nrows)));
    cfg.blockDim = dim3(X7T);
    cfg.dynamicSmemBytes = shm;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (prof) TRY(prof_begin(ctx));
    CK(cudaLaunchKernelEx(&cfg, kern, a));
    TRY(last_launch(ctx));
    if (prof) TRY(prof_end(ctx, PRS_K_XPASS, (double)B * (double)ctx->vol * (16.0 + (coef ? 8.0 : 0.0))));
    return PRS_OK;
}

static int launch_xpass(prs_ctx *ctx, int scheme, const TauFactors &f, const double *in, double *out,
                        long long B, const TimeArgs &ta, bool prof) {
    if (ctx->p.dim == 2 && ctx->p.n == X7N && ctx->ss == ctx->vol)
        return launch_xpass7(ctx, scheme, f, in, out, B, ta, prof);
    if (xpass3_ok(ctx, B)) return launch_xpass3(ctx, scheme, f, in, out, B, ta, prof);
    const int n = ctx->p.n, dim = ctx->p.dim;
    XArgs a{};
    a.in = in;
    a.out = out;
    a.vol = ctx->vol;
    a.n = n;
    a.lines_per_state = (dim == 2) ? n : n * n;
    a.nlines = B * a.lines_per_state;
    a.P = next_pow2((n + LCH - 1) / LCH);
    a.S = cpad_host(n);
    a.St = cpad_host(n + 1);
    a.dim = dim;
    a.tau = f.tau;
    a.h2inv = ctx->h2inv;
    a.creact = ctx->creact;
    a.src_amp = ctx->src_amp;
    a.sinpi = ctx->srcsin;
    a.ta = ta;
    a.tab = CoefTab{f.tab, f.tab ? f.tab + n : nullptr, f.tab ? f.tab + 2 * n : nullptr};
    a.invd = f.invdx;
    a.s2n = ctx->s2n;
    a.s2f = ctx->s2f;
    const int threads_target = 256;
    const int lpb = (a.P >= threads_target) ? 1 : threads_target / a.P;
    const int threads = lpb * a.P;
    const int dr = (scheme == PRS_DR) ? 1 : 0;
    const int coef = ctx->p.coef_kind;
    const int src = ctx->p.source_kind != 0;
    const size_t shm = sizeof(double) * xpass_smem_doubles(lpb, a.S, a.St, coef, threads);
    const long long blocks = (a.nlines + lpb - 1) / lpb;
    void (*kern)(XArgs) = nullptr;
#define XK(C, D, S_) if (coef == C && dr == D && src == S_) kern = xpass_kernel<C, D, S_>;
    XK(0, 0, 0) XK(0, 0, 1) XK(0, 1, 0) XK(0, 1, 1) XK(1, 0, 0) XK(1, 0, 1) XK(1, 1, 0) XK(1, 1, 1)
#undef XK
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    if (prof) TRY(prof_begin(ctx));
    kern<<<(unsigned)blocks, threads, shm, ctx->stream>>>(a);
    TRY(last_launch(ctx));
    if (prof) {
        double bytes = (double)B * (double)ctx->vol * (16.0 + (coef ? 8.0 : 0.0));
        TRY(prof_end(ctx, PRS_K_XPASS, bytes));
    }
    return PRS_OK;
}

// persistent pipelined strided pass (lpass3.cuh): n = 16 * 2^k in [64, 4096]
static int launch_lpass3(prs_ctx *ctx, int axis, const TauFactors &f, const double *in, double *out, long long B,
                         const EpiArgs &ep, bool prof) {
    const int n = ctx->p.n, dim = ctx->p.dim;
    L3Args a{};
    a.in = in;
    a.out = out;
    a.vol = ctx->vol;
    a.n = n;
    if (axis == 1) {
        a.Sl = n;
        a.nq = (dim == 2) ? 1 : n;
        a.Sq = (long long)n * n;
    } else {
        a.Sl = (long long)n * n;
        a.nq = n;
        a.Sq = n;
    }
    a.CL = std::max(1, n / 512);
    a.R = n / a.CL;
    a.CP = a.R / LCH;
    a.PW = L3T / a.CP;
    a.nwb = n / a.PW;
    a.npanels = B * a.nq * a.nwb;
    a.tau = f.tau;
    a.h2inv = ctx->h2inv;
    a.tab = CoefTab{f.tab, f.tab ? f.tab + n : nullptr, f.tab ? f.tab + 2 * n : nullptr};
    a.invd = f.invdy;
    a.s2n = ctx->s2n;
    a.s2f = ctx->s2f;
    a.e_gc = ep.gc;
    a.e_gcache = ep.gcache;
    a.e_delta = ep.delta;
    a.e_traj = ep.traj;
    a.e_red = ctx->red;
    const int coef = ctx->p.coef_kind;
    // clusters (long lines): one exchange of composed tuples per panel, hidden behind the
    // previous panel (lpass4); single-CTA lines: lpass3
    const bool use4 = a.CL > 1;
    const size_t shm = use4 ? lpass4_smem_bytes(a.PW, a.R, a.CL, coef) : lpass3_smem_bytes(a.PW, a.R, a.CL, coef);
    void (*kern)(L3Args) = nullptr;
#define LK(W, C, E)                                                   \
    if (a.PW == W && coef == C && ep.kind == E)                       \
        kern = use4 ? lpass4_kernel<W, C, E> : lpass3_kernel<W, C, E>;
#define LKW(W) LK(W, 0, 0) LK(W, 0, 1) LK(W, 0, 2) LK(W, 0, 3) LK(W, 1, 0) LK(W, 1, 1) LK(W, 1, 2) LK(W, 1, 3)
    LKW(8) LKW(16) LKW(32) LKW(64)
#undef LKW
#undef LK
    if (!kern) {
        ctx->err = "lpass3: unsupported panel width";
        return PRS_EUNSUPPORTED;
    }
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    if (a.CL > 1) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const long long nclusters = std::min<long long>(std::max(1, ctx->num_sms / a.CL), a.npanels);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(nclusters * a.CL));
    cfg.blockDim = dim3(L3T);
    cfg.dynamicSmemBytes = shm;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (prof) TRY(prof_begin(ctx));
    CK(cudaLaunchKernelEx(&cfg, kern, a));
    TRY(last_launch(ctx));
    if (prof) {
        double per = 16.0 + (coef ? 8.0 : 0.0);
        if (ep.kind == EPI_DELTA) per += 8.0;
        TRY(prof_end(ctx, PRS_K_LPASS, (double)B * (double)ctx->vol * per));
    }
    return PRS_OK;
}

// long strided lines (n >= 2048): tuple / scan / finish over 64 x 64 tiles (lpass5.cuh)
// the lp8 finish instantiation for a coefficient kind, epilogue and register width
static void (*lp8_finish_fn(int coef, int kind))(L5Args) {
    void (*f8)(L5Args) = nullptr;
#define LK(C, E) if (coef == C && kind == E) f8 = lp8_kernel<C, E, 1, 1>;
    LK(0, 0) LK(0, 1) LK(0, 2) LK(0, 3) LK(1, 0) LK(1, 1) LK(1, 2) LK(1, 3)
#undef LK
    return f8;
}

static int launch_lpass5(prs_ctx *ctx, int axis, const TauFactors &f, const double *in, double *out, long long B,
                         const EpiArgs &ep, bool prof) {
    const int n = ctx->p.n, dim = ctx->p.dim;
    L5Args a{};
    a.in = in;
    a.out = out;
    a.vol = ctx->vol;
    a.n = n;
    if (axis == 1) {
        a.Sl = n;
        a.nq = (dim == 2) ? 1 : n;
        a.Sq = (long long)n * n;
    } else {
        a.Sl = (long long)n * n;
        a.nq = n;
        a.Sq = n;
    }
    a.nrb = n / L5RB;
    a.ncb = n / L5W;
    a.ntiles = B * a.nq * a.nrb * a.ncb;
    a.tau = f.tau;
    a.h2inv = ctx->h2inv;
    a.tab = CoefTab{f.tab, f.tab ? f.tab + n : nullptr, f.tab ? f.tab + 2 * n : nullptr};
    a.invd = f.invdy;
    a.s2n = ctx->s2n;
    a.s2f = ctx->s2f;
    a.tstride = B * a.nq * a.nrb * (long long)n;
    const size_t need = sizeof(double) * 7 * (size_t)a.tstride;
    if (ctx->l5_bytes < need) {
        if (ctx->l5buf) CK(cudaFree(ctx->l5buf));
        ctx->l5buf = nullptr;
        CK(cudaMalloc(&ctx->l5buf, need));
        ctx->l5_bytes = need;
        ++ctx->scratch_gen;
    }
    a.tt = ctx->l5buf;
    a.yx = ctx->l5buf + 5 * a.tstride;
    a.e_gc = ep.gc;
    a.e_gcache = ep.gcache;
    a.e_delta = ep.delta;
    a.e_traj = ep.traj;
    a.e_red = ctx->red;
    const int coef = ctx->p.coef_kind;
    void (*k1)(L5Args) = coef ? lp5_tuples_kernel<1> : lp5_tuples_kernel<0>;
    void (*k3)(L5Args) = nullptr;
#define LK(C, E) if (coef == C && ep.kind == E) k3 = lp5_finish_kernel<C, E>;
    LK(0, 0) LK(0, 1) LK(0, 2) LK(0, 3) LK(1, 0) LK(1, 1) LK(1, 2) LK(1, 3)
#undef LK
    const long long ncols = B * a.nq * (long long)n;
    const bool use8 = a.nq == 1;
    if (prof) TRY(prof_begin(ctx));
    if (use8) {
        // persistent over slice groups: coefficients once per tile position, state tiles
        // through a cp.async ring
        a.nsq = B;
        a.s8 = (int)std::min<long long>(B, 16);
        a.nsg8 = (int)((B + a.s8 - 1) / a.s8);
        const long long grid = (long long)a.nrb * a.ncb * a.nsg8;
        const size_t shm = lpass8_smem_bytes(0), shmf = lpass8_smem_bytes(1);
        void (*t8)(L5Args) = coef ? lp8_kernel<1, 0, 0> : lp8_kernel<0, 0, 0>;
        void (*f8)(L5Args) = lp8_finish_fn(coef, ep.kind);
        CK(cudaFuncSetAttribute(t8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        CK(cudaFuncSetAttribute(f8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmf));
        t8<<<(unsigned)grid, L5T, shm, ctx->stream>>>(a);
        TRY(last_launch(ctx));
        lp5_scan_kernel<<<(unsigned)((ncols + 255) / 256), 256, 0, ctx->stream>>>(a, ncols);
        TRY(last_launch(ctx));
        f8<<<(unsigned)grid, L5T, shmf, ctx->stream>>>(a);
        TRY(last_launch(ctx));
    } else {
        k1<<<(unsigned)a.ntiles, L5T, 0, ctx->stream>>>(a);
        TRY(last_launch(ctx));
        lp5_scan_kernel<<<(unsigned)((ncols + 255) / 256), 256, 0, ctx->stream>>>(a, ncols);
        TRY(last_launch(ctx));
        k3<<<(unsigned)a.ntiles, L5T, 0, ctx->stream>>>(a);
        TRY(last_launch(ctx));
    }
    if (prof) {
        double per = 16.0 + (coef ? 8.0 : 0.0);
        if (ep.kind == EPI_DELTA) per += 8.0;
        TRY(prof_end(ctx, PRS_K_LPASS, (double)B * (double)ctx->vol * per));
    }
    return PRS_OK;
}

// strided pass along axis d (1 = y, 2 = z) over B states in place (in == out allowed)
static int launch_lpass(prs_ctx *ctx, int axis, const TauFactors &f, const double *in, double *out,
                        long long B, const EpiArgs &ep, bool prof) {
    const int n = ctx->p.n, dim = ctx->p.dim;
    if (n >= 2048 && n <= 4096 && (n & (n - 1)) == 0)
        return launch_lpass5(ctx, axis, f, in, out, B, ep, prof);
    if (n >= 64 && n <= 4096 && (n & (n - 1)) == 0)
        return launch_lpass3(ctx, axis, f, in, out, B, ep, prof);
    LArgs a{};
    a.in = in;
    a.out = out;
    a.vol = ctx->vol;
    a.n = n;
    if (axis == 1) {
        a.Sl = n;
        a.nq = (dim == 2) ? 1 : n;
        a.Sq = (long long)n * n;
    } else {
        a.Sl = (long long)n * n;
        a.nq = n;
        a.Sq = n;
    }
    const int coef = ctx->p.coef_kind;
    const int PWc = coef ? 8 : 16;  // variable kappa stages pivots too: narrower panels, more CTAs/SM
    a.nwb = (n + PWc - 1) / PWc;
    a.npanels = B * a.nq * a.nwb;
    int CL = 1;
    while ((n + CL - 1) / CL > 32 * LCH) CL *= 2;
    if (CL > 8) {
        ctx->err = "strided line longer than 8 * 512 is not supported";
        return PRS_EUNSUPPORTED;
    }
    a.CL = CL;
    a.R = (n + CL - 1) / CL;
    a.CP = next_pow2((a.R + LCH - 1) / LCH);
    a.S = cpad_host(a.R);
    a.St = cpad_host(a.R + 1);
    a.tau = f.tau;
    a.h2inv = ctx->h2inv;
    a.tab = CoefTab{f.tab, f.tab ? f.tab + n : nullptr, f.tab ? f.tab + 2 * n : nullptr};
    a.invd = f.invdy;
    a.s2n = ctx->s2n;
    a.s2f = ctx->s2f;
    a.e_gc = ep.gc;
    a.e_gcache = ep.gcache;
    a.e_delta = ep.delta;
    a.e_traj = ep.traj;
    a.e_red = ctx->red;
    const int threads = PWc * a.CP;
    const size_t shm = sizeof(double) * lpass_smem_doubles(PWc, a.S, a.St, coef);
    void (*kern)(LArgs) = nullptr;
#define LK(C, E) if (coef == C && ep.kind == E) kern = lpass_kernel<(C ? 8 : 16), C, E>;
    LK(0, 0) LK(0, 1) LK(0, 2) LK(0, 3) LK(1, 0) LK(1, 1) LK(1, 2) LK(1, 3)
#undef LK
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    if (CL > 1) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(a.npanels * CL));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = shm;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (prof) TRY(prof_begin(ctx));
    CK(cudaLaunchKernelEx(&cfg, kern, a));
    TRY(last_launch(ctx));
    if (prof) {
        double per = 16.0 + (coef ? 8.0 : 0.0);
        if (ep.kind == EPI_DELTA) per += 8.0;
        TRY(prof_end(ctx, PRS_K_LPASS, (double)B * (double)ctx->vol * per));
    }
    return PRS_OK;
}

// One step of `scheme` on B consecutive states: in -> out (out holds the result, or the
// epilogue consumes it).  tmp must be distinct from in when scheme is DR.
static int ie_step(prs_ctx *ctx, double tau, const double *in, double *out, long long B, const TimeArgs &ta,
                   const EpiArgs &ep, bool prof);
static int run_step(prs_ctx *ctx, int scheme, const TauFactors &f, const double *in, double *out,
                    long long B, const TimeArgs &ta_in, const EpiArgs &ep, bool prof, long long stride) {
    TimeArgs ta = ta_in;
    ta.gk = ctx->p.source_kind == 2 ? 1 : 0;
    ta.gc = 8.0 * M_PI * M_PI + ctx->p.c;
    if (scheme == PRS_IE) {
        if (stride != ctx->vol) {
            ctx->err = "internal: padded slice stride on the IE path";
            return PRS_EUNSUPPORTED;
        }
        return ie_step(ctx, f.tau, in, out, B, ta, ep, prof);
    }
    if (ctx->p.split == 1)
        return dd_step(ctx->dd, scheme, (int)(&f - ctx->fac), in, out, B, ta, ep.kind, ep.gc, ep.gcache,
                       ep.delta, ep.traj, ctx->red, ctx->stream, prof ? ctx : nullptr, ctx->err, ctx->launches,
                       ctx->src_amp, ctx->p.source_kind != 0);
    if (stride != ctx->vol) {
        ctx->err = "internal: padded slice stride on a path without stride support";
        return PRS_EUNSUPPORTED;
    }
    if (ctx->p.dim == 3 && ctx->p.n == XY_N && ctx->p.coef_kind == 0 && scheme == PRS_FIE && !ctx->no_xy) {
        // x and y stages fused per z-plane (xy3.cuh), then the z stage
        XYArgs x{};
        x.in = in;
        x.out = out;
        x.vol = ctx->vol;
        x.nplanes = B * XY_N;
        x.tau = f.tau;
        x.src_amp = ctx->src_amp;
        x.sinpi = ctx->srcsin;
        x.ta = ta;
        x.tab = CoefTab{f.tab, f.tab + XY_N, f.tab + 2 * XY_N};
        x.offd = -f.tau * ctx->h2inv;  // as setup_const_tab forms it
        void (*kx)(XYArgs) = ctx->p.source_kind ? xy3_kernel<1> : xy3_kernel<0>;
        const size_t shm = xy3_smem_bytes();
        CK(cudaFuncSetAttribute(kx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(2 * x.nplanes));
        cfg.blockDim = dim3(XY_T);
        cfg.dynamicSmemBytes = shm;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (prof) TRY(prof_begin(ctx));
        CK(cudaLaunchKernelEx(&cfg, kx, x));
        TRY(last_launch(ctx));
        if (prof) TRY(prof_end(ctx, PRS_K_XPASS, (double)B * (double)ctx->vol * 16.0));
        return launch_lpass(ctx, 2, f, out, out, B, ep, prof);
    }
    TRY(launch_xpass(ctx, scheme, f, in, out, B, ta, prof));
    if (ctx->p.dim == 2) return launch_lpass(ctx, 1, f, out, out, B, ep, prof);
    EpiArgs st;
    TRY(launch_lpass(ctx, 1, f, out, out, B, st, prof));
    return launch_lpass(ctx, 2, f, out, out, B, ep, prof);
}

// One unsplit implicit-Euler step (ie.cuh) on B consecutive states: dim forward sine transforms
// (the first forms U + tau F on its loads, the last divides by 1 + tau (c + sum mu) and
// normalises), dim inverse transforms (the last carries the epilogue).  Scratch alternates
// between two batches, so `in` may alias `out`.
static int ie_step(prs_ctx *ctx, double tau, const double *in, double *out, long long B, const TimeArgs &ta,
                   const EpiArgs &ep, bool prof) {
    const int n = ctx->p.n, dim = ctx->p.dim;
    if (B > ctx->ie_cap) {
        if (ctx->ie_w1) CK(cudaFree(ctx->ie_w1));
        if (ctx->ie_w2) CK(cudaFree(ctx->ie_w2));
        ctx->ie_w1 = ctx->ie_w2 = nullptr;
        ctx->ie_cap = 0;
        const long long cap = std::max<long long>(B, ctx->count);
        CK(cudaMalloc(&ctx->ie_w1, ctx->sbytes * cap));
        CK(cudaMalloc(&ctx->ie_w2, ctx->sbytes * cap));
        ctx->ie_cap = cap;
        ctx->scratch_gen++;  // captured graphs hold the old scratch pointers
    }
    IEArgs a{};
    a.S = ctx->ie_S;
    a.mu = ctx->ie_mu;
    a.vol = ctx->vol;
    a.ncols = B * (ctx->vol / n);
    a.n = n;
    a.dim = dim;
    a.src = ctx->p.source_kind != 0;
    a.tau = tau;
    a.src_amp = ctx->src_amp;
    a.sinpi = ctx->srcsin;
    a.ta = ta;
    a.creact = ctx->p.c;
    a.norm = std::pow(2.0 / (double)(n + 1), dim);
    a.e_gc = ep.gc;
    a.e_gcache = ep.gcache;
    a.e_delta = ep.delta;
    a.e_traj = ep.traj;
    a.e_red = ctx->red;
    const long long gy = (a.ncols + IE_BN - 1) / IE_BN;
    if (gy > 65535) {
        ctx->err = "IE step: more than 65535 x 64 lines per batch";
        return PRS_EUNSUPPORTED;
    }
    const dim3 grid((unsigned)((n + IE_BM - 1) / IE_BM), (unsigned)gy);
    double *w[2] = {ctx->ie_w1, ctx->ie_w2};
    const double *src = in;
    if (prof) TRY(prof_begin(ctx));
    for (int pass = 0; pass < 2 * dim; ++pass) {
        const int axis = pass % dim;
        const bool last = pass == 2 * dim - 1;
        a.in = src;
        a.out = last ? out : w[pass & 1];
        a.inner = 1;
        for (int d = 0; d < axis; ++d) a.inner *= n;
        if (pass == 0) ie_axis_kernel<1, EPI_STORE><<<grid, IE_T, 0, ctx->stream>>>(a);
        else if (pass == dim - 1) ie_axis_kernel<0, IE_SCALE><<<grid, IE_T, 0, ctx->stream>>>(a);
        else if (!last) ie_axis_kernel<0, EPI_STORE><<<grid, IE_T, 0, ctx->stream>>>(a);
        else if (ep.kind == EPI_DELTA) ie_axis_kernel<0, EPI_DELTA><<<grid, IE_T, 0, ctx->stream>>>(a);
        else if (ep.kind == EPI_CORRECT) ie_axis_kernel<0, EPI_CORRECT><<<grid, IE_T, 0, ctx->stream>>>(a);
        else if (ep.kind == EPI_INIT) ie_axis_kernel<0, EPI_INIT><<<grid, IE_T, 0, ctx->stream>>>(a);
        else ie_axis_kernel<0, EPI_STORE><<<grid, IE_T, 0, ctx->stream>>>(a);
        TRY(last_launch(ctx));
        src = a.out;
    }
    // fp64 flops: 2 dim transforms, each n multiply-adds per output element
    if (prof) TRY(prof_end(ctx, PRS_K_IE, 2.0 * dim * 2.0 * n * (double)B * (double)ctx->vol));
    return PRS_OK;
}

// hook for dd.cuh profiling
int prs_internal_prof_begin(prs_ctx *ctx) { return prof_begin(ctx); }
int prs_internal_prof_end(prs_ctx *ctx, int kind, double bytes) { return prof_end(ctx, kind, bytes); }

static double *state(prs_ctx *ctx, double *base, long long i) { return base + i * ctx->ss; }

// global index of local slice i; the rank owning global slice n; the end state of local slice i
static long long gslice(const prs_ctx *ctx, long long i) {
    return ctx->cyclic ? ctx->rank + i * ctx->nranks : ctx->first + i;
}
static int owner_of(const prs_ctx *ctx, int n) {
    if (ctx->cyclic) return n % ctx->nranks;
    for (int q = 0; q < ctx->nranks; ++q) {
        int f = 0, c = 0;
        prs_partition(ctx->p.N, ctx->nranks, q, &f, &c);
        if (n >= f && n < f + c) return q;
    }
    return -1;
}
static double *end_state(prs_ctx *ctx, long long i) {
    return ctx->cyclic ? state(ctx, ctx->tend, i) : state(ctx, ctx->traj, i + 1);
}
static long long slice_stride(const prs_ctx *ctx) { return ctx->cyclic ? ctx->nranks : 1; }

// ==================================================================== C ABI =========
extern "C" {

int prs_partition(int N, int nranks, int rank, int *first, int *count) {
    if (N < 1 || nranks < 1 || rank < 0 || rank >= nranks || nranks > N) return PRS_EINVAL;
    const int base = N / nranks, rem = N % nranks;
    *count = base + (rank < rem ? 1 : 0);
    *first = rank * base + (rank < rem ? rank : rem);
    return PRS_OK;
}

int prs_nccl_unique_id(void *uid128) {
    std::string err;
    if (!g_nccl.load(err)) return PRS_ENCCL;
    ncclUniqueId id;
    if (g_nccl.GetUniqueId(&id) != ncclSuccess) return PRS_ENCCL;
    memcpy(uid128, &id, sizeof(id));
    return PRS_OK;
}

static int validate(const prs_problem *p, std::string &err) {
    if (!p) { err = "null problem"; return PRS_EINVAL; }
    if (p->dim != 2 && p->dim != 3) { err = "dim must be 2 or 3"; return PRS_EINVAL; }
    if (p->n < 1) { err = "n must be >= 1"; return PRS_EINVAL; }
    if (!(p->c >= 0.0) || !(p->T > 0.0)) { err = "need c >= 0 and T > 0"; return PRS_EINVAL; }
    if (p->N < 1 || p->s < 1) { err = "need N >= 1 and s >= 1"; return PRS_EINVAL; }
    if ((p->G != PRS_FIE && p->G != PRS_DR && p->G != PRS_IE) ||
        (p->F != PRS_FIE && p->F != PRS_DR && p->F != PRS_IE)) {
        err = "schemes must be PRS_FIE, PRS_DR or PRS_IE";
        return PRS_EINVAL;
    }
    if ((p->G == PRS_IE || p->F == PRS_IE) && p->coef_kind != 0) {
        err = "the unsplit implicit Euler (PRS_IE) solves in the sine basis: constant coefficients "
              "(coef_kind 0, the paper's D = I problem of PAPER.md:449) only on the GPU path";
        return PRS_EUNSUPPORTED;
    }
    if (p->coef_kind == 2 && (p->split != 1 || p->dim != 2)) {
        err = "the full diffusion tensor (coef_kind 2, PAPER.md:520-546) needs the 2-D DD split (mixed "
              "derivatives: dimensional splitting does not apply, SPEC.md:128)";
        return PRS_EUNSUPPORTED;
    }
    if (p->coef_kind < 0 || p->coef_kind > 2) { err = "coef_kind must be 0, 1 or 2"; return PRS_EINVAL; }
    if (p->source_kind < 0 || p->source_kind > 2) { err = "source_kind must be 0, 1 or 2"; return PRS_EINVAL; }
    if (p->source_kind == 2 && (p->dim != 2 || p->coef_kind != 0)) {
        err = "source_kind 2 (the section-5.1 solution sin(2 pi t) sin(2 pi x) sin(2 pi y), PAPER.md:444-449) "
              "is defined for the 2-D problem with D = I (coef_kind 0)";
        return PRS_EINVAL;
    }
    if (p->split != 0 && p->split != 1) { err = "split must be 0 or 1"; return PRS_EINVAL; }
    if (p->split == 1) {
        if (p->dim != 2) { err = "DD splitting is 2-D"; return PRS_EUNSUPPORTED; }
        if (p->dd_strips < 1 || p->n % p->dd_strips != 0) {
            err = "n must be a multiple of dd_strips";
            return PRS_EINVAL;
        }
        if (p->dd_overlap < 0 || p->dd_overlap % 2 != 0 || p->dd_overlap >= p->n / p->dd_strips) {
            err = "dd_overlap must be even and smaller than the strip width";
            return PRS_EINVAL;
        }
        if (p->dd_ramp != 0 && p->dd_ramp != 1) { err = "dd_ramp must be 0 or 1"; return PRS_EINVAL; }
    }
    if (p->dim == 3 && p->coef_kind != 0) { err = "variable kappa is 2-D only"; return PRS_EUNSUPPORTED; }
    if (p->dim == 3 && (p->G == PRS_DR || p->F == PRS_DR)) {
        err = "3-D Douglas-Rachford (M = 3) is not implemented on the GPU path";
        return PRS_EUNSUPPORTED;
    }
    if (p->split == 0 && p->n > 16 * 256) { err = "n > 4096 is not supported by the line kernels"; return PRS_EUNSUPPORTED; }
    return PRS_OK;
}

void prs_destroy(prs_ctx *ctx);

// the context on `rank` of `nranks`, exchanging through `tr` (owned; nranks > 1)
static int create_impl(const prs_problem *prob, int rank, int nranks, Transport *tr, void *cuda_stream,
                       prs_ctx **out) {
    prs_ctx *ctx = new prs_ctx();
    ctx->tr = tr;
    int first = 0, count = 0;
    prs_partition(prob->N, nranks, rank, &first, &count);
    ctx->p = *prob;
    ctx->rank = rank;
    ctx->nranks = nranks;
    ctx->first = first;
    ctx->count = count;
    const int n = prob->n;
    ctx->vol = (prob->dim == 2) ? (long long)n * n : (long long)n * n * n;
    ctx->sbytes = sizeof(double) * (size_t)ctx->vol;
    ctx->M = (prob->split == 1) ? 2 : prob->dim;
    ctx->h = 1.0 / (double)(n + 1);
    ctx->h2inv = (double)(n + 1) * (double)(n + 1);
    ctx->creact = prob->c / (double)ctx->M;
    ctx->dT = prob->T / (double)prob->N;
    ctx->dt = prob->T / ((double)prob->N * (double)prob->s);
    *out = ctx;
#define CKC(call)                                                                \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);       \
            fprintf(stderr, "prs_create: %s\n", ctx->err.c_str());               \
            prs_destroy(ctx);                                                    \
            *out = nullptr;                                                      \
            return PRS_ECUDA;                                                    \
        }                                                                        \
    } while (0)
    CKC(cudaGetDevice(&ctx->device));
    CKC(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
    {
        const char *swv = getenv("PRS_SWEEP2");
        ctx->no_sweep2 = swv && swv[0] == '0';
        const char *xyv = getenv("PRS_XY");
        ctx->no_xy = xyv && xyv[0] == '0';
        const char *sv = getenv("PRS_SKIP");
        ctx->skip_converged = sv ? (sv[0] == '1') : (ctx->vol >= (1LL << 18));
        const char *lg = getenv("PRS_LAG");
        ctx->lag = !(lg && lg[0] == '0');
        const char *gv = getenv("PRS_GRAPHS");
        ctx->graphs = !(gv && gv[0] == '0');
        const char *tv = getenv("PRS_X7TMA");
        ctx->x7_tma = !(tv && tv[0] == '0');
    }
    if (cuda_stream) {
        ctx->stream = (cudaStream_t)cuda_stream;
    } else {
        // a blocking stream: it orders with the legacy default stream, on which callers that
        // pass no stream (e.g. PyTorch's default stream) fill the input buffers
        CKC(cudaStreamCreate(&ctx->stream));
        ctx->own_stream = true;
    }
    ctx->ss = ctx->vol;
    const size_t sb = sizeof(double) * (size_t)ctx->ss;
    CKC(cudaMalloc(&ctx->traj, sb * (count + 1)));
    CKC(cudaMalloc(&ctx->fa, sb * count));
    CKC(cudaMalloc(&ctx->fb, sb * count));
    CKC(cudaMalloc(&ctx->gcache, sb * count));
    CKC(cudaMalloc(&ctx->gtmp, sb));
    CKC(cudaMalloc(&ctx->u0, sb));
    CKC(cudaMalloc(&ctx->sinpi, sizeof(double) * n));
    CKC(cudaMalloc(&ctx->s2n, sizeof(double) * n));
    CKC(cudaMalloc(&ctx->s2f, sizeof(double) * (n + 1)));
    CKC(cudaMalloc(&ctx->red_base, sizeof(unsigned long long) * 8));
    CKC(cudaMallocHost(&ctx->red_host, sizeof(unsigned long long) * 8));
    ctx->red = ctx->red_base;
    setup_sines<<<(n + 1 + 255) / 256, 256, 0, ctx->stream>>>(n, ctx->h, ctx->sinpi, ctx->s2n, ctx->s2f);
    ctx->launches++;
    ctx->src_amp = prob->source_kind == 2 ? 1.0 : (double)prob->dim * M_PI * M_PI + prob->c - 1.0;
    ctx->srcsin = prob->source_kind == 2 ? ctx->s2n : ctx->sinpi;
    CKC(cudaGetLastError());
    if (prob->split == 1) {
        int drc = dd_init(ctx->dd, *prob, ctx->h, ctx->h2inv, ctx->stream, ctx->err);
        if (drc != PRS_OK) {
            fprintf(stderr, "prs_create: %s\n", ctx->err.c_str());
            prs_destroy(ctx);
            *out = nullptr;
            return drc;
        }
        ctx->dd.sinpi = ctx->srcsin;
    }
    if (prob->G == PRS_IE || prob->F == PRS_IE) {
        CKC(cudaMalloc(&ctx->ie_S, sizeof(double) * (size_t)n * n));
        CKC(cudaMalloc(&ctx->ie_mu, sizeof(double) * n));
        const long long ne = (long long)n * n;
        ie_setup_kernel<<<(unsigned)((ne + 255) / 256), 256, 0, ctx->stream>>>(n, ctx->h2inv, ctx->ie_S, ctx->ie_mu);
        ctx->launches++;
        CKC(cudaGetLastError());
    }
    int frc = ensure_factors(ctx, 0, ctx->dT);
    if (frc == PRS_OK) frc = ensure_factors(ctx, 1, ctx->dt);
    if (frc != PRS_OK) {
        fprintf(stderr, "prs_create: %s\n", ctx->err.c_str());
        prs_destroy(ctx);
        *out = nullptr;
        return frc;
    }
    CKC(cudaStreamSynchronize(ctx->stream));
#undef CKC
    return PRS_OK;
}

static int precreate(const prs_problem *prob, int rank, int nranks, prs_ctx **out) {
    if (!out) return PRS_EINVAL;
    *out = nullptr;
    std::string verr;
    int rc = validate(prob, verr);
    if (rc != PRS_OK) {
        fprintf(stderr, "prs_create: %s\n", verr.c_str());
        return rc;
    }
    int first = 0, count = 0;
    if (prs_partition(prob->N, nranks, rank, &first, &count) != PRS_OK) return PRS_EINVAL;
    return PRS_OK;
}

int prs_create(const prs_problem *prob, int rank, int nranks, const void *nccl_uid, void *cuda_stream,
               prs_ctx **out) {
    TRY(precreate(prob, rank, nranks, out));
    if (nranks > 1 && !nccl_uid) return PRS_EINVAL;
    NcclTransport *tr = nullptr;
    if (nranks > 1) {
        tr = new NcclTransport();
        tr->my_rank = rank;
        if (tr->init(nccl_uid, nranks, rank) != PRS_OK) {
            fprintf(stderr, "prs_create: %s\n", tr->err.c_str());
            delete tr;
            return PRS_ENCCL;
        }
    }
    return create_impl(prob, rank, nranks, tr, cuda_stream, out);
}

int prs_local_world_create(int nranks, void **world) {
    if (!world || nranks < 1) return PRS_EINVAL;
    *world = new LocalWorld(nranks);
    return PRS_OK;
}

void prs_local_world_destroy(void *world) { delete static_cast<LocalWorld *>(world); }

int prs_create_local(const prs_problem *prob, int rank, void *world, void *cuda_stream, prs_ctx **out) {
    if (!world) return PRS_EINVAL;
    LocalWorld *w = static_cast<LocalWorld *>(world);
    TRY(precreate(prob, rank, w->P, out));
    return create_impl(prob, rank, w->P, w->P > 1 ? new LocalTransport(w, rank) : nullptr, cuda_stream, out);
}

static void pipe_free(prs_ctx *ctx) {
    for (auto st : ctx->psF) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    if (ctx->psC) {
        cudaStreamSynchronize(ctx->psC);
        cudaStreamDestroy(ctx->psC);
    }
    for (auto e : ctx->pevF) cudaEventDestroy(e);
    for (auto e : ctx->pevC) cudaEventDestroy(e);
    for (cudaEvent_t e : {ctx->pev0, ctx->pevRed[0], ctx->pevRed[1]})
        if (e) cudaEventDestroy(e);
    if (ctx->traj2) cudaFree(ctx->traj2);
    if (ctx->gcache2) cudaFree(ctx->gcache2);
    if (ctx->pred) cudaFree(ctx->pred);
    if (ctx->pred_host) cudaFreeHost(ctx->pred_host);
    ctx->psF.clear();
    ctx->pevF.clear();
    ctx->pevC.clear();
    ctx->psC = nullptr;
    ctx->pev0 = ctx->pevRed[0] = ctx->pevRed[1] = nullptr;
    ctx->traj2 = ctx->gcache2 = nullptr;
    ctx->pred = ctx->pred_host = nullptr;
    ctx->pipe = 0;
}

void prs_destroy(prs_ctx *ctx) {
    if (!ctx) return;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
#ifdef PRS_DD_TIMING
    {
        unsigned long long h[4] = {0, 0, 0, 0};
        cudaMemcpyFromSymbol(h, prs::g_dd_timing, sizeof(h));
        if (h[3])
            fprintf(stderr, "DD timing: %llu tasks, per task %.1f us, forward wait %.1f us, backward wait %.1f us\n",
                    h[3], h[2] / 1e3 / h[3], h[0] / 1e3 / h[3], h[1] / 1e3 / h[3]);
        unsigned long long g[9];
        cudaMemcpyFromSymbol(g, prs::g_dd2_timing, sizeof(g));
        if (g[7] && g[8])
            fprintf(stderr,
                    "DD split timing (us per task, thread 0): p1 %llu tasks: load %.2f gemm(+turn) %.2f store+walk %.2f "
                    "| p2 %llu tasks: load+walk %.2f gemm(+turn) %.2f store %.2f\n",
                    g[7], g[0] / 1e3 / g[7], g[1] / 1e3 / g[7], g[2] / 1e3 / g[7], g[8], g[3] / 1e3 / g[8],
                    g[4] / 1e3 / g[8], g[5] / 1e3 / g[8]);
    }
#endif
#ifdef PRS_X7_TIMING
    {
        unsigned long long h[2][10];
        cudaMemcpyFromSymbol(h, prs::g_x7_timing, sizeof(h));
        static const char *ph[9] = {"cp.async wait", "barrier", "loads+stencil", "F1+scan", "fwd msg", "F3+scan",
                                    "bwd msg", "B3+store", "scalars+issue"};
        for (int r = 0; r < 2; ++r)
            if (h[r][9]) {
                fprintf(stderr, "x7 timing rank %d: %llu rows, cycles per row:", r, h[r][9]);
                double tot = 0;
                for (int p = 0; p < 9; ++p) tot += (double)h[r][p] / h[r][9];
                for (int p = 0; p < 9; ++p) fprintf(stderr, " %s %.0f", ph[p], (double)h[r][p] / h[r][9]);
                fprintf(stderr, " | total %.0f\n", tot);
            }
    }
#endif
    delete ctx->tr;
    double *bufs[] = {ctx->traj, ctx->fa, ctx->fb, ctx->gcache, ctx->gtmp, ctx->u0, ctx->cyc2,
                      ctx->sinpi, ctx->s2n, ctx->s2f, ctx->tend};
    for (double *b : bufs)
        if (b) cudaFree(b);
    for (auto &f : ctx->fac) {
        if (f.tab) cudaFree(f.tab);
        if (f.invdx) cudaFree(f.invdx);
        if (f.invdy) cudaFree(f.invdy);
    }
    dd_free(ctx->dd);
    if (ctx->red_base) cudaFree(ctx->red_base);
    if (ctx->red_host) cudaFreeHost(ctx->red_host);
    if (ctx->ctl) {
        cudaStreamSynchronize(ctx->ctl);
        cudaStreamDestroy(ctx->ctl);
    }
    for (cudaEvent_t e : {ctx->ev_chain[0], ctx->ev_chain[1], ctx->ev_red[0], ctx->ev_red[1]})
        if (e) cudaEventDestroy(e);
    if (ctx->l5buf) cudaFree(ctx->l5buf);
    if (ctx->fine_exec) cudaGraphExecDestroy(ctx->fine_exec);
    {
        for (double *q : {ctx->ie_S, ctx->ie_mu, ctx->ie_w1, ctx->ie_w2})
            if (q) cudaFree(q);
        double *gb[] = {ctx->gb_u, ctx->gb_d, ctx->gb_gc, ctx->gb_v, ctx->gb_tt, ctx->gb_tot, ctx->gb_yx};
        for (double *b : gb)
            if (b) cudaFree(b);
    }
    if (ctx->corr_exec) cudaGraphExecDestroy(ctx->corr_exec);
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    pipe_free(ctx);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char *prs_last_error(const prs_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int prs_set_initial(prs_ctx *ctx, const double *u0, int u0_on_device) {
    if (!ctx || !u0) return PRS_EINVAL;
    CK(cudaMemcpyAsync(ctx->u0, u0, ctx->sbytes, u0_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       ctx->stream));
    if (ctx->rank == 0) CK(cudaMemcpyAsync(ctx->traj, ctx->u0, ctx->sbytes, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->red_base + 2, 0, sizeof(unsigned long long), ctx->stream));
    absmax_kernel<<<148 * 4, 256, 0, ctx->stream>>>(ctx->u0, ctx->vol, ctx->red_base + 2);
    TRY(last_launch(ctx));
    CK(cudaMemcpyAsync(ctx->red_host + 2, ctx->red_base + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    double nrm;
    memcpy(&nrm, ctx->red_host + 2, sizeof(double));
    ctx->u0norm = (nrm > 0.0) ? nrm : 1.0;
    ctx->have_initial = true;
    ctx->have_coarse = false;
    ctx->gb_valid = false;
    return PRS_OK;
}

static bool sweep2_ok(const prs_ctx *ctx);
static int launch_chain2(prs_ctx *ctx, int i0, int epi);
static int chain2_cyclic_one(prs_ctx *ctx, int i, int epi);

static TimeArgs coarse_time(prs_ctx *ctx, int slice) {
    TimeArgs ta;
    ta.slice0 = slice;
    ta.tmul = 1;
    ta.toff = 1;
    ta.tstep = ctx->dT;
    return ta;
}

int prs_coarse_sweep(prs_ctx *ctx) {
    if (!ctx) return PRS_EINVAL;
    if (!ctx->have_initial) { ctx->err = "prs_set_initial first"; return PRS_EINVAL; }
    TRY(ensure_factors(ctx, 0, ctx->dT));
    if (ctx->cyclic) {
        // slice n on rank n mod P: receive U^0_n from the previous slice's rank, one G step with
        // the initial-guess epilogue, hand U^0_{n+1} to the next slice's rank
        for (int i = 0; i < ctx->count; ++i) {
            const int n = (int)gslice(ctx, i);
            if (n > 0) NK(ctx->tr->recv(state(ctx, ctx->traj, i), (size_t)ctx->vol, owner_of(ctx, n - 1), ctx->stream));
            if (sweep2_ok(ctx)) {
                TRY(chain2_cyclic_one(ctx, i, EPI_INIT));
            } else {
                EpiArgs ep;
                ep.kind = EPI_INIT;
                ep.gcache = state(ctx, ctx->gcache, i);
                ep.traj = end_state(ctx, i);
                TRY(run_step(ctx, ctx->p.G, ctx->fac[0], state(ctx, ctx->traj, i), ctx->gtmp, 1, coarse_time(ctx, n),
                             ep, false, ctx->ss));
            }
            if (n + 1 < ctx->p.N)
                NK(ctx->tr->send(end_state(ctx, i), (size_t)ctx->vol, owner_of(ctx, n + 1), ctx->stream));
        }
        ctx->have_coarse = true;
        return PRS_OK;
    }
    if (ctx->nranks > 1 && ctx->rank > 0) NK(ctx->tr->recv(ctx->traj, (size_t)ctx->vol, ctx->rank - 1, ctx->stream));
    if (sweep2_ok(ctx)) TRY(launch_chain2(ctx, 0, EPI_INIT));
    for (int i = sweep2_ok(ctx) ? ctx->count : 0; i < ctx->count; ++i) {
        EpiArgs ep;
        ep.kind = EPI_INIT;
        ep.gcache = state(ctx, ctx->gcache, i);
        ep.traj = state(ctx, ctx->traj, i + 1);
        TRY(run_step(ctx, ctx->p.G, ctx->fac[0], state(ctx, ctx->traj, i), ctx->gtmp, 1,
                     coarse_time(ctx, ctx->first + i), ep, false, ctx->ss));
    }
    if (ctx->nranks > 1 && ctx->rank < ctx->nranks - 1)
        NK(ctx->tr->send(state(ctx, ctx->traj, ctx->count), (size_t)ctx->vol, ctx->rank + 1, ctx->stream));
    ctx->have_coarse = true;
    ctx->gb_valid = false;
    return PRS_OK;
}

// first local slice that still needs work (prs_iterate's converged prefix, else 0)
static int local_start(const prs_ctx *ctx) {
    if (ctx->cyclic) {  // local slices with rank + i P < kconv
        const int k = ctx->kconv - ctx->rank;
        const int i0 = k <= 0 ? 0 : (k + ctx->nranks - 1) / ctx->nranks;
        return i0 > ctx->count ? ctx->count : i0;
    }
    const int k = ctx->kconv - ctx->first;
    return k <= 0 ? 0 : (k > ctx->count ? ctx->count : k);
}

// small 2-D slices (kappa = 1, n = 32 / 64 / 128 / 256): the whole sweep on chip (sweep2.cuh)
static bool sweep2_ok(const prs_ctx *ctx) {
    const int n = ctx->p.n;
    return !ctx->no_sweep2 && ctx->p.dim == 2 && ctx->p.split == 0 && ctx->p.coef_kind == 0 &&
           ctx->p.G != PRS_IE && ctx->p.F != PRS_IE && ctx->p.source_kind != 2 &&
           (n == 32 || n == 64 || n == 128 || n == 256);
}

static int launch_sweep2(prs_ctx *ctx, const double *in, double *out, const double *gc, long long B, long long slice0,
                         int steps, cudaStream_t st = nullptr) {
    const int n = ctx->p.n;
    const TauFactors &f = ctx->fac[1];
    SWArgs a{};
    a.in = in;
    a.out = out;
    a.gc = gc;
    a.vol = ctx->ss;
    a.s = steps;
    a.tau = f.tau;
    a.h2inv = ctx->h2inv;
    a.creact = ctx->creact;
    a.src_amp = ctx->src_amp;
    a.sinpi = ctx->srcsin;
    a.slice0 = slice0;
    a.sstride = slice_stride(ctx);
    a.dt = ctx->dt;
    a.tab = CoefTab{f.tab, f.tab + n, f.tab + 2 * n};
    const int dr = (ctx->p.F == PRS_DR) ? 1 : 0, src = ctx->p.source_kind != 0, epi = gc ? EPI_DELTA : EPI_STORE;
    void (*k)(SWArgs) = nullptr;
    size_t shm = 0;
#define SK(N_, D, S_, E)                                                   \
    if (n == N_ && dr == D && src == S_ && epi == E) {                     \
        k = sweep2_kernel<N_, D, S_, E>;                                   \
        shm = sizeof(double) * sweep2_smem_doubles<N_>();                   \
    }
#define SKN(N_) SK(N_, 0, 0, 0) SK(N_, 0, 1, 0) SK(N_, 1, 0, 0) SK(N_, 1, 1, 0) \
                SK(N_, 0, 0, 1) SK(N_, 0, 1, 1) SK(N_, 1, 0, 1) SK(N_, 1, 1, 1)
    SKN(32) SKN(64) SKN(128) SKN(256)
#undef SKN
#undef SK
    const int CL = n / SW_R;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(B * CL));
    cfg.blockDim = dim3(SW_T);
    cfg.dynamicSmemBytes = shm;
    cfg.stream = st ? st : ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (ctx->prof) TRY(prof_begin(ctx));
    CK(cudaLaunchKernelEx(&cfg, k, a));
    TRY(last_launch(ctx));
    // 32 B per update for a 2-D step; on chip here, so the rate is an effective one
    if (ctx->prof) TRY(prof_end(ctx, PRS_K_XPASS, (double)B * (double)ctx->vol * ctx->p.s * 32.0));
    return PRS_OK;
}

// the coarse chain of local slices i0 .. i1-1 on chip (sweep2 with CHAIN = 1): one cluster.
// traj / gcache / delta are batch buffers (slice stride ss); U_{i0} is read from traj.
static int launch_chain2x(prs_ctx *ctx, double *traj, double *gcache, const double *delta, int i0, int i1, int epi,
                          unsigned long long *red, cudaStream_t st, const double *trajold = nullptr,
                          long long slice0 = -1) {
    const int n = ctx->p.n, cnt = i1 - i0;
    if (cnt <= 0) return PRS_OK;
    const TauFactors &f = ctx->fac[0];
    SWArgs a{};
    a.in = state(ctx, traj, i0);
    a.traj = state(ctx, traj, i0);
    a.trajold = trajold ? state(ctx, const_cast<double *>(trajold), i0) : nullptr;
    a.gcache = state(ctx, gcache, i0);
    a.delta = (epi == EPI_CORRECT) ? state(ctx, const_cast<double *>(delta), i0) : nullptr;
    a.red = red;
    a.vol = ctx->ss;
    a.s = cnt;
    a.tau = f.tau;
    a.h2inv = ctx->h2inv;
    a.creact = ctx->creact;
    a.src_amp = ctx->src_amp;
    a.sinpi = ctx->srcsin;
    a.slice0 = slice0 >= 0 ? slice0 : ctx->first + i0;
    a.sstride = 1;
    a.dt = ctx->dT;
    a.tab = CoefTab{f.tab, f.tab + n, f.tab + 2 * n};
    const int dr = (ctx->p.G == PRS_DR) ? 1 : 0, src = ctx->p.source_kind != 0;
    void (*k)(SWArgs) = nullptr;
    size_t shm = 0;
#define SK(N_, D, S_, E)                                                   \
    if (n == N_ && dr == D && src == S_ && epi == E) {                     \
        k = sweep2_kernel<N_, D, S_, E, 1>;                                \
        shm = sizeof(double) * sweep2_smem_doubles<N_>();                   \
    }
#define SKN(N_) SK(N_, 0, 0, EPI_CORRECT) SK(N_, 0, 1, EPI_CORRECT) SK(N_, 1, 0, EPI_CORRECT) \
                SK(N_, 1, 1, EPI_CORRECT) SK(N_, 0, 0, EPI_INIT) SK(N_, 0, 1, EPI_INIT)       \
                SK(N_, 1, 0, EPI_INIT) SK(N_, 1, 1, EPI_INIT)
    SKN(32) SKN(64) SKN(128) SKN(256)
#undef SKN
#undef SK
    if (!k) {
        ctx->err = "chain2: unsupported shape";
        return PRS_EUNSUPPORTED;
    }
    const int CL = n / SW_R;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)CL);
    cfg.blockDim = dim3(SW_T);
    cfg.dynamicSmemBytes = shm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k, a));
    return last_launch(ctx);
}

static int launch_chain2(prs_ctx *ctx, int i0, int epi) {
    return launch_chain2x(ctx, ctx->traj, ctx->gcache, ctx->delta, i0, ctx->count, epi, ctx->red, ctx->stream);
}

// cyclic ownership, on-chip shapes: the G step (+ epilogue) of local slice i by the same on-chip
// chain kernel as contiguous ownership (so the results stay bitwise those of one rank): the chain
// runs on a two-state scratch [U_i, U_{i+1}]; U_{i+1} (and, for the update norm, the old end
// state) live in tend[i]
static int chain2_cyclic_one(prs_ctx *ctx, int i, int epi) {
    if (!ctx->cyc2) CK(cudaMalloc(&ctx->cyc2, sizeof(double) * 2 * ctx->ss));
    double *te = const_cast<double *>(end_state(ctx, i));
    CK(cudaMemcpyAsync(ctx->cyc2, state(ctx, ctx->traj, i), sizeof(double) * ctx->vol, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    TRY(launch_chain2x(ctx, ctx->cyc2, state(ctx, ctx->gcache, i), epi == EPI_CORRECT ? state(ctx, ctx->delta, i) : nullptr,
                       0, 1, epi, ctx->red, ctx->stream, epi == EPI_CORRECT ? te - ctx->ss : nullptr, gslice(ctx, i)));
    CK(cudaMemcpyAsync(te, ctx->cyc2 + ctx->ss, sizeof(double) * ctx->vol, cudaMemcpyDeviceToDevice, ctx->stream));
    return PRS_OK;
}

static int enqueue_fine_sweep(prs_ctx *ctx) {
    const int s = ctx->p.s;
    const int i0 = local_start(ctx);
    const long long B = ctx->count - i0;
    if (B <= 0) return PRS_OK;
    if (sweep2_ok(ctx))
        return launch_sweep2(ctx, state(ctx, ctx->traj, i0), state(ctx, (s & 1) ? ctx->fa : ctx->fb, i0),
                             state(ctx, ctx->gcache, i0), B, gslice(ctx, i0), s);
    const double *src = state(ctx, ctx->traj, i0);
    double *bufs[2] = {state(ctx, ctx->fa, i0), state(ctx, ctx->fb, i0)};
    for (int j = 0; j < s; ++j) {
        double *dst = bufs[j & 1];
        TimeArgs ta;
        ta.slice0 = gslice(ctx, i0);
        ta.sstride = slice_stride(ctx);
        ta.tmul = s;
        ta.toff = j + 1;
        ta.tstep = ctx->dt;
        EpiArgs ep;
        if (j == s - 1) {
            ep.kind = EPI_DELTA;
            ep.gc = state(ctx, ctx->gcache, i0);
        }
        TRY(run_step(ctx, ctx->p.F, ctx->fac[1], src, dst, B, ta, ep, ctx->prof, ctx->ss));
        src = dst;
    }
    return PRS_OK;
}

// Run `enqueue` directly, or (single rank, profiling off, from the second call on) as a replay
// of its captured CUDA graph.  Kernel arguments are the context's fixed buffers, so one
// capture serves every later call.
static int run_graphed(prs_ctx *ctx, int (*enqueue)(prs_ctx *), int &calls, cudaGraphExec_t &exec,
                       long long &per_replay, int &gen) {
    // (graphs are captured for the full batch: a converged prefix launches directly)
    const bool use = ctx->graphs && ctx->nranks == 1 && !ctx->prof && local_start(ctx) == 0;
    if (!use || calls++ == 0) return enqueue(ctx);
    if (exec && gen != ctx->scratch_gen + ctx->dd.gen) {
        // scratch reallocated since the capture: the graph is stale; this call launches
        // directly (sizing the scratch again), the next one captures anew
        CK(cudaGraphExecDestroy(exec));
        exec = nullptr;
        return enqueue(ctx);
    }
    if (!exec) {
        const long long l0 = ctx->launches;
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        const int rc = enqueue(ctx);
        cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
        if (rc != PRS_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e != cudaSuccess) {
            ctx->err = std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e);
            return PRS_ECUDA;
        }
        e = cudaGraphInstantiate(&exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            exec = nullptr;
            ctx->err = std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e);
            return PRS_ECUDA;
        }
        per_replay = ctx->launches - l0;
        ctx->launches = l0;
        gen = ctx->scratch_gen + ctx->dd.gen;
    }
    CK(cudaGraphLaunch(exec, ctx->stream));
    ctx->launches += per_replay;
    return PRS_OK;
}

int prs_fine_sweep(prs_ctx *ctx) {
    if (!ctx) return PRS_EINVAL;
    if (!ctx->have_coarse) { ctx->err = "prs_coarse_sweep first"; return PRS_EINVAL; }
    TRY(ensure_factors(ctx, 1, ctx->dt));
    TRY(run_graphed(ctx, enqueue_fine_sweep, ctx->fine_calls, ctx->fine_exec, ctx->fine_glaunch, ctx->fine_gen));
    ctx->delta = (ctx->p.s & 1) ? ctx->fa : ctx->fb;
    if (ctx->prof) TRY(prof_flush(ctx));
    return PRS_OK;
}

// ---------------------------------------------------------- space-parallel G -------
static L5Args gp_l5(prs_ctx *ctx, int b) {
    const int n = ctx->p.n, nrb = ctx->gnb / L5RB;
    const TauFactors &f = ctx->fac[0];
    L5Args a{};
    a.vol = (long long)ctx->gnb * n;
    a.n = n;
    a.Sl = n;
    a.nq = 1;
    a.Sq = a.vol;
    a.nrb = nrb;
    a.ncb = n / L5W;
    a.nsq = 1;
    a.ntiles = (long long)nrb * a.ncb;
    a.tau = f.tau;
    a.h2inv = ctx->h2inv;
    a.tab = CoefTab{f.tab, f.tab ? f.tab + n : nullptr, f.tab ? f.tab + 2 * n : nullptr};
    a.invd = f.invdy;
    a.s2n = ctx->s2n;
    a.s2f = ctx->s2f;
    a.tstride = (long long)nrb * n;
    a.tt = ctx->gb_tt + (long long)b * 7 * a.tstride;
    a.yx = a.tt + 5 * a.tstride;
    a.row0 = b * ctx->gnb;
    a.ybeg = ctx->gb_yx + (long long)b * 2 * n;
    a.xend = a.ybeg + n;
    a.e_red = ctx->red;
    return a;
}

// phase 1 of band b's G step for slice `slice`: x stage (row-local) into v, the band's y block
// tuples and its band tuple (gb_tot[b])
static int gp_phase1(prs_ctx *ctx, int b, const double *in, double *v, int slice) {
    const int n = ctx->p.n;
    const TauFactors &f = ctx->fac[0];
    X3Args x{};
    x.in = in;
    x.out = v;
    x.vol = (long long)ctx->gnb * n;
    x.n = n;
    x.P = n / LCH;
    x.lines_per_state = ctx->gnb;
    x.ngroups = (long long)ctx->gnb * n / 4096;
    x.nstates = 1;
    x.nranges = 0;
    x.dim = 2;
    x.row0 = b * ctx->gnb;
    x.tau = f.tau;
    x.h2inv = ctx->h2inv;
    x.creact = ctx->creact;
    x.src_amp = ctx->src_amp;
    x.sinpi = ctx->srcsin;
    x.ta = coarse_time(ctx, slice);
    x.tab = CoefTab{f.tab, f.tab ? f.tab + n : nullptr, f.tab ? f.tab + 2 * n : nullptr};
    x.invd = f.invdx;
    x.s2n = ctx->s2n;
    x.s2f = ctx->s2f;
    const int coef = ctx->p.coef_kind, src = ctx->p.source_kind != 0;
    void (*kx)(X3Args) = nullptr;
#define XK(C, S_) if (coef == C && src == S_) kx = xpass3_kernel<C, 0, S_>;
    XK(0, 0) XK(0, 1) XK(1, 0) XK(1, 1)
#undef XK
    const size_t shm = xpass3_smem_bytes(coef);
    CK(cudaFuncSetAttribute(kx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    kx<<<(unsigned)std::min<long long>(ctx->num_sms, x.ngroups), X3T, shm, ctx->stream>>>(x);
    TRY(last_launch(ctx));
    L5Args a = gp_l5(ctx, b);
    a.in = v;
    a.out = v;
    (coef ? lp5_tuples_kernel<1> : lp5_tuples_kernel<0>)<<<(unsigned)a.ntiles, L5T, 0, ctx->stream>>>(a);
    TRY(last_launch(ctx));
    gp_band_total_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(a, ctx->gb_tot + (long long)b * 5 * n);
    TRY(last_launch(ctx));
    return PRS_OK;
}

// phase 2 of band b: boundary values from all band tuples, scan, finish with the fused
// correction epilogue on the band's rows of U_{n+1}, the G cache and Delta_n
static int gp_phase2(prs_ctx *ctx, int b, double *v, double *traj_next, double *gcache, const double *delta) {
    const int n = ctx->p.n;
    L5Args a = gp_l5(ctx, b);
    a.in = v;
    a.out = v;
    a.e_traj = traj_next;
    a.e_gcache = gcache;
    a.e_delta = delta;
    gp_boundary_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(ctx->gb_tot, ctx->gP, b, n,
                                                                 const_cast<double *>(a.ybeg),
                                                                 const_cast<double *>(a.xend));
    TRY(last_launch(ctx));
    lp5_scan_kernel<<<(n + 255) / 256, 256, 0, ctx->stream>>>(a, (long long)n);
    TRY(last_launch(ctx));
    (ctx->p.coef_kind ? lp5_finish_kernel<1, EPI_CORRECT> : lp5_finish_kernel<0, EPI_CORRECT>)
        <<<(unsigned)a.ntiles, L5T, 0, ctx->stream>>>(a);
    TRY(last_launch(ctx));
    return PRS_OK;
}

// The band exchange of space-parallel G over P = nranks ranks as a list of point-to-point
// operations (host logic, also exported as prs_gpar_plan for the multi-process tests): each op is
// {kind (0 send, 1 recv, 2 local copy), what (0 Delta_slice, 1 U_{slice+1}, 2 Gcache_slice),
//  slice, band, peer, local index of the owner-side state}; the ops between any two ranks come
// in the same order on both sides (NCCL group / in-order matching).
//   phase 0 (scatter): band p of Delta_sl from owner(sl) to rank p;
//   phase 1 (gather) : band p of U_{sl+1} to owner(sl) (its end state) and, at a rank edge, to
//                      owner(sl+1) (its incoming state, local index 0); band p of Gcache_sl to
//                      owner(sl);
//   phase 2 (seed)   : band p of U_{sl+1} from owner(sl) to rank p (what = 1): the bands of the
//                      current iterate, before the first band chain after the trajectory was
//                      written elsewhere (the chain's update norm compares against them).
static int gpar_plan(int N, int nranks, int me, int phase, std::vector<int> &ops) {
    ops.clear();
    const int P = nranks;
    std::vector<int> own(N), first(P);
    for (int q = 0; q < P; ++q) {
        int f0 = 0, c0 = 0;
        if (prs_partition(N, P, q, &f0, &c0) != PRS_OK) return PRS_EINVAL;
        first[q] = f0;
        for (int sl = f0; sl < f0 + c0; ++sl) own[sl] = q;
    }
    auto push = [&](int kind, int what, int sl, int band, int peer, int lidx) {
        ops.insert(ops.end(), {kind, what, sl, band, peer, lidx});
    };
    if (phase == 0 || phase == 2) {
        const int what = (phase == 0) ? 0 : 1, off = (phase == 0) ? 0 : 1;
        for (int sl = 0; sl < N; ++sl) {
            const int q = own[sl];
            if (q == me) {
                for (int p = 0; p < P; ++p) push(p == me ? 2 : 0, what, sl, p, p, sl + off - first[q]);
            } else {
                push(1, what, sl, me, q, -1);
            }
        }
        return PRS_OK;
    }
    for (int sl = 0; sl < N; ++sl) {
        const int q = own[sl];
        const int qn = (sl + 1 < N) ? own[sl + 1] : -1;
        for (int p = 0; p < P; ++p) {
            const int dsts[2] = {q, (qn != q) ? qn : -1};
            for (int dst : dsts) {
                if (dst < 0) continue;
                const int lidx = (dst == q) ? sl + 1 - first[q] : 0;
                if (p == me && dst == me) push(2, 1, sl, p, me, lidx);
                else if (p == me) push(0, 1, sl, p, dst, lidx);
                else if (dst == me) push(1, 1, sl, p, p, lidx);
            }
            if (p == me && q == me) push(2, 2, sl, p, me, sl - first[q]);
            else if (p == me) push(0, 2, sl, p, q, sl - first[q]);
            else if (q == me) push(1, 2, sl, p, p, sl - first[q]);
        }
    }
    return PRS_OK;
}

// the correction chain with space-parallel G.  One process: every slice, all P bands are
// views into the full states.  P ranks: this rank's band of every state, Delta bands
// scattered from the slice owners first, U / G-cache bands gathered back afterwards.
static int gp_correct(prs_ctx *ctx) {
    const int n = ctx->p.n, P = ctx->gP;
    const long long bvol = (long long)ctx->gnb * n;
    const size_t bbytes = sizeof(double) * (size_t)bvol;
    CK(cudaMemsetAsync(ctx->red, 0, sizeof(unsigned long long) * 2, ctx->stream));
    if (ctx->nranks == 1) {
        for (int i = local_start(ctx); i < ctx->count; ++i) {
            for (int b = 0; b < P; ++b)
                TRY(gp_phase1(ctx, b, state(ctx, ctx->traj, i) + b * bvol, ctx->gb_v + b * bvol, ctx->first + i));
            for (int b = 0; b < P; ++b)
                TRY(gp_phase2(ctx, b, ctx->gb_v + b * bvol, state(ctx, ctx->traj, i + 1) + b * bvol,
                              state(ctx, ctx->gcache, i) + b * bvol, state(ctx, ctx->delta, i) + b * bvol));
        }
        return PRS_OK;
    }
    const int me = ctx->rank, N = ctx->p.N;
    // U_0's band (U^{k+1}_0 = U_0)
    CK(cudaMemcpyAsync(ctx->gb_u, ctx->u0 + (long long)me * bvol, bbytes, cudaMemcpyDeviceToDevice, ctx->stream));
    // phase 2 (seed, when stale): band p of U^k_{n+1} from owner(n) to rank p;
    // phase 0 (scatter): band p of Delta_n from owner(n) to rank p
    std::vector<int> ops;
    for (int phase : {2, 0}) {
        if (phase == 2 && ctx->gb_valid) continue;
        TRY(gpar_plan(N, ctx->nranks, me, phase, ops));
        double *mine = (phase == 0) ? ctx->gb_d : ctx->gb_u + bvol;  // band of slice sl at + sl * bvol
        const double *src = (phase == 0) ? ctx->delta : ctx->traj;
        NK(ctx->tr->group_start());
        for (size_t o = 0; o < ops.size(); o += 6) {
            const int kind = ops[o], sl = ops[o + 2], band = ops[o + 3], peer = ops[o + 4], lidx = ops[o + 5];
            if (kind == 1) {
                NK(ctx->tr->recv(mine + sl * bvol, (size_t)bvol, peer, ctx->stream));
            } else {
                const double *d = state(ctx, const_cast<double *>(src), lidx) + band * bvol;
                if (kind == 2)
                    CK(cudaMemcpyAsync(mine + sl * bvol, d, bbytes, cudaMemcpyDeviceToDevice, ctx->stream));
                else
                    NK(ctx->tr->send(d, (size_t)bvol, peer, ctx->stream));
            }
        }
        NK(ctx->tr->group_end());
    }
    // the chain on this rank's band: exchange the band tuples after phase 1 of every step
    for (int sl = 0; sl < N; ++sl) {
        TRY(gp_phase1(ctx, me, ctx->gb_u + sl * bvol, ctx->gb_v, sl));
        NK(ctx->tr->allgather_inplace(ctx->gb_tot, (size_t)5 * n, ctx->stream));
        TRY(gp_phase2(ctx, me, ctx->gb_v, ctx->gb_u + (sl + 1) * bvol, ctx->gb_gc + sl * bvol,
                      ctx->gb_d + sl * bvol));
    }
    // gather: U_{n+1} and Gcache_n bands to the owner of slice n, and U_first to this rank
    TRY(gpar_plan(N, ctx->nranks, me, 1, ops));
    NK(ctx->tr->group_start());
    for (size_t o = 0; o < ops.size(); o += 6) {
        const int kind = ops[o], what = ops[o + 1], sl = ops[o + 2], band = ops[o + 3], peer = ops[o + 4],
                  lidx = ops[o + 5];
        double *mine = (what == 1) ? ctx->gb_u + (sl + 1) * bvol : ctx->gb_gc + sl * bvol;  // this rank's band
        double *dst = ((what == 1) ? state(ctx, ctx->traj, lidx) : state(ctx, ctx->gcache, lidx)) + band * bvol;
        if (kind == 2)
            CK(cudaMemcpyAsync(dst, mine, bbytes, cudaMemcpyDeviceToDevice, ctx->stream));
        else if (kind == 0)
            NK(ctx->tr->send(mine, (size_t)bvol, peer, ctx->stream));
        else
            NK(ctx->tr->recv(dst, (size_t)bvol, peer, ctx->stream));
    }
    NK(ctx->tr->group_end());
    ctx->gb_valid = true;  // gb_u[1..N] = this rank's bands of U^{k+1}, as gathered into traj
    return PRS_OK;
}

// the local part of the coarse correction chain: G step + fused correction
// epilogue for every local slice, in time order
static int enqueue_correct_chain(prs_ctx *ctx) {
    CK(cudaMemsetAsync(ctx->red, 0, sizeof(unsigned long long) * 2, ctx->stream));
    if (sweep2_ok(ctx)) return launch_chain2(ctx, local_start(ctx), EPI_CORRECT);
    for (int i = local_start(ctx); i < ctx->count; ++i) {
        EpiArgs ep;
        ep.kind = EPI_CORRECT;
        ep.gcache = state(ctx, ctx->gcache, i);
        ep.delta = state(ctx, ctx->delta, i);
        ep.traj = state(ctx, ctx->traj, i + 1);
        TRY(run_step(ctx, ctx->p.G, ctx->fac[0], state(ctx, ctx->traj, i), ctx->gtmp, 1,
                     coarse_time(ctx, ctx->first + i), ep, false, ctx->ss));
    }
    return PRS_OK;
}

// The multi-rank coarse chain of one iteration on the context stream (owner-G: receive
// U^{k+1}_first from the previous rank, G steps with the fused correction over the local slices,
// send U^{k+1}_last on; space-parallel G: the band chain of gp_correct); the update / flag
// maxima land in ctx->red (this rank's part).
static int enqueue_chain_mr(prs_ctx *ctx) {
    if (ctx->gpar) return gp_correct(ctx);
    CK(cudaMemsetAsync(ctx->red, 0, sizeof(unsigned long long) * 2, ctx->stream));
    if (ctx->cyclic) {
        // slices in time order; the first active one (global kconv) starts from the converged,
        // frozen U^k_kconv it holds, every later one receives U^{k+1}_n from the previous slice's rank
        for (int i = local_start(ctx); i < ctx->count; ++i) {
            const int n = (int)gslice(ctx, i);
            if (n > ctx->kconv)
                NK(ctx->tr->recv(state(ctx, ctx->traj, i), (size_t)ctx->vol, owner_of(ctx, n - 1), ctx->stream));
            if (sweep2_ok(ctx)) {
                TRY(chain2_cyclic_one(ctx, i, EPI_CORRECT));
            } else {
                EpiArgs ep;
                ep.kind = EPI_CORRECT;
                ep.gcache = state(ctx, ctx->gcache, i);
                ep.delta = state(ctx, ctx->delta, i);
                ep.traj = end_state(ctx, i);
                TRY(run_step(ctx, ctx->p.G, ctx->fac[0], state(ctx, ctx->traj, i), ctx->gtmp, 1, coarse_time(ctx, n),
                             ep, false, ctx->ss));
            }
            if (n + 1 < ctx->p.N)
                NK(ctx->tr->send(end_state(ctx, i), (size_t)ctx->vol, owner_of(ctx, n + 1), ctx->stream));
        }
        return PRS_OK;
    }
    if (ctx->rank > 0) NK(ctx->tr->recv(ctx->traj, (size_t)ctx->vol, ctx->rank - 1, ctx->stream));
    if (sweep2_ok(ctx)) TRY(launch_chain2(ctx, local_start(ctx), EPI_CORRECT));
    for (int i = sweep2_ok(ctx) ? ctx->count : local_start(ctx); i < ctx->count; ++i) {
        EpiArgs ep;
        ep.kind = EPI_CORRECT;
        ep.gcache = state(ctx, ctx->gcache, i);
        ep.delta = state(ctx, ctx->delta, i);
        ep.traj = state(ctx, ctx->traj, i + 1);
        TRY(run_step(ctx, ctx->p.G, ctx->fac[0], state(ctx, ctx->traj, i), ctx->gtmp, 1,
                     coarse_time(ctx, ctx->first + i), ep, false, ctx->ss));
    }
    if (ctx->rank < ctx->nranks - 1)
        NK(ctx->tr->send(state(ctx, ctx->traj, ctx->count), (size_t)ctx->vol, ctx->rank + 1, ctx->stream));
    return PRS_OK;
}

// (update, flag) pair at host `h` -> normalised update; PRS_EDIVERGED on a non-finite value
static int read_update(prs_ctx *ctx, const unsigned long long *h, double *update_out) {
    double upd;
    memcpy(&upd, h, sizeof(double));
    if (update_out) *update_out = upd / ctx->u0norm;
    if (h[1]) {
        ctx->err = "non-finite value in the parareal iterate";
        return PRS_EDIVERGED;
    }
    return PRS_OK;
}

int prs_parareal_correct(prs_ctx *ctx, double *update_out) {
    if (!ctx) return PRS_EINVAL;
    if (!ctx->delta) { ctx->err = "prs_fine_sweep first"; return PRS_EINVAL; }
    if (ctx->nranks > 1) {
        TRY(enqueue_chain_mr(ctx));
        NK(ctx->tr->allreduce_max_u64(ctx->red, 2, ctx->stream, 1));
    } else if (ctx->gpar) {
        TRY(gp_correct(ctx));
    } else {
        TRY(run_graphed(ctx, enqueue_correct_chain, ctx->corr_calls, ctx->corr_exec, ctx->corr_glaunch, ctx->corr_gen));
    }
    CK(cudaMemcpyAsync(ctx->red_host, ctx->red, sizeof(unsigned long long) * 2, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->delta = nullptr;
    return read_update(ctx, ctx->red_host, update_out);
}

// prs_iterate over several ranks with a lagged stop test:
// the stop-test all-reduce of iteration k runs on its own stream (and NCCL communicator) once
// this rank's chain of k is done, while the context stream already runs the fine sweep of
// iteration k + 1 (it needs only U^{k+1}_n); the host reads iteration k's
// update while that sweep runs.  On a stop, the lookahead sweep has written only the Delta
// scratch: trajectory, k and update history are those of the unlagged loop.  The (update,
// flag) words alternate between two parities so chain k + 1 never clears the pair the
// all-reduce of k still reads.
static int iterate_lagged(prs_ctx *ctx, int K, double tol, int *k_out, double *hist) {
    if (!ctx->have_coarse) { ctx->err = "prs_coarse_sweep first"; return PRS_EINVAL; }
    if (!ctx->ctl) {
        CK(cudaStreamCreateWithFlags(&ctx->ctl, cudaStreamNonBlocking));
        for (int p = 0; p < 2; ++p) {
            CK(cudaEventCreateWithFlags(&ctx->ev_chain[p], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_red[p], cudaEventDisableTiming | cudaEventBlockingSync));
        }
    }
    TRY(ensure_factors(ctx, 0, ctx->dT));
    TRY(ensure_factors(ctx, 1, ctx->dt));
    int k = 0, rc = PRS_OK;
    ctx->kconv = 0;
    if (K > 0) {
        rc = enqueue_fine_sweep(ctx);
        ctx->delta = (ctx->p.s & 1) ? ctx->fa : ctx->fb;
    }
    while (rc == PRS_OK && k < K) {
        const int p = k & 1;
        ctx->red = ctx->red_base + 4 * p;
        rc = enqueue_chain_mr(ctx);
        if (rc != PRS_OK) break;
        CK(cudaEventRecord(ctx->ev_chain[p], ctx->stream));
        CK(cudaStreamWaitEvent(ctx->ctl, ctx->ev_chain[p], 0));
        rc = ctx->tr->allreduce_max_u64(ctx->red, 2, ctx->ctl, 1);
        if (rc != PRS_OK) {
            ctx->err = ctx->tr->err;
            break;
        }
        CK(cudaMemcpyAsync(ctx->red_host + 4 * p, ctx->red, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           ctx->ctl));
        CK(cudaEventRecord(ctx->ev_red[p], ctx->ctl));
        if (k + 1 < K) {  // lookahead: iteration k+1's fine sweep (slices n < k+1 converged)
            ctx->kconv = ctx->skip_converged ? k + 1 : 0;
            rc = enqueue_fine_sweep(ctx);
            if (rc != PRS_OK) break;
        }
        CK(cudaEventSynchronize(ctx->ev_red[p]));
        double upd = 0.0;
        rc = read_update(ctx, ctx->red_host + 4 * p, &upd);
        if (hist) hist[k] = upd;
        ++k;
        if (rc != PRS_OK || upd <= tol) break;
    }
    // drain (a lookahead sweep wrote only the Delta scratch)
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->ctl);
    ctx->red = ctx->red_base;
    ctx->kconv = 0;
    ctx->delta = nullptr;
    if (k_out) *k_out = k;
    return rc;
}

// ---------------------------------------------------------- pipelined parareal -------
// Iteration k (U^k -> U^{k+1}) as a per-block dependency graph on streams:
//   fine(k, b)  : Delta_i = F^s(U^k_i) - G(U^k_i) for the slices of block b (sweep2), once the
//                 chain of iteration k-1 has produced U^k and G(U^k) of that block;
//   chain(k, b) : G step + fused correction of block b's slices, in time order, once fine(k, b)
//                 is done and chain(k, b-1) has produced U^{k+1} of the block's first slice.
// So the fine sweeps of iteration k+1 start block by block while the chain of iteration k is
// still correcting later blocks, and the chain of k+1 follows the fine sweeps as they land
// (F on slice n needs only U^{k+1}_n).  Iteration k reads the parity-(k & 1)
// trajectory / G cache and writes the other parity, so an iteration started before the stop
// test of the previous one (one iteration of lookahead) never touches the converged iterate;
// it is drained and discarded.  The kernels and their inputs are those of the unpipelined
// path, so trajectories and update histories are bitwise identical to it.
static int pipe_enqueue(prs_ctx *ctx, int k) {
    const int G = ctx->pipe, cnt = ctx->count, s = ctx->p.s, p = k & 1, q = p ^ 1;
    double *T[2] = {ctx->traj, ctx->traj2}, *GC[2] = {ctx->gcache, ctx->gcache2};
    double *D = ctx->fa;
    for (int b = 0; b < G; ++b) {
        const int lo = (int)((long long)b * cnt / G), hi = (int)((long long)(b + 1) * cnt / G);
        if (k > 0) CK(cudaStreamWaitEvent(ctx->psF[b], ctx->pevC[b], 0));
        if (hi > lo)
            TRY(launch_sweep2(ctx, state(ctx, T[p], lo), state(ctx, D, lo), state(ctx, GC[p], lo), hi - lo,
                              ctx->first + lo, s, ctx->psF[b]));
        CK(cudaEventRecord(ctx->pevF[b], ctx->psF[b]));
    }
    CK(cudaMemsetAsync(ctx->pred + 2 * p, 0, 2 * sizeof(unsigned long long), ctx->psC));
    for (int b = 0; b < G; ++b) {
        const int lo = (int)((long long)b * cnt / G), hi = (int)((long long)(b + 1) * cnt / G);
        CK(cudaStreamWaitEvent(ctx->psC, ctx->pevF[b], 0));
        TRY(launch_chain2x(ctx, T[q], GC[q], D, lo, hi, EPI_CORRECT, ctx->pred + 2 * p, ctx->psC, T[p]));
        CK(cudaEventRecord(ctx->pevC[b], ctx->psC));
    }
    CK(cudaMemcpyAsync(ctx->pred_host + 2 * p, ctx->pred + 2 * p, 2 * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, ctx->psC));
    CK(cudaEventRecord(ctx->pevRed[p], ctx->psC));
    return PRS_OK;
}

static int pipe_iterate(prs_ctx *ctx, int K, double tol, int *k_out, double *hist) {
    TRY(ensure_factors(ctx, 0, ctx->dT));
    TRY(ensure_factors(ctx, 1, ctx->dt));
    // parity 1 starts from the same U_0 (slice 0 of every iterate)
    CK(cudaMemcpyAsync(ctx->traj2, ctx->traj, ctx->sbytes, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaEventRecord(ctx->pev0, ctx->stream));
    for (auto st : ctx->psF) CK(cudaStreamWaitEvent(st, ctx->pev0, 0));
    CK(cudaStreamWaitEvent(ctx->psC, ctx->pev0, 0));
    int k = 0, rc = PRS_OK;
    if (K > 0) rc = pipe_enqueue(ctx, 0);
    while (rc == PRS_OK && k < K) {
        if (k + 1 < K) {
            rc = pipe_enqueue(ctx, k + 1);  // lookahead: runs while iteration k's chain finishes
            if (rc != PRS_OK) break;
        }
        const int p = k & 1;
        CK(cudaEventSynchronize(ctx->pevRed[p]));
        double upd;
        memcpy(&upd, ctx->pred_host + 2 * p, sizeof(double));
        const bool bad = ctx->pred_host[2 * p + 1] != 0;
        upd /= ctx->u0norm;
        if (hist) hist[k] = upd;
        ++k;
        if (bad) {
            ctx->err = "non-finite value in the parareal iterate";
            rc = PRS_EDIVERGED;
            break;
        }
        if (upd <= tol) break;
    }
    // drain the lookahead iteration (it wrote only the other parity and the Delta scratch)
    for (auto st : ctx->psF) CK(cudaStreamSynchronize(st));
    CK(cudaStreamSynchronize(ctx->psC));
    if (k & 1) {  // U^k and G(U^k) are in parity 1: make parity 0 (ctx->traj / gcache) current
        CK(cudaMemcpyAsync(ctx->traj, ctx->traj2, ctx->ss * sizeof(double) * (size_t)(ctx->count + 1),
                           cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->gcache, ctx->gcache2, ctx->ss * sizeof(double) * (size_t)ctx->count,
                           cudaMemcpyDeviceToDevice, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->delta = nullptr;
    if (k_out) *k_out = k;
    return rc;
}

int prs_set_pipeline(prs_ctx *ctx, int blocks) {
    if (!ctx || blocks < 0) return PRS_EINVAL;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    pipe_free(ctx);
    if (blocks == 0) return PRS_OK;
    if (ctx->nranks != 1 || !sweep2_ok(ctx) || ctx->gpar) {
        ctx->err = "pipelined parareal: one rank, 2-D dimensional split with kappa = 1 and n in {32, 64, 128, 256} "
                   "(the on-chip sweep kernels), owner-G coarse mode";
        return PRS_EUNSUPPORTED;
    }
    const int G = blocks < ctx->count ? blocks : ctx->count;
    CK(cudaMalloc(&ctx->traj2, ctx->ss * sizeof(double) * (size_t)(ctx->count + 1)));
    CK(cudaMalloc(&ctx->gcache2, ctx->ss * sizeof(double) * (size_t)ctx->count));
    CK(cudaMalloc(&ctx->pred, 4 * sizeof(unsigned long long)));
    CK(cudaMallocHost(&ctx->pred_host, 4 * sizeof(unsigned long long)));
    ctx->psF.resize(G);
    ctx->pevF.resize(G);
    ctx->pevC.resize(G);
    for (int b = 0; b < G; ++b) {
        CK(cudaStreamCreateWithFlags(&ctx->psF[b], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->pevF[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->pevC[b], cudaEventDisableTiming));
    }
    CK(cudaStreamCreateWithFlags(&ctx->psC, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->pev0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->pevRed[0], cudaEventDisableTiming | cudaEventBlockingSync));
    CK(cudaEventCreateWithFlags(&ctx->pevRed[1], cudaEventDisableTiming | cudaEventBlockingSync));
    ctx->pipe = G;
    return PRS_OK;
}

int prs_iterate(prs_ctx *ctx, int kmax, double tol, int *k_out, double *hist) {
    if (!ctx || kmax < 0) return PRS_EINVAL;
    if (ctx->nranks > 1 && ctx->lag) return iterate_lagged(ctx, kmax < ctx->p.N ? kmax : ctx->p.N, tol, k_out, hist);
    if (ctx->pipe && !ctx->gpar) {  // (space-parallel G takes the unpipelined chain)
        if (!ctx->have_coarse) { ctx->err = "prs_coarse_sweep first"; return PRS_EINVAL; }
        return pipe_iterate(ctx, kmax < ctx->p.N ? kmax : ctx->p.N, tol, k_out, hist);
    }
    const int K = kmax < ctx->p.N ? kmax : ctx->p.N;
    int k = 0;
    int rc = PRS_OK;
    for (; k < K;) {
        // iteration k computes U^{k+1}; slices n < k are converged (see kconv)
        ctx->kconv = ctx->skip_converged ? k : 0;
        rc = prs_fine_sweep(ctx);
        if (rc != PRS_OK) break;
        double upd = 0.0;
        rc = prs_parareal_correct(ctx, &upd);
        if (hist) hist[k] = upd;
        ++k;
        if (rc != PRS_OK) break;
        if (upd <= tol) break;
    }
    ctx->kconv = 0;
    if (k_out) *k_out = k;
    return rc;
}

int prs_get_slice(prs_ctx *ctx, int n, double *out, int out_on_device) {
    if (!ctx || !out || n < 0 || n > ctx->p.N) return PRS_EINVAL;
    const double *src = nullptr;
    if (ctx->cyclic) {  // U_n is slice n's start (rank n mod P) and slice n-1's end state
        if (n < ctx->p.N && n % ctx->nranks == ctx->rank) src = state(ctx, ctx->traj, n / ctx->nranks);
        else if (n > 0 && (n - 1) % ctx->nranks == ctx->rank) src = state(ctx, ctx->tend, (n - 1) / ctx->nranks);
    } else {
        const int i = n - ctx->first;
        if (i >= 0 && i <= ctx->count) src = state(ctx, ctx->traj, i);
    }
    if (!src) { ctx->err = "slice not owned by this rank"; return PRS_EINVAL; }
    CK(cudaMemcpyAsync(out, src, ctx->sbytes,
                       out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return PRS_OK;
}

int prs_step(prs_ctx *ctx, int scheme, double tau, double t_next, const double *in, double *out) {
    if (!ctx || !in || !out || in == out || !(tau > 0.0)) return PRS_EINVAL;
    if (scheme != PRS_FIE && scheme != PRS_DR && scheme != PRS_IE) return PRS_EINVAL;
    if (ctx->p.dim == 3 && scheme == PRS_DR) return PRS_EUNSUPPORTED;
    if (scheme == PRS_IE && !ctx->ie_S) {
        ctx->err = "PRS_IE steps need a context created with G or F = PRS_IE";
        return PRS_EINVAL;
    }
    if (scheme == PRS_IE) {
        TimeArgs ta;
        ta.slice0 = 0;
        ta.tmul = 0;
        ta.toff = 1;
        ta.tstep = t_next;
        ta.gk = ctx->p.source_kind == 2 ? 1 : 0;
        ta.gc = 8.0 * M_PI * M_PI + ctx->p.c;
        EpiArgs ep;
        TRY(ie_step(ctx, tau, in, out, 1, ta, ep, false));
        CK(cudaStreamSynchronize(ctx->stream));
        return PRS_OK;
    }
    int slot = 2;
    if (tau == ctx->fac[0].tau) slot = 0;
    else if (tau == ctx->fac[1].tau) slot = 1;
    TRY(ensure_factors(ctx, slot, tau));
    TimeArgs ta;
    ta.slice0 = 0;
    ta.tmul = 0;
    ta.toff = 1;
    ta.tstep = t_next;
    EpiArgs ep;
    TRY(run_step(ctx, scheme, ctx->fac[slot], in, out, 1, ta, ep, false, ctx->vol));
    CK(cudaStreamSynchronize(ctx->stream));
    return PRS_OK;
}

int prs_step_batch(prs_ctx *ctx, int which, int slice0, int j, const double *in, double *out, int B) {
    if (!ctx || !in || !out || in == out || B < 1 || (which != 0 && which != 1)) return PRS_EINVAL;
    TRY(ensure_factors(ctx, which, which == 0 ? ctx->dT : ctx->dt));
    TimeArgs ta;
    ta.slice0 = slice0;
    ta.tmul = (which == 0) ? 1 : ctx->p.s;
    ta.toff = (which == 0) ? 1 : j + 1;
    ta.tstep = (which == 0) ? ctx->dT : ctx->dt;
    EpiArgs ep;
    TRY(run_step(ctx, which == 0 ? ctx->p.G : ctx->p.F, ctx->fac[which], in, out, B, ta, ep, false, ctx->vol));
    CK(cudaStreamSynchronize(ctx->stream));
    return PRS_OK;
}

int prs_fine_solve(prs_ctx *ctx, const double *u0, int u0_on_device, int nslices, double *out, int out_on_device) {
    if (!ctx || !u0 || !out || nslices < 0 || nslices > ctx->p.N) return PRS_EINVAL;
    TRY(ensure_factors(ctx, 1, ctx->dt));
    double *buf[2] = {ctx->fa, ctx->fb};  // the fine-sweep work buffers (slot 0 of each)
    ctx->delta = nullptr;                 // a pending fine sweep is invalidated
    CK(cudaMemcpyAsync(buf[0], u0, ctx->sbytes, u0_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       ctx->stream));
    int cur = 0;
    const int s = ctx->p.s;
    if (sweep2_ok(ctx) && nslices > 0) {
        // small 2-D states: all nslices * s steps in one on-chip sweep (source times (j+1) dt)
        TRY(launch_sweep2(ctx, buf[0], buf[1], nullptr, 1, 0, nslices * s));
        cur = 1;
        nslices = 0;
    }
    for (int n = 0; n < nslices; ++n) {
        for (int j = 0; j < s; ++j) {
            TimeArgs ta;
            ta.slice0 = n;
            ta.tmul = s;
            ta.toff = j + 1;
            ta.tstep = ctx->dt;
            EpiArgs ep;
            TRY(run_step(ctx, ctx->p.F, ctx->fac[1], buf[cur], buf[cur ^ 1], 1, ta, ep, false, ctx->ss));
            cur ^= 1;
        }
    }
    CK(cudaMemcpyAsync(out, buf[cur], ctx->sbytes, out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return PRS_OK;
}

int prs_gpar_plan(int N, int nranks, int rank, int phase, int *ops, int max_ops) {
    if (N < 1 || nranks < 1 || rank < 0 || rank >= nranks || phase < 0 || phase > 2 || max_ops < 0) return -1;
    std::vector<int> v;
    if (gpar_plan(N, nranks, rank, phase, v) != PRS_OK) return -1;
    const int cnt = (int)(v.size() / 6);
    if (ops)
        for (int i = 0; i < cnt && i < max_ops; ++i)
            for (int f = 0; f < 6; ++f) ops[6 * i + f] = v[6 * i + f];
    return cnt;
}

int prs_set_coarse_mode(prs_ctx *ctx, int mode, int bands) {
    if (!ctx || (mode != 0 && mode != 1)) return PRS_EINVAL;
    if (mode == 0) {
        ctx->gpar = 0;
        return PRS_OK;
    }
    const int n = ctx->p.n;
    const int P = (ctx->nranks > 1) ? ctx->nranks : bands;
    const bool pow2 = P >= 1 && (P & (P - 1)) == 0 && (n & (n - 1)) == 0;
    if (ctx->cyclic) {
        ctx->err = "space-parallel G: contiguous slice ownership only";
        return PRS_EUNSUPPORTED;
    }
    if (ctx->p.source_kind == 2) {
        ctx->err = "space-parallel G: source_kind 0 or 1";
        return PRS_EUNSUPPORTED;
    }
    if (ctx->p.dim != 2 || ctx->p.split != 0 || ctx->p.G != PRS_FIE || !pow2 || n > 4096 || n % (L5RB * P) != 0 ||
        (long long)n * n / P < 4096) {
        ctx->err = "space-parallel G: 2-D dimensional split, G = FIE, P a power of two, n a power of two "
                   "<= 4096 with n % (64 P) == 0";
        return PRS_EUNSUPPORTED;
    }
    if (ctx->nranks > 1 && bands != ctx->nranks && bands != 0) {
        ctx->err = "space-parallel G over ranks: one band per rank";
        return PRS_EINVAL;
    }
    ctx->gP = P;
    ctx->gnb = n / P;
    ctx->gb_valid = false;
    const long long bvol = (long long)ctx->gnb * n, nrb = ctx->gnb / L5RB;
    double **bufs[] = {&ctx->gb_u, &ctx->gb_d, &ctx->gb_gc, &ctx->gb_v, &ctx->gb_tt, &ctx->gb_tot, &ctx->gb_yx};
    for (double **b : bufs)
        if (*b) {
            CK(cudaFree(*b));
            *b = nullptr;
        }
    if (ctx->nranks > 1) {
        const int N = ctx->p.N;
        CK(cudaMalloc(&ctx->gb_u, sizeof(double) * bvol * (N + 1)));
        CK(cudaMalloc(&ctx->gb_d, sizeof(double) * bvol * N));
        CK(cudaMalloc(&ctx->gb_gc, sizeof(double) * bvol * N));
        CK(cudaMalloc(&ctx->gb_v, sizeof(double) * bvol));
    } else {
        CK(cudaMalloc(&ctx->gb_v, sizeof(double) * bvol * P));
    }
    CK(cudaMalloc(&ctx->gb_tt, sizeof(double) * 7 * nrb * n * P));
    CK(cudaMalloc(&ctx->gb_tot, sizeof(double) * 5 * (size_t)n * P));
    CK(cudaMalloc(&ctx->gb_yx, sizeof(double) * 2 * (size_t)n * P));
    ctx->gpar = 1;
    return PRS_OK;
}

int prs_set_ownership(prs_ctx *ctx, int mode) {
    if (!ctx || (mode != 0 && mode != 1)) return PRS_EINVAL;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (mode == 1 && (ctx->gpar || ctx->pipe)) {
        ctx->err = "cyclic ownership: owner-G coarse chain, unpipelined (prs_set_coarse_mode 0, prs_set_pipeline 0)";
        return PRS_EUNSUPPORTED;
    }
    const int cyc = (mode == 1 && ctx->nranks > 1) ? 1 : 0;  // one rank: the same layout either way
    if (cyc == ctx->cyclic) return PRS_OK;
    int first = 0, count = 0;
    if (cyc) {
        first = ctx->rank;
        count = (ctx->p.N - ctx->rank + ctx->nranks - 1) / ctx->nranks;
    } else {
        prs_partition(ctx->p.N, ctx->nranks, ctx->rank, &first, &count);
    }
    const size_t sb = sizeof(double) * (size_t)ctx->ss;
    double **bufs[] = {&ctx->traj, &ctx->fa, &ctx->fb, &ctx->gcache, &ctx->tend};
    for (double **b : bufs)
        if (*b) {
            CK(cudaFree(*b));
            *b = nullptr;
        }
    CK(cudaMalloc(&ctx->traj, sb * (count + 1)));
    CK(cudaMalloc(&ctx->fa, sb * count));
    CK(cudaMalloc(&ctx->fb, sb * count));
    CK(cudaMalloc(&ctx->gcache, sb * count));
    if (cyc) CK(cudaMalloc(&ctx->tend, sb * count));
    ctx->cyclic = cyc;
    ctx->first = first;
    ctx->count = count;
    ctx->delta = nullptr;
    ctx->have_coarse = false;
    if (ctx->have_initial && ctx->rank == 0)
        CK(cudaMemcpyAsync(ctx->traj, ctx->u0, ctx->sbytes, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return PRS_OK;
}

int prs_set_profiling(prs_ctx *ctx, int on) {
    if (!ctx) return PRS_EINVAL;
    ctx->prof = on != 0;
    for (int k = 0; k < 4; ++k) {
        ctx->k_launch[k] = 0;
        ctx->k_ms[k] = 0;
        ctx->k_bytes[k] = 0;
    }
    return PRS_OK;
}

long long prs_launches(const prs_ctx *ctx) { return ctx ? ctx->launches : -1; }

int prs_kernel_stats(prs_ctx *ctx, int kind, long long *launches, double *ms, double *bytes) {
    if (!ctx || kind < 0 || kind > 3) return PRS_EINVAL;
    TRY(prof_flush(ctx));
    if (launches) *launches = ctx->k_launch[kind];
    if (ms) *ms = ctx->k_ms[kind];
    if (bytes) *bytes = ctx->k_bytes[kind];
    return PRS_OK;
}

}  // extern "C"
