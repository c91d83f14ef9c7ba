// transport.cuh -- the rank-to-rank data plane of the parareal driver.
//
// The driver's multi-rank steps -- the slice hand-off along the owner-G chain (PAPER.md:203:
// U^{k+1}_{n+1} needs U^{k+1}_n from the previous slice's owner), the max all-reduce of the
// stop test, the band scatter / gather / all-gather of space-parallel G -- are
// issued through this interface, as stream-ordered operations on the caller's CUDA stream.
// Two implementations:
//   NcclTransport  -- production: NCCL over NVLink / NVSwitch, one communicator per channel
//                     (channel 0: data; channel 1: the stop-test all-reduce, so a lagged stop
//                     test on its own stream never orders against the data plane);
//   LocalTransport -- P ranks as P contexts of ONE process on one device, driven by P host
//                     threads (tests): messages are device-to-device copies ordered by CUDA
//                     events, matching happens on the host, so no kernel ever waits on
//                     another rank (B200_PROFILING.md: no spinning ranks on one GPU).
// Semantics (both): per (channel, ordered pair of ranks) point-to-point messages match in issue
// order; a send's buffer may be rewritten by later work on the sender's stream; group_start /
// group_end bracket point-to-point ops that may depend on one another (as an NCCL group);
// collectives are issued by every rank in the same order per channel.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

namespace prs {

struct Transport {
    virtual ~Transport() {}
    virtual int group_start() = 0;
    virtual int group_end() = 0;
    virtual int send(const double *buf, size_t count, int peer, cudaStream_t st, int ch = 0) = 0;
    virtual int recv(double *buf, size_t count, int peer, cudaStream_t st, int ch = 0) = 0;
    // in place, element-wise max over ranks of `count` unsigned 64-bit words
    virtual int allreduce_max_u64(unsigned long long *buf, size_t count, cudaStream_t st, int ch = 0) = 0;
    // in place: rank r's segment recv[r count, (r+1) count) to every rank
    virtual int allgather_inplace(double *recv, size_t count, cudaStream_t st, int ch = 0) = 0;
    std::string err;
};

// ------------------------------------------------------------------------ local world
__global__ void local_max_u64_kernel(const unsigned long long *const *ptrs, int P, int count,
                                     unsigned long long *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    unsigned long long m = 0;
    for (int r = 0; r < P; ++r) m = max(m, ptrs[r][i]);
    out[i] = m;
}

struct LocalWorld {
    int P;
    std::mutex mu;
    std::condition_variable cv;
    std::chrono::seconds timeout{300};
    struct Msg {
        const double *ptr;
        size_t count;
        cudaEvent_t ready, done;
        bool consumed = false;
    };
    // (channel, src, dst) -> FIFO of messages
    std::map<std::tuple<int, int, int>, std::deque<std::shared_ptr<Msg>>> q;
    // collectives per channel: one rendezvous at a time
    struct Coll {
        long long gen = 0;
        int arrived = 0, staged = 0, left = 0;
        std::vector<const void *> ptr;
        std::vector<cudaEvent_t> ready, read;
    };
    std::map<int, Coll> coll;
    explicit LocalWorld(int P_) : P(P_) {}
    bool wait(std::unique_lock<std::mutex> &lk, const std::function<bool()> &pred) {
        return cv.wait_for(lk, timeout, pred);
    }
};

struct LocalTransport : Transport {
    LocalWorld *w;
    int me;
    bool in_group = false;
    struct PendingRecv {
        double *buf;
        size_t count;
        int peer, ch;
        cudaStream_t st;
    };
    std::vector<PendingRecv> precv;
    std::vector<std::pair<std::shared_ptr<LocalWorld::Msg>, cudaStream_t>> psend;
    unsigned long long *d_max = nullptr;  // scratch: P pointers + result
    size_t d_max_cap = 0;

    LocalTransport(LocalWorld *w_, int me_) : w(w_), me(me_) {}
    ~LocalTransport() override {
        if (d_max) cudaFree(d_max);
    }
    int fail(const std::string &m) {
        err = "local transport (rank " + std::to_string(me) + "): " + m;
        return 6;  // PRS_ENCCL: a data-plane failure
    }
    int group_start() override {
        in_group = true;
        return 0;
    }
    int group_end() override {
        in_group = false;
        for (auto &r : precv)
            if (int rc = do_recv(r.buf, r.count, r.peer, r.st, r.ch)) return rc;
        precv.clear();
        for (auto &s : psend)
            if (int rc = wait_sent(s.first, s.second)) return rc;
        psend.clear();
        return 0;
    }
    int send(const double *buf, size_t count, int peer, cudaStream_t st, int ch) override {
        auto m = std::make_shared<LocalWorld::Msg>();
        m->ptr = buf;
        m->count = count;
        if (cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&m->done, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventRecord(m->ready, st) != cudaSuccess)
            return fail("event");
        {
            std::lock_guard<std::mutex> lk(w->mu);
            w->q[{ch, me, peer}].push_back(m);
        }
        w->cv.notify_all();
        if (in_group) {
            psend.push_back({m, st});
            return 0;
        }
        return wait_sent(m, st);
    }
    int wait_sent(const std::shared_ptr<LocalWorld::Msg> &m, cudaStream_t st) {
        std::unique_lock<std::mutex> lk(w->mu);
        if (!w->wait(lk, [&] { return m->consumed; })) return fail("send not matched (timeout)");
        lk.unlock();
        // the sender's later writes to the buffer wait for the receiver's copy
        if (cudaStreamWaitEvent(st, m->done, 0) != cudaSuccess) return fail("wait event");
        cudaEventDestroy(m->ready);
        cudaEventDestroy(m->done);
        return 0;
    }
    int recv(double *buf, size_t count, int peer, cudaStream_t st, int ch) override {
        if (in_group) {
            precv.push_back({buf, count, peer, ch, st});
            return 0;
        }
        return do_recv(buf, count, peer, st, ch);
    }
    int do_recv(double *buf, size_t count, int peer, cudaStream_t st, int ch) {
        std::shared_ptr<LocalWorld::Msg> m;
        {
            std::unique_lock<std::mutex> lk(w->mu);
            auto &qq = w->q[{ch, peer, me}];
            if (!w->wait(lk, [&] { return !qq.empty(); })) return fail("recv not matched (timeout)");
            m = qq.front();
            qq.pop_front();
        }
        if (m->count != count) return fail("message size mismatch");
        if (cudaStreamWaitEvent(st, m->ready, 0) != cudaSuccess ||
            cudaMemcpyAsync(buf, m->ptr, count * sizeof(double), cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
            cudaEventRecord(m->done, st) != cudaSuccess)
            return fail("copy");
        {
            std::lock_guard<std::mutex> lk(w->mu);
            m->consumed = true;
        }
        w->cv.notify_all();
        return 0;
    }
    // rendezvous of all P ranks on channel ch: register (ptr, ready event), wait for all
    template <class Body>
    int collective(const void *ptr, cudaStream_t st, int ch, Body body) {
        cudaEvent_t ready, read;
        if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&read, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(ready, st))
            return fail("event");
        std::unique_lock<std::mutex> lk(w->mu);
        LocalWorld::Coll &c = w->coll[ch];
        // a previous rendezvous still being left by slower ranks
        if (!w->wait(lk, [&] { return c.left == 0; })) return fail("collective (timeout)");
        if (c.arrived == 0) {
            c.ptr.assign(w->P, nullptr);
            c.ready.assign(w->P, nullptr);
            c.read.assign(w->P, nullptr);
        }
        c.ptr[me] = ptr;
        c.ready[me] = ready;
        c.read[me] = read;
        const long long gen = c.gen;
        if (++c.arrived == w->P) w->cv.notify_all();
        if (!w->wait(lk, [&] { return c.arrived == w->P || c.gen != gen; })) return fail("collective (timeout)");
        std::vector<const void *> ptrs = c.ptr;
        std::vector<cudaEvent_t> readies = c.ready, reads = c.read;
        lk.unlock();
        for (int r = 0; r < w->P; ++r)
            if (cudaStreamWaitEvent(st, readies[r], 0) != cudaSuccess) return fail("wait event");
        if (int rc = body(ptrs)) return rc;
        if (cudaEventRecord(read, st) != cudaSuccess) return fail("event");
        lk.lock();
        if (++c.staged == w->P) w->cv.notify_all();
        if (!w->wait(lk, [&] { return c.staged == w->P || c.gen != gen; })) return fail("collective (timeout)");
        lk.unlock();
        // nobody rewrites its buffer before every rank has read it
        for (int r = 0; r < w->P; ++r)
            if (cudaStreamWaitEvent(st, reads[r], 0) != cudaSuccess) return fail("wait event");
        lk.lock();
        if (c.gen == gen) {  // the first to leave closes the rendezvous
            c.gen++;
            c.arrived = 0;
            c.staged = 0;
            c.left = w->P;
        }
        if (--c.left == 0) {
            for (int r = 0; r < w->P; ++r) {
                cudaEventDestroy(readies[r]);
                cudaEventDestroy(reads[r]);
            }
        }
        w->cv.notify_all();
        return 0;
    }
    int allreduce_max_u64(unsigned long long *buf, size_t count, cudaStream_t st, int ch) override {
        const size_t need = (size_t)w->P + 2 * count;
        if (d_max_cap < need) {
            if (d_max) cudaFree(d_max);
            if (cudaMalloc(&d_max, need * sizeof(unsigned long long)) != cudaSuccess) return fail("malloc");
            d_max_cap = need;
        }
        unsigned long long *pp = d_max, *res = d_max + w->P;
        int rc = collective(buf, st, ch, [&](const std::vector<const void *> &ptrs) {
            if (cudaMemcpyAsync(pp, ptrs.data(), sizeof(void *) * w->P, cudaMemcpyHostToDevice, st) != cudaSuccess)
                return fail("copy");
            local_max_u64_kernel<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(
                reinterpret_cast<const unsigned long long *const *>(pp), w->P, (int)count, res);
            return cudaGetLastError() == cudaSuccess ? 0 : fail("max kernel");
        });
        if (rc) return rc;
        // (pageable H2D above is synchronous w.r.t. the host buffer; the result lands in buf
        // only after every rank has read every buf)
        return cudaMemcpyAsync(buf, res, count * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st) ==
                       cudaSuccess
                   ? 0
                   : fail("copy");
    }
    int allgather_inplace(double *recv, size_t count, cudaStream_t st, int ch) override {
        return collective(recv, st, ch, [&](const std::vector<const void *> &ptrs) {
            for (int r = 0; r < w->P; ++r) {
                if (r == me) continue;
                const double *src = static_cast<const double *>(ptrs[r]) + (size_t)r * count;
                if (cudaMemcpyAsync(recv + (size_t)r * count, src, count * sizeof(double), cudaMemcpyDeviceToDevice,
                                    st) != cudaSuccess)
                    return fail("copy");
            }
            return 0;
        });
    }
};

}  // namespace prs
