// comm.hpp -- the two data-path collectives of the multi-rank path behind one
// interface (host side of libdogip.so):
//   exchange       each rank sends its two slab-interface planes of partial sums to
//                  the z-1 / z+1 neighbours and receives theirs (A8, once per apply);
//   allreduce_sum  the CG scalars p.q and r.r (twice per iteration).
// Backends:
//   NcclComm      NCCL over NVLink / NVSwitch, one process per GPU (the product path);
//                 libnccl is resolved at run time (dlopen), so libdogip.so has no
//                 link-time NCCL dependency and reuses the copy torch already loaded.
//   LoopbackComm  several ranks of ONE process (one host thread per rank), planes and
//                 scalars moved with cudaMemcpyAsync between the ranks' buffers; the
//                 host threads rendezvous per collective, the streams are ordered by
//                 events, and no kernel ever waits on another rank's kernel.  It runs
//                 the multi-rank data path (boundary layers first, exchange, plane add,
//                 all-reduced CG dots) on a single GPU with REAL neighbour partials.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

namespace dogip {

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's copy if loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { api.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror(); return; }
#define DOGIP_SYM(field, name)                                           \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));   \
    if (!api.field) { api.err = std::string("missing NCCL symbol ") + name; return; }
        DOGIP_SYM(GetUniqueId, "ncclGetUniqueId")
        DOGIP_SYM(CommInitRank, "ncclCommInitRank")
        DOGIP_SYM(CommDestroy, "ncclCommDestroy")
        DOGIP_SYM(CommAbort, "ncclCommAbort")
        DOGIP_SYM(CommGetAsyncError, "ncclCommGetAsyncError")
        DOGIP_SYM(Send, "ncclSend")
        DOGIP_SYM(Recv, "ncclRecv")
        DOGIP_SYM(GroupStart, "ncclGroupStart")
        DOGIP_SYM(GroupEnd, "ncclGroupEnd")
        DOGIP_SYM(AllReduce, "ncclAllReduce")
        DOGIP_SYM(GetErrorString, "ncclGetErrorString")
#undef DOGIP_SYM
        api.ok = true;
    });
    return api;
}

// seconds a blocking wait on a peer may take before the communicator is declared dead
inline double comm_timeout_s() {
    static const double t = [] {
        const char* e = std::getenv("DOGIP_COMM_TIMEOUT_S");
        const double v = e ? std::atof(e) : 0.0;
        return v > 0 ? v : 600.0;
    }();
    return t;
}

// Return codes: 0 OK, else a DOGIP_E_* value (-8 = E_NCCL, -7 = E_CUDA) with `err` set.
class Comm {
public:
    int rank = 0, nranks = 1;
    std::string err;
    virtual ~Comm() = default;
    virtual const char* kind() const = 0;
    // Enqueued on st: send lo_send (P doubles) to rank-1 and hi_send to rank+1, receive
    // rank-1's plane into lo_recv and rank+1's into hi_recv.  The send buffers may be
    // modified by work enqueued on st after this call.
    virtual int exchange(const double* lo_send, const double* hi_send, double* lo_recv, double* hi_recv,
                         int64_t P, cudaStream_t st) = 0;
    // in place sum over ranks of n doubles, enqueued on st; every rank gets the same bits
    virtual int allreduce_sum(double* v, int64_t n, cudaStream_t st) = 0;
    // non-zero once the communicator failed asynchronously (peer died, network error)
    virtual int async_error() = 0;
    virtual void abort() = 0;
    // collectives may be captured into a CUDA graph
    virtual bool capturable() const = 0;

protected:
    int bad(int code, const std::string& m) {
        err = m;
        return code;
    }
};

class NcclComm final : public Comm {
public:
    ncclComm_t c = nullptr;
    ~NcclComm() override {
        if (c && nccl().ok) nccl().CommDestroy(c);
    }
    const char* kind() const override { return "nccl"; }
    int init(const void* id128, int r, int n) {
        auto& api = nccl();
        if (!api.ok) return bad(-8, api.err);
        rank = r;
        nranks = n;
        ncclUniqueId id;
        static_assert(sizeof id == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(&id, id128, sizeof id);
        const ncclResult_t e = api.CommInitRank(&c, n, id, r);
        if (e != ncclSuccess) { c = nullptr; return bad(-8, std::string("ncclCommInitRank: ") + api.GetErrorString(e)); }
        return 0;
    }
    int exchange(const double* lo_send, const double* hi_send, double* lo_recv, double* hi_recv, int64_t P,
                 cudaStream_t st) override {
        auto& api = nccl();
        ncclResult_t e = api.GroupStart();
        if (e == ncclSuccess && rank > 0) {
            e = api.Send(lo_send, P, ncclDouble, rank - 1, c, st);
            if (e == ncclSuccess) e = api.Recv(lo_recv, P, ncclDouble, rank - 1, c, st);
        }
        if (e == ncclSuccess && rank < nranks - 1) {
            e = api.Send(hi_send, P, ncclDouble, rank + 1, c, st);
            if (e == ncclSuccess) e = api.Recv(hi_recv, P, ncclDouble, rank + 1, c, st);
        }
        const ncclResult_t e2 = api.GroupEnd();
        if (e == ncclSuccess) e = e2;
        return e == ncclSuccess ? 0 : bad(-8, std::string("NCCL exchange: ") + api.GetErrorString(e));
    }
    int allreduce_sum(double* v, int64_t n, cudaStream_t st) override {
        auto& api = nccl();
        const ncclResult_t e = api.AllReduce(v, v, n, ncclDouble, ncclSum, c, st);
        return e == ncclSuccess ? 0 : bad(-8, std::string("ncclAllReduce: ") + api.GetErrorString(e));
    }
    int async_error() override {
        if (!c) return bad(-8, "NCCL communicator was aborted");
        ncclResult_t a = ncclSuccess;
        const ncclResult_t e = nccl().CommGetAsyncError(c, &a);
        if (e != ncclSuccess) return bad(-8, std::string("ncclCommGetAsyncError: ") + nccl().GetErrorString(e));
        if (a != ncclSuccess && a != ncclInProgress)
            return bad(-8, std::string("NCCL asynchronous error: ") + nccl().GetErrorString(a));
        return 0;
    }
    void abort() override {
        if (c) nccl().CommAbort(c);
        c = nullptr;
    }
    bool capturable() const override { return true; }
};

// ------------------------------------------------------------------ loopback
struct LoopbackGroup {
    struct Msg {
        int64_t gen = 0;
        const double* ptr = nullptr;
        cudaEvent_t ev = nullptr;
    };
    int nranks = 0, device = 0;
    std::mutex mu;
    std::condition_variable cv;
    bool dead = false;
    std::vector<Msg> sendbox, donebox;   // [src * nranks + dst]
    std::vector<Msg> arbox;              // [rank]
    double* slots = nullptr;             // [2][nranks][SLOT] device scratch of the all-reduce
    static constexpr int64_t SLOT = 64;
    int members = 0;                     // meshes attached
    std::vector<char> rank_used;         // one mesh per rank (collectives match by call order)

    // wait (host) until pred() holds; false on timeout or a dead group
    template <class Pred>
    bool wait(std::unique_lock<std::mutex>& lk, Pred pred) {
        const auto until = std::chrono::steady_clock::now() +
                           std::chrono::milliseconds((int64_t)(comm_timeout_s() * 1000.0));
        while (!pred()) {
            if (dead) return false;
            if (cv.wait_until(lk, until) == std::cv_status::timeout && !pred()) {
                dead = true;
                cv.notify_all();
                return false;
            }
        }
        return true;
    }
};

cudaError_t launch_sum_slots(const double* slots, int nranks, int64_t stride, int64_t n, double* out,
                             cudaStream_t st);

class LoopbackComm final : public Comm {
public:
    LoopbackGroup* g = nullptr;
    int64_t xgen = 0, argen = 0;
    cudaEvent_t ev_send = nullptr, ev_done = nullptr, ev_ar = nullptr;

    const char* kind() const override { return "loopback"; }
    int init(LoopbackGroup* grp, int r, int n) {
        if (!grp || grp->nranks != n) return bad(-10, "loopback group size differs from nranks");
        g = grp;
        rank = r;
        nranks = n;
        {
            std::lock_guard<std::mutex> lk(g->mu);
            if ((int)g->rank_used.size() < n) g->rank_used.resize(n, 0);
            if (g->rank_used[r]) { g = nullptr; return bad(-10, "loopback group already has a mesh for this rank"); }
            g->rank_used[r] = 1;
            ++g->members;
        }
        for (cudaEvent_t* e : {&ev_send, &ev_done, &ev_ar})
            if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return bad(-7, "event create");
        return 0;
    }
    ~LoopbackComm() override {
        for (cudaEvent_t e : {ev_send, ev_done, ev_ar})
            if (e) cudaEventDestroy(e);
        if (g) {
            std::lock_guard<std::mutex> lk(g->mu);
            --g->members;
            g->rank_used[rank] = 0;
        }
    }
    int exchange(const double* lo_send, const double* hi_send, double* lo_recv, double* hi_recv, int64_t P,
                 cudaStream_t st) override {
        const int64_t gen = ++xgen;
        const int n = nranks, r = rank;
        if (cudaEventRecord(ev_send, st) != cudaSuccess) return bad(-7, "loopback: event record");
        LoopbackGroup::Msg lo, hi;
        {
            std::unique_lock<std::mutex> lk(g->mu);
            if (r > 0) g->sendbox[r * n + r - 1] = {gen, lo_send, ev_send};
            if (r < n - 1) g->sendbox[r * n + r + 1] = {gen, hi_send, ev_send};
            g->cv.notify_all();
            const bool ok = g->wait(lk, [&] {
                return (r == 0 || g->sendbox[(r - 1) * n + r].gen >= gen) &&
                       (r == n - 1 || g->sendbox[(r + 1) * n + r].gen >= gen);
            });
            if (!ok) return bad(-8, "loopback exchange: peer did not arrive (timeout or dead group)");
            if (r > 0) lo = g->sendbox[(r - 1) * n + r];
            if (r < n - 1) hi = g->sendbox[(r + 1) * n + r];
        }
        cudaError_t e = cudaSuccess;
        if (r > 0) {
            e = cudaStreamWaitEvent(st, lo.ev, 0);
            if (e == cudaSuccess) e = cudaMemcpyAsync(lo_recv, lo.ptr, sizeof(double) * P, cudaMemcpyDefault, st);
        }
        if (e == cudaSuccess && r < n - 1) {
            e = cudaStreamWaitEvent(st, hi.ev, 0);
            if (e == cudaSuccess) e = cudaMemcpyAsync(hi_recv, hi.ptr, sizeof(double) * P, cudaMemcpyDefault, st);
        }
        if (e == cudaSuccess) e = cudaEventRecord(ev_done, st);
        if (e != cudaSuccess) return bad(-7, std::string("loopback exchange: ") + cudaGetErrorString(e));
        // the neighbours' send planes are read: wait until they have read ours too, so a
        // later write to our planes on st cannot race their copies
        LoopbackGroup::Msg dlo, dhi;
        {
            std::unique_lock<std::mutex> lk(g->mu);
            if (r > 0) g->donebox[r * n + r - 1] = {gen, nullptr, ev_done};
            if (r < n - 1) g->donebox[r * n + r + 1] = {gen, nullptr, ev_done};
            g->cv.notify_all();
            const bool ok = g->wait(lk, [&] {
                return (r == 0 || g->donebox[(r - 1) * n + r].gen >= gen) &&
                       (r == n - 1 || g->donebox[(r + 1) * n + r].gen >= gen);
            });
            if (!ok) return bad(-8, "loopback exchange: peer did not finish (timeout or dead group)");
            if (r > 0) dlo = g->donebox[(r - 1) * n + r];
            if (r < n - 1) dhi = g->donebox[(r + 1) * n + r];
        }
        if (r > 0) e = cudaStreamWaitEvent(st, dlo.ev, 0);
        if (e == cudaSuccess && r < n - 1) e = cudaStreamWaitEvent(st, dhi.ev, 0);
        return e == cudaSuccess ? 0 : bad(-7, std::string("loopback exchange: ") + cudaGetErrorString(e));
    }
    // every rank copies its n values into slot[rank] of a double-buffered scratch, then
    // (after all ranks' copies, by events) sums the slots in rank order 0..nranks-1 into v:
    // the same bits on every rank.  A rank reuses a buffer two generations later, which its
    // stream reaches only after waiting on every rank's next copy event -- recorded after
    // that rank's sum over the buffer was enqueued -- so no reader is overtaken.
    int allreduce_sum(double* v, int64_t n, cudaStream_t st) override {
        if (n > LoopbackGroup::SLOT) return bad(-10, "loopback all-reduce: too many values");
        const int64_t gen = ++argen;
        double* buf = g->slots + (gen & 1) * (int64_t)nranks * LoopbackGroup::SLOT;
        cudaError_t e = cudaMemcpyAsync(buf + rank * LoopbackGroup::SLOT, v, sizeof(double) * n,
                                        cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess) e = cudaEventRecord(ev_ar, st);
        if (e != cudaSuccess) return bad(-7, std::string("loopback all-reduce: ") + cudaGetErrorString(e));
        std::vector<cudaEvent_t> evs(nranks);
        {
            std::unique_lock<std::mutex> lk(g->mu);
            g->arbox[rank] = {gen, nullptr, ev_ar};
            g->cv.notify_all();
            const bool ok = g->wait(lk, [&] {
                for (int k = 0; k < nranks; ++k)
                    if (g->arbox[k].gen < gen) return false;
                return true;
            });
            if (!ok) return bad(-8, "loopback all-reduce: peer did not arrive (timeout or dead group)");
            for (int k = 0; k < nranks; ++k) evs[k] = g->arbox[k].ev;
        }
        for (int k = 0; k < nranks && e == cudaSuccess; ++k)
            if (k != rank) e = cudaStreamWaitEvent(st, evs[k], 0);
        if (e == cudaSuccess) e = launch_sum_slots(buf, nranks, LoopbackGroup::SLOT, n, v, st);
        return e == cudaSuccess ? 0 : bad(-7, std::string("loopback all-reduce: ") + cudaGetErrorString(e));
    }
    int async_error() override {
        std::lock_guard<std::mutex> lk(g->mu);
        return g->dead ? bad(-8, "loopback group is dead (a peer timed out or aborted)") : 0;
    }
    void abort() override {
        std::lock_guard<std::mutex> lk(g->mu);
        g->dead = true;
        g->cv.notify_all();
    }
    bool capturable() const override { return false; }   // host rendezvous per collective
};

}  // namespace dogip
