// Communicator backends (see comm.hpp).
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include <chrono>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <thread>

#include "comm.hpp"

namespace be {

void Comm::sync(cudaStream_t s) { BE_CUDA(cudaStreamSynchronize(s)); }

namespace {

// NCCL is resolved at run time (dlopen), not linked: the process may already
// hold the NCCL that torch bundles, and pinning the system libnccl.so.2 under
// the same soname first would break torch's import. Order: an NCCL already
// loaded in the process; $BE_NCCL_LIB; the default libnccl.so.2.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

const NcclApi& nccl() {
    static std::once_flag once;
    static NcclApi api;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            if (const char* e = std::getenv("BE_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p && err.empty()) err = std::string("libnccl.so.2 lacks ") + n;
            return p;
        };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.ReduceScatter = reinterpret_cast<decltype(api.ReduceScatter)>(sym("ncclReduceScatter"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
        api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    });
    if (!err.empty()) fail(BE_ERR_NCCL, err);
    return api;
}

#define BE_NCCL(call)                                                                                  \
    do {                                                                                               \
        ncclResult_t r_ = (call);                                                                      \
        if (r_ != ncclSuccess) ::be::fail(BE_ERR_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
    } while (0)

constexpr int kMaxLocalRanks = 16;

template <typename T>
struct Ptrs {
    const T* p[kMaxLocalRanks];
};

// out[i] = (((in_0[i] + in_1[i]) + in_2[i]) + ...) : ascending rank order
template <typename T>
__global__ void k_sum_ranks(Ptrs<T> in, int nin, T* __restrict__ out, std::size_t count) {
    for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
        T s = in.p[0][i];
        for (int q = 1; q < nin; ++q) s += in.p[q][i];
        out[i] = s;
    }
}

int sum_grid(std::size_t count) {
    return static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>((count + 255) / 256, 148 * 8)));
}

class NcclComm final : public Comm {
  public:
    NcclComm(int dev, const unsigned char id[128], int r, int w) {
        rank = r;
        world = w;
        device = dev;
        ncclUniqueId uid;
        static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
        std::memcpy(uid.internal, id, 128);
        BE_CUDA(cudaSetDevice(dev));
        BE_NCCL(nccl().CommInitRank(&comm_, w, uid, r));
    }
    ~NcclComm() override {
        if (comm_) nccl().CommDestroy(comm_);
    }
    void sync(cudaStream_t s) override {
        const auto t0 = std::chrono::steady_clock::now();
        double limit = 600.0;
        if (const char* e = std::getenv("BE_COMM_TIMEOUT_S")) limit = std::atof(e);
        for (int spin = 0;; ++spin) {
            const cudaError_t q = cudaStreamQuery(s);
            if (q == cudaSuccess) return;
            if (q != cudaErrorNotReady) BE_CUDA(q);
            ncclResult_t ae = ncclSuccess;
            BE_NCCL(nccl().CommGetAsyncError(comm_, &ae));
            const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if ((ae != ncclSuccess && ae != ncclInProgress) || el > limit) {
                const std::string why = ae != ncclSuccess && ae != ncclInProgress
                                            ? std::string("asynchronous NCCL error: ") + nccl().GetErrorString(ae)
                                            : "no progress in " + std::to_string(limit) + " s";
                nccl().CommAbort(comm_);
                comm_ = nullptr;
                fail(BE_ERR_PROTOCOL_DEADLOCK, "distributed collective: a rank is missing (" + why + ")");
            }
            if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
    void allreduce_f64(double* buf, std::size_t count, cudaStream_t s) override {
        BE_NCCL(nccl().AllReduce(buf, buf, count, ncclDouble, ncclSum, comm_, s));
        ++calls;
        bytes_moved += static_cast<std::int64_t>(2 * (world - 1) * count * sizeof(double) / std::max(world, 1));
    }
    void allgather_f32(const float* send, float* recv, std::size_t count, cudaStream_t s) override {
        BE_NCCL(nccl().AllGather(send, recv, count, ncclFloat, comm_, s));
        ++calls;
        bytes_moved += static_cast<std::int64_t>((world - 1) * count * sizeof(float));
    }
    void reduce_scatter_f32(const float* send, float* recv, std::size_t count, cudaStream_t s) override {
        BE_NCCL(nccl().ReduceScatter(send, recv, count, ncclFloat, ncclSum, comm_, s));
        ++calls;
        bytes_moved += static_cast<std::int64_t>((world - 1) * count * sizeof(float));
    }
    void p2p(const std::vector<P2POp>& ops, cudaStream_t s) override {
        if (ops.empty()) return;
        BE_NCCL(nccl().GroupStart());
        for (const auto& o : ops) {
            if (o.send) {
                BE_NCCL(nccl().Send(o.ptr, o.bytes, ncclChar, o.peer, comm_, s));
            } else {
                BE_NCCL(nccl().Recv(o.ptr, o.bytes, ncclChar, o.peer, comm_, s));
                bytes_moved += static_cast<std::int64_t>(o.bytes);
            }
        }
        BE_NCCL(nccl().GroupEnd());
        ++calls;
    }
    const char* backend() const override { return "nccl"; }

  private:
    ncclComm_t comm_ = nullptr;
};

class LocalComm final : public Comm {
  public:
    LocalComm(int dev, LocalGroup* g, int r) : g_(g) {
        if (r < 0 || r >= g->world) fail(BE_ERR_BAD_PARAMS, "local comm: rank out of range");
        rank = r;
        world = g->world;
        device = dev;
        BE_CUDA(cudaSetDevice(dev));
        BE_CUDA(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
        BE_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
        {
            std::lock_guard<std::mutex> lk(g->mu);
            g->slots[static_cast<std::size_t>(r)].device = dev;
            g->slots[static_cast<std::size_t>(r)].ready = ready_;
            g->slots[static_cast<std::size_t>(r)].done = done_;
        }
        g->barrier();  // every rank registered its device and events
        for (int q = 0; q < world; ++q) {
            const int pd = g->slots[static_cast<std::size_t>(q)].device;
            if (pd == dev) continue;
            int ok = 0;
            BE_CUDA(cudaDeviceCanAccessPeer(&ok, dev, pd));
            if (!ok) fail(BE_ERR_BAD_PARAMS, "local comm: devices without peer access");
            const cudaError_t e = cudaDeviceEnablePeerAccess(pd, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) BE_CUDA(e);
            cudaGetLastError();
        }
    }
    ~LocalComm() override {
        if (ready_) cudaEventDestroy(ready_);
        if (done_) cudaEventDestroy(done_);
        if (scratch_) cudaFree(scratch_);
    }

    void allreduce_f64(double* buf, std::size_t count, cudaStream_t s) override {
        if (scratch_bytes_ < count * sizeof(double)) {
            if (scratch_) cudaFree(scratch_);
            scratch_ = nullptr;
            BE_CUDA(cudaMalloc(&scratch_, count * sizeof(double)));
            scratch_bytes_ = count * sizeof(double);
        }
        double* tmp = static_cast<double*>(scratch_);
        run(buf, buf, s, [&](const std::vector<LocalGroup::Slot>& sl) {
            Ptrs<double> in{};
            for (int q = 0; q < world; ++q) in.p[q] = static_cast<const double*>(sl[static_cast<std::size_t>(q)].send);
            k_sum_ranks<double><<<sum_grid(count), 256, 0, s>>>(in, world, tmp, count);
            BE_CUDA(cudaGetLastError());
        });
        // peers have finished reading buf: overwrite it with the sum
        BE_CUDA(cudaMemcpyAsync(buf, tmp, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
        bytes_moved += static_cast<std::int64_t>(2 * (world - 1) * count * sizeof(double) / std::max(world, 1));
    }
    void allgather_f32(const float* send, float* recv, std::size_t count, cudaStream_t s) override {
        run(send, recv, s, [&](const std::vector<LocalGroup::Slot>& sl) {
            for (int q = 0; q < world; ++q) {
                float* dst = recv + static_cast<std::size_t>(q) * count;
                const void* src = sl[static_cast<std::size_t>(q)].send;
                if (src == dst || count == 0) continue;
                BE_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(float), cudaMemcpyDefault, s));
            }
        });
        bytes_moved += static_cast<std::int64_t>((world - 1) * count * sizeof(float));
    }
    void reduce_scatter_f32(const float* send, float* recv, std::size_t count, cudaStream_t s) override {
        run(send, recv, s, [&](const std::vector<LocalGroup::Slot>& sl) {
            Ptrs<float> in{};
            for (int q = 0; q < world; ++q)
                in.p[q] = static_cast<const float*>(sl[static_cast<std::size_t>(q)].send) +
                          static_cast<std::size_t>(rank) * count;
            if (count) k_sum_ranks<float><<<sum_grid(count), 256, 0, s>>>(in, world, recv, count);
            BE_CUDA(cudaGetLastError());
        });
        bytes_moved += static_cast<std::int64_t>((world - 1) * count * sizeof(float));
    }
    void p2p(const std::vector<P2POp>& ops, cudaStream_t s) override {
        std::vector<P2POp> sends, recvs;
        for (const auto& o : ops) (o.send ? sends : recvs).push_back(o);
        {
            std::lock_guard<std::mutex> lk(g_->mu);
            g_->slots[static_cast<std::size_t>(rank)].sends = sends;
        }
        run(nullptr, nullptr, s, [&](const std::vector<LocalGroup::Slot>& sl) {
            std::vector<int> taken(static_cast<std::size_t>(world), 0);  // k-th receive from p <- k-th send of p to me
            for (const auto& r : recvs) {
                const auto& ps = sl[static_cast<std::size_t>(r.peer)].sends;
                int k = taken[static_cast<std::size_t>(r.peer)]++, seen = 0;
                const P2POp* match = nullptr;
                for (const auto& x : ps)
                    if (x.peer == rank && seen++ == k) {
                        match = &x;
                        break;
                    }
                if (!match || match->bytes != r.bytes)
                    fail(BE_ERR_PROTOCOL_DEADLOCK, "local comm: unmatched point-to-point receive");
                if (r.bytes) BE_CUDA(cudaMemcpyAsync(r.ptr, match->ptr, r.bytes, cudaMemcpyDefault, s));
                bytes_moved += static_cast<std::int64_t>(r.bytes);
            }
        });
    }
    const char* backend() const override { return "local"; }

  private:
    // publish -> barrier -> wait peers' ready -> body -> record done ->
    // barrier -> wait peers' done (so no rank reuses a buffer a peer still reads) -> barrier
    template <class F>
    void run(const void* send, void* recv, cudaStream_t s, F&& body) {
        if (world > kMaxLocalRanks) fail(BE_ERR_BAD_PARAMS, "local comm: more than 16 ranks");
        BE_CUDA(cudaSetDevice(device));
        {
            std::lock_guard<std::mutex> lk(g_->mu);
            auto& sl = g_->slots[static_cast<std::size_t>(rank)];
            sl.send = send;
            sl.recv = recv;
        }
        BE_CUDA(cudaEventRecord(ready_, s));
        g_->barrier();
        std::vector<LocalGroup::Slot> sl;
        {
            std::lock_guard<std::mutex> lk(g_->mu);
            sl = g_->slots;
        }
        for (int q = 0; q < world; ++q)
            if (q != rank) BE_CUDA(cudaStreamWaitEvent(s, sl[static_cast<std::size_t>(q)].ready, 0));
        body(sl);
        BE_CUDA(cudaEventRecord(done_, s));
        g_->barrier();
        for (int q = 0; q < world; ++q)
            if (q != rank) BE_CUDA(cudaStreamWaitEvent(s, sl[static_cast<std::size_t>(q)].done, 0));
        // every rank has enqueued its waits on the peers' events before any rank leaves: a rank
        // that returned first could otherwise destroy its events (comm close) or re-record them
        // while a slower peer is still about to wait on them
        g_->barrier();
        ++calls;
    }

    LocalGroup* g_;
    cudaEvent_t ready_ = nullptr, done_ = nullptr;
    void* scratch_ = nullptr;
    std::size_t scratch_bytes_ = 0;
};

}  // namespace

LocalGroup::LocalGroup(int w) : world(w), slots(static_cast<std::size_t>(w)) {
    if (w < 1 || w > kMaxLocalRanks) fail(BE_ERR_BAD_PARAMS, "local comm group: world must be in [1, 16]");
    if (const char* e = std::getenv("BE_COMM_TIMEOUT_S")) timeout_s = std::atof(e);
}

void LocalGroup::barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) fail(BE_ERR_PROTOCOL_DEADLOCK, "local comm: the group was aborted by a failing rank");
    const std::uint64_t gen = generation;
    if (++arrived == world) {
        arrived = 0;
        ++generation;
        cv.notify_all();
        return;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                [&] { return generation != gen || aborted; });
    if (generation != gen) return;
    aborted = true;  // a missing or failed peer: release everybody
    cv.notify_all();
    fail(BE_ERR_PROTOCOL_DEADLOCK, ok ? "local comm: the group was aborted by a failing rank"
                                      : "local comm: a rank is missing from the collective (timeout)");
}

void LocalGroup::abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
}

std::unique_ptr<Comm> make_nccl_comm(int device, const unsigned char id[128], int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) fail(BE_ERR_BAD_PARAMS, "nccl comm: bad rank / world");
    return std::make_unique<NcclComm>(device, id, rank, world);
}

void nccl_unique_id(unsigned char id[128]) {
    ncclUniqueId uid;
    BE_NCCL(nccl().GetUniqueId(&uid));
    std::memcpy(id, uid.internal, 128);
}

std::unique_ptr<Comm> make_local_comm(int device, LocalGroup* group, int rank) {
    if (!group) fail(BE_ERR_BAD_PARAMS, "local comm: null group");
    return std::make_unique<LocalComm>(device, group, rank);
}

}  // namespace be
