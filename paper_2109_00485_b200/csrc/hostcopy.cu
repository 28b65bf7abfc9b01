// Large host <-> device copies of caller-owned (pageable) buffers: a
// persistent pool of host worker threads, each running its own pipeline over
// one contiguous slice of the transfer -- host memcpy between the caller's
// pages and the worker's two pinned staging chunks, DMA on the worker's own
// stream -- so the host-side memcpy of every worker and all copy engines run
// concurrently. The driver's own pageable path does the same with one thread
// (~5 GB/s on the B200 hosts); the round-1 version spawned threads per chunk
// and kept one pipeline (16 GB/s).
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hostcopy.hpp"

namespace be {
namespace {

constexpr std::size_t kChunk = 4u << 20;   // bytes per staging chunk (x2 per worker: 128 MB pinned for 16 workers)
constexpr std::size_t kDirect = 8u << 20;  // below this the driver's path is as good
constexpr std::size_t kMinSlice = 4u << 20;

struct Worker {
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaEvent_t done = nullptr;
    cudaStream_t stream = nullptr;
    bool used[2] = {false, false};
};

// The pool: workers sleep on a condition variable; run() hands every worker a
// job index and returns when all finished. One transfer at a time (the mutex
// of copy()).
class Pool {
  public:
    static Pool& get() {
        // process-wide, created on first use and never destroyed: the detached workers stay
        // parked on a live condition variable until the process exits (a static object's
        // destructor would tear the mutex down under them and hang the exit)
        static Pool* p = new Pool();
        return *p;
    }
    int size() const { return static_cast<int>(threads_.size()); }
    void run(const std::function<void(int)>& job) {
        std::unique_lock<std::mutex> lk(mu_);
        job_ = &job;
        pending_ = size();
        ++gen_;
        cv_.notify_all();
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }
    std::mutex copy_mu;  // serialises transfers (the workers' staging buffers are shared)
    std::vector<Worker> workers;
    int device = -1;

  private:
    Pool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const int n = static_cast<int>(std::min(16u, hw));
        workers.resize(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) threads_.emplace_back([this, i] { loop(i); });
        for (auto& t : threads_) t.detach();
    }
    void loop(int i) {
        std::uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* job = nullptr;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                job = job_;
            }
            if (job) (*job)(i);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* job_ = nullptr;
    int pending_ = 0;
    std::uint64_t gen_ = 0;
};

void ensure(Pool& p, int device) {
    if (p.device == device) return;
    for (auto& w : p.workers) {
        if (w.buf[0]) {  // streams / events belong to another device: recreate them here
            for (auto& e : w.ev) cudaEventDestroy(e);
            for (auto& b : w.buf) cudaFreeHost(b);
            cudaEventDestroy(w.done);
            cudaStreamDestroy(w.stream);
        }
        for (auto& b : w.buf) BE_CUDA(cudaHostAlloc(&b, kChunk, cudaHostAllocPortable));
        for (auto& e : w.ev) BE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        BE_CUDA(cudaEventCreateWithFlags(&w.done, cudaEventDisableTiming));
        BE_CUDA(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
        w.used[0] = w.used[1] = false;
    }
    p.device = device;
}

// worker slices: contiguous, 64-byte aligned boundaries
void slice(std::size_t bytes, int nw, int i, std::size_t& b, std::size_t& e) {
    const std::size_t per = ((bytes + static_cast<std::size_t>(nw) - 1) / nw + 63) & ~std::size_t{63};
    b = std::min(bytes, per * static_cast<std::size_t>(i));
    e = std::min(bytes, b + per);
}

}  // namespace

void hostcopy_prepare(int device) {
    auto& p = Pool::get();
    std::lock_guard<std::mutex> lk(p.copy_mu);
    ensure(p, device);
}

void h2d_large(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
    if (bytes < kDirect) {
        BE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    int dev = 0;
    BE_CUDA(cudaGetDevice(&dev));
    auto& p = Pool::get();
    std::lock_guard<std::mutex> lk(p.copy_mu);
    ensure(p, dev);
    const int nw = static_cast<int>(std::clamp<std::size_t>(bytes / kMinSlice, 1, p.workers.size()));
    std::vector<cudaError_t> err(static_cast<std::size_t>(nw), cudaSuccess);
    p.run([&](int i) {
        if (i >= nw) return;
        auto& w = p.workers[static_cast<std::size_t>(i)];
        cudaError_t e = cudaSetDevice(dev);
        std::size_t b0, e0;
        slice(bytes, nw, i, b0, e0);
        for (std::size_t off = b0, c = 0; off < e0 && e == cudaSuccess; off += kChunk, ++c) {
            const int k = static_cast<int>(c & 1);
            const std::size_t len = std::min(kChunk, e0 - off);
            if (w.used[k]) e = cudaEventSynchronize(w.ev[k]);  // its previous DMA is done
            if (e != cudaSuccess) break;
            std::memcpy(w.buf[k], static_cast<const char*>(src) + off, len);
            e = cudaMemcpyAsync(static_cast<char*>(dst) + off, w.buf[k], len, cudaMemcpyHostToDevice, w.stream);
            if (e == cudaSuccess) e = cudaEventRecord(w.ev[k], w.stream);
            w.used[k] = true;
        }
        if (e == cudaSuccess) e = cudaEventRecord(w.done, w.stream);
        err[static_cast<std::size_t>(i)] = e;
    });
    for (auto e : err) BE_CUDA(e);
    for (int i = 0; i < nw; ++i) BE_CUDA(cudaStreamWaitEvent(s, p.workers[static_cast<std::size_t>(i)].done, 0));
}

void d2h_large(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
    if (bytes < kDirect) {
        BE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaStreamSynchronize(s));
        return;
    }
    int dev = 0;
    BE_CUDA(cudaGetDevice(&dev));
    auto& p = Pool::get();
    std::lock_guard<std::mutex> lk(p.copy_mu);
    ensure(p, dev);
    cudaEvent_t ready = nullptr;  // the producer of src on s is done
    BE_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    BE_CUDA(cudaEventRecord(ready, s));
    const int nw = static_cast<int>(std::clamp<std::size_t>(bytes / kMinSlice, 1, p.workers.size()));
    std::vector<cudaError_t> err(static_cast<std::size_t>(nw), cudaSuccess);
    p.run([&](int i) {
        if (i >= nw) return;
        auto& w = p.workers[static_cast<std::size_t>(i)];
        cudaError_t e = cudaSetDevice(dev);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(w.stream, ready, 0);
        std::size_t b0, e0;
        slice(bytes, nw, i, b0, e0);
        const std::size_t nch = (e0 - b0 + kChunk - 1) / kChunk;
        auto issue = [&](std::size_t c) {
            const int k = static_cast<int>(c & 1);
            const std::size_t off = b0 + c * kChunk, len = std::min(kChunk, e0 - off);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(w.buf[k], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, w.stream);
            if (e == cudaSuccess) e = cudaEventRecord(w.ev[k], w.stream);
            w.used[k] = true;
        };
        if (nch > 0) issue(0);
        for (std::size_t c = 0; c < nch && e == cudaSuccess; ++c) {
            const int k = static_cast<int>(c & 1);
            e = cudaEventSynchronize(w.ev[k]);
            if (e != cudaSuccess) break;
            if (c + 1 < nch) issue(c + 1);  // the other buffer was drained in the previous round
            const std::size_t off = b0 + c * kChunk, len = std::min(kChunk, e0 - off);
            std::memcpy(static_cast<char*>(dst) + off, w.buf[k], len);
        }
        err[static_cast<std::size_t>(i)] = e;
    });
    cudaEventDestroy(ready);
    for (auto e : err) BE_CUDA(e);
}

}  // namespace be
