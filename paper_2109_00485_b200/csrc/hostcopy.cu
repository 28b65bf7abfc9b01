// Large host <-> device copies of caller-owned (pageable) buffers: the
// caller's bytes go through two pinned staging chunks; host threads move
// each chunk between the caller's pages and the staging buffer while the copy
// engine moves the other chunk. The driver's own pageable path does the same
// with one thread (~5 GB/s on the B200 hosts); here the host side runs on up
// to 8 threads.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "hostcopy.hpp"

namespace be {
namespace {

constexpr std::size_t kChunk = 16u << 20;  // bytes per staging chunk
constexpr std::size_t kDirect = 8u << 20;  // below this the driver's path is as good

struct Staging {
    std::mutex mu;
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int device = -1;
};

Staging& staging() {
    static Staging st;  // process-wide, allocated on first use, never freed
    return st;
}

void ensure(Staging& st, int device) {
    if (st.buf[0] && st.device == device) return;
    if (st.buf[0]) {  // events belong to another device: recreate them there
        for (auto& e : st.ev) cudaEventDestroy(e);
        for (auto& b : st.buf) cudaFreeHost(b);
    }
    for (auto& b : st.buf) BE_CUDA(cudaHostAlloc(&b, kChunk, cudaHostAllocPortable));
    for (auto& e : st.ev) BE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    st.device = device;
}

// dst[0, n) = src[0, n) on up to `nt` threads
void par_memcpy(void* dst, const void* src, std::size_t n) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const std::size_t nt = std::min<std::size_t>({8, hw, std::max<std::size_t>(1, n >> 20)});
    if (nt <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    const std::size_t per = (n + nt - 1) / nt;
    for (std::size_t t = 1; t < nt; ++t) {
        const std::size_t b = t * per, e = std::min(n, b + per);
        if (b < e)
            th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b); });
    }
    std::memcpy(dst, src, std::min(n, per));
    for (auto& x : th) x.join();
}

}  // namespace

void h2d_large(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
    if (bytes < kDirect) {
        BE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    int dev = 0;
    BE_CUDA(cudaGetDevice(&dev));
    auto& st = staging();
    std::lock_guard<std::mutex> lk(st.mu);
    ensure(st, dev);
    bool used[2] = {false, false};
    for (std::size_t off = 0, c = 0; off < bytes; off += kChunk, ++c) {
        const int b = static_cast<int>(c & 1);
        const std::size_t len = std::min(kChunk, bytes - off);
        if (used[b]) BE_CUDA(cudaEventSynchronize(st.ev[b]));  // its previous DMA is done
        par_memcpy(st.buf[b], static_cast<const char*>(src) + off, len);
        BE_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, st.buf[b], len, cudaMemcpyHostToDevice, s));
        BE_CUDA(cudaEventRecord(st.ev[b], s));
        used[b] = true;
    }
    for (int b = 0; b < 2; ++b)  // the staging buffers are free again when this returns
        if (used[b]) BE_CUDA(cudaEventSynchronize(st.ev[b]));
}

void d2h_large(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
    if (bytes < kDirect) {
        BE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaStreamSynchronize(s));
        return;
    }
    int dev = 0;
    BE_CUDA(cudaGetDevice(&dev));
    auto& st = staging();
    std::lock_guard<std::mutex> lk(st.mu);
    ensure(st, dev);
    const std::size_t nchunk = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](std::size_t c) {
        const int b = static_cast<int>(c & 1);
        const std::size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
        BE_CUDA(cudaMemcpyAsync(st.buf[b], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaEventRecord(st.ev[b], s));
    };
    issue(0);
    for (std::size_t c = 0; c < nchunk; ++c) {
        const int b = static_cast<int>(c & 1);
        BE_CUDA(cudaEventSynchronize(st.ev[b]));
        if (c + 1 < nchunk) issue(c + 1);  // the other buffer was drained in the previous round
        const std::size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
        par_memcpy(static_cast<char*>(dst) + off, st.buf[b], len);
    }
}

}  // namespace be
