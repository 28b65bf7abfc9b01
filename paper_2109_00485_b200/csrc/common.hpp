// Internal plumbing shared by the host and device translation units of
// libblockeig_b200.so: the exception type that carries a be_status across the
// C ABI, CUDA error checks, and small host utilities (thread fan-out).
#pragma once

#include <cstdint>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "blockeig_b200.h"

namespace be {

using index_t = std::int64_t;

// Thrown inside the library; caught at the C ABI edge (abi.cpp) and turned
// into a status code + thread-local message. `code` follows errors.hpp 1:1.
struct Failure : std::runtime_error {
    be_status code;
    int pivot;
    Failure(be_status c, const std::string& m, int p = -1) : std::runtime_error(m), code(c), pivot(p) {}
};

[[noreturn]] inline void fail(be_status c, const std::string& m, int pivot = -1) { throw Failure(c, m, pivot); }

inline int hw_threads() {
    unsigned t = std::thread::hardware_concurrency();
    return t == 0 ? 1 : static_cast<int>(t);
}

// Run fn(w) for w in [0, nw) on nw threads (w = 0 on the caller).
inline void fan_out(int nw, const std::function<void(int)>& fn) {
    if (nw <= 1) {
        fn(0);
        return;
    }
    std::vector<std::thread> ts;
    ts.reserve(static_cast<std::size_t>(nw - 1));
    std::exception_ptr err;
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(nw));
    for (int w = 1; w < nw; ++w)
        ts.emplace_back([&, w] {
            try {
                fn(w);
            } catch (...) {
                errs[static_cast<std::size_t>(w)] = std::current_exception();
            }
        });
    try {
        fn(0);
    } catch (...) {
        errs[0] = std::current_exception();
    }
    for (auto& t : ts) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

// Dynamic job loop over [0, njobs) on nw threads.
void parallel_for_dynamic(int nw, index_t njobs, const std::function<void(index_t, int)>& fn);

}  // namespace be

#ifdef __CUDACC__
#include <cuda_runtime.h>
#define BE_CUDA(call)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            ::be::fail(e_ == cudaErrorMemoryAllocation ? BE_ERR_OUT_OF_MEMORY : BE_ERR_CUDA,   \
                       std::string(#call) + ": " + cudaGetErrorString(e_));                    \
    } while (0)
#endif
