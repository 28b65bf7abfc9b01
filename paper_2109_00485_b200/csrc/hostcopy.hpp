// Staged, multi-threaded copies between pageable host memory and the device.
#pragma once

#include <cstddef>

#include <cuda_runtime.h>

#include "device.hpp"

namespace be {

// The worker pool and its pinned staging buffers for `device` (context setup,
// so the first large copy of a solve call does not pay for them).
void hostcopy_prepare(int device);
// Both return with the copy complete (src / dst may be reused immediately).
void h2d_large(void* dst, const void* src, std::size_t bytes, cudaStream_t s);
void d2h_large(void* dst, const void* src, std::size_t bytes, cudaStream_t s);

}  // namespace be
