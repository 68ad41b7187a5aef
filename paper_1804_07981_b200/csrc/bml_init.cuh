// Internal interface of bml_init.cu (device-side init_grid); used by bml_dev.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace bml_init {

// Zero rows [0, row_end - row_begin) of `planes` (uint2 {L, T} words, `pitch`
// words per row) and set the vehicles the reference init_grid({n, rho, seed})
// places in rows [row_begin, row_end). Requires n*n <= 2^32. `reject_mask` is
// a test hook (0 in production): draws with (r & mask) == 0 are also rejected,
// to exercise the rejection fix-up path the reference rule reaches < once per
// 2^32 draws. Synchronises `stream`. Returns 0, 2 (CUDA error) or 3 (out of
// device memory); *msg describes the failure.
int init_planes(uint2* planes, int pitch, int n, int row_begin, int row_end, double rho,
                uint64_t seed, uint64_t reject_mask, cudaStream_t stream, int sms,
                std::string* msg);

}  // namespace bml_init
