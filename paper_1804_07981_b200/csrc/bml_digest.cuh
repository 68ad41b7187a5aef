// Internal interface of bml_digest.cu (device-side FNV-1a grid digest); used by bml_dev.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace bml_digest {

// Hash segment of `rows` rows of bit planes (row-major cells, n per row):
// seg = {p^cells, B(0), B(1), B(2), B(3), packed s_out}. Synchronises `stream`.
// Returns 0, 2 (CUDA error) or 3 (out of memory).
int segment(const uint2* planes, int n, int W, int pitch, int rows, cudaStream_t stream, int sms,
            uint64_t seg[6], std::string* msg);

// FNV-1a digest of the concatenation of `count` segments (host arithmetic).
uint64_t finish(const uint64_t* segs, int count);

}  // namespace bml_digest
