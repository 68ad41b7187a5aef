// paper_1804_07981_b200/csrc/bml_digest.cu — device-side grid_digest (FNV-1a-64
// over the interior cell bytes, row-major), bit-identical to the reference's
// sequential hash (/root/reference/proj/src/digest.cpp:5-14,
// include/bml/digest.hpp:13-20). SURVEY.md §8(f) item 2 (readback/format).
//
// FNV-1a is a serial chain h <- (h ^ b) * p, but the cell bytes b are 0, 1 or
// 2, so the XOR only touches the low two bits of h:
//     h ^ b = h + d,   d = (s ^ b) - s,   s = h mod 4,
// and the low two bits of a product depend only on the low two bits of the
// factors (p mod 4 = 3), so s evolves by itself: s' = ((s ^ b) * 3) mod 4.
// Given s, the step is affine, h' = (h + d) * p, and a run of m cells maps
//     h  ->  h * p^m + B(s_in),   s_in -> s_out(s_in),
// a "segment" that depends only on the 4 possible incoming low-bit states.
// Segments compose associatively: (X then Y)(s) = { s_out: Y.s_out[X.s_out[s]],
// B: X.B[s] * Y.p^m + Y.B[X.s_out[s]], p^m: X.p^m * Y.p^m }. Threads hash
// chunks of words for all 4 incoming states, blocks and then one block reduce
// the segments in order; the host finishes h = basis * p^n² + B[basis mod 4].
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "bml_digest.cuh"

namespace bml_digest {
namespace {

constexpr uint64_t kPrime = 0x100000001b3ull;
constexpr int kThreads = 256;

struct Seg {
    uint64_t pw;    // p^m
    uint64_t b[4];  // B(s_in)
    uint32_t out;   // s_out(s_in) packed 2 bits per s_in
};

__host__ __device__ __forceinline__ Seg identity() {
    Seg s;
    s.pw = 1;
    s.b[0] = s.b[1] = s.b[2] = s.b[3] = 0;
    s.out = 0u | (1u << 2) | (2u << 4) | (3u << 6);
    return s;
}

__host__ __device__ __forceinline__ Seg combine(const Seg& x, const Seg& y) {
    Seg r;
    r.pw = x.pw * y.pw;
    r.out = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const uint32_t m = (x.out >> (2 * s)) & 3u;
        r.b[s] = x.b[s] * y.pw + y.b[m];
        r.out |= ((y.out >> (2 * m)) & 3u) << (2 * s);
    }
    return r;
}

// Append `cells` cells of one bit-plane word (bit i: LR, T bit i: TB).
__device__ __forceinline__ void hash_word(Seg& g, uint32_t l, uint32_t t, int cells) {
    uint32_t st[4] = {g.out & 3u, (g.out >> 2) & 3u, (g.out >> 4) & 3u, (g.out >> 6) & 3u};
    for (int i = 0; i < cells; ++i) {
        const uint32_t byte = ((l >> i) & 1u) | (((t >> i) & 1u) << 1);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const uint32_t x = st[s] ^ byte;
            const uint64_t d = static_cast<uint64_t>(static_cast<int64_t>(x) - static_cast<int64_t>(st[s]));
            g.b[s] = (g.b[s] + d) * kPrime;
            st[s] = (x * 3u) & 3u;
        }
        g.pw *= kPrime;
    }
    g.out = st[0] | (st[1] << 2) | (st[2] << 4) | (st[3] << 6);
}

// In-order tree reduction of one segment per thread; thread 0 returns the result.
__device__ Seg block_reduce(Seg mine, Seg* sh) {
    sh[threadIdx.x] = mine;
    __syncthreads();
    for (int d = 1; d < blockDim.x; d <<= 1) {
        if ((threadIdx.x % (2 * d)) == 0 && threadIdx.x + d < blockDim.x)
            sh[threadIdx.x] = combine(sh[threadIdx.x], sh[threadIdx.x + d]);
        __syncthreads();
    }
    return sh[0];
}

__global__ void __launch_bounds__(kThreads) segment_kernel(const uint2* __restrict__ planes, int W, int pitch,
                                                           long long words, uint32_t last_cells,
                                                           Seg* __restrict__ block_out) {
    __shared__ Seg sh[kThreads];
    const long long threads = static_cast<long long>(gridDim.x) * blockDim.x;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long chunk = (words + threads - 1) / threads;
    const long long lo = min(words, t * chunk), hi = min(words, lo + chunk);
    Seg g = identity();
    for (long long idx = lo; idx < hi; ++idx) {
        const long long r = idx / W;
        const int w = static_cast<int>(idx - r * W);
        const uint2 x = __ldg(planes + r * pitch + w);
        hash_word(g, x.x, x.y, w == W - 1 ? static_cast<int>(last_cells) : 32);
    }
    const Seg b = block_reduce(g, sh);
    if (threadIdx.x == 0) block_out[blockIdx.x] = b;
}

__global__ void __launch_bounds__(kThreads) finish_kernel(const Seg* __restrict__ parts, int count,
                                                          uint64_t* __restrict__ out) {
    __shared__ Seg sh[kThreads];
    const int chunk = (count + blockDim.x - 1) / blockDim.x;
    const int lo = min(count, static_cast<int>(threadIdx.x) * chunk), hi = min(count, lo + chunk);
    Seg g = identity();
    for (int i = lo; i < hi; ++i) g = combine(g, parts[i]);
    const Seg b = block_reduce(g, sh);
    if (threadIdx.x == 0) {
        out[0] = b.pw;
        for (int s = 0; s < 4; ++s) out[1 + s] = b.b[s];
        out[5] = b.out;
    }
}

}  // namespace

int segment(const uint2* planes, int n, int W, int pitch, int rows, cudaStream_t stream, int sms,
            uint64_t seg[6], std::string* msg) {
    const long long words = static_cast<long long>(rows) * W;
    const uint32_t last_cells = static_cast<uint32_t>(n - 32 * (W - 1));
    const int blocks = sms * 4;
    Seg* parts = nullptr;
    uint64_t* out = nullptr;
    cudaError_t e = cudaMalloc(&parts, blocks * sizeof(Seg));
    if (e == cudaSuccess) e = cudaMalloc(&out, 6 * sizeof(uint64_t));
    if (e == cudaSuccess) {
        segment_kernel<<<blocks, kThreads, 0, stream>>>(planes, W, pitch, words, last_cells, parts);
        finish_kernel<<<1, kThreads, 0, stream>>>(parts, blocks, out);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(seg, out, 6 * sizeof(uint64_t), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    cudaFree(parts);
    cudaFree(out);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        if (msg) *msg = std::string("digest: ") + cudaGetErrorString(e);
        return e == cudaErrorMemoryAllocation ? 3 : 2;
    }
    return 0;
}

uint64_t finish(const uint64_t* segs, int count) {
    Seg acc = identity();
    for (int i = 0; i < count; ++i) {
        Seg s;
        s.pw = segs[6 * i];
        for (int k = 0; k < 4; ++k) s.b[k] = segs[6 * i + 1 + k];
        s.out = static_cast<uint32_t>(segs[6 * i + 5]);
        acc = combine(acc, s);
    }
    const uint64_t basis = 0xcbf29ce484222325ull;  // kFnvOffsetBasis, digest.hpp
    return basis * acc.pw + acc.b[basis & 3u];
}

}  // namespace bml_digest
