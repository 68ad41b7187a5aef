// paper_1804_07981_b200/csrc/bml_init.cu — device-side init_grid, bit-identical
// to the reference's sequential shuffle.
//
// Reference (/root/reference/proj): init_grid src/seeding.cpp:26-51 draws, for
// i = n²-1 down to 1, j_i = bounded(rng, i+1) (src/seeding.cpp:11-19, SplitMix64
// include/bml/seeding.hpp:11-24) and swaps cells[i] <-> cells[j_i]; the first k
// shuffled indices become LR vehicles, the next k TB vehicles. The host loop
// is serial and random-access bound (≈10 min and 32 GiB at n = 65536).
//
// Here the same permutation is computed in parallel, in four passes:
//
//  1. draws. SplitMix64 is a counter generator: the t-th output (t from 0) is
//     mix(seed + (t+1)·γ). Step i consumes draw t = (n²-1-i) + R(i), R(i) =
//     rejections at steps > i. Rejections (r >= 2^64 - (2^64 mod m)) have
//     probability < m/2^64 per draw, so the pass assumes none, records the
//     first (largest-i) rejected step with an atomicMax, and the host repeats
//     the pass below that step with the offset bumped — expected < 1 repeat
//     even at n = 65536.
//  2. group the steps by target: a stable radix sort of (j_i, i) pairs, keyed
//     on j (CUB onesweep; input is in ascending i, so each key's run lists its
//     steps in ascending i).
//  3. links. With V(x) = the value at position x once every step > x has run,
//     V(x) = V(first[x]) if some step > x swapped into x (first[x] = the
//     smallest such step), else x. Position i is final after step i, where it
//     receives the value position j_i holds after the steps > i:
//        final[i] = V(s) for s = the next step after i with the same target
//                   j_i (the successor of i in j_i's run), else j_i itself;
//        final[0] = V(0).
//     One pass over the sorted runs writes first[] (head of each run, skipping
//     the self-swap j_x = x) and, for i < 2k, link[i] = successor (> i) or j_i
//     (<= i) — the two cases are told apart by comparing with i.
//  4. resolve + scatter: follow first[] chains (expected length O(log)) for
//     the 2k placed vehicles and set their bits straight in the bit planes.
//
// Everything is integer and exact; the result equals the reference for every
// (n, rho, seed) with n² <= 2^32 (n <= 65536), which keeps indices in 32 bits.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "bml_init.cuh"

namespace bml_init {
namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t counter) {
    uint64_t z = seed + counter * kGamma;  // state after `counter` increments
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Draws for steps i in [1, hi], offset `off` rejections already consumed.
// keys[i-1] = j_i, vals[i-1] = i. `reject_mask` is a TEST hook: a draw with
// (r & mask) == 0 is treated as rejected too (0 = the reference's rule only).
__global__ void draw_kernel(uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                            uint64_t count, uint64_t seed, uint64_t hi, uint64_t off,
                            uint64_t reject_mask, unsigned long long* rejected) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = 1 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= hi;
         i += stride) {
        const uint64_t t = (count - 1 - i) + off;
        const uint64_t r = splitmix_at(seed, t + 1);
        const uint64_t m = i + 1;
        bool rej = reject_mask != 0 && (r & reject_mask) == 0;
        if (r > ~0ull - m) {  // r >= 2^64 - m: the only range a rejection can hit
            const uint64_t excess = (0ull - m) % m;  // 2^64 mod m
            rej |= excess != 0 && r >= 0ull - excess;
        }
        if (rej) atomicMax(rejected, static_cast<unsigned long long>(i));
        keys[i - 1] = static_cast<uint32_t>(r % m);
        vals[i - 1] = static_cast<uint32_t>(i);
    }
}

// Sorted runs (keys ascending, vals ascending within a key) -> first[], link[].
__global__ void links_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                             uint64_t items, uint64_t two_k, uint32_t* __restrict__ first,
                             uint32_t* __restrict__ link) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t m = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; m < items;
         m += stride) {
        const uint32_t q = keys[m], i = vals[m];
        const uint32_t nxt = (m + 1 < items && keys[m + 1] == q) ? vals[m + 1] : 0u;
        if (m == 0 || keys[m - 1] != q) first[q] = (i > q) ? i : nxt;
        if (i < two_k) link[i] = nxt ? nxt : q;
    }
}

__device__ __forceinline__ uint32_t settle(const uint32_t* __restrict__ first, uint32_t x) {
    for (uint32_t f = first[x]; f != 0u; f = first[x]) x = f;
    return x;
}

// Place vehicle i (LR for i < k, TB for k <= i < 2k) at its final cell, for
// rows [row_begin, row_end) of the band; plane words are uint2 {L, T}.
__global__ void scatter_kernel(const uint32_t* __restrict__ first, const uint32_t* __restrict__ link,
                               uint64_t k, int n, int row_begin, int row_end, int pitch,
                               uint2* planes) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < 2 * k;
         i += stride) {
        uint32_t v;
        if (i == 0) {
            v = settle(first, 0u);
        } else {
            const uint32_t l = link[i];
            v = (l > i) ? settle(first, l) : l;
        }
        const int r = static_cast<int>(v / static_cast<uint32_t>(n));
        const int c = static_cast<int>(v - static_cast<uint32_t>(r) * static_cast<uint32_t>(n));
        if (r < row_begin || r >= row_end) continue;
        uint32_t* word = reinterpret_cast<uint32_t*>(
            planes + static_cast<long long>(r - row_begin) * pitch + (c >> 5));
        atomicOr(word + (i < k ? 0 : 1), 1u << (c & 31));
    }
}

int cuda_err(cudaError_t e, const char* what, std::string* msg) {
    (void)cudaGetLastError();
    if (msg) *msg = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? 3 : 2;
}

}  // namespace

int init_planes(uint2* planes, int pitch, int n, int row_begin, int row_end, double rho,
                uint64_t seed, uint64_t reject_mask, cudaStream_t stream, int sms,
                std::string* msg) {
#define BI_CUDA(call)                                        \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) {                             \
            release();                                       \
            return cuda_err(e_, #call, msg);                 \
        }                                                    \
    } while (0)
    const uint64_t count = static_cast<uint64_t>(n) * static_cast<uint64_t>(n);
    // vehicles_per_species (src/seeding.cpp:21-24), same double arithmetic
    const uint64_t k = static_cast<uint64_t>(
        std::floor(rho * static_cast<double>(n) * static_cast<double>(n) / 2.0));
    uint32_t* buf[4] = {nullptr, nullptr, nullptr, nullptr};
    void* temp = nullptr;
    unsigned long long* rej = nullptr;
    auto release = [&]() {
        for (auto*& p : buf) {
            if (p) cudaFree(p);
            p = nullptr;
        }
        if (temp) cudaFree(temp);
        if (rej) cudaFree(rej);
        temp = nullptr;
        rej = nullptr;
    };

    const int rows = row_end - row_begin;
    BI_CUDA(cudaMemsetAsync(planes, 0, static_cast<size_t>(rows) * pitch * sizeof(uint2), stream));
    if (k == 0) return 0;

    const uint64_t items = count - 1;  // steps i = 1 .. n²-1 (k > 0 implies n >= 2)
    for (auto*& p : buf) BI_CUDA(cudaMalloc(&p, count * sizeof(uint32_t)));
    BI_CUDA(cudaMalloc(&rej, sizeof(unsigned long long)));

    // 1. draws, with the rejection fix-up passes
    const unsigned grid = static_cast<unsigned>(sms) * 8;
    uint64_t hi = items, off = 0;
    for (;;) {
        BI_CUDA(cudaMemsetAsync(rej, 0, sizeof(unsigned long long), stream));
        draw_kernel<<<grid, 256, 0, stream>>>(buf[0], buf[1], count, seed, hi, off, reject_mask, rej);
        BI_CUDA(cudaGetLastError());
        unsigned long long h = 0;
        BI_CUDA(cudaMemcpyAsync(&h, rej, sizeof h, cudaMemcpyDeviceToHost, stream));
        BI_CUDA(cudaStreamSynchronize(stream));
        if (h == 0) break;
        hi = h;     // steps above h drew correctly; step h redraws one counter later
        off += 1;
    }

    // 2. stable sort of (j_i, i) by j_i
    int end_bit = 1;
    while (end_bit < 32 && (uint64_t{1} << end_bit) < count) ++end_bit;
    cub::DoubleBuffer<uint32_t> dk(buf[0], buf[2]), dv(buf[1], buf[3]);
    size_t temp_bytes = 0;
    BI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, dk, dv,
                                            static_cast<int64_t>(items), 0, end_bit, stream));
    BI_CUDA(cudaMalloc(&temp, temp_bytes));
    BI_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, dk, dv, static_cast<int64_t>(items),
                                            0, end_bit, stream));

    // 3. links; the sort's alternate buffers become first[] and link[]
    uint32_t* first = dk.Alternate();
    uint32_t* link = dv.Alternate();
    BI_CUDA(cudaMemsetAsync(first, 0, count * sizeof(uint32_t), stream));
    links_kernel<<<grid, 256, 0, stream>>>(dk.Current(), dv.Current(), items, 2 * k, first, link);
    BI_CUDA(cudaGetLastError());

    // 4. resolve + scatter into the bit planes
    scatter_kernel<<<grid, 256, 0, stream>>>(first, link, k, n, row_begin, row_end, pitch, planes);
    BI_CUDA(cudaGetLastError());
    BI_CUDA(cudaStreamSynchronize(stream));
    release();
    return 0;
#undef BI_CUDA
}

}  // namespace bml_init
