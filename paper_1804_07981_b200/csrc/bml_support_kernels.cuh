// paper_1804_07981_b200/csrc/bml_support_kernels.cuh — single-phase, pack/unpack, PPM, ghost-row and count kernels.
// Part of libbml_dev.so: included once, by bml_dev.cu (see its header comment).
#pragma once

#include "bml_kernels_common.cuh"

namespace bml_k {

// ------------------------------------------------------------ single phases
// One thread per (row, word) of the band; used by step_phase (bml_dev_phase).
struct PhaseArgs {
    const uint2* src;
    uint2* dst;
    int n, W, pitch, rows;
    uint32_t last_mask;
    unsigned long long* moved;
};

__device__ __forceinline__ void put_with_images(const PhaseArgs& a, int r, int w, uint32_t l,
                                                uint32_t t) {
    put(a.dst + static_cast<long long>(r) * a.pitch + w, l, t);
    for (int h = r - a.n; h >= -kHalo; h -= a.n) put(a.dst + static_cast<long long>(h) * a.pitch + w, l, t);
    for (int h = r + a.n; h < a.rows + kHalo; h += a.n) put(a.dst + static_cast<long long>(h) * a.pitch + w, l, t);
}

__global__ void phase_h_kernel(const PhaseArgs a) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = idx < static_cast<long long>(a.rows) * a.W;
    uint32_t moved = 0;
    if (live) {
        const int r = static_cast<int>(idx / a.W), w = static_cast<int>(idx % a.W);
        const uint2* row = a.src + static_cast<long long>(r) * a.pitch;
        const int c = 32 * w;
        const uint2 x = gather_window(row, c, a.n);
        const uint2 left = gather_window(row, ((c - 32) % a.n + a.n) % a.n, a.n);
        const uint2 right = gather_window(row, (c + 32) % a.n, a.n);
        const uint32_t E = ~(x.x | x.y);
        const uint32_t Er = ~(right.x | right.y);
        const uint32_t prevL = __funnelshift_l(left.x, x.x, 1);
        const uint32_t nextE = __funnelshift_r(E, Er, 1);
        const uint32_t valid = (w == a.W - 1) ? a.last_mask : kFull;
        const uint32_t vac = x.x & nextE & valid;
        const uint32_t Lp = ((prevL & E) | (x.x & ~nextE)) & valid;
        moved = __popc(vac);
        put_with_images(a, r, w, Lp, x.y & valid);
    }
    moved = __reduce_add_sync(kFull, moved);
    if ((threadIdx.x & 31) == 0 && moved) atomicAdd(a.moved, static_cast<unsigned long long>(moved));
}

__global__ void phase_v_kernel(const PhaseArgs a) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = idx < static_cast<long long>(a.rows) * a.W;
    uint32_t moved = 0;
    if (live) {
        const int r = static_cast<int>(idx / a.W), w = static_cast<int>(idx % a.W);
        const uint2 up = a.src[static_cast<long long>(r - 1) * a.pitch + w];
        const uint2 x = a.src[static_cast<long long>(r) * a.pitch + w];
        const uint2 dn = a.src[static_cast<long long>(r + 1) * a.pitch + w];
        const uint32_t E = ~(x.x | x.y);
        const uint32_t Ed = ~(dn.x | dn.y);
        const uint32_t valid = (w == a.W - 1) ? a.last_mask : kFull;
        const uint32_t vac = x.y & Ed & valid;
        const uint32_t Tp = ((up.y & E) | (x.y & ~Ed)) & valid;
        moved = __popc(vac);
        put_with_images(a, r, w, x.x & valid, Tp);
    }
    moved = __reduce_add_sync(kFull, moved);
    if ((threadIdx.x & 31) == 0 && moved) atomicAdd(a.moved, static_cast<unsigned long long>(moved));
}

// ------------------------------------------------------------ pack / unpack
// Byte lattice (0/1/2 per cell, `bpitch` bytes per row) <-> bit planes.
__device__ __forceinline__ uint32_t gather4(uint32_t x) {  // bit 0 of 4 bytes -> 4 bits
    return ((x & 0x01010101u) * 0x01020408u) >> 24;
}
__device__ __forceinline__ uint32_t spread4(uint32_t nib) {  // 4 bits -> bit 0 of 4 bytes
    return (nib * 0x00204081u) & 0x01010101u;
}

__global__ void pack_kernel(const uint8_t* __restrict__ bytes, long long bpitch, uint2* dst,
                            int n, int W, int pitch, int rows, int* bad) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(rows) * W) return;
    const int r = static_cast<int>(idx / W), w = static_cast<int>(idx % W);
    const uint8_t* p = bytes + r * bpitch + 32LL * w;
    const int cells = min(32, n - 32 * w);
    uint32_t l = 0, t = 0, badbits = 0;
    if (cells == 32 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
        const uint4 v0 = *reinterpret_cast<const uint4*>(p);
        const uint4 v1 = *reinterpret_cast<const uint4*>(p + 16);
        const uint32_t v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            l |= gather4(v[i]) << (4 * i);
            t |= gather4(v[i] >> 1) << (4 * i);
            badbits |= (v[i] & 0xfcfcfcfcu) | (v[i] & (v[i] >> 1) & 0x01010101u);
        }
    } else {
        for (int i = 0; i < cells; ++i) {
            const uint32_t b = p[i];
            l |= (b & 1u) << i;
            t |= ((b >> 1) & 1u) << i;
            badbits |= (b > 2u);
        }
    }
    if (badbits) atomicExch(bad, 1);
    dst[static_cast<long long>(r) * pitch + w] = make_uint2(l, t);
}

__global__ void unpack_kernel(const uint2* __restrict__ src, uint8_t* bytes, long long bpitch,
                              int n, int W, int pitch, int rows) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(rows) * W) return;
    const int r = static_cast<int>(idx / W), w = static_cast<int>(idx % W);
    const uint2 x = src[static_cast<long long>(r) * pitch + w];
    uint8_t* p = bytes + r * bpitch + 32LL * w;
    const int cells = min(32, n - 32 * w);
    if (cells == 32 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
        uint32_t v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            v[i] = spread4((x.x >> (4 * i)) & 15u) | (spread4((x.y >> (4 * i)) & 15u) << 1);
        *reinterpret_cast<uint4*>(p) = make_uint4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<uint4*>(p + 16) = make_uint4(v[4], v[5], v[6], v[7]);
    } else {
        for (int i = 0; i < cells; ++i)
            p[i] = static_cast<uint8_t>(((x.x >> i) & 1u) | (((x.y >> i) & 1u) << 1));
    }
}

// Bit planes -> binary-PPM pixels (snapshot.cpp:21-36, snapshot.hpp kLrColor /
// kTbColor / kEmptyColor): LR (255,0,0), TB (0,0,255), empty (255,255,255), so
// R = ~T, G = empty, B = ~L per cell. One thread per 32-cell word.
__global__ void ppm_kernel(const uint2* __restrict__ src, uint8_t* rgb, long long rpitch, int n,
                           int W, int pitch, int rows) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(rows) * W) return;
    const int r = static_cast<int>(idx / W), w = static_cast<int>(idx % W);
    const uint2 x = src[static_cast<long long>(r) * pitch + w];
    uint8_t* p = rgb + r * rpitch + 96LL * w;
    const int cells = min(32, n - 32 * w);
    for (int i = 0; i < cells; ++i) {
        const uint32_t l = (x.x >> i) & 1u, t = (x.y >> i) & 1u;
        p[3 * i + 0] = t ? 0 : 255;
        p[3 * i + 1] = (l | t) ? 0 : 255;
        p[3 * i + 2] = l ? 0 : 255;
    }
}

// Ghost rows of a single band: row h in [-kHalo,0) U [rows, rows+kHalo) is
// the image of row (h mod n).
__global__ void fill_images_kernel(uint2* buf, int n, int W, int pitch, int rows) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= 2 * kHalo * W) return;
    const int g = idx / W, w = idx % W;
    const int h = g < kHalo ? g - kHalo : rows + (g - kHalo);
    const int src = ((h % n) + n) % n;
    buf[static_cast<long long>(h) * pitch + w] = buf[static_cast<long long>(src) * pitch + w];
}

// Multi-band: publish the band's first/last kHalo rows into the neighbours'
// ghost rows of the same parity and raise their flags (one signal per warp
// column, matching the step kernel's accounting).
__global__ void push_halo_kernel(const uint2* buf, int W, int pitch, int rows, uint2* up_halo,
                                 uint2* down_halo, unsigned long long* up_flag,
                                 unsigned long long* down_flag, int ncols) {
    for (int idx = threadIdx.x; idx < kHalo * W; idx += blockDim.x) {
        const int r = idx / W, w = idx % W;
        up_halo[static_cast<long long>(r) * pitch + w] = buf[static_cast<long long>(r) * pitch + w];
        const int rb = rows - kHalo + r;
        down_halo[static_cast<long long>(rb - rows) * pitch + w] =
            buf[static_cast<long long>(rb) * pitch + w];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd_system(up_flag, static_cast<unsigned long long>(ncols));
        atomicAdd_system(down_flag, static_cast<unsigned long long>(ncols));
    }
}

__global__ void counts_kernel(const uint2* __restrict__ buf, int W, int pitch, int rows,
                              unsigned long long* out) {
    unsigned long long lr = 0, tb = 0;
    const long long total = static_cast<long long>(rows) * W;
    for (long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(idx / W), w = static_cast<int>(idx % W);
        const uint2 x = buf[static_cast<long long>(r) * pitch + w];
        lr += __popc(x.x);
        tb += __popc(x.y);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lr += __shfl_xor_sync(kFull, lr, o);
        tb += __shfl_xor_sync(kFull, tb, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (lr) atomicAdd(out, lr);
        if (tb) atomicAdd(out + 1, tb);
    }
}


// ------------------------------------------------------------ even/odd layout
// The wide kernel's EO mode (bml_wide_kernel.cuh) keeps each 64-cell group
// (words 2g, 2g+1) as its even cells, then its odd cells. These convert a
// whole buffer (every row including the ghost rows) in place, one thread per
// word pair, both planes; 16-byte accesses, HBM-bound (one read + one write).
__device__ __forceinline__ uint32_t even_bits(uint32_t x) {  // bits 0,2,..,30 -> 0..15
    x &= 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    return (x | (x >> 8)) & 0x0000FFFFu;
}
__device__ __forceinline__ uint32_t spread_bits(uint32_t x) {  // bits 0..15 -> 0,2,..,30
    x &= 0x0000FFFFu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    return (x | (x << 1)) & 0x55555555u;
}
// (a, b) = cells 0..31, 32..63 of a group  <->  (e, o) = its even, odd cells
__device__ __forceinline__ void to_eo(uint32_t a, uint32_t b, uint32_t& e, uint32_t& o) {
    e = even_bits(a) | (even_bits(b) << 16);
    o = even_bits(a >> 1) | (even_bits(b >> 1) << 16);
}
__device__ __forceinline__ void from_eo(uint32_t e, uint32_t o, uint32_t& a, uint32_t& b) {
    a = spread_bits(e) | (spread_bits(o) << 1);
    b = spread_bits(e >> 16) | (spread_bits(o >> 16) << 1);
}
template <bool TO_EO>
__device__ __forceinline__ void eo_convert_pair(uint4* q) {
    const uint4 v = __ldcg(q);  // {L0, T0, L1, T1}
    uint4 w;
    if (TO_EO) {
        to_eo(v.x, v.z, w.x, w.z);
        to_eo(v.y, v.w, w.y, w.w);
    } else {
        from_eo(v.x, v.z, w.x, w.z);
        from_eo(v.y, v.w, w.y, w.w);
    }
    *q = w;
}
template <bool TO_EO>
__global__ void eo_convert_kernel(uint2* base, long long rows_total, int pitch, int pairs) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= rows_total * pairs) return;
    const long long r = idx / pairs;
    const int p = static_cast<int>(idx - r * pairs);
    eo_convert_pair<TO_EO>(reinterpret_cast<uint4*>(base + r * pitch + 2 * p));
}
// A connected band's ghost rows are written by its neighbours' kernels: convert
// them only once the neighbour has published every launch so far (its flag has
// reached `expect`, the band's running sum, see StepArgs::expect). blockIdx.y = 0:
// the kHalo rows above the band (from the up neighbour, top flag), 1: below.
template <bool TO_EO>
__global__ void eo_convert_ghost_kernel(uint2* row0, int pitch, int pairs, int rows, const unsigned long long* top_flag,
                                        const unsigned long long* bot_flag, unsigned long long expect, int* err) {
    const bool below = blockIdx.y != 0;
    if (threadIdx.x < 32) wait_flag(below ? bot_flag : top_flag, expect, err);
    __syncthreads();
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(kHalo) * pairs) return;
    const int r = static_cast<int>(idx / pairs);
    const int p = static_cast<int>(idx - static_cast<long long>(r) * pairs);
    const long long row = below ? rows + r : r - kHalo;
    eo_convert_pair<TO_EO>(reinterpret_cast<uint4*>(row0 + row * pitch + 2 * p));
}

// TEST HOOK (bml_dev_debug_fault): toggle one cell, Empty <-> LR, TB -> Empty.
__global__ void debug_toggle_kernel(uint2* row0, int pitch, int row, int col) {
    if (threadIdx.x != 0) return;
    uint2* w = row0 + static_cast<long long>(row) * pitch + (col >> 5);
    const uint32_t bit = 1u << (col & 31);
    uint2 v = *w;
    if (v.y & bit)
        v.y &= ~bit;
    else
        v.x ^= bit;
    *w = v;
}

}  // namespace bml_k
