// paper_1804_07981_b200/csrc/bml_kernels_common.cuh — constants, kernel arguments and
// device helpers shared by the sm_100a kernels of libbml_dev.so (included by bml_dev.cu).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

namespace bml_k {

constexpr int kHalo = 16;       // ghost rows per side == max steps fused per launch
// zero rows allocated after the lower ghost rows: the wide kernel's ring reads
// (don't-care) rows up to rows + 2K + 8 <= rows + 40 without clamping the address
constexpr int kLoadPad = 32;
constexpr int kMaxWarpsPerCta = 12;  // step kernel: one CTA per SM, up to 3 warps per SMSP
constexpr int kOutWords = 30;      // output words per warp in the haloed modes
constexpr int kSeamOutWords = 28;  // kSeam: output words per warp (two ghost words per side)
constexpr unsigned kFull = 0xffffffffu;

#ifndef BML_PDL
#define BML_PDL 1  // step kernel: programmatic dependent launch between consecutive blocks
#endif
#ifndef BML_IMAD_OR
#define BML_IMAD_OR 1
#endif

// kGeneric: n % 32 != 0 with rows narrower than a warp's span (n < 993): cells
//   gathered across the seam, register prefetch. kSeam: n % 32 != 0, W >= 32:
//   aligned row words through the cp.async ring, seam windows rebuilt with two
//   shuffles and a funnel shift (28 output words per warp, 2 ghost words per
//   side). kAligned: n % 32 == 0. kFullRow: W == 32 (one warp per row).
enum Mode { kGeneric = 0, kAligned = 1, kFullRow = 2, kSeam = 3 };

// ---------------------------------------------------------------- kernel args
struct StepArgs {
    const uint2* src;  // row 0 of the source buffer (ghost rows at negative rows)
    uint2* dst;        // row 0 of the destination buffer
    int n;             // torus side
    int W;             // words per row
    int pitch;         // words between rows
    int rows;          // rows in this band
    int strip_rows;    // unused by the kernel (rows are split evenly over nstrips)
    int nstrips;
    int ncols;         // warp columns per strip
    int items;         // nstrips * ncols
    uint32_t last_mask;
    int single_band;   // ghost rows are images of this band's own rows
    uint2* up_halo;    // multi-band: output row r < kHalo also goes to up_halo + r*pitch
    uint2* down_halo;  // multi-band: row r >= rows-kHalo also goes to down_halo + (r-rows)*pitch
    unsigned long long* up_flag;    // +1 per warp after publishing to up
    unsigned long long* down_flag;  // +1 per warp after publishing to down
    const unsigned long long* top_flag;  // wait before reading ghost rows above
    const unsigned long long* bot_flag;  // wait before reading ghost rows below
    unsigned long long expect;
    unsigned long long* metrics;  // [4][stride]: lr_moved, tb_moved, lr_count, tb_count
    int metrics_stride;
    int step_base;
    int* error_flag;
    uint32_t one;        // 1, at run time: IMAD-issued ORs of disjoint planes (BML_IMAD_OR)
    long long top_delta;  // words from row o's slot to its upper image (ghost row rows+o / up peer)
    long long bot_delta;  // words from row o's slot to its lower image (ghost row o-rows / down peer)
};

// --------------------------------------------------------------- device utils
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Spin until *flag >= expect (peer publication of ghost rows). Bounded so a
// broken peer cannot hang the GPU: after ~4 s the error flag is raised.
__device__ void wait_flag(const unsigned long long* flag, unsigned long long expect, int* err) {
    if (threadIdx.x % 32 == 0) {
        const long long t0 = clock64();
        while (ld_acquire_sys(flag) < expect) {
            __nanosleep(256);
            if (clock64() - t0 > 8000000000LL) {
                atomicExch(err, 2);
                break;
            }
        }
    }
    __syncwarp();
}

__device__ __forceinline__ void publish(unsigned long long* flag) {
    __threadfence_system();
    __syncwarp();
    if (threadIdx.x % 32 == 0) atomicAdd_system(flag, 1ull);
}

// 32 cells starting at cell c0 of a row (0 <= c0 < n), wrapping at n.
// Fast path: an aligned full word. Slow path (row end, n % 32 != 0, tiny n):
// gather bit runs across words and across the wrap.
__device__ __noinline__ uint2 gather_window(const uint2* __restrict__ row, int c0, int n) {
    uint32_t l = 0, t = 0;
    int got = 0, c = c0;
    while (got < 32) {
        const int q = c >> 5, o = c & 31;
        int take = min(32 - o, n - c);
        take = min(take, 32 - got);
        const uint2 w = __ldcg(row + q);
        const uint32_t m = (take == 32) ? kFull : ((1u << take) - 1u);
        l |= ((w.x >> o) & m) << got;
        t |= ((w.y >> o) & m) << got;
        got += take;
        c += take;
        if (c >= n) c = 0;
    }
    return make_uint2(l, t);
}

template <int MODE>
__device__ __forceinline__ uint2 load_cells(const uint2* row, int word, int c0, int n,
                                            bool coherent) {
    if (MODE == kGeneric) {
        if ((c0 & 31) == 0 && c0 + 32 <= n) return coherent ? __ldcg(row + (c0 >> 5)) : __ldg(row + (c0 >> 5));
        return gather_window(row, c0, n);
    }
    return coherent ? __ldcg(row + word) : __ldg(row + word);
}

__device__ __forceinline__ void put(uint2* p, uint32_t l, uint32_t t) { *p = make_uint2(l, t); }

__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Asynchronous 8-byte global->shared copies (LDGSTS) feeding a per-warp ring of
// input rows, so each warp keeps kRing-1 rows of loads in flight.
constexpr int kRing = 6;  // == the main loop's unroll factor: every slot index is a compile-time constant
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

}  // namespace bml_k
