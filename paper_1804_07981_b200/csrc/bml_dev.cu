// paper_1804_07981_b200/csrc/bml_dev.cu — B200-native BML lattice engine (sm_100a).
//
// Implements include/bml_dev.h. The reference (/root/reference/proj) keeps one
// byte per cell and runs each phase as a separate pass (src/engine.cpp:68-120,
// src/lanes.cpp:59-88). Here the lattice stays resident in HBM as two bit
// planes (bit j of word w of row i: plane L = "LR vehicle", plane T = "TB
// vehicle"), 32 cells per 32-bit word, the two planes interleaved as uint2.
// That is 2 bits/cell instead of 8, and both phase rules become a handful of
// LOP3/funnel-shift instructions per 32 cells:
//
//   LR phase (engine.hpp:32-36, lanes.cpp:52-57), on one row:
//     E      = ~(L | T)                               empty cells
//     prevL  = L shifted one cell right (cell j sees cell j-1), torus wrap
//     nextE  = E shifted one cell left  (cell j sees cell j+1), torus wrap
//     vacate = L & nextE                              moved_in_phase mask
//     L'     = (prevL & E) | (L & ~nextE)
//   TB phase (engine.hpp:38-42), rows i-1, i, i+1 after the LR phase:
//     T'(i)  = (T(i-1) & E(i)) | (T(i) & ~E(i+1)),    vacate = T(i) & E(i+1)
//
// The step kernel (step_block_kernel) is temporally blocked: one warp walks
// down a strip of rows, and K full steps (2K phases) are pipelined in
// registers, so each launch reads the lattice once and writes it once for K
// steps. Column wrap uses warp shuffles; each warp owns 30 output words plus
// one halo word on each side (the dependency cone grows one cell per step,
// K <= 32). Vertical wrap and band decomposition use kHalo ghost rows above
// and below the band, which the kernel itself refreshes for the NEXT launch
// (directly into a neighbour GPU's buffer over NVLink for row bands).

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <iterator>
#include <mutex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include "bml_dev.h"
#include "bml_digest.cuh"
#include "bml_init.cuh"

namespace {

constexpr int kHalo = 16;       // ghost rows per side == max steps fused per launch
constexpr int kMaxWarpsPerCta = 12;  // step kernel: one CTA per SM, up to 3 warps per SMSP
constexpr int kOutWords = 30;   // output words per warp in the haloed modes
constexpr unsigned kFull = 0xffffffffu;

#ifndef BML_PDL
#define BML_PDL 1  // step kernel: programmatic dependent launch between consecutive blocks
#endif
#ifndef BML_IMAD_OR
#define BML_IMAD_OR 1
#endif

enum Mode { kGeneric = 0, kAligned = 1, kFullRow = 2 };

// ---------------------------------------------------------------- error state
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    (void)cudaGetLastError();  // clear sticky-free errors
    const int code = (e == cudaErrorMemoryAllocation) ? BML_ENOMEM : BML_ECUDA;
    return fail(code, std::string(what) + ": " + cudaGetErrorString(e));
}

#define BML_CUDA(call)                                  \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

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

// ------------------------------------------------------- temporally blocked step
//
// Warp w handles (strip, col). Lane l stands for the 32 cells starting at
// cell 32*(30*col + l - 1) (mod n): lanes 1..30 are outputs, lanes 0 and 31
// are ghost words whose outer bits go stale by one cell per step. In
// kFullRow mode (W == 32) lane l is word l and shuffles wrap exactly.
//
// Software pipeline: stage s (step s+1 of the block) at loop index j consumes
// row j-2s at time s (produced by stage s-1 one iteration earlier, so all K
// stages of an iteration are independent) and emits row j-2s-1 at time s+1.
// Stage K-1 therefore emits row j-2K+1 at time K. The loop is unrolled by two
// and the TB window's two T registers swap roles by iteration parity, so the
// loop-carried state never moves between registers.
// Pipeline state. Values live in modulo-indexed register slots so that the
// loop (unrolled by 6 = lcm of the 3- and 2-iteration lifetimes) never moves a
// value between registers:
//   nt[s][j%3]  TB output T of stage s at iteration j  (stage s+1 reads it at
//               j+1 as its T, at j+2 as tB, at j+3 as tA)
//   lp[s][j%2]  LR output L of stage s at iteration j  (emitted as row L at
//               j+1, read by stage s+1 at j+2)
//   oc[s]       occupancy after LR of the row stage s saw last iteration
//   xt[j%3]     T of the row loaded at iteration j (stage 0's TB window)
template <int K>
struct PipeState {
    uint32_t nt[K][3];
    uint32_t lp[K][2];
    uint32_t oc[K];
    uint32_t xt[3];
    uint32_t cm[K], cc[K];  // packed 16-bit counters (COUNT only)
};

struct StripCtx {
    int lane, r_lo, r_hi, out_word;
    uint32_t valid;
    unsigned span;  // rows this lane stores (r_hi - r_lo, or 0 for ghost lanes)
    uint2* outp;    // aligned modes: this lane's word of the row emitted next
};

// Final-stage output of row o: the row itself plus its ghost images (the
// band's own ghost rows for a single band, or the neighbours' ghost rows for
// connected bands). Aligned modes have n >= 32 > kHalo, so each row has at
// most one image per side and every store is a predicated STG (no branches
// around the shuffles of the next stage).
template <int MODE>
__device__ __forceinline__ void store_row(const StepArgs& a, StripCtx& c, int o, uint32_t l,
                                          uint32_t t) {
    const bool st = static_cast<unsigned>(o - c.r_lo) < c.span;
    if (MODE != kGeneric) {
        // aligned modes: valid is 0 (ghost lane, span 0) or all ones, so no
        // masking; one running row pointer, images at fixed deltas from it
        // (ghost-row images are copied after the strip, copy_images)
        if (st) *c.outp = make_uint2(l, t);  // (st.global.cg / inline st.global measured 2-4% slower)
        c.outp += a.pitch;
        return;
    }
    const uint2 v = make_uint2(l & c.valid, t & c.valid);
    if (MODE != kGeneric) {
        const long long off = static_cast<long long>(o) * a.pitch + c.out_word;
        if (st) a.dst[off] = v;
        {
            uint2* top_img = a.single_band ? a.dst + static_cast<long long>(a.rows) * a.pitch : a.up_halo;
            uint2* bot_img = a.single_band ? a.dst - static_cast<long long>(a.rows) * a.pitch
                                           : a.down_halo - static_cast<long long>(a.rows) * a.pitch;
            if (st && o < kHalo) top_img[off] = v;            // row o -> ghost row rows+o (or up peer)
            if (st && o >= a.rows - kHalo) bot_img[off] = v;  // row o -> ghost row o-rows (or down peer)
        }
        return;
    }
    const long long off = static_cast<long long>(o) * a.pitch + c.out_word;
    {
        if (st) {
            a.dst[off] = v;
            if (a.single_band) {
                for (int h = o - a.n; h >= -kHalo; h -= a.n)
                    a.dst[static_cast<long long>(h) * a.pitch + c.out_word] = v;
                for (int h = o + a.n; h < a.rows + kHalo; h += a.n)
                    a.dst[static_cast<long long>(h) * a.pitch + c.out_word] = v;
            } else {
                if (o < kHalo) a.up_halo[off] = v;
                if (o >= a.rows - kHalo) a.down_halo[off - static_cast<long long>(a.rows) * a.pitch] = v;
            }
        }
    }
}

// Aligned modes: after a strip, its rows among the band's first / last kHalo
// rows are copied (re-read from L2, this thread's own stores) to their ghost
// images: the band's own ghost rows (single band) or the neighbours' (peer
// stores over NVLink), then the neighbour's flag is raised. Keeps the per-row
// store in the pipeline a single predicated STG.
__device__ __noinline__ void copy_images(const StepArgs& a, int r_lo, int r_hi, int out_word,
                                         bool stores) {
    const int top_end = min(r_hi, kHalo);
    const int bot_begin = max(r_lo, a.rows - kHalo);
    for (int o = r_lo; o < top_end; ++o) {
        const long long off = static_cast<long long>(o) * a.pitch + out_word;
        if (stores) a.dst[off + a.top_delta] = __ldcg(a.dst + off);  // -> ghost row rows+o (or up peer)
    }
    for (int o = bot_begin; o < r_hi; ++o) {
        const long long off = static_cast<long long>(o) * a.pitch + out_word;
        if (stores) a.dst[off + a.bot_delta] = __ldcg(a.dst + off);  // -> ghost row o-rows (or down peer)
    }
    if (!a.single_band) {
        if (r_lo == 0) publish(a.up_flag);
        if (r_hi == a.rows) publish(a.down_flag);
    }
}

template <int K, int MODE, bool COUNT, int P>
__device__ __forceinline__ void pipe_iter(PipeState<K>& q, const uint2 x, const int j,
                                          const StepArgs& a, StripCtx& c) {
    constexpr int P3 = P % 3, P2 = P % 2;
    q.xt[P3] = x.y;
#pragma unroll
    for (int s = K - 1; s >= 0; --s) {
        const uint32_t L = (s == 0) ? x.x : q.lp[s > 0 ? s - 1 : 0][P2];
        const uint32_t T = (s == 0) ? x.y : q.nt[s > 0 ? s - 1 : 0][(P3 + 2) % 3];
        const uint32_t tB = (s == 0) ? q.xt[(P3 + 2) % 3] : q.nt[s > 0 ? s - 1 : 0][(P3 + 1) % 3];
        const uint32_t tA = (s == 0) ? q.xt[(P3 + 1) % 3] : q.nt[s > 0 ? s - 1 : 0][P3];
        // ---- LR phase on row rho = j - 2s
#if BML_IMAD_OR
        // L and T are disjoint planes (a cell holds one vehicle), so L | T ==
        // L + T: issue it as IMAD on the FMA pipe (runtime multiplier 1 keeps
        // ptxas from folding it back into an ALU LOP3/IADD3).
        const uint32_t O = imad(L, a.one, T);
#else
        const uint32_t O = L | T;
#endif
        // (funnel shifts stay on the ALU pipe: moving them to the FMA pipe as
        // IMAD / IMAD.HI measured 13-24% slower, profiles/r1_sweep_fma_shifts_rejected.jsonl)
        const uint32_t Ll = MODE == kFullRow ? __shfl_sync(kFull, L, (c.lane + 31) & 31)
                                             : __shfl_up_sync(kFull, L, 1);
        const uint32_t Or = MODE == kFullRow ? __shfl_sync(kFull, O, (c.lane + 1) & 31)
                                             : __shfl_down_sync(kFull, O, 1);
        const uint32_t prevL = __funnelshift_l(Ll, L, 1);
        const uint32_t nextO = __funnelshift_r(O, Or, 1);
        const uint32_t Lp = (prevL & ~O) | (L & nextO);
#if BML_IMAD_OR
        const uint32_t Op = imad(Lp, a.one, T);  // Lp, T disjoint after the LR phase
#else
        const uint32_t Op = Lp | T;
#endif
        // ---- TB phase emits row rho - 1
        const uint32_t newT = (tA & ~q.oc[s]) | (tB & Op);
        const uint32_t newL = q.lp[s][(P2 + 1) % 2];
        if (COUNT) {
            const int rho = j - 2 * s;
            const unsigned span = static_cast<unsigned>(c.r_hi - c.r_lo);
            if (static_cast<unsigned>(rho - c.r_lo) < span) q.cm[s] += __popc(L & ~nextO & c.valid);
            if (static_cast<unsigned>(rho - 1 - c.r_lo) < span) {
                q.cm[s] += static_cast<uint32_t>(__popc(tB & ~Op & c.valid)) << 16;
                q.cc[s] += __popc(newL & c.valid) +
                           (static_cast<uint32_t>(__popc(newT & c.valid)) << 16);
            }
        }
        q.oc[s] = Op;
        q.lp[s][P2] = Lp;
        if (s < K - 1) {
            q.nt[s][P3] = newT;
        } else {
            store_row<MODE>(a, c, j - 2 * K + 1, newL, newT);
        }
    }
}

// MAXT: launch bound. The default instantiation fits 3 warps per SMSP in the
// register file (<= 168 registers); the 256-thread one (at most two warps per
// SMSP, the latency-bound regime of mid-size lattices) may use up to 255
// registers, and ptxas schedules it with fewer moves (+4% at N=8192).
template <int K, int MODE, bool COUNT, int MAXT = kMaxWarpsPerCta * 32>
__global__ void __launch_bounds__(MAXT, 1)
step_block_kernel(const StepArgs a) {
    if (BML_PDL) {
        asm volatile("griddepcontrol.launch_dependents;");
        asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous launch's rows are final
    }
    const int lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int warps_total = gridDim.x * nwarps;
    __shared__ uint2 ring[MAXT / 32][kRing][32];
    uint2 (*my_ring)[32] = ring[threadIdx.x >> 5];

    // One CTA per SM, 4u warps (u per SM sub-partition: warp w runs on SMSP
    // w % 4). Warp-major item order: items 0..grid-1 go to warp 0 of every CTA,
    // the next grid items to warp 1, ..., so a launch with fewer items than
    // warps still spreads them evenly over the SMs and their sub-partitions.
    for (int item = (threadIdx.x >> 5) * gridDim.x + blockIdx.x; item < a.items; item += warps_total) {
        const int strip = item / a.ncols;
        const int col = item - strip * a.ncols;
        StripCtx c;
        c.lane = lane;
        // rows split evenly: strip i owns [i*rows/nstrips, (i+1)*rows/nstrips)
        c.r_lo = static_cast<int>(static_cast<long long>(strip) * a.rows / a.nstrips);
        c.r_hi = static_cast<int>(static_cast<long long>(strip + 1) * a.rows / a.nstrips);

        int word = lane, c0 = 0;
        c.out_word = lane;
        c.valid = kFull;
        if (MODE != kFullRow) {
            const int w = col * kOutWords + lane - 1;
            const bool is_out = lane >= 1 && lane <= kOutWords && w < a.W;
            c.out_word = w;
            c.valid = is_out ? (w == a.W - 1 ? a.last_mask : kFull) : 0u;
            word = ((w % a.W) + a.W) % a.W;
            long long cc = (32LL * w) % a.n;
            if (cc < 0) cc += a.n;
            c0 = static_cast<int>(cc);
        }

        c.span = c.valid ? static_cast<unsigned>(c.r_hi - c.r_lo) : 0u;

        if (!a.single_band) {
            if (c.r_lo == 0) wait_flag(a.top_flag, a.expect, a.error_flag);
            if (c.r_hi == a.rows) wait_flag(a.bot_flag, a.expect, a.error_flag);
        }

        PipeState<K> q;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            q.nt[s][0] = q.nt[s][1] = q.nt[s][2] = 0u;
            q.lp[s][0] = q.lp[s][1] = 0u;
            q.oc[s] = 0u;
            q.cm[s] = q.cc[s] = 0u;
        }
        q.xt[0] = q.xt[1] = q.xt[2] = 0u;

        const int j_begin = c.r_lo - K;
        const int j_load_end = c.r_hi + K;
        // r_hi + 2K - 1 iterations drain the pipeline; round up to a multiple of 6
        const int iters = c.r_hi + 2 * K - 1 - j_begin;
        const int j_end = j_begin + (iters + 5) / 6 * 6;
        const bool coherent = !a.single_band;

        auto fetch = [&](int j) -> uint2 {
            if (j >= j_load_end) return make_uint2(0u, 0u);
            const uint2* row = a.src + static_cast<long long>(j) * a.pitch;
            return load_cells<MODE>(row, word, c0, a.n, coherent && (j < 0 || j >= a.rows));
        };
        // cp.async ring: row j lands in slot (j - j_begin) % kRing; kRing == the
        // unroll factor, so every slot index below is a compile-time constant
        const uint2* gsrc = a.src + static_cast<long long>(j_begin) * a.pitch + word;
        c.outp = a.dst + static_cast<long long>(j_begin - 2 * K + 1) * a.pitch + c.out_word;
        int j_issue = j_begin;
        auto issue_to = [&](int slot_idx) {
            if (j_issue < j_load_end) cp_async8(&my_ring[slot_idx][lane], gsrc);
            cp_async_commit();
            ++j_issue;
            gsrc += a.pitch;
        };
        auto next_row = [&](auto p_const, uint2& nx0, uint2& nx1) -> uint2 {
            constexpr int P = decltype(p_const)::value;
            uint2 x;
            if (MODE == kGeneric) {
                x = nx0;
                nx0 = nx1;
                nx1 = fetch(j_issue);
                ++j_issue;
            } else {
                cp_async_wait<kRing - 2>();
                x = my_ring[P][lane];
                issue_to((P + kRing - 1) % kRing);
            }
            return x;
        };

        uint2 nx0 = make_uint2(0u, 0u), nx1 = make_uint2(0u, 0u);
        if (MODE == kGeneric) {
            nx0 = fetch(j_begin);
            nx1 = fetch(j_begin + 1);
            j_issue = j_begin + 2;
        } else {
            __syncwarp();
#pragma unroll
            for (int i = 0; i < kRing - 1; ++i) issue_to(i);
        }
        using P0 = std::integral_constant<int, 0>;
        using P1 = std::integral_constant<int, 1>;
        using P2 = std::integral_constant<int, 2>;
        using P3 = std::integral_constant<int, 3>;
        using P4 = std::integral_constant<int, 4>;
        using P5 = std::integral_constant<int, 5>;
        for (int j = j_begin; j < j_end; j += 6) {
            pipe_iter<K, MODE, COUNT, 0>(q, next_row(P0{}, nx0, nx1), j, a, c);
            pipe_iter<K, MODE, COUNT, 1>(q, next_row(P1{}, nx0, nx1), j + 1, a, c);
            pipe_iter<K, MODE, COUNT, 2>(q, next_row(P2{}, nx0, nx1), j + 2, a, c);
            pipe_iter<K, MODE, COUNT, 3>(q, next_row(P3{}, nx0, nx1), j + 3, a, c);
            pipe_iter<K, MODE, COUNT, 4>(q, next_row(P4{}, nx0, nx1), j + 4, a, c);
            pipe_iter<K, MODE, COUNT, 5>(q, next_row(P5{}, nx0, nx1), j + 5, a, c);
            if (MODE == kGeneric && !a.single_band) {
                // rows j-2K+1 .. j-2K+6 were just stored (with their images)
                const int o_last = j - 2 * K + 6;
                if (c.r_lo == 0 && o_last >= kHalo - 1 && o_last - 6 < kHalo - 1) publish(a.up_flag);
                if (c.r_hi == a.rows && o_last >= a.rows - 1 && o_last - 6 < a.rows - 1)
                    publish(a.down_flag);
            }
        }
        if (MODE != kGeneric && (c.r_lo < kHalo || c.r_hi > a.rows - kHalo))
            copy_images(a, c.r_lo, c.r_hi, c.out_word, c.span != 0u);

        if (MODE != kGeneric) cp_async_wait<0>();
        if (COUNT) {
#pragma unroll
            for (int s = 0; s < K; ++s) {
                const unsigned v0 = __reduce_add_sync(kFull, q.cm[s] & 0xffffu);
                const unsigned v1 = __reduce_add_sync(kFull, q.cm[s] >> 16);
                const unsigned v2 = __reduce_add_sync(kFull, q.cc[s] & 0xffffu);
                const unsigned v3 = __reduce_add_sync(kFull, q.cc[s] >> 16);
                if (lane == 0) {
                    unsigned long long* m = a.metrics + a.step_base + s;
                    if (v0) atomicAdd(m, static_cast<unsigned long long>(v0));
                    if (v1) atomicAdd(m + a.metrics_stride, static_cast<unsigned long long>(v1));
                    if (v2) atomicAdd(m + 2 * a.metrics_stride, static_cast<unsigned long long>(v2));
                    if (v3) atomicAdd(m + 3 * a.metrics_stride, static_cast<unsigned long long>(v3));
                }
            }
        }
    }
}

// ------------------------------------------------------------ cluster mbarrier helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint32_t bar, uint32_t tx_bytes) {
    asm volatile(
        "{ .reg .b64 st; mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1; }" ::"r"(bar),
        "r"(tx_bytes)
        : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
// Bounded wait: a lost handoff raises the error flag after ~2 s instead of
// hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int* err) {
    if (mbar_try(bar, parity)) return;
    if (*reinterpret_cast<volatile int*>(err)) return;  // already failed: do not wait again
    const long long t0 = clock64();
    while (!mbar_try(bar, parity)) {
        if (clock64() - t0 > 4000000000LL) {
            atomicExch(err, 3);
            return;
        }
    }
}
__device__ __forceinline__ void st_async_u64(uint32_t remote_addr, uint32_t lo, uint32_t hi,
                                             uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.u32 [%0], {%1, %2}, [%3];" ::"r"(
                     remote_addr),
                 "r"(lo), "r"(hi), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void st_async_u32(uint32_t remote_addr, uint32_t v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(remote_addr),
                 "r"(v), "r"(remote_bar)
                 : "memory");
}

// ------------------------------------------------------------ resident cluster kernel
//
// Small lattices (n % 32 == 0, W = n/32 <= 32) are latency-bound in the
// streaming kernel (a few microseconds of work per launch). Here ONE thread-
// block cluster keeps the whole lattice in registers for the entire run:
// CTA c of C owns rows [c*B, (c+1)*B), B = n/C, and additionally carries
// G ghost rows above and below (its "extended window", E = B + 2G rows,
// RPW rows per warp, lane = word). Each step is computed on the whole
// window in registers; adjacent warps exchange one boundary row per phase
// through shared memory (one __syncthreads per step). Every G steps each CTA
// pushes its first and last G owned rows into the two neighbour CTAs' ghost
// buffers with st.async (DSMEM), completing bytes on the receiver's mbarrier;
// only the warps holding ghost rows wait, and only for their two neighbours.
struct ResidentArgs {
    uint32_t one;  // 1 at run time (IMAD-issued ORs of disjoint planes, BML_IMAD_OR)
    const uint2* src;
    uint2* dst;
    int n, W, pitch;
    int ghost;   // G
    long long steps;
    unsigned long long* metrics;
    int metrics_stride;
    int* error_flag;
};

constexpr int kResidentMaxWarps = 32;
constexpr int kResidentMaxGhost = 16;

template <int RPW, bool COUNT>
__global__ void __launch_bounds__(1024, 1) resident_kernel(const ResidentArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int C = static_cast<int>(cluster.num_blocks());
    const int c = static_cast<int>(cluster.block_rank());
    const int G = a.ghost;
    const int B = a.n / C;
    const int r0 = c * B;
    const int NW = blockDim.x >> 5;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = a.W;
    const bool lane_ok = lane < W;
    const int left = lane == 0 ? W - 1 : lane - 1;
    const int right = lane + 1 >= W ? 0 : lane + 1;

    __shared__ uint32_t xT[2][kResidentMaxWarps][32];  // last row's T of each warp
    __shared__ uint32_t xO[2][kResidentMaxWarps][32];  // first row's occupancy after LR
    __shared__ uint2 ghostb[2][2 * kResidentMaxGhost][32];  // [0,G): rows above, [G,2G): rows below
    __shared__ unsigned long long cnt[4][kResidentMaxGhost];
    // ghost rows arrive by st.async from the two neighbours, completing bytes on
    // gbar[block parity]: only those two CTAs synchronise, no cluster barrier
    __shared__ __align__(8) unsigned long long gbar[2];
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&gbar[0]), 1);
        mbar_init(smem_u32(&gbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint32_t ghost_bytes = 2u * static_cast<uint32_t>(G) * 32u * sizeof(uint2);
    const int up_rank = (c + C - 1) % C, dn_rank = (c + 1) % C;
    cluster.sync();  // every CTA's barriers are initialised before the first remote store

    uint32_t L[RPW], T[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int e = w * RPW + i;
        int row = (r0 - G + e) % a.n;
        if (row < 0) row += a.n;
        const uint2 x = lane_ok ? a.src[static_cast<long long>(row) * a.pitch + lane] : make_uint2(0u, 0u);
        L[i] = x.x;
        T[i] = x.y;
    }
    if (COUNT) {
        for (int i = threadIdx.x; i < 4 * kResidentMaxGhost; i += blockDim.x) (&cnt[0][0])[i] = 0ull;
        __syncthreads();
    }

    const uint32_t valid = lane_ok ? kFull : 0u;
    int par = 0, bp = 0;
    long long blk = 0;
    for (long long done = 0; done < a.steps;) {
        const int kb = static_cast<int>(min(static_cast<long long>(G), a.steps - done));
        if (threadIdx.x == 0) mbar_arm(smem_u32(&gbar[bp]), ghost_bytes);  // this block's pushes
        if (done > 0) {
            // the previous block's ghost rows: only warps holding ghost rows wait
            const bool holds_ghost = w * RPW < G || (w + 1) * RPW > G + B;
            if (holds_ghost) mbar_wait(smem_u32(&gbar[bp ^ 1]), static_cast<uint32_t>(((blk - 1) >> 1) & 1), a.error_flag);
            // ghost rows pushed into this CTA's shared memory by the neighbours
            // before the last cluster barrier (local loads only)
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int e = w * RPW + i;
                if (e < G) {
                    const uint2 x = ghostb[bp ^ 1][e][lane];
                    L[i] = x.x;
                    T[i] = x.y;
                } else if (e >= G + B) {
                    const uint2 x = ghostb[bp ^ 1][G + (e - G - B)][lane];
                    L[i] = x.x;
                    T[i] = x.y;
                }
            }
        }
        for (int s = 0; s < kb; ++s) {
            uint32_t Op[RPW];
            uint32_t lr_moved = 0;
#pragma unroll
            for (int i = 0; i < RPW; ++i) {  // LR phase, row-local
                const uint32_t O = BML_IMAD_OR ? imad(L[i], a.one, T[i]) : (L[i] | T[i]);
                const uint32_t Ll = __shfl_sync(kFull, L[i], left);
                const uint32_t Or = __shfl_sync(kFull, O, right);
                const uint32_t prevL = __funnelshift_l(Ll, L[i], 1);
                const uint32_t nextO = __funnelshift_r(O, Or, 1);
                const uint32_t inc = prevL & ~O;
                const uint32_t vac = L[i] & ~nextO;
                if (COUNT) {
                    const int e = w * RPW + i;
                    if (e >= G && e < G + B) lr_moved += __popc(vac & valid);
                }
                L[i] = inc | (L[i] & nextO);
                Op[i] = BML_IMAD_OR ? imad(L[i], a.one, T[i]) : (L[i] | T[i]);
            }
            xT[par][w][lane] = T[RPW - 1];
            xO[par][w][lane] = Op[0];
            uint32_t tb_moved = 0, lr_cnt = 0, tb_cnt = 0;
            auto tb_row = [&](int i, uint32_t above, uint32_t below) {  // TB phase, one row
                const uint32_t nt = (above & ~Op[i]) | (T[i] & below);
                if (COUNT) {
                    const int e = w * RPW + i;
                    if (e >= G && e < G + B) {
                        tb_moved += __popc(T[i] & ~below & valid);
                        lr_cnt += __popc(L[i] & valid);
                        tb_cnt += __popc(nt & valid);
                    }
                }
                T[i] = nt;
            };
            __syncthreads();
            const uint32_t t_up = w > 0 ? xT[par][w - 1][lane] : 0u;
            const uint32_t o_dn = w < NW - 1 ? xO[par][w + 1][lane] : kFull;
#pragma unroll
            for (int i = RPW - 1; i >= 0; --i)  // top-down neighbours
                tb_row(i, i > 0 ? T[i - 1] : t_up, i < RPW - 1 ? Op[i + 1] : o_dn);
            if (COUNT) {
                const unsigned v0 = __reduce_add_sync(kFull, lr_moved);
                const unsigned v1 = __reduce_add_sync(kFull, tb_moved);
                const unsigned v2 = __reduce_add_sync(kFull, lr_cnt);
                const unsigned v3 = __reduce_add_sync(kFull, tb_cnt);
                if (lane == 0) {
                    if (v0) atomicAdd(&cnt[0][s], static_cast<unsigned long long>(v0));
                    if (v1) atomicAdd(&cnt[1][s], static_cast<unsigned long long>(v1));
                    if (v2) atomicAdd(&cnt[2][s], static_cast<unsigned long long>(v2));
                    if (v3) atomicAdd(&cnt[3][s], static_cast<unsigned long long>(v3));
                }
            }
            par ^= 1;
        }
        // push owned boundary rows into the neighbours' ghost buffers (DSMEM
        // stores, made visible by the release/acquire cluster barrier below):
        // first G owned rows -> the CTA above's rows-below slots, last G owned
        // rows -> the CTA below's rows-above slots
        {
            const uint32_t base = smem_u32(&ghostb[bp][0][0]);
            const uint32_t up_base = mapa_u32(base, up_rank), dn_base = mapa_u32(base, dn_rank);
            const uint32_t up_bar = mapa_u32(smem_u32(&gbar[bp]), up_rank);
            const uint32_t dn_bar = mapa_u32(smem_u32(&gbar[bp]), dn_rank);
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int e = w * RPW + i;
                if (e >= G && e < 2 * G)
                    st_async_u64(up_base + static_cast<uint32_t>((e * 32 + lane) * 8), L[i], T[i], up_bar);
                if (e >= B && e < B + G)
                    st_async_u64(dn_base + static_cast<uint32_t>(((e - B) * 32 + lane) * 8), L[i], T[i], dn_bar);
            }
        }
        if (COUNT) {
            __syncthreads();
            for (int t = threadIdx.x; t < 4 * kb; t += blockDim.x) {
                const int q = t / kb, s = t % kb;
                const unsigned long long v = cnt[q][s];
                if (v) atomicAdd(a.metrics + static_cast<long long>(q) * a.metrics_stride + done + s, v);
                cnt[q][s] = 0ull;
            }
        }
        bp ^= 1;
        done += kb;
        ++blk;
    }
    cluster.sync();  // no CTA leaves while a neighbour may still store into its shared memory
    // owned rows back to global, plus the single-band ghost images
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int e = w * RPW + i;
        if (e >= G && e < G + B && lane_ok) {
            const int row = r0 + e - G;
            const uint2 v = make_uint2(L[i], T[i]);
            a.dst[static_cast<long long>(row) * a.pitch + lane] = v;
            for (int h = row - a.n; h >= -kHalo; h -= a.n) a.dst[static_cast<long long>(h) * a.pitch + lane] = v;
            for (int h = row + a.n; h < a.n + kHalo; h += a.n) a.dst[static_cast<long long>(h) * a.pitch + lane] = v;
        }
    }
}

// ------------------------------------------------------------ resident kernel, p2p variant
//
// Same residency as resident_kernel, but no ghost rows: every step the CTA
// hands its first row's post-LR occupancy to the CTA above and its last row's
// T plane to the CTA below with st.async remote stores that complete_tx on the
// receiver's mbarrier (256 B per step per CTA). Only the two boundary warps
// ever wait, and only for their two neighbours: no cluster-wide barrier, no
// redundant ghost-row arithmetic.

template <int RPW, bool COUNT>
__global__ void __launch_bounds__(1024, 1) resident_p2p_kernel(const ResidentArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int C = static_cast<int>(cluster.num_blocks());
    const int c = static_cast<int>(cluster.block_rank());
    const int B = a.n / C;
    const int r0 = c * B;
    const int NW = blockDim.x >> 5;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = a.W;
    const bool lane_ok = lane < W;
    const int left = lane == 0 ? W - 1 : lane - 1;
    const int right = lane + 1 >= W ? 0 : lane + 1;
    const int up_rank = (c + C - 1) % C, dn_rank = (c + 1) % C;

    __shared__ uint32_t xT[2][kResidentMaxWarps][32];
    __shared__ uint32_t xO[2][kResidentMaxWarps][32];
    __shared__ uint32_t mT[2][32];  // T of the row above this CTA's first row (from the CTA above)
    __shared__ uint32_t mO[2][32];  // occupancy after LR of the row below the last row (from below)
    __shared__ __align__(8) unsigned long long mbar[2];
    __shared__ unsigned long long cnt[2][4][16];

    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&mbar[0]), 1);
        mbar_init(smem_u32(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (COUNT)
        for (int i = threadIdx.x; i < 2 * 4 * 16; i += blockDim.x) (&cnt[0][0][0])[i] = 0ull;

    uint32_t L[RPW], T[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int row = r0 + w * RPW + i;
        const uint2 x = lane_ok ? a.src[static_cast<long long>(row) * a.pitch + lane] : make_uint2(0u, 0u);
        L[i] = x.x;
        T[i] = x.y;
    }
    cluster.sync();  // every CTA's mbarriers are initialised before the first remote store

    // remote destinations (constant for the run)
    const uint32_t up_mO0 = mapa_u32(smem_u32(&mO[0][lane]), up_rank);
    const uint32_t up_mO1 = mapa_u32(smem_u32(&mO[1][lane]), up_rank);
    const uint32_t dn_mT0 = mapa_u32(smem_u32(&mT[0][lane]), dn_rank);
    const uint32_t dn_mT1 = mapa_u32(smem_u32(&mT[1][lane]), dn_rank);
    const uint32_t up_bar0 = mapa_u32(smem_u32(&mbar[0]), up_rank);
    const uint32_t up_bar1 = mapa_u32(smem_u32(&mbar[1]), up_rank);
    const uint32_t dn_bar0 = mapa_u32(smem_u32(&mbar[0]), dn_rank);
    const uint32_t dn_bar1 = mapa_u32(smem_u32(&mbar[1]), dn_rank);
    const uint32_t my_bar0 = smem_u32(&mbar[0]), my_bar1 = smem_u32(&mbar[1]);

    const uint32_t valid = lane_ok ? kFull : 0u;
    for (long long s = 0; s < a.steps; ++s) {
        const int p = static_cast<int>(s & 1);
        const uint32_t ph = static_cast<uint32_t>((s >> 1) & 1);
        const uint32_t my_bar = p ? my_bar1 : my_bar0;
        if (threadIdx.x == 0) mbar_arm(my_bar, 2 * 32 * 4);
        uint32_t Op[RPW];
        uint32_t lr_moved = 0;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {  // LR phase
            const uint32_t O = BML_IMAD_OR ? imad(L[i], a.one, T[i]) : (L[i] | T[i]);
            const uint32_t Ll = __shfl_sync(kFull, L[i], left);
            const uint32_t Or = __shfl_sync(kFull, O, right);
            const uint32_t prevL = __funnelshift_l(Ll, L[i], 1);
            const uint32_t nextO = __funnelshift_r(O, Or, 1);
            if (COUNT) lr_moved += __popc(L[i] & ~nextO & valid);
            L[i] = (prevL & ~O) | (L[i] & nextO);
            Op[i] = BML_IMAD_OR ? imad(L[i], a.one, T[i]) : (L[i] | T[i]);
        }
        if (w == 0) st_async_u32(p ? up_mO1 : up_mO0, Op[0], p ? up_bar1 : up_bar0);
        if (w == NW - 1) st_async_u32(p ? dn_mT1 : dn_mT0, T[RPW - 1], p ? dn_bar1 : dn_bar0);
        xT[p][w][lane] = T[RPW - 1];
        xO[p][w][lane] = Op[0];
        __syncthreads();
        if (w == 0 || w == NW - 1) mbar_wait(my_bar, ph, a.error_flag);
        const uint32_t t_up = w > 0 ? xT[p][w - 1][lane] : mT[p][lane];
        const uint32_t o_dn = w < NW - 1 ? xO[p][w + 1][lane] : mO[p][lane];
        uint32_t tb_moved = 0, lr_cnt = 0, tb_cnt = 0;
#pragma unroll
        for (int i = RPW - 1; i >= 0; --i) {  // TB phase
            const uint32_t above = i > 0 ? T[i - 1] : t_up;
            const uint32_t below = i < RPW - 1 ? Op[i + 1] : o_dn;
            const uint32_t nt = (above & ~Op[i]) | (T[i] & below);
            if (COUNT) {
                tb_moved += __popc(T[i] & ~below & valid);
                lr_cnt += __popc(L[i] & valid);
                tb_cnt += __popc(nt & valid);
            }
            T[i] = nt;
        }
        if (COUNT) {
            const int chunk = static_cast<int>((s >> 4) & 1), slot = static_cast<int>(s & 15);
            const unsigned v0 = __reduce_add_sync(kFull, lr_moved);
            const unsigned v1 = __reduce_add_sync(kFull, tb_moved);
            const unsigned v2 = __reduce_add_sync(kFull, lr_cnt);
            const unsigned v3 = __reduce_add_sync(kFull, tb_cnt);
            if (lane == 0) {
                if (v0) atomicAdd(&cnt[chunk][0][slot], static_cast<unsigned long long>(v0));
                if (v1) atomicAdd(&cnt[chunk][1][slot], static_cast<unsigned long long>(v1));
                if (v2) atomicAdd(&cnt[chunk][2][slot], static_cast<unsigned long long>(v2));
                if (v3) atomicAdd(&cnt[chunk][3][slot], static_cast<unsigned long long>(v3));
            }
            if (slot == 15 || s == a.steps - 1) {
                __syncthreads();
                const long long base = s - slot;
                for (int t = threadIdx.x; t < 4 * (slot + 1); t += blockDim.x) {
                    const int q = t / (slot + 1), k = t % (slot + 1);
                    const unsigned long long v = cnt[chunk][q][k];
                    if (v) atomicAdd(a.metrics + static_cast<long long>(q) * a.metrics_stride + base + k, v);
                    cnt[chunk][q][k] = 0ull;
                }
            }
        }
    }
    cluster.sync();  // no CTA leaves while a neighbour may still address its shared memory
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        if (!lane_ok) continue;
        const int row = r0 + w * RPW + i;
        const uint2 v = make_uint2(L[i], T[i]);
        a.dst[static_cast<long long>(row) * a.pitch + lane] = v;
        for (int h = row - a.n; h >= -kHalo; h -= a.n) a.dst[static_cast<long long>(h) * a.pitch + lane] = v;
        for (int h = row + a.n; h < a.n + kHalo; h += a.n) a.dst[static_cast<long long>(h) * a.pitch + lane] = v;
    }
}

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

// ------------------------------------------------------------ dispatch table
using StepKernel = void (*)(const StepArgs);

template <int MODE, bool COUNT>
StepKernel pick_k(int k) {
    switch (k) {
        case 1: return step_block_kernel<1, MODE, COUNT>;
        case 2: return step_block_kernel<2, MODE, COUNT>;
        case 4: return step_block_kernel<4, MODE, COUNT>;
        case 8: return step_block_kernel<8, MODE, COUNT>;
        case 16: return step_block_kernel<16, MODE, COUNT>;
        default: return nullptr;
    }
}

// u <= 2 (at most two warps per SMSP) variant of the K = 16 hot path, see step_block_kernel
StepKernel pick_narrow(int k, int mode, bool count) {
    if (k != 16 || count) return nullptr;
    if (mode == kFullRow) return step_block_kernel<16, kFullRow, false, 256>;
    if (mode == kAligned) return step_block_kernel<16, kAligned, false, 256>;
    return nullptr;
}

// Warps per SMSP the register file allows for a kernel (memoised: the
// attribute query costs host time on every launch otherwise).
int warps_per_smsp(StepKernel kern) {
    static std::mutex mu;
    static std::vector<std::pair<StepKernel, int>> cache;
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& kv : cache)
        if (kv.first == kern) return kv.second;
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    const int regs = std::max(1, (fa.numRegs + 7) / 8 * 8);
    const int u = std::max(1, std::min(kMaxWarpsPerCta / 4, 65536 / (regs * 128)));
    cache.emplace_back(kern, u);
    return u;
}

StepKernel pick(int k, int mode, bool count) {
    if (mode == kFullRow) return count ? pick_k<kFullRow, true>(k) : pick_k<kFullRow, false>(k);
    if (mode == kAligned) return count ? pick_k<kAligned, true>(k) : pick_k<kAligned, false>(k);
    return count ? pick_k<kGeneric, true>(k) : pick_k<kGeneric, false>(k);
}

int largest_block_at_most(long long remaining, int cap) {
    int k = 16;
    while (k > 1 && (k > remaining || k > cap)) k >>= 1;
    return k;
}

struct IpcBlob {
    uint32_t magic;
    int32_t n, row_begin, row_end, pitch, W;
    int32_t pid;
    int32_t device;
    cudaIpcMemHandle_t buf[2];
    cudaIpcMemHandle_t flags;
};
static_assert(sizeof(IpcBlob) <= BML_EXPORT_BYTES, "blob too large");
constexpr uint32_t kBlobMagic = 0xB200B31Eu;

}  // namespace

// ================================================================ handle
struct bml_dev {
    int n = 0, W = 0, pitch = 0;
    int row_begin = 0, row_end = 0, rows = 0;
    int device = 0;
    uint32_t last_mask = kFull;
    int mode = kGeneric;
    int block_steps = 16;
    int strip_rows = 0;      // 0 = auto (choose_nstrips); < 0: exactly -strip_rows strips
    int resident = 1;        // 1: use the cluster-resident kernel when the lattice qualifies
    int resident_cluster = 0;  // cluster size actually used by the last resident launch
    int last_nstrips = 0, last_grid = 0, last_items = 0;  // last streaming launch
    int ns_cache_k[kHalo + 1] = {};        // memoised choose_nstrips per block depth
    int ns_cache_setting[kHalo + 1] = {};  // the strip_rows setting it was computed for
    int sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    uint2* buf[2] = {nullptr, nullptr};  // allocation bases
    int cur = 0;
    uint8_t* staging = nullptr;          // rows * n bytes
    unsigned long long* scratch = nullptr;  // 4 words: counts / moved
    int* err = nullptr;                  // [0]: bad upload cell, [1]: flag timeout
    unsigned long long* flags = nullptr;  // [0]: top (from up), [1]: bottom (from down)
    unsigned long long* metrics = nullptr;
    long long metrics_cap = 0;
    // multi-band links
    bool connected = false;
    uint2* up_halo[2] = {nullptr, nullptr};
    uint2* down_halo[2] = {nullptr, nullptr};
    unsigned long long* up_flag = nullptr;    // neighbour above: its bottom flag
    unsigned long long* down_flag = nullptr;  // neighbour below: its top flag
    std::vector<void*> ipc_opened;
    unsigned long long pubs = 0;
    // timing
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    long long launches = 0;
    double kernel_ms = 0.0;

    uint2* row0(int parity) const { return buf[parity] + static_cast<long long>(kHalo) * pitch; }
    bool single_band() const { return rows == n && row_begin == 0; }
    int ncols() const { return mode == kFullRow ? 1 : (W + kOutWords - 1) / kOutWords; }
};

namespace {

int check(bml_dev* d) {
    if (!d) return fail(BML_EINVAL, "null bml_dev handle");
    cudaError_t e = cudaSetDevice(d->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    return BML_OK;
}

cudaEvent_t take_event(bml_dev* d) {
    if (!d->ev_pool.empty()) {
        cudaEvent_t e = d->ev_pool.back();
        d->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void harvest_timing(bml_dev* d) {
    for (auto& pr : d->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) d->kernel_ms += ms;
        d->ev_pool.push_back(pr.first);
        d->ev_pool.push_back(pr.second);
    }
    d->pending.clear();
}

int ensure_metrics(bml_dev* d, long long steps) {
    const long long need = 4 * steps;
    if (need <= d->metrics_cap) return BML_OK;
    if (d->metrics) cudaFree(d->metrics);
    d->metrics = nullptr;
    d->metrics_cap = 0;
    BML_CUDA(cudaMalloc(&d->metrics, need * sizeof(unsigned long long)));
    d->metrics_cap = need;
    return BML_OK;
}

int fill_images(bml_dev* d, int parity) {
    const int total = 2 * kHalo * d->W;
    fill_images_kernel<<<(total + 255) / 256, 256, 0, d->stream>>>(d->row0(parity), d->n, d->W,
                                                                   d->pitch, d->rows);
    BML_CUDA(cudaGetLastError());
    return BML_OK;
}

int create_common(int n, int row_begin, int row_end, int device, bml_dev** out) {
    if (!out) return fail(BML_EINVAL, "bml_dev_create: out is null");
    *out = nullptr;
    if (n < 1) return fail(BML_EINVAL, "bml_dev_create: n must be >= 1");
    if (row_begin < 0 || row_end > n || row_begin >= row_end)
        return fail(BML_EINVAL, "bml_dev_create_band: need 0 <= row_begin < row_end <= n");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0) {
        e = cudaGetDevice(&device);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    }
    if (device < 0 || device >= count)
        return fail(BML_EINVAL, "bml_dev_create: device " + std::to_string(device) + " out of range");
    e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");

    bml_dev* d = new (std::nothrow) bml_dev;
    if (!d) return fail(BML_ENOMEM, "host allocation failed");
    d->n = n;
    d->W = (n + 31) / 32;
    d->pitch = (d->W + 15) / 16 * 16;  // 128-byte aligned rows
    d->row_begin = row_begin;
    d->row_end = row_end;
    d->rows = row_end - row_begin;
    d->device = device;
    const int nb = n - 32 * (d->W - 1);
    d->last_mask = nb == 32 ? kFull : ((1u << nb) - 1u);
    d->mode = (n % 32 != 0) ? kGeneric : (d->W == 32 ? kFullRow : kAligned);
    cudaDeviceGetAttribute(&d->sms, cudaDevAttrMultiProcessorCount, device);

    auto bail = [&](cudaError_t err, const char* what) {
        bml_dev_destroy(d);
        return cuda_fail(err, what);
    };
    const size_t words = static_cast<size_t>(d->rows + 2 * kHalo) * d->pitch;
    for (int p = 0; p < 2; ++p) {
        if ((e = cudaMalloc(&d->buf[p], words * sizeof(uint2))) != cudaSuccess)
            return bail(e, "cudaMalloc(lattice)");
        if ((e = cudaMemset(d->buf[p], 0, words * sizeof(uint2))) != cudaSuccess)
            return bail(e, "cudaMemset(lattice)");
    }
    if ((e = cudaMalloc(&d->staging, static_cast<size_t>(d->rows) * n)) != cudaSuccess)
        return bail(e, "cudaMalloc(staging)");
    if ((e = cudaMalloc(&d->scratch, 4 * sizeof(unsigned long long))) != cudaSuccess)
        return bail(e, "cudaMalloc(scratch)");
    if ((e = cudaMalloc(&d->err, 4 * sizeof(int))) != cudaSuccess) return bail(e, "cudaMalloc(err)");
    if ((e = cudaMemset(d->err, 0, 4 * sizeof(int))) != cudaSuccess) return bail(e, "cudaMemset(err)");
    if ((e = cudaMalloc(&d->flags, 2 * sizeof(unsigned long long))) != cudaSuccess)
        return bail(e, "cudaMalloc(flags)");
    if ((e = cudaMemset(d->flags, 0, 2 * sizeof(unsigned long long))) != cudaSuccess)
        return bail(e, "cudaMemset(flags)");
    if ((e = cudaStreamCreateWithFlags(&d->own_stream, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(e, "cudaStreamCreate");
    d->stream = d->own_stream;
    *out = d;
    return BML_OK;
}

int check_errors(bml_dev* d) {
    int h[4] = {0, 0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(h, d->err, sizeof h, cudaMemcpyDeviceToHost, d->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(d->stream);
    if (e != cudaSuccess) return cuda_fail(e, "error-flag readback");
    if (h[1]) {
        cudaMemsetAsync(d->err, 0, 4 * sizeof(int), d->stream);
        return fail(BML_ECUDA, h[1] == 3 ? "resident kernel: DSMEM handoff timed out"
                                         : "halo flag wait timed out (neighbour band stalled)");
    }
    return BML_OK;
}

// Strips per launch. A strip of R rows costs R + 3K - 1 pipeline iterations
// of K stages (2K ghost rows + K-1 drain) plus about 16 iterations' worth of
// per-item setup. Items (strips x warp columns) are spread evenly over the SMs
// and their four sub-partitions (SMSPs; one CTA per SM, warp-major order, see
// step_block_kernel). Per-SMSP time model, in clocks for one pipeline iteration
// of each of its u warps at K = 16, measured on B200
// (profiles/r1_sweep_narrow_u1.jsonl, r1_sweep_u2big.jsonl): u = 1: 330 (one
// warp's K independent stage chains cannot fill the issue slots), u = 2: 515
// (the 255-register instantiation), u = 3: 780 (~260 per warp: ALU pipe and
// issue slots near saturation). An SM runs ceil(items / SMs) warps' items in
// rounds of at most warps_per_sm. Rows are split evenly over the strips.
long long smsp_round_cost(long long w) {
    const long long u = (w + 3) / 4;
    if (u <= 1) return 330;
    if (u == 2) return 515;
    return 780 + (u - 3) * 260;
}

int choose_nstrips(const bml_dev* d, int k, int warps_per_sm) {
    const int min_rows = d->connected ? kHalo : 1;
    if (d->strip_rows > 0) return std::max(1, d->rows / std::max(d->strip_rows, min_rows));
    if (d->strip_rows < 0) return std::max(1, std::min(-d->strip_rows, d->rows / min_rows));
    const long long cols = d->ncols();
    const int max_strips = std::max(1, d->rows / min_rows);
    long long best_cost = -1;
    int best = 1;
    for (int ns = 1; ns <= max_strips; ++ns) {
        const long long r = (d->rows + ns - 1) / ns;
        const long long per_sm = (ns * cols + d->sms - 1) / d->sms;
        const long long full = per_sm / warps_per_sm, last = per_sm % warps_per_sm;
        const long long cost = (r + 3 * k + 16) * (full * smsp_round_cost(warps_per_sm) +
                                              (last ? smsp_round_cost(last) : 0));
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = ns;
        }
    }
    return best;
}

int launch_block(bml_dev* d, int k, bool count, int step_base, int metrics_stride) {
    StepKernel kern = pick(k, d->mode, count);
    if (!kern) return fail(BML_EINVAL, "unsupported block depth " + std::to_string(k));
    const int u_max = warps_per_smsp(kern);  // 3 at <= 168 registers/thread
    // every strip has >= min(strip_rows, 16) rows, so for connected bands the
    // ghost-row sources of a band never straddle strips
    // the model scans every strip count: memoised per (k, strip setting)
    if (d->ns_cache_k[k] <= 0 || d->ns_cache_setting[k] != d->strip_rows) {
        d->ns_cache_k[k] = choose_nstrips(d, k, 4 * u_max);
        d->ns_cache_setting[k] = d->strip_rows;
    }
    const int nstrips = d->ns_cache_k[k];
    const int strip = d->rows / nstrips;
    StepArgs a{};
    a.src = d->row0(d->cur);
    a.dst = d->row0(d->cur ^ 1);
    a.n = d->n;
    a.W = d->W;
    a.pitch = d->pitch;
    a.rows = d->rows;
    a.strip_rows = strip;
    a.nstrips = nstrips;
    a.ncols = d->ncols();
    a.items = nstrips * a.ncols;
    a.last_mask = d->last_mask;
    a.single_band = d->connected ? 0 : 1;
    const int nxt = d->cur ^ 1;
    a.up_halo = d->up_halo[nxt];
    a.down_halo = d->down_halo[nxt];
    a.up_flag = d->up_flag;
    a.down_flag = d->down_flag;
    a.top_flag = d->flags;
    a.bot_flag = d->flags + 1;
    a.expect = d->pubs * static_cast<unsigned long long>(a.ncols);
    a.metrics = d->metrics;
    a.metrics_stride = metrics_stride;
    a.step_base = step_base;
    a.error_flag = d->err + 1;
    a.one = 1u;
    {
        // image slots relative to a row's own slot (flat 64-bit address space,
        // so the distance to a peer's buffer is a plain pointer difference)
        const long long rp = static_cast<long long>(d->rows) * d->pitch;
        const auto words_between = [](const uint2* from, const uint2* to) {
            return static_cast<long long>(reinterpret_cast<intptr_t>(to) - reinterpret_cast<intptr_t>(from)) /
                   static_cast<long long>(sizeof(uint2));
        };
        a.top_delta = d->connected ? words_between(a.dst, a.up_halo) : rp;
        a.bot_delta = d->connected ? words_between(a.dst, a.down_halo) - rp : -rp;
    }

    // one CTA per SM with 4u warps, u = the warps per SMSP the items need
    const int u = std::min(u_max, std::max(1, (a.items + 4 * d->sms - 1) / (4 * d->sms)));
    const int grid = std::max(1, std::min(d->sms, a.items));
    const int threads = 4 * u * 32;
    if (u <= 2) {
        if (StepKernel narrow = pick_narrow(k, d->mode, count)) kern = narrow;
    }
    d->last_nstrips = nstrips;
    d->last_grid = grid;
    d->last_items = a.items;

    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (d->timing) {
        e0 = take_event(d);
        e1 = take_event(d);
        cudaEventRecord(e0, d->stream);
    }
    cudaError_t e;
    if (BML_PDL) {
        // programmatic dependent launch: this grid may be scheduled while the
        // previous one drains; the kernel waits (griddepcontrol.wait) before
        // touching the lattice, so only the launch gap is hidden
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(static_cast<unsigned>(threads));
        cfg.stream = d->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, a);
    } else {
        kern<<<grid, threads, 0, d->stream>>>(a);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return cuda_fail(e, "step_block_kernel launch");
    if (d->timing) {
        cudaEventRecord(e1, d->stream);
        d->pending.emplace_back(e0, e1);
    }
    ++d->launches;
    d->cur ^= 1;
    if (d->connected) ++d->pubs;
    return BML_OK;
}

using ResidentKernel = void (*)(const ResidentArgs);

template <bool COUNT>
ResidentKernel pick_p2p(int rpw) {
    switch (rpw) {
        case 1: return resident_p2p_kernel<1, COUNT>;
        case 2: return resident_p2p_kernel<2, COUNT>;
        case 4: return resident_p2p_kernel<4, COUNT>;
        case 8: return resident_p2p_kernel<8, COUNT>;
        default: return nullptr;
    }
}

template <bool COUNT>
ResidentKernel pick_resident(int rpw) {
    switch (rpw) {
        case 1: return resident_kernel<1, COUNT>;
        case 2: return resident_kernel<2, COUNT>;
        case 3: return resident_kernel<3, COUNT>;
        case 4: return resident_kernel<4, COUNT>;
        case 5: return resident_kernel<5, COUNT>;
        case 6: return resident_kernel<6, COUNT>;
        case 8: return resident_kernel<8, COUNT>;
        default: return nullptr;
    }
}

// Geometry of the resident launch, or false if the lattice does not qualify.
bool resident_plan(const bml_dev* d, int cluster, int* ghost, int* rpw, int* warps) {
    if (!d->resident || !d->single_band() || d->connected) return false;
    if (d->n % 32 != 0 || d->W > 32 || d->n % cluster != 0) return false;
    const int B = d->n / cluster;
    if (d->resident == 2) {  // p2p variant: no ghost rows, B = warps * rpw
        for (int r : {4, 2, 8, 1}) {
            if (B % r == 0 && B / r <= kResidentMaxWarps) {
                *ghost = 0;
                *rpw = r;
                *warps = B / r;
                return true;
            }
        }
        return false;
    }
    const int G = std::min(kResidentMaxGhost, std::max(1, d->block_steps));
    if (B < G) return false;
    const int E = B + 2 * G;
    for (int r : {5, 4, 6, 3, 8, 2, 1}) {
        if (E % r == 0 && E / r <= kResidentMaxWarps && E / r >= 1) {
            *ghost = G;
            *rpw = r;
            *warps = E / r;
            return true;
        }
    }
    return false;
}

int launch_resident(bml_dev* d, long long steps, bool count, bool* used) {
    *used = false;
    for (int cluster : {16, 8, 4, 2, 1}) {
        int G = 0, rpw = 0, nw = 0;
        if (!resident_plan(d, cluster, &G, &rpw, &nw)) continue;
        ResidentKernel kern = d->resident == 2
                                  ? (count ? pick_p2p<true>(rpw) : pick_p2p<false>(rpw))
                                  : (count ? pick_resident<true>(rpw) : pick_resident<false>(rpw));
        if (!kern) continue;
        if (cluster > 8) {
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                cudaSuccess) {
                (void)cudaGetLastError();
                continue;
            }
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(cluster));
        cfg.blockDim = dim3(static_cast<unsigned>(32 * nw));
        cfg.dynamicSmemBytes = 0;
        cfg.stream = d->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int max_clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) {
            (void)cudaGetLastError();
            continue;
        }
        ResidentArgs ra{};
        ra.one = 1u;
        ra.src = d->row0(d->cur);
        ra.dst = d->row0(d->cur ^ 1);
        ra.n = d->n;
        ra.W = d->W;
        ra.pitch = d->pitch;
        ra.ghost = G;
        ra.steps = steps;
        ra.metrics = d->metrics;
        ra.metrics_stride = static_cast<int>(steps);
        ra.error_flag = d->err + 1;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (d->timing) {
            e0 = take_event(d);
            e1 = take_event(d);
            cudaEventRecord(e0, d->stream);
        }
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ra);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            if (d->timing) {
                d->ev_pool.push_back(e0);
                d->ev_pool.push_back(e1);
            }
            continue;
        }
        if (d->timing) {
            cudaEventRecord(e1, d->stream);
            d->pending.emplace_back(e0, e1);
        }
        ++d->launches;
        d->cur ^= 1;
        d->resident_cluster = cluster;
        *used = true;
        return BML_OK;
    }
    return BML_OK;
}

}  // namespace

// ================================================================ C-ABI
extern "C" {

const char* bml_dev_last_error(void) { return g_last_error.c_str(); }

const char* bml_dev_version(void) { return "bml_dev 0.1.0 sm_100a bitplane-temporal"; }

int bml_dev_device_count(int* count) {
    if (!count) return fail(BML_EINVAL, "bml_dev_device_count: null pointer");
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
        (void)cudaGetLastError();
        *count = 0;
        return BML_OK;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    return BML_OK;
}

int bml_dev_create(int n, int device, bml_dev** out) {
    return create_common(n, 0, n, device, out);
}

int bml_dev_create_band(int n, int row_begin, int row_end, int device, bml_dev** out) {
    if (row_end - row_begin < kHalo && !(row_begin == 0 && row_end == n))
        return fail(BML_EINVAL, "bml_dev_create_band: a band needs >= 16 rows");
    return create_common(n, row_begin, row_end, device, out);
}

int bml_dev_destroy(bml_dev* d) {
    if (!d) return BML_OK;
    cudaSetDevice(d->device);
    if (d->stream) cudaStreamSynchronize(d->stream);
    for (void* p : d->ipc_opened) cudaIpcCloseMemHandle(p);
    for (int p = 0; p < 2; ++p) cudaFree(d->buf[p]);
    cudaFree(d->staging);
    cudaFree(d->scratch);
    cudaFree(d->err);
    cudaFree(d->flags);
    cudaFree(d->metrics);
    for (auto& pr : d->pending) {
        d->ev_pool.push_back(pr.first);
        d->ev_pool.push_back(pr.second);
    }
    for (cudaEvent_t e : d->ev_pool) cudaEventDestroy(e);
    if (d->own_stream) cudaStreamDestroy(d->own_stream);
    delete d;
    return BML_OK;
}

int bml_dev_set_stream(bml_dev* d, void* stream) {
    if (int rc = check(d)) return rc;
    d->stream = stream ? static_cast<cudaStream_t>(stream) : d->own_stream;
    return BML_OK;
}

int bml_dev_sync(bml_dev* d) {
    if (int rc = check(d)) return rc;
    BML_CUDA(cudaStreamSynchronize(d->stream));
    return check_errors(d);
}

int bml_dev_configure(bml_dev* d, int block_steps, int strip_rows) {
    if (int rc = check(d)) return rc;
    if (block_steps) {
        if (block_steps != 1 && block_steps != 2 && block_steps != 4 && block_steps != 8 &&
            block_steps != 16)
            return fail(BML_EINVAL, "block_steps must be one of 1, 2, 4, 8, 16");
        d->block_steps = block_steps;
    }
    if (strip_rows) {
        if (strip_rows < -65536 || strip_rows > 65536)
            return fail(BML_EINVAL, "strip_rows must be in [1, 65536], -1 (auto) or -ns (ns >= 2 strips)");
        if (strip_rows == -1) strip_rows = 0;
        if (d->connected && strip_rows > 0 && strip_rows < kHalo)
            return fail(BML_EINVAL, "connected bands need strip_rows >= 16");
        d->strip_rows = strip_rows;
    }
    return BML_OK;
}

int bml_dev_set_resident(bml_dev* d, int mode) {
    if (int rc = check(d)) return rc;
    if (mode < 0 || mode > 2) return fail(BML_EINVAL, "bml_dev_set_resident: mode must be 0, 1 or 2");
    d->resident = mode;
    return BML_OK;
}

int bml_dev_path(bml_dev* d, int* resident_cluster) {
    if (!d) return fail(BML_EINVAL, "null bml_dev handle");
    if (resident_cluster) *resident_cluster = d->resident_cluster;
    return BML_OK;
}

int bml_dev_last_launch(bml_dev* d, int* nstrips, int* items, int* grid) {
    if (!d) return fail(BML_EINVAL, "null bml_dev handle");
    if (nstrips) *nstrips = d->last_nstrips;
    if (items) *items = d->last_items;
    if (grid) *grid = d->last_grid;
    return BML_OK;
}

int bml_dev_info(bml_dev* d, int* n, int* row_begin, int* row_end, int* block_steps,
                 int* strip_rows, size_t* device_bytes) {
    if (!d) return fail(BML_EINVAL, "null bml_dev handle");
    if (n) *n = d->n;
    if (row_begin) *row_begin = d->row_begin;
    if (row_end) *row_end = d->row_end;
    if (block_steps) *block_steps = d->block_steps;
    if (strip_rows) *strip_rows = d->strip_rows;
    if (device_bytes)
        *device_bytes = 2 * static_cast<size_t>(d->rows + 2 * kHalo) * d->pitch * sizeof(uint2) +
                        static_cast<size_t>(d->rows) * d->n;
    return BML_OK;
}

int bml_dev_enable_timing(bml_dev* d, int enable) {
    if (int rc = check(d)) return rc;
    d->timing = enable != 0;
    return BML_OK;
}

int bml_dev_kernel_stats(bml_dev* d, int64_t* launches, double* kernel_ms, int reset) {
    if (int rc = check(d)) return rc;
    BML_CUDA(cudaStreamSynchronize(d->stream));
    harvest_timing(d);
    if (launches) *launches = d->launches;
    if (kernel_ms) *kernel_ms = d->kernel_ms;
    if (reset) {
        d->launches = 0;
        d->kernel_ms = 0.0;
    }
    return BML_OK;
}

int bml_dev_upload(bml_dev* d, const uint8_t* src, size_t src_pitch) {
    if (int rc = check(d)) return rc;
    if (!src) return fail(BML_EINVAL, "bml_dev_upload: src is null");
    if (src_pitch < static_cast<size_t>(d->n))
        return fail(BML_EINVAL, "bml_dev_upload: pitch smaller than a row");
    BML_CUDA(cudaMemsetAsync(d->err, 0, 4 * sizeof(int), d->stream));
    BML_CUDA(cudaMemcpy2DAsync(d->staging, d->n, src, src_pitch, d->n, d->rows,
                               cudaMemcpyDefault, d->stream));
    const long long total = static_cast<long long>(d->rows) * d->W;
    pack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, d->stream>>>(
        d->staging, d->n, d->row0(d->cur), d->n, d->W, d->pitch, d->rows, d->err);
    BML_CUDA(cudaGetLastError());
    if (d->single_band()) {
        if (int rc = fill_images(d, d->cur)) return rc;
    }
    int bad = 0;
    BML_CUDA(cudaMemcpyAsync(&bad, d->err, sizeof(int), cudaMemcpyDeviceToHost, d->stream));
    BML_CUDA(cudaStreamSynchronize(d->stream));
    if (bad) return fail(BML_EINVAL, "bml_dev_upload: cell value outside {0,1,2}");
    return BML_OK;
}

int bml_dev_download(bml_dev* d, uint8_t* dst, size_t dst_pitch) {
    if (int rc = check(d)) return rc;
    if (!dst) return fail(BML_EINVAL, "bml_dev_download: dst is null");
    if (dst_pitch < static_cast<size_t>(d->n))
        return fail(BML_EINVAL, "bml_dev_download: pitch smaller than a row");
    const long long total = static_cast<long long>(d->rows) * d->W;
    unpack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, d->stream>>>(
        d->row0(d->cur), d->staging, d->n, d->n, d->W, d->pitch, d->rows);
    BML_CUDA(cudaGetLastError());
    BML_CUDA(cudaMemcpy2DAsync(dst, dst_pitch, d->staging, d->n, d->n, d->rows,
                               cudaMemcpyDefault, d->stream));
    BML_CUDA(cudaStreamSynchronize(d->stream));
    return check_errors(d);
}

int bml_dev_init_random_masked(bml_dev* d, double rho, uint64_t seed, uint64_t reject_mask) {
    if (int rc = check(d)) return rc;
    if (!(rho >= 0.0 && rho <= 1.0))
        return fail(BML_EINVAL, "init_grid: density must be in [0, 1]");
    if (static_cast<unsigned long long>(d->n) * d->n > (1ull << 32))
        return fail(BML_EINVAL, "bml_dev_init_random: device init supports n <= 65536");
    std::string msg;
    const int rc = bml_init::init_planes(d->row0(d->cur), d->pitch, d->n, d->row_begin,
                                         d->row_end, rho, seed, reject_mask, d->stream, d->sms,
                                         &msg);
    if (rc == 3) return fail(BML_ENOMEM, "bml_dev_init_random: " + msg);
    if (rc != 0) return fail(BML_ECUDA, "bml_dev_init_random: " + msg);
    if (d->single_band()) {
        if (int r2 = fill_images(d, d->cur)) return r2;
    }
    BML_CUDA(cudaStreamSynchronize(d->stream));
    return BML_OK;
}

int bml_dev_init_random(bml_dev* d, double rho, uint64_t seed) {
    return bml_dev_init_random_masked(d, rho, seed, 0);
}

int bml_dev_encode_ppm(bml_dev* d, uint8_t* dst, size_t dst_pitch) {
    if (int rc = check(d)) return rc;
    if (!dst) return fail(BML_EINVAL, "bml_dev_encode_ppm: dst is null");
    const size_t row_bytes = 3 * static_cast<size_t>(d->n);
    if (dst_pitch < row_bytes) return fail(BML_EINVAL, "bml_dev_encode_ppm: pitch smaller than a row");
    uint8_t* rgb = nullptr;
    BML_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rgb), row_bytes * d->rows, d->stream));
    const long long total = static_cast<long long>(d->rows) * d->W;
    ppm_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, d->stream>>>(
        d->row0(d->cur), rgb, static_cast<long long>(row_bytes), d->n, d->W, d->pitch, d->rows);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(dst, dst_pitch, rgb, row_bytes, row_bytes, d->rows, cudaMemcpyDefault,
                              d->stream);
    cudaFreeAsync(rgb, d->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(d->stream);
    if (e != cudaSuccess) return cuda_fail(e, "bml_dev_encode_ppm");
    return BML_OK;
}

int bml_dev_digest_segment(bml_dev* d, uint64_t seg[6]) {
    if (int rc = check(d)) return rc;
    if (!seg) return fail(BML_EINVAL, "bml_dev_digest_segment: seg is null");
    std::string msg;
    const int rc = bml_digest::segment(d->row0(d->cur), d->n, d->W, d->pitch, d->rows, d->stream,
                                       d->sms, seg, &msg);
    if (rc == 3) return fail(BML_ENOMEM, msg);
    if (rc != 0) return fail(BML_ECUDA, msg);
    return BML_OK;
}

int bml_dev_digest(bml_dev* d, uint64_t* digest) {
    if (int rc = check(d)) return rc;
    if (!digest) return fail(BML_EINVAL, "bml_dev_digest: digest is null");
    if (!d->single_band())
        return fail(BML_EINVAL, "bml_dev_digest: a row band hashes only its rows; combine "
                                "bml_dev_digest_segment() of all bands with bml_digest_finish()");
    uint64_t seg[6];
    if (int rc = bml_dev_digest_segment(d, seg)) return rc;
    *digest = bml_digest::finish(seg, 1);
    return BML_OK;
}

int bml_digest_finish(const uint64_t* segs, int count, uint64_t* digest) {
    if (!digest || count < 0 || (count > 0 && !segs))
        return fail(BML_EINVAL, "bml_digest_finish: bad arguments");
    *digest = bml_digest::finish(segs, count);
    return BML_OK;
}

int bml_dev_counts(bml_dev* d, int64_t* lr, int64_t* tb) {
    if (int rc = check(d)) return rc;
    BML_CUDA(cudaMemsetAsync(d->scratch, 0, 2 * sizeof(unsigned long long), d->stream));
    counts_kernel<<<d->sms * 4, 256, 0, d->stream>>>(d->row0(d->cur), d->W, d->pitch, d->rows,
                                                     d->scratch);
    BML_CUDA(cudaGetLastError());
    unsigned long long h[2];
    BML_CUDA(cudaMemcpyAsync(h, d->scratch, sizeof h, cudaMemcpyDeviceToHost, d->stream));
    BML_CUDA(cudaStreamSynchronize(d->stream));
    if (lr) *lr = static_cast<int64_t>(h[0]);
    if (tb) *tb = static_cast<int64_t>(h[1]);
    return BML_OK;
}

int bml_dev_phase(bml_dev* d, int phase, int64_t* moved) {
    if (int rc = check(d)) return rc;
    if (phase != BML_PHASE_HORIZONTAL && phase != BML_PHASE_VERTICAL)
        return fail(BML_EINVAL, "bml_dev_phase: phase must be 0 (horizontal) or 1 (vertical)");
    if (!d->single_band())
        return fail(BML_EINVAL, "bml_dev_phase: single phases need a single-band handle");
    BML_CUDA(cudaMemsetAsync(d->scratch, 0, sizeof(unsigned long long), d->stream));
    PhaseArgs a{};
    a.src = d->row0(d->cur);
    a.dst = d->row0(d->cur ^ 1);
    a.n = d->n;
    a.W = d->W;
    a.pitch = d->pitch;
    a.rows = d->rows;
    a.last_mask = d->last_mask;
    a.moved = d->scratch;
    const long long total = static_cast<long long>(d->rows) * d->W;
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    if (phase == BML_PHASE_HORIZONTAL)
        phase_h_kernel<<<grid, 256, 0, d->stream>>>(a);
    else
        phase_v_kernel<<<grid, 256, 0, d->stream>>>(a);
    BML_CUDA(cudaGetLastError());
    d->cur ^= 1;
    if (moved) {
        unsigned long long h = 0;
        BML_CUDA(cudaMemcpyAsync(&h, d->scratch, sizeof h, cudaMemcpyDeviceToHost, d->stream));
        BML_CUDA(cudaStreamSynchronize(d->stream));
        *moved = static_cast<int64_t>(h);
    }
    return BML_OK;
}

int bml_dev_step(bml_dev* d, int64_t steps, int64_t* lr_moved, int64_t* tb_moved,
                 int64_t* lr_count, int64_t* tb_count) {
    if (int rc = check(d)) return rc;
    if (steps < 0) return fail(BML_EINVAL, "bml_dev_step: steps must be >= 0");
    if (steps == 0) return BML_OK;
    const bool count = lr_moved || tb_moved || lr_count || tb_count;
    if (count && steps > (1LL << 26))
        return fail(BML_EINVAL, "bml_dev_step: at most 2^26 steps per call with metrics");
    int64_t lr0 = 0, tb0 = 0;
    const bool check_conservation = (lr_count || tb_count) && d->single_band();
    if (check_conservation) {
        if (int rc = bml_dev_counts(d, &lr0, &tb0)) return rc;
    }
    if (count) {
        if (int rc = ensure_metrics(d, steps)) return rc;
        BML_CUDA(cudaMemsetAsync(d->metrics, 0, 4 * steps * sizeof(unsigned long long), d->stream));
    }
    d->resident_cluster = 0;
    bool resident_used = false;
    if (int rc = launch_resident(d, steps, count, &resident_used)) return rc;
    long long done = resident_used ? steps : 0;
    while (done < steps) {
        const int k = largest_block_at_most(steps - done, d->block_steps);
        if (int rc = launch_block(d, k, count, static_cast<int>(done), static_cast<int>(steps)))
            return rc;
        done += k;
    }
    if (count) {
        std::vector<unsigned long long> h(static_cast<size_t>(4 * steps));
        BML_CUDA(cudaMemcpyAsync(h.data(), d->metrics, h.size() * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, d->stream));
        BML_CUDA(cudaStreamSynchronize(d->stream));
        for (int64_t s = 0; s < steps; ++s) {
            if (lr_moved) lr_moved[s] = static_cast<int64_t>(h[s]);
            if (tb_moved) tb_moved[s] = static_cast<int64_t>(h[steps + s]);
            if (lr_count) lr_count[s] = static_cast<int64_t>(h[2 * steps + s]);
            if (tb_count) tb_count[s] = static_cast<int64_t>(h[3 * steps + s]);
        }
        if (check_conservation) {
            for (int64_t s = 0; s < steps; ++s) {
                if (static_cast<int64_t>(h[2 * steps + s]) != lr0 ||
                    static_cast<int64_t>(h[3 * steps + s]) != tb0) {
                    return fail(BML_ECONSERVE,
                                "conservation violated at step " + std::to_string(s + 1) +
                                    ": lr " + std::to_string(h[2 * steps + s]) + "/" +
                                    std::to_string(lr0) + ", tb " +
                                    std::to_string(h[3 * steps + s]) + "/" + std::to_string(tb0));
                }
            }
        }
        return check_errors(d);
    }
    return BML_OK;
}

// ---------------------------------------------------------------- multi-band
int bml_dev_export(bml_dev* d, void* blob, size_t* size) {
    if (int rc = check(d)) return rc;
    if (!blob || !size || *size < sizeof(IpcBlob))
        return fail(BML_EINVAL, "bml_dev_export: blob buffer too small");
    IpcBlob b{};
    b.magic = kBlobMagic;
    b.n = d->n;
    b.row_begin = d->row_begin;
    b.row_end = d->row_end;
    b.pitch = d->pitch;
    b.W = d->W;
    b.device = d->device;
    for (int p = 0; p < 2; ++p) BML_CUDA(cudaIpcGetMemHandle(&b.buf[p], d->buf[p]));
    BML_CUDA(cudaIpcGetMemHandle(&b.flags, d->flags));
    std::memcpy(blob, &b, sizeof b);
    *size = sizeof b;
    return BML_OK;
}

namespace {

int link_peer(bml_dev* d, uint2* const peer_buf[2], unsigned long long* peer_flags, int peer_rows,
              bool is_up) {
    for (int p = 0; p < 2; ++p) {
        uint2* peer_row0 = peer_buf[p] + static_cast<long long>(kHalo) * d->pitch;
        if (is_up)
            d->up_halo[p] = peer_row0 + static_cast<long long>(peer_rows) * d->pitch;  // its bottom ghosts
        else
            d->down_halo[p] = peer_row0;  // row (r - rows) in [-kHalo, 0): its top ghosts
    }
    if (is_up)
        d->up_flag = peer_flags + 1;  // the neighbour above waits on its bottom flag
    else
        d->down_flag = peer_flags;  // the neighbour below waits on its top flag
    return BML_OK;
}

int validate_neighbours(bml_dev* d, int up_end, int up_n, int up_pitch, int dn_begin, int dn_n,
                        int dn_pitch) {
    if (up_n != d->n || dn_n != d->n || up_pitch != d->pitch || dn_pitch != d->pitch)
        return fail(BML_EINVAL, "bml_dev_connect: neighbour lattice geometry differs");
    if (up_end % d->n != d->row_begin)
        return fail(BML_EINVAL, "bml_dev_connect: up neighbour does not end where this band begins");
    if (dn_begin != d->row_end % d->n)
        return fail(BML_EINVAL, "bml_dev_connect: down neighbour does not begin where this band ends");
    if (d->strip_rows > 0 && d->strip_rows < kHalo) d->strip_rows = kHalo;
    return BML_OK;
}

}  // namespace

int bml_dev_connect(bml_dev* d, const void* up_blob, const void* down_blob) {
    if (int rc = check(d)) return rc;
    if (!up_blob || !down_blob) return fail(BML_EINVAL, "bml_dev_connect: null blob");
    IpcBlob up, dn;
    std::memcpy(&up, up_blob, sizeof up);
    std::memcpy(&dn, down_blob, sizeof dn);
    if (up.magic != kBlobMagic || dn.magic != kBlobMagic)
        return fail(BML_EINVAL, "bml_dev_connect: not a bml_dev export blob");
    if (int rc = validate_neighbours(d, up.row_end, up.n, up.pitch, dn.row_begin, dn.n, dn.pitch))
        return rc;
    const bool same = std::memcmp(&up.buf[0], &dn.buf[0], sizeof(cudaIpcMemHandle_t)) == 0;
    auto open = [&](const cudaIpcMemHandle_t& h, void** p) -> int {
        cudaError_t e = cudaIpcOpenMemHandle(p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
        d->ipc_opened.push_back(*p);
        return BML_OK;
    };
    void *ub[2], *uf, *db[2], *df;
    for (int p = 0; p < 2; ++p)
        if (int rc = open(up.buf[p], &ub[p])) return rc;
    if (int rc = open(up.flags, &uf)) return rc;
    if (same) {
        db[0] = ub[0];
        db[1] = ub[1];
        df = uf;
    } else {
        for (int p = 0; p < 2; ++p)
            if (int rc = open(dn.buf[p], &db[p])) return rc;
        if (int rc = open(dn.flags, &df)) return rc;
    }
    uint2* ubp[2] = {static_cast<uint2*>(ub[0]), static_cast<uint2*>(ub[1])};
    uint2* dbp[2] = {static_cast<uint2*>(db[0]), static_cast<uint2*>(db[1])};
    link_peer(d, ubp, static_cast<unsigned long long*>(uf), up.row_end - up.row_begin, true);
    link_peer(d, dbp, static_cast<unsigned long long*>(df), dn.row_end - dn.row_begin, false);
    d->connected = true;
    std::fill(std::begin(d->ns_cache_k), std::end(d->ns_cache_k), 0);  // strip limits changed
    return BML_OK;
}

int bml_dev_connect_local(bml_dev* d, bml_dev* up, bml_dev* down) {
    if (int rc = check(d)) return rc;
    if (!up || !down) return fail(BML_EINVAL, "bml_dev_connect_local: null neighbour");
    if (int rc = validate_neighbours(d, up->row_end, up->n, up->pitch, down->row_begin, down->n,
                                     down->pitch))
        return rc;
    for (bml_dev* peer : {up, down}) {
        if (peer->device != d->device) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, d->device, peer->device);
            if (!can) return fail(BML_ECUDA, "bml_dev_connect_local: no peer access between devices");
            cudaError_t e = cudaDeviceEnablePeerAccess(peer->device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return cuda_fail(e, "cudaDeviceEnablePeerAccess");
            (void)cudaGetLastError();
        }
    }
    link_peer(d, up->buf, up->flags, up->rows, true);
    link_peer(d, down->buf, down->flags, down->rows, false);
    d->connected = true;
    std::fill(std::begin(d->ns_cache_k), std::end(d->ns_cache_k), 0);  // strip limits changed
    return BML_OK;
}

int bml_dev_exchange_halos(bml_dev* d) {
    if (int rc = check(d)) return rc;
    if (!d->connected) return fill_images(d, d->cur);
    push_halo_kernel<<<1, 1024, 0, d->stream>>>(d->row0(d->cur), d->W, d->pitch, d->rows,
                                                d->up_halo[d->cur], d->down_halo[d->cur],
                                                d->up_flag, d->down_flag, d->ncols());
    BML_CUDA(cudaGetLastError());
    ++d->pubs;
    return BML_OK;
}

}  // extern "C"
