// paper_1804_07981_b200/csrc/bml_step_kernel.cuh — the temporally blocked streaming step kernel (step_block_kernel).
// Part of libbml_dev.so: included once, by bml_dev.cu (see its header comment).
#pragma once

#include "bml_kernels_common.cuh"

namespace bml_k {

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
// Stage K-1 therefore emits row j-2K+1 at time K.
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
    // kSeam: this lane's window = funnel_r(lo, hi, sh) with lo = own word <<
    // pre (or the left lane's word), hi = the right lane's word (or own word)
    int seam_pre, seam_sh;
    bool seam_left;
    unsigned span;  // rows this lane stores (r_hi - r_lo, or 0 for ghost lanes)
    uint2* outp;    // aligned modes: this lane's word of the row emitted next
};

// Final-stage output of row o (rows outside the strip, and ghost lanes, are
// not stored).
//  - Aligned modes: valid is 0 (ghost lane, span 0) or all ones, so no
//    masking; one predicated store through a running row pointer. The ghost
//    images of the band's first/last kHalo rows are written after the strip
//    (copy_images). st.global.cg / inline st.global measured 2-4% slower.
//  - Generic mode (n % 32 != 0): masked words, and each row's images (tiny n
//    can have several per side) are stored here.
template <int MODE>
__device__ __forceinline__ void store_row(const StepArgs& a, StripCtx& c, int o, uint32_t l,
                                          uint32_t t) {
    const bool st = static_cast<unsigned>(o - c.r_lo) < c.span;
    if (MODE != kGeneric) {
        if (MODE == kSeam) {  // the last word is partial: keep its padding bits zero
            if (st) *c.outp = make_uint2(l & c.valid, t & c.valid);
        } else {
            if (st) *c.outp = make_uint2(l, t);
        }
        c.outp += a.pitch;
        return;
    }
    if (!st) return;
    const uint2 v = make_uint2(l & c.valid, t & c.valid);
    const long long off = static_cast<long long>(o) * a.pitch + c.out_word;
    a.dst[off] = v;
    if (a.single_band) {
        for (int h = o - a.n; h >= -kHalo; h -= a.n) a.dst[static_cast<long long>(h) * a.pitch + c.out_word] = v;
        for (int h = o + a.n; h < a.rows + kHalo; h += a.n)
            a.dst[static_cast<long long>(h) * a.pitch + c.out_word] = v;
    } else {
        if (o < kHalo) a.up_halo[off] = v;
        if (o >= a.rows - kHalo) a.down_halo[off - static_cast<long long>(a.rows) * a.pitch] = v;
    }
}

// kSeam: rebuild this lane's 32-cell window across the torus seam from its own
// aligned row word and its neighbours' (see StripCtx).
__device__ __forceinline__ uint32_t seam_window(uint32_t v, const StripCtx& c) {
    const uint32_t right = __shfl_down_sync(kFull, v, 1);
    const uint32_t left = __shfl_up_sync(kFull, v, 1);
    const uint32_t lo = c.seam_left ? left : (v << c.seam_pre);
    const uint32_t hi = c.seam_left ? v : right;
    return __funnelshift_r(lo, hi, c.seam_sh);
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

// Stages [S0, S1) of one pipeline iteration (the whole pipeline by default;
// step_split_kernel runs the two halves in two warps). Stage S0 > 0 reads the
// stage-(S0-1) state slots, which the caller fills.
template <int K, int MODE, int COUNT, int P, int S0 = 0, int S1 = K>
__device__ __forceinline__ void pipe_iter(PipeState<K>& q, const uint2 x, const int j,
                                          const StepArgs& a, StripCtx& c) {
    constexpr int P3 = P % 3, P2 = P % 2;
    if (S0 == 0) q.xt[P3] = x.y;
#pragma unroll
    for (int s = S1 - 1; s >= S0; --s) {
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
                // vehicle census of the emitted row after every step (COUNT 2: row
                // bands, whose counts change as TB vehicles cross band edges, and the
                // strict single-band mode); COUNT 1 takes it at the store below
                if (COUNT == 2)
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
            if (COUNT == 1) {  // census after the launch's last step: the stored row
                // (aligned modes store whole words: span is 0 for ghost lanes, so the
                // stored-row test alone selects the counted cells; branch-free select)
                const bool st = static_cast<unsigned>(j - 2 * K + 1 - c.r_lo) < c.span;
                const uint32_t cl = MODE == kAligned || MODE == kFullRow ? newL : (newL & c.valid);
                const uint32_t ct = MODE == kAligned || MODE == kFullRow ? newT : (newT & c.valid);
                const uint32_t add = __popc(cl) + (static_cast<uint32_t>(__popc(ct)) << 16);
                q.cc[K - 1] += st ? add : 0u;
            }
        }
    }
}

// MAXT: launch bound. The default instantiation fits 3 warps per SMSP in the
// register file (<= 168 registers); the 256-thread one (at most two warps per
// SMSP, the latency-bound regime of mid-size lattices) may use up to 255
// registers, and ptxas schedules it with fewer moves (+4% at N=8192).
// COUNT: 0 no metrics; 1 moved counts per step + the vehicle census after the
// launch's last step; 2 moved counts + the census after every step (row bands,
// strict single-band mode; see bml_dev_step)
template <int K, int MODE, int COUNT, int MAXT = kMaxWarpsPerCta * 32>
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
        const int order = item / a.ncols;
        const int col = item - order * a.ncols;
        // connected bands run boundary-first: the band's top and bottom strips are
        // items of the first round, so both neighbours' ghost rows are published
        // early and the interior strips overlap their wait (order 0 -> strip 0,
        // order 1 -> the last strip, order k -> strip k-1)
        const int strip = (a.single_band || a.nstrips < 2 || order == 0)
                              ? order
                              : (order == 1 ? a.nstrips - 1 : order - 1);
        StripCtx c;
        c.lane = lane;
        // rows split evenly: strip i owns [i*rows/nstrips, (i+1)*rows/nstrips)
        c.r_lo = static_cast<int>(static_cast<long long>(strip) * a.rows / a.nstrips);
        c.r_hi = static_cast<int>(static_cast<long long>(strip + 1) * a.rows / a.nstrips);

        int word = lane, c0 = 0;
        c.out_word = lane;
        c.valid = kFull;
        c.seam_pre = c.seam_sh = 0;
        c.seam_left = false;
        if (MODE != kFullRow) {
            constexpr int kOut = MODE == kSeam ? kSeamOutWords : kOutWords;
            constexpr int kLead = MODE == kSeam ? 2 : 1;  // ghost words on each side
            const int w = col * kOut + lane - kLead;
            const bool is_out = lane >= kLead && lane < kLead + kOut && w < a.W;
            c.out_word = w;
            c.valid = is_out ? (w == a.W - 1 ? a.last_mask : kFull) : 0u;
            word = ((w % a.W) + a.W) % a.W;
            if (MODE == kGeneric) {
                long long cc = (32LL * w) % a.n;
                if (cc < 0) cc += a.n;
                c0 = static_cast<int>(cc);
            }
            if (MODE == kSeam) {
                // window of cells [32w, 32w + 32) mod n from the aligned row words;
                // nb = cells in the last (partial) word. W >= 32, so a warp wraps once.
                const int nb = a.n - 32 * (a.W - 1);
                if (w == a.W - 1) {  // last word, then the row's first cells
                    c.seam_pre = 32 - nb;
                    c.seam_sh = 32 - nb;
                } else if (w >= a.W) {  // past the end: word w-W shifted by 32-nb
                    c.seam_sh = 32 - nb;
                } else if (w == -1) {  // before the start: the row's last 32 cells
                    c.seam_left = true;
                    c.seam_sh = nb;
                }
            }
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
                if (MODE == kSeam) x = make_uint2(seam_window(x.x, c), seam_window(x.y, c));
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
                const bool census = COUNT == 2 || s == K - 1;
                const unsigned v2 = census ? __reduce_add_sync(kFull, q.cc[s] & 0xffffu) : 0u;
                const unsigned v3 = census ? __reduce_add_sync(kFull, q.cc[s] >> 16) : 0u;
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


}  // namespace bml_k
