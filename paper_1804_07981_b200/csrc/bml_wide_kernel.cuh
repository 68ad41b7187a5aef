// paper_1804_07981_b200/csrc/bml_wide_kernel.cuh — the wide-lane streaming step kernel
// (step_wide_kernel). Part of libbml_dev.so: included once, by bml_dev.cu.
#pragma once

#include "bml_kernels_common.cuh"

namespace bml_k {

// ------------------------------------------------------- wide-lane temporally blocked step
//
// Same temporal pipeline as step_block_kernel (K full steps per launch, stage
// s of iteration j works on row j - 2s; see bml_step_kernel.cuh), but every
// lane carries 64 cells: two consecutive row words. Per 32 cells and step that
// halves the warp shuffles (1 instead of 2: the LR phase needs one word from
// each neighbouring lane, not one per 32 cells) and the per-row load / store /
// ring bookkeeping, which ncu showed queueing with the shuffles in the LSU/MIO
// pipe (60% busy next to an 80%-busy ALU pipe at configs[4]); the ALU work per
// cell is unchanged (4 LOP3 + 2 funnel shifts per 32 cells per step).
//
// Geometry (n % 64 == 0, W >= 64): column `col` is the 64-word window starting
// at word a = 62*col - 2 (even, taken mod W: a 16-byte-aligned pair per lane).
// The first and last word of the window are ghosts (their stale edge grows one
// cell per step, K <= 16 < 32); the 62 words in between are outputs, so the
// windows' outputs tile the row from word W-1 (column 0's first output) onward;
// outputs past word W-2 repeat column 0's and are not stored.
//
// Rows reach shared memory by TMA bulk copies (cp.async.bulk, one elected lane,
// 512 B per row per warp in at most two pieces across the torus seam) into a
// per-warp ring of kWideRing slots, each completed on its own mbarrier; the
// lanes wait on the slot's barrier and read their 16-byte pair with one LDS.
constexpr int kWideOut = 62;   // output words per warp window
constexpr int kEoOut = 60;     // even/odd layout: output words per window (lanes 1..30)
constexpr int kWideRing = 6;   // == the loop unroll factor (slot index compile-time)
constexpr int kWideSlotWords = 64;

__device__ __forceinline__ void wide_mbar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
// One elected lane arms the slot's barrier for 512 bytes and issues the row's
// one or two bulk copies. Predicated inside the asm: no branch in the loop body,
// so ptxas keeps the warp provably converged for the shuffles around it.
__device__ __forceinline__ void wide_issue_row(bool leader, uint32_t bar, uint32_t dst, const void* src1,
                                               uint32_t bytes1, const void* src2, uint32_t bytes2) {
    asm volatile(
        "{\n .reg .pred p, q;\n"
        " setp.ne.u32 p, %0, 0;\n"
        " setp.ne.and.u32 q, %6, 0, p;\n"
        " @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], 512;\n"
        " @p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %4, [%1];\n"
        " @q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%5], [%7], %6, [%1];\n"
        "}" ::"r"(static_cast<uint32_t>(leader)),
        "r"(bar), "r"(dst), "l"(src1), "r"(bytes1), "r"(dst + bytes1), "r"(bytes2), "l"(src2)
        : "memory");
}
// All lanes spin on the slot's barrier inside one asm block (a single
// straight-line statement for the compiler; the loop is PTX-local).
__device__ __forceinline__ void wide_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred done;\n"
        " WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
        " @!done bra WAIT_%=;\n"
        "}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

template <int K>
struct WideState {
    uint32_t nt[K][3][2];
    uint32_t lp[K][2][2];
    uint32_t oc[K][2];
    uint32_t xt[3][2];
    uint32_t cm[K], cc[K];  // packed 16-bit counters (COUNT only)
};

struct WideCtx {
    int lane, r_lo, r_hi;
    uint32_t v0, v1;      // output masks of the lane's two words (0 or all ones)
    int kind;             // stored words: 0 none, 1 low, 2 high, 3 both
    unsigned span;        // rows stored (r_hi - r_lo, or 0)
    uint2* outp;          // this lane's pair in the row emitted next
};

// Final-stage output: one predicated 16-byte store for a full pair, one 8-byte
// store for a half pair (the lanes next to the ghost words). The even/odd layout
// only has whole pairs: the 8-byte forms (and the register moves that build
// their aligned operand pairs) are left out.
// OFF >= 0 (even/odd layout, compile-time pitch): the row is c.outp + OFF bytes,
// an immediate offset; the caller advances c.outp once per unrolled loop.
template <bool EO, int OFF = -1>
__device__ __forceinline__ void wide_store(const StepArgs& a, WideCtx& c, int o, const uint32_t l[2],
                                           const uint32_t t[2], int pitch) {
    const bool st = static_cast<unsigned>(o - c.r_lo) < c.span;
    if (EO && OFF >= 0) {
        asm volatile(
            "{\n .reg .pred pf;\n"
            " setp.ne.u32 pf, %0, 0;\n"
            " @pf st.global.v4.u32 [%1+%6], {%2, %3, %4, %5};\n"
            "}" ::"r"(static_cast<uint32_t>(st)),
            "l"(c.outp), "r"(l[0]), "r"(t[0]), "r"(l[1]), "r"(t[1]), "n"(OFF)
            : "memory");
        return;
    }
    if (EO) {
        asm volatile(
            "{\n .reg .pred pf;\n"
            " setp.ne.u32 pf, %0, 0;\n"
            " @pf st.global.v4.u32 [%1], {%2, %3, %4, %5};\n"
            "}" ::"r"(static_cast<uint32_t>(st)),
            "l"(c.outp), "r"(l[0]), "r"(t[0]), "r"(l[1]), "r"(t[1])
            : "memory");
        c.outp += pitch;
        return;
    }
    const uint32_t full = st && c.kind == 3, lo = st && c.kind == 1, hi = st && c.kind == 2;
    asm volatile(
        "{\n .reg .pred pf, pl, ph;\n"
        " setp.ne.u32 pf, %0, 0;\n"
        " setp.ne.u32 pl, %1, 0;\n"
        " setp.ne.u32 ph, %2, 0;\n"
        " @pf st.global.v4.u32 [%3], {%4, %5, %6, %7};\n"
        " @pl st.global.v2.u32 [%3], {%4, %5};\n"
        " @ph st.global.v2.u32 [%3+8], {%6, %7};\n"
        "}" ::"r"(full),
        "r"(lo), "r"(hi), "l"(c.outp), "r"(l[0]), "r"(t[0]), "r"(l[1]), "r"(t[1])
        : "memory");
    c.outp += pitch;
}

// EO (even/odd layout, see eo_convert_kernel): a lane's two words are the EVEN
// and the ODD cells of its 64-cell group (bit b of word 0 is cell 64g + 2b, of
// word 1 cell 64g + 2b + 1). An odd cell's left neighbour and an even cell's
// right neighbour are then the same bit of the lane's other word, so the LR
// phase needs 2 funnel shifts per 64 cells instead of 4 (5 ALU-pipe
// instructions per 32 cells and step instead of 6):
//   even cell 2b:   left 2b-1 = odd bit b-1 (bit 31 of the left lane's odd word for b = 0),
//                   right 2b+1 = odd bit b
//   odd cell 2b+1:  left 2b = even bit b,
//                   right 2b+2 = even bit b+1 (bit 0 of the right lane's even word for b = 31)
// TBD: the first TBD words of the pair run the TB phase in departures form,
// D = T & ~Op(below), newT = T - D + D(above) (1 LOP3 + 2 IMAD instead of 2 LOP3:
// moves ALU-pipe work to the FMA pipe); their oc slot carries D(above).
// DL (bit h): word h (if not TBD) carries the departures too but combines them
// with LOP3s, newT = (T & Op(below)) | D(above): the same 2 LOP3 as the plain
// form, without the T(i-1) register (tA) per stage.
template <int K, int COUNT, int P, bool EO = false, int TBD = 0, int PITCH = 0, int DL = 0>
__device__ __forceinline__ void wide_iter(WideState<K>& q, const uint4 x, const int j, const StepArgs& a,
                                          WideCtx& c) {
    constexpr int P3 = P % 3, P2 = P % 2;
    q.xt[P3][0] = x.y;
    q.xt[P3][1] = x.w;
#pragma unroll
    for (int s = K - 1; s >= 0; --s) {
        const int sp = s > 0 ? s - 1 : 0;
        uint32_t L[2], T[2], tB[2], tA[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            L[h] = (s == 0) ? (h ? x.z : x.x) : q.lp[sp][P2][h];
            T[h] = (s == 0) ? (h ? x.w : x.y) : q.nt[sp][(P3 + 2) % 3][h];
            tB[h] = (s == 0) ? q.xt[(P3 + 2) % 3][h] : q.nt[sp][(P3 + 1) % 3][h];
            tA[h] = (s == 0) ? q.xt[(P3 + 1) % 3][h] : q.nt[sp][P3][h];
        }
        // ---- LR phase on row j - 2s (cells: bit b of word w is cell 32w + b)
        const uint32_t O0 = BML_IMAD_OR ? imad(L[0], a.one, T[0]) : (L[0] | T[0]);
        const uint32_t O1 = BML_IMAD_OR ? imad(L[1], a.one, T[1]) : (L[1] | T[1]);
        const uint32_t Ll = __shfl_up_sync(kFull, L[1], 1);    // left lane's high (odd) word
        const uint32_t Or = __shfl_down_sync(kFull, O0, 1);    // right lane's low (even) word
        const uint32_t prevL0 = __funnelshift_l(Ll, EO ? L[1] : L[0], 1);
        const uint32_t prevL1 = EO ? L[0] : __funnelshift_l(L[0], L[1], 1);
        const uint32_t nextO0 = EO ? O1 : __funnelshift_r(O0, O1, 1);
        const uint32_t nextO1 = __funnelshift_r(EO ? O0 : O1, Or, 1);
        uint32_t Lp[2], Op[2], newT[2], D[2];
        Lp[0] = (prevL0 & ~O0) | (L[0] & nextO0);
        Lp[1] = (prevL1 & ~O1) | (L[1] & nextO1);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            Op[h] = BML_IMAD_OR ? imad(Lp[h], a.one, T[h]) : (Lp[h] | T[h]);
            // ---- TB phase emits row j - 2s - 1
            if (h < TBD) {
                D[h] = tB[h] & ~Op[h];
                newT[h] = imad(q.oc[s][h], a.one, imad(D[h], 0u - a.one, tB[h]));
            } else if (DL & (1 << h)) {  // departures carried, plain LOP3s: no T(i-1) slot
                D[h] = tB[h] & ~Op[h];
                newT[h] = (tB[h] & Op[h]) | q.oc[s][h];
            } else {
                newT[h] = (tA[h] & ~q.oc[s][h]) | (tB[h] & Op[h]);
            }
        }
        if (COUNT) {
            const int rho = j - 2 * s;
            const unsigned span = static_cast<unsigned>(c.r_hi - c.r_lo);
            if (static_cast<unsigned>(rho - c.r_lo) < span)
                q.cm[s] += __popc(L[0] & ~nextO0 & c.v0) + __popc(L[1] & ~nextO1 & c.v1);
            if (static_cast<unsigned>(rho - 1 - c.r_lo) < span) {
                q.cm[s] += static_cast<uint32_t>(__popc(tB[0] & ~Op[0] & c.v0) + __popc(tB[1] & ~Op[1] & c.v1))
                           << 16;
                if (COUNT == 2) {
                    const uint32_t* nl = q.lp[s][(P2 + 1) % 2];
                    q.cc[s] += __popc(nl[0] & c.v0) + __popc(nl[1] & c.v1) +
                               (static_cast<uint32_t>(__popc(newT[0] & c.v0) + __popc(newT[1] & c.v1)) << 16);
                }
            }
        }
        if (s == K - 1) {
            const uint32_t* nl = q.lp[s][(P2 + 1) % 2];
            wide_store<EO, (EO && PITCH) ? P * PITCH * 8 : -1>(a, c, j - 2 * K + 1, nl, newT, PITCH ? PITCH : a.pitch);
            if (COUNT == 1) {  // census after the launch's last step: the stored row (branch-free)
                const bool st = static_cast<unsigned>(j - 2 * K + 1 - c.r_lo) < c.span;
                const uint32_t add = __popc(nl[0] & c.v0) + __popc(nl[1] & c.v1) +
                                     (static_cast<uint32_t>(__popc(newT[0] & c.v0) + __popc(newT[1] & c.v1)) << 16);
                q.cc[K - 1] += st ? add : 0u;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            q.oc[s][h] = (h < TBD || (DL & (1 << h))) ? D[h] : Op[h];
            q.lp[s][P2][h] = Lp[h];
            if (s < K - 1) q.nt[s][P3][h] = newT[h];
        }
    }
}

// After a strip: its rows among the band's first / last kHalo rows go to their
// ghost images (own ghost rows, or the neighbours' over NVLink), then the
// neighbour's flag is raised (see copy_images in bml_step_kernel.cuh).
__device__ __noinline__ void wide_copy_images(const StepArgs& a, int r_lo, int r_hi, long long off0,
                                              uint32_t v0, uint32_t v1) {
    const int top_end = min(r_hi, kHalo);
    const int bot_begin = max(r_lo, a.rows - kHalo);
    for (int o = r_lo; o < top_end; ++o) {
        const long long off = static_cast<long long>(o) * a.pitch + off0;
        if (v0) a.dst[off + a.top_delta] = __ldcg(a.dst + off);
        if (v1) a.dst[off + 1 + a.top_delta] = __ldcg(a.dst + off + 1);
    }
    for (int o = bot_begin; o < r_hi; ++o) {
        const long long off = static_cast<long long>(o) * a.pitch + off0;
        if (v0) a.dst[off + a.bot_delta] = __ldcg(a.dst + off);
        if (v1) a.dst[off + 1 + a.bot_delta] = __ldcg(a.dst + off + 1);
    }
    if (!a.single_band) {
        if (r_lo == 0) publish(a.up_flag);
        if (r_hi == a.rows) publish(a.down_flag);
    }
}

// TMA: rows by bulk copies into the mbarrier ring (true), or by per-lane 16-byte
// cp.async (LDGSTS) into a commit-group ring like step_block_kernel's (false).
// PITCH: the row pitch in words at compile time (0: StepArgs::pitch), so the
// unrolled loop addresses its six rows with immediate offsets
template <int K, int COUNT, bool TMA = true, int MAXT = 256, bool EO = false, int TBD = 0, int PITCH = 0, int DL = 0>
__global__ void __launch_bounds__(MAXT, 1) step_wide_kernel(const StepArgs a) {
    static_assert(!(EO && TMA), "the even/odd layout uses the LDGSTS ring");
    if (BML_PDL) {
        asm volatile("griddepcontrol.launch_dependents;");
        asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous launch's rows are final
    }
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int warps_total = gridDim.x * nwarps;
    __shared__ __align__(128) uint4 ring[MAXT / 32][kWideRing][kWideSlotWords / 2];
    __shared__ __align__(8) unsigned long long bars[MAXT / 32][kWideRing];
    const uint32_t ring_base = static_cast<uint32_t>(__cvta_generic_to_shared(&ring[wid][0][0]));
    const uint32_t bar_base = static_cast<uint32_t>(__cvta_generic_to_shared(&bars[wid][0]));
    constexpr uint32_t kSlotBytes = kWideSlotWords * sizeof(uint2);
    if (TMA && lane == 0) {
#pragma unroll
        for (int i = 0; i < kWideRing; ++i) wide_mbar_init(bar_base + 8u * i);
        // the previous launch's (generic-proxy) row stores before this launch's TMA reads
        fence_proxy_async();
    }
    __syncwarp();
    uint32_t phase_bits = 0;  // bit i: parity of slot i's next completion

    for (int item = wid * gridDim.x + blockIdx.x; item < a.items; item += warps_total) {
        const int order = item / a.ncols;
        const int col = item - order * a.ncols;
        // connected bands run boundary-first: the band's top and bottom strips are
        // items of the first round, so both neighbours' ghost rows are published
        // early and the interior strips overlap their wait (order 0 -> strip 0,
        // order 1 -> the last strip, order k -> strip k-1)
        const int strip = (a.single_band || a.nstrips < 2 || order == 0)
                              ? order
                              : (order == 1 ? a.nstrips - 1 : order - 1);
        WideCtx c;
        c.lane = lane;
        c.r_lo = static_cast<int>(static_cast<long long>(strip) * a.rows / a.nstrips);
        c.r_hi = static_cast<int>(static_cast<long long>(strip + 1) * a.rows / a.nstrips);
        const int win = (EO ? kEoOut : kWideOut) * col - 2;  // window start (may be -2)
        const int g0 = win + 2 * lane;                 // this lane's first word, unwrapped
        // outputs: window words 1..62, unwrapped index in [-1, W-2]; EO: whole
        // 64-cell groups, lanes 1..30 (words 2..61, unwrapped index in [0, W-1])
        const bool o0 = EO ? (lane > 0 && lane < 31 && g0 <= a.W - 2) : (lane > 0 && g0 <= a.W - 2);
        const bool o1 = EO ? o0 : (lane < 31 && g0 + 1 <= a.W - 2);
        c.v0 = o0 ? kFull : 0u;
        c.v1 = o1 ? kFull : 0u;
        c.span = (o0 || o1) ? static_cast<unsigned>(c.r_hi - c.r_lo) : 0u;
        c.kind = (o0 ? 1 : 0) | (o1 ? 2 : 0);
        // wrapped first word (even). EO: fully mod W, since the ghost group right
        // of the last output group must hold the row's first cells
        const int w0 = EO ? (g0 < 0 ? g0 + a.W : (g0 >= a.W ? g0 - a.W : g0)) : (g0 < 0 ? g0 + a.W : g0);

        if (!a.single_band) {
            if (c.r_lo == 0) wait_flag(a.top_flag, a.expect, a.error_flag);
            if (c.r_hi == a.rows) wait_flag(a.bot_flag, a.expect, a.error_flag);
            if (TMA && lane == 0) fence_proxy_async();  // peer ghost rows (generic) before TMA reads
            __syncwarp();
        }

        WideState<K> q;
#pragma unroll
        for (int s = 0; s < K; ++s) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                q.nt[s][0][h] = q.nt[s][1][h] = q.nt[s][2][h] = 0u;
                q.lp[s][0][h] = q.lp[s][1][h] = 0u;
                q.oc[s][h] = 0u;
            }
            q.cm[s] = q.cc[s] = 0u;
        }
        q.xt[0][0] = q.xt[1][0] = q.xt[2][0] = q.xt[0][1] = q.xt[1][1] = q.xt[2][1] = 0u;

        const int j_begin = c.r_lo - K;
        const int j_load_end = c.r_hi + K;
        const int iters = c.r_hi + 2 * K - 1 - j_begin;
        const int j_end = j_begin + (iters + 5) / 6 * 6;

        // the window as at most two contiguous pieces of a row (torus seam)
        const int wa = win < 0 ? win + a.W : win;      // first window word, wrapped
        const int piece1 = min(kWideSlotWords, a.W - wa);  // words before the seam
        const uint32_t bytes1 = static_cast<uint32_t>(piece1) * 8u;
        const uint32_t bytes2 = kSlotBytes - bytes1;
        const uint2* gsrc = a.src + static_cast<long long>(j_begin) * a.pitch;
        c.outp = a.dst + static_cast<long long>(j_begin - 2 * K + 1) * a.pitch + w0;
        int j_issue = j_begin;
        // rows past j_load_end feed only stage inputs outside every stored row's
        // dependency cone: their slots are filled with row j_load_end - 1 (so every
        // slot is issued and waited on, branch-free), and the data is don't-care
        const uint2* glast = a.src + static_cast<long long>(j_load_end - 1) * a.pitch;
        auto issue_to = [&](int slot) {
            // EO: rows past the band end read the zero pad rows (kLoadPad), no select
            const uint2* row = EO ? gsrc : (j_issue < j_load_end ? gsrc : glast);
            if (TMA) {
                wide_issue_row(lane == 0, bar_base + 8u * slot, ring_base + slot * kSlotBytes, row + wa, bytes1,
                               row, bytes2);
            } else {
                const unsigned sm = ring_base + slot * kSlotBytes + 16u * lane;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sm), "l"(row + w0) : "memory");
                cp_async_commit();
            }
            ++j_issue;
            gsrc += PITCH ? PITCH : a.pitch;
        };
        auto next_row = [&](auto p_const) -> uint4 {
            constexpr int P = decltype(p_const)::value;
            if (TMA) {
                wide_mbar_wait(bar_base + 8u * P, (phase_bits >> P) & 1u);
                phase_bits ^= 1u << P;
            } else {
                cp_async_wait<kWideRing - 2>();
            }
            const uint4 x = ring[wid][P][lane];
            if (TMA) __syncwarp();  // every lane has read slot P before it is refilled
            // EO refills the slot read one iteration earlier AFTER the iteration's
            // stages (refill_after): the LDS and the LDGSTS are then far apart, and
            // ptxas needs no padding between them
            if (!EO) issue_to((P + kWideRing - 1) % kWideRing);
            return x;
        };
        auto refill_after = [&](auto p_const) {
            constexpr int P = decltype(p_const)::value;
            if (EO && PITCH && !TMA) {  // row gsrc + P rows: an immediate offset, gsrc advances per loop
                const unsigned sm = ring_base + ((P + kWideRing - 1) % kWideRing) * kSlotBytes + 16u * lane;
                asm volatile("cp.async.cg.shared.global [%0], [%1+%2], 16;" ::"r"(sm), "l"(gsrc + w0),
                             "n"(P * PITCH * 8)
                             : "memory");
                cp_async_commit();
            } else if (EO) {
                issue_to((P + kWideRing - 1) % kWideRing);
            }
        };
#pragma unroll
        for (int i = 0; i < kWideRing - 1; ++i) issue_to(i);
        using P0 = std::integral_constant<int, 0>;
        using P1 = std::integral_constant<int, 1>;
        using P2 = std::integral_constant<int, 2>;
        using P3 = std::integral_constant<int, 3>;
        using P4 = std::integral_constant<int, 4>;
        using P5 = std::integral_constant<int, 5>;
        for (int j = j_begin; j < j_end; j += 6) {
            wide_iter<K, COUNT, 0, EO, TBD, PITCH, DL>(q, next_row(P0{}), j, a, c);
            refill_after(P0{});
            wide_iter<K, COUNT, 1, EO, TBD, PITCH, DL>(q, next_row(P1{}), j + 1, a, c);
            refill_after(P1{});
            wide_iter<K, COUNT, 2, EO, TBD, PITCH, DL>(q, next_row(P2{}), j + 2, a, c);
            refill_after(P2{});
            wide_iter<K, COUNT, 3, EO, TBD, PITCH, DL>(q, next_row(P3{}), j + 3, a, c);
            refill_after(P3{});
            wide_iter<K, COUNT, 4, EO, TBD, PITCH, DL>(q, next_row(P4{}), j + 4, a, c);
            refill_after(P4{});
            wide_iter<K, COUNT, 5, EO, TBD, PITCH, DL>(q, next_row(P5{}), j + 5, a, c);
            refill_after(P5{});
            if (EO && PITCH) {
                gsrc += 6 * PITCH;
                c.outp += 6 * PITCH;
            }
        }
        // the last kWideRing - 1 issues (rows j_end .. j_end + 4) were never
        // consumed: wait for them so every slot's parity is in step for the next item
        if (TMA) {
#pragma unroll
            for (int P = 0; P < kWideRing - 1; ++P) {
                wide_mbar_wait(bar_base + 8u * P, (phase_bits >> P) & 1u);
                phase_bits ^= 1u << P;
            }
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        if (c.r_lo < kHalo || c.r_hi > a.rows - kHalo)
            wide_copy_images(a, c.r_lo, c.r_hi, w0, c.span ? c.v0 : 0u, c.span ? c.v1 : 0u);

        if (COUNT) {
#pragma unroll
            for (int s = 0; s < K; ++s) {
                const unsigned m0 = __reduce_add_sync(kFull, q.cm[s] & 0xffffu);
                const unsigned m1 = __reduce_add_sync(kFull, q.cm[s] >> 16);
                const bool census = COUNT == 2 || s == K - 1;
                const unsigned m2 = census ? __reduce_add_sync(kFull, q.cc[s] & 0xffffu) : 0u;
                const unsigned m3 = census ? __reduce_add_sync(kFull, q.cc[s] >> 16) : 0u;
                if (lane == 0) {
                    unsigned long long* m = a.metrics + a.step_base + s;
                    if (m0) atomicAdd(m, static_cast<unsigned long long>(m0));
                    if (m1) atomicAdd(m + a.metrics_stride, static_cast<unsigned long long>(m1));
                    if (m2) atomicAdd(m + 2 * a.metrics_stride, static_cast<unsigned long long>(m2));
                    if (m3) atomicAdd(m + 3 * a.metrics_stride, static_cast<unsigned long long>(m3));
                }
            }
        }
    }
}

}  // namespace bml_k
