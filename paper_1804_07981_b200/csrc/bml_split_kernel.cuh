// paper_1804_07981_b200/csrc/bml_split_kernel.cuh — the stage-split streaming kernel
// (step_split_kernel). Part of libbml_dev.so: included once, by bml_dev.cu.
#pragma once

#include "bml_kernels_common.cuh"
#include "bml_step_kernel.cuh"

namespace bml_k {

// ------------------------------------------------------- stage-split temporally blocked step
//
// step_block_kernel gives every (strip, column) item to one warp, which runs all
// K pipeline stages. For a fixed number of warps (about two per SM sub-partition)
// that fixes the strip length R, and each strip pays a pipeline fill and drain of
// 3K - 1 iterations: 2.4% at configs[4] (R = 3855) but 10% on the 8192-row bands
// of an 8-GPU split and 37% at configs[2] (R = 126, one warp per SMSP).
//
// Here a PAIR of warps shares an item: the front warp loads the rows (cp.async
// ring) and runs stages 0 .. K/2-1; after every iteration it hands its last
// stage's outputs (the L row and the T row it emitted, 8 bytes per lane) to the
// back warp through shared memory; the back warp runs stages K/2 .. K-1 and
// stores. For the same number of warps, strips are twice as long, so the fill
// and drain weigh half as much, and each warp carries half the pipeline state.
// The handoff is batched by the loop's 6-iteration unroll into two shared-memory
// halves, each guarded by a "full" and an "empty" mbarrier (one arrival each).
// The two warps of a pair sit on different SM sub-partitions (warps 2p, 2p+1).
constexpr int kSplitBatch = 6;  // == the unroll factor

__device__ __forceinline__ void split_mbar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void split_mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// The spin loop lives inside one asm block, so the compiler sees straight-line,
// warp-converged code around it.
__device__ __forceinline__ void split_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred done;\n"
        " SPLIT_WAIT_%=:\n"
        " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1;\n"
        " @!done bra SPLIT_WAIT_%=;\n"
        "}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

template <int K, int MODE, int COUNT, int MAXT = 256>
__global__ void __launch_bounds__(MAXT, 1) step_split_kernel(const StepArgs a) {
    static_assert(K % 2 == 0 && K >= 2, "split kernel needs an even block depth");
    static_assert(MODE == kAligned, "split kernel: aligned rows only");
    constexpr int H = K / 2;
    if (BML_PDL) {
        asm volatile("griddepcontrol.launch_dependents;");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int pair = wid >> 1;
    const bool front = (wid & 1) == 0;
    const int npairs = blockDim.x >> 6;
    const int pairs_total = gridDim.x * npairs;
    __shared__ uint2 ring[MAXT / 64][kRing][32];
    __shared__ uint2 hand[MAXT / 64][2][kSplitBatch][32];
    __shared__ __align__(8) unsigned long long hbar[MAXT / 64][4];  // full[2], empty[2]
    uint2 (*my_ring)[32] = ring[pair];
    const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(&hbar[pair][0]));
    auto full_bar = [&](int h) { return bar0 + 8u * h; };
    auto empty_bar = [&](int h) { return bar0 + 8u * (2 + h); };
    if (front && lane == 0) {
        for (int i = 0; i < 4; ++i) split_mbar_init(bar0 + 8u * i);
    }
    __syncthreads();
    uint32_t par = 0;  // bit h: parity of the next completion of this warp's barrier h

    for (int item = pair * gridDim.x + blockIdx.x; item < a.items; item += pairs_total) {
        const int order = item / a.ncols;
        const int col = item - order * a.ncols;
        const int strip = (a.single_band || a.nstrips < 2 || order == 0)
                              ? order
                              : (order == 1 ? a.nstrips - 1 : order - 1);  // boundary first
        StripCtx c;
        c.lane = lane;
        c.r_lo = static_cast<int>(static_cast<long long>(strip) * a.rows / a.nstrips);
        c.r_hi = static_cast<int>(static_cast<long long>(strip + 1) * a.rows / a.nstrips);
        const int w = col * kOutWords + lane - 1;
        const bool is_out = lane >= 1 && lane < 1 + kOutWords && w < a.W;
        c.out_word = w;
        c.valid = is_out ? kFull : 0u;
        const int word = ((w % a.W) + a.W) % a.W;
        c.seam_pre = c.seam_sh = 0;
        c.seam_left = false;
        c.span = c.valid ? static_cast<unsigned>(c.r_hi - c.r_lo) : 0u;

        if (front && !a.single_band) {  // the front warp reads the ghost rows
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
        const int iters = c.r_hi + 2 * K - 1 - j_begin;
        const int nbatch = (iters + kSplitBatch - 1) / kSplitBatch;
        using P0 = std::integral_constant<int, 0>;
        using P1 = std::integral_constant<int, 1>;
        using P2 = std::integral_constant<int, 2>;
        using P3 = std::integral_constant<int, 3>;
        using P4 = std::integral_constant<int, 4>;
        using P5 = std::integral_constant<int, 5>;

        if (front) {
            const uint2* gsrc = a.src + static_cast<long long>(j_begin) * a.pitch + word;
            int j_issue = j_begin;
            auto issue_to = [&](int slot_idx) {
                if (j_issue < j_load_end) cp_async8(&my_ring[slot_idx][lane], gsrc);
                cp_async_commit();
                ++j_issue;
                gsrc += a.pitch;
            };
            __syncwarp();
#pragma unroll
            for (int i = 0; i < kRing - 1; ++i) issue_to(i);
            auto step_front = [&](auto p_const, int j, int h) {
                constexpr int P = decltype(p_const)::value;
                cp_async_wait<kRing - 2>();
                const uint2 x = my_ring[P][lane];
                issue_to((P + kRing - 1) % kRing);
                pipe_iter<K, MODE, COUNT, P, 0, H>(q, x, j, a, c);
                hand[pair][h][P][lane] = make_uint2(q.lp[H - 1][P % 2], q.nt[H - 1][P % 3]);
            };
            for (int b = 0; b < nbatch; ++b) {
                const int h = b & 1;
                if (b >= 2) {  // the back warp has consumed batch b - 2 from this half
                    split_mbar_wait(empty_bar(h), (par >> h) & 1u);
                    par ^= 1u << h;
                }
                const int j = j_begin + kSplitBatch * b;
                step_front(P0{}, j, h);
                step_front(P1{}, j + 1, h);
                step_front(P2{}, j + 2, h);
                step_front(P3{}, j + 3, h);
                step_front(P4{}, j + 4, h);
                step_front(P5{}, j + 5, h);
                __syncwarp();
                if (lane == 0) split_mbar_arrive(full_bar(h));
            }
            // the back warp's releases of the last two batches: consume them so every
            // barrier phase is waited on exactly once
            for (int b = (nbatch >= 2 ? nbatch - 2 : 0); b < nbatch; ++b) {
                const int h = b & 1;
                split_mbar_wait(empty_bar(h), (par >> h) & 1u);
                par ^= 1u << h;
            }
            cp_async_wait<0>();
        } else {
            c.outp = a.dst + static_cast<long long>(j_begin - 2 * K + 1) * a.pitch + c.out_word;
            const uint2 none = make_uint2(0u, 0u);
            auto step_back = [&](auto p_const, int j, int h) {
                constexpr int P = decltype(p_const)::value;
                const uint2 hv = hand[pair][h][P][lane];
                pipe_iter<K, MODE, COUNT, P, H, K>(q, none, j, a, c);
                q.lp[H - 1][P % 2] = hv.x;  // stage H-1's state update, as if it ran here
                q.nt[H - 1][P % 3] = hv.y;
            };
            for (int b = 0; b < nbatch; ++b) {
                const int h = b & 1;
                split_mbar_wait(full_bar(h), (par >> h) & 1u);
                par ^= 1u << h;
                const int j = j_begin + kSplitBatch * b;
                step_back(P0{}, j, h);
                step_back(P1{}, j + 1, h);
                step_back(P2{}, j + 2, h);
                step_back(P3{}, j + 3, h);
                step_back(P4{}, j + 4, h);
                step_back(P5{}, j + 5, h);
                __syncwarp();
                if (lane == 0) split_mbar_arrive(empty_bar(h));
            }
            if (c.r_lo < kHalo || c.r_hi > a.rows - kHalo)
                copy_images(a, c.r_lo, c.r_hi, c.out_word, c.span != 0u);
        }

        if (COUNT) {
#pragma unroll
            for (int s = 0; s < K; ++s) {
                if ((s < H) != front) continue;  // each warp reports its own stages
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
