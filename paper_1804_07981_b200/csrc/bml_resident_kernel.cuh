// paper_1804_07981_b200/csrc/bml_resident_kernel.cuh — the cluster-resident small-lattice kernels (resident_kernel, resident_p2p_kernel).
// Part of libbml_dev.so: included once, by bml_dev.cu (see its header comment).
#pragma once

#include "bml_kernels_common.cuh"

namespace bml_k {

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
#ifndef BML_RESIDENT_GHOST
#define BML_RESIDENT_GHOST 8
#endif
constexpr int kResidentGhost = BML_RESIDENT_GHOST;  // default ghost depth G (bml_dev.cu resident_plan)

// PACK: rows per register. A lattice narrower than a warp (W = 32 / PACK words,
// n = 256 -> PACK 4) packs PACK rows into the 32 lanes: lane = segment * W +
// word, segment s of register i holding window row w * RPW * PACK + s * RPW + i.
// Column wrap stays inside a segment; the row above / below an edge register
// comes from the neighbouring segment by a W-lane shuffle, and only the first /
// last segment talks to the neighbouring warps through shared memory.
template <int RPW, bool COUNT, int PACK = 1>
__global__ void __launch_bounds__(1024, 1) resident_kernel(const ResidentArgs a) {
    constexpr int SEG = 32 / PACK;  // lanes per row segment
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int C = static_cast<int>(cluster.num_blocks());
    const int c = static_cast<int>(cluster.block_rank());
    const int G = a.ghost;
    const int B = a.n / C;
    const int r0 = c * B;
    const int NW = blockDim.x >> 5;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = a.W;  // == SEG when PACK > 1
    const int seg = lane / SEG, word = lane % SEG;
    const bool lane_ok = word < W;
    const int left = seg * SEG + (word == 0 ? W - 1 : word - 1);
    const int right = seg * SEG + (word + 1 >= W ? 0 : word + 1);
    constexpr int RW = RPW * PACK;  // window rows per warp
    auto erow = [&](int i) { return w * RW + seg * RPW + i; };  // this lane's window row of register i

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
    const uint32_t ghost_bytes = 2u * static_cast<uint32_t>(G) * (PACK == 1 ? 32u : SEG) * sizeof(uint2);
    const int up_rank = (c + C - 1) % C, dn_rank = (c + 1) % C;
    cluster.sync();  // every CTA's barriers are initialised before the first remote store

    uint32_t L[RPW], T[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int e = erow(i);
        int row = (r0 - G + e) % a.n;
        if (row < 0) row += a.n;
        const uint2 x = lane_ok ? a.src[static_cast<long long>(row) * a.pitch + word] : make_uint2(0u, 0u);
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
            const bool holds_ghost = w * RW < G || (w + 1) * RW > G + B;
            if (holds_ghost) mbar_wait(smem_u32(&gbar[bp ^ 1]), static_cast<uint32_t>(((blk - 1) >> 1) & 1), a.error_flag);
            // ghost rows pushed into this CTA's shared memory by the neighbours
            // before the last cluster barrier (local loads only)
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int e = erow(i);
                if (e < G) {
                    const uint2 x = ghostb[bp ^ 1][e][word];
                    L[i] = x.x;
                    T[i] = x.y;
                } else if (e >= G + B) {
                    const uint2 x = ghostb[bp ^ 1][G + (e - G - B)][word];
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
                    const int e = erow(i);
                    if (e >= G && e < G + B) lr_moved += __popc(vac & valid);
                }
                L[i] = inc | (L[i] & nextO);
                Op[i] = BML_IMAD_OR ? imad(L[i], a.one, T[i]) : (L[i] | T[i]);
            }
            if (seg == PACK - 1) xT[par][w][word] = T[RPW - 1];  // the warp's last row
            if (seg == 0) xO[par][w][word] = Op[0];              // the warp's first row
            uint32_t tb_moved = 0, lr_cnt = 0, tb_cnt = 0;
            auto tb_row = [&](int i, uint32_t above, uint32_t below) {  // TB phase, one row
                const uint32_t nt = (above & ~Op[i]) | (T[i] & below);
                if (COUNT) {
                    const int e = erow(i);
                    if (e >= G && e < G + B) {  // owned rows: moved, and the census after the step
                        tb_moved += __popc(T[i] & ~below & valid);
                        lr_cnt += __popc(L[i] & valid);
                        tb_cnt += __popc(nt & valid);
                    }
                }
                T[i] = nt;
            };
            // rows across segment boundaries (PACK > 1): W-lane shuffles
            const uint32_t t_seg = PACK > 1 ? __shfl_up_sync(kFull, T[RPW - 1], SEG) : 0u;
            const uint32_t o_seg = PACK > 1 ? __shfl_down_sync(kFull, Op[0], SEG) : 0u;
            __syncthreads();
            const uint32_t t_up = seg > 0 ? t_seg : (w > 0 ? xT[par][w - 1][word] : 0u);
            const uint32_t o_dn = seg < PACK - 1 ? o_seg : (w < NW - 1 ? xO[par][w + 1][word] : kFull);
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
                const int e = erow(i);
                if (e >= G && e < 2 * G)
                    st_async_u64(up_base + static_cast<uint32_t>((e * 32 + word) * 8), L[i], T[i], up_bar);
                if (e >= B && e < B + G)
                    st_async_u64(dn_base + static_cast<uint32_t>(((e - B) * 32 + word) * 8), L[i], T[i], dn_bar);
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
        const int e = erow(i);
        if (e >= G && e < G + B && lane_ok) {
            const int row = r0 + e - G;
            const uint2 v = make_uint2(L[i], T[i]);
            a.dst[static_cast<long long>(row) * a.pitch + word] = v;
            for (int h = row - a.n; h >= -kHalo; h -= a.n) a.dst[static_cast<long long>(h) * a.pitch + word] = v;
            for (int h = row + a.n; h < a.n + kHalo; h += a.n) a.dst[static_cast<long long>(h) * a.pitch + word] = v;
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
            if (COUNT) {  // moved, and the census after the step
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


}  // namespace bml_k
