// scripts/probe/dsmem_pingpong.cu — latency of the resident kernel's ghost handoff
// primitive: st.async into a neighbour CTA's shared memory completing bytes on its
// mbarrier, measured as a ping-pong between CTA pairs of one 16-CTA cluster.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probe/dsmem_pingpong scripts/probe/dsmem_pingpong.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ void arm(uint32_t bar, uint32_t tx) {
    asm volatile("{ .reg .b64 s; mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 s, [%0], %1; }" ::"r"(bar), "r"(tx) : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(bar),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void st_async(uint32_t addr, uint32_t v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(addr), "r"(v), "r"(bar) : "memory");
}

__global__ void pingpong(long long* out, int iters, int stride) {
    __shared__ __align__(8) unsigned long long bar;
    __shared__ uint32_t buf[32];
    cg::cluster_group cluster = cg::this_cluster();
    const int c = static_cast<int>(cluster.block_rank());
    // partner: the neighbouring rank (stride 1) or a farther one in the same cluster
    const int partner = (c / stride) % 2 == 0 ? c + stride : c - stride;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();
    if (threadIdx.x == 0) {
        const uint32_t me = smem_u32(&bar);
        const uint32_t rbar = mapa(me, partner), rbuf = mapa(smem_u32(&buf[0]), partner);
        const bool lead = (c / stride) % 2 == 0;
        long long t0 = 0;
        for (int i = 0; i < iters + 16; ++i) {
            if (i == 16) t0 = clock64();
            arm(me, 4);
            if (lead) {
                st_async(rbuf, i, rbar);
                wait(me, i & 1);
            } else {
                wait(me, i & 1);
                st_async(rbuf, i, rbar);
            }
        }
        out[blockIdx.x] = (clock64() - t0) / iters;
    }
    cluster.sync();
}

int main() {
    long long* d;
    long long h[16];
    cudaMalloc(&d, sizeof(h));
    cudaFuncSetAttribute(pingpong, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int stride : {1, 2, 4, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(32);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, pingpong, d, 20000, stride);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        long long mn = h[0], mx = h[0], sum = 0;
        for (long long v : h) {
            mn = v < mn ? v : mn;
            mx = v > mx ? v : mx;
            sum += v;
        }
        printf("{\"probe\": \"dsmem st.async+mbarrier ping-pong\", \"rank_stride\": %d, \"round_trip_cycles_mean\": %.1f, \"min\": %lld, \"max\": %lld}\n",
               stride, sum / 16.0, mn, mx);
    }
    return 0;
}
