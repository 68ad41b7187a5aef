// Probe: which SM / warp slot (%warpid, SMSP = %warpid % 4 presumably) each warp lands on.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__global__ void probe(int* out, int spin) {
    unsigned smid, warpid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(warpid));
    long long t0 = clock64();
    while (clock64() - t0 < spin) {}
    if ((threadIdx.x & 31) == 0) {
        int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
        out[2 * w] = smid;
        out[2 * w + 1] = warpid;
    }
}
int main() {
    for (auto cfg : std::vector<std::pair<int,int>>{{148, 128}, {148, 256}, {296, 128}, {148, 384}, {444, 128}}) {
        int grid = cfg.first, threads = cfg.second, nw = grid * threads / 32;
        int* d; cudaMalloc(&d, nw * 2 * sizeof(int));
        probe<<<grid, threads>>>(d, 200000);
        std::vector<int> h(nw * 2);
        cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
        printf("grid %d threads %d\n", grid, threads);
        for (int b = 0; b < 6; ++b) {
            printf("  cta %d:", b);
            for (int w = 0; w < threads / 32; ++w) printf(" (sm%d,w%d)", h[2 * (b * threads / 32 + w)], h[2 * (b * threads / 32 + w) + 1]);
            printf("\n");
        }
        for (int b = 148; b < 150 && b < grid; ++b) {
            printf("  cta %d:", b);
            for (int w = 0; w < threads / 32; ++w) printf(" (sm%d,w%d)", h[2 * (b * threads / 32 + w)], h[2 * (b * threads / 32 + w) + 1]);
            printf("\n");
        }
        cudaFree(d);
    }
}
