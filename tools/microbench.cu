// tools/microbench.cu -- B200 latency facts the engine design depends on:
// grid-barrier cost vs grid size, back-to-back launch cost, block barrier
// cost, dependent-load latency (L2-resident and HBM).  Not part of the
// product.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__global__ void k_gridsync(int iters, unsigned* sink) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
    if (g.thread_rank() == 0) sink[0] = iters;
}
__global__ void k_blocksync(int iters, unsigned* sink) {
    for (int i = 0; i < iters; ++i) __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = iters;
}
__global__ void k_empty(unsigned* sink) {
    if (threadIdx.x == 0 && blockIdx.x == 0) sink[1] += 1;
}
__global__ void k_chase(const unsigned* __restrict__ next, int steps, unsigned* out) {
    unsigned p = 0;
    for (int i = 0; i < steps; ++i) p = next[p];
    out[0] = p;
}

int main() {
    unsigned* sink;
    cudaMalloc(&sink, 1 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bps : {1, 2, 4, 8}) {
        int grid = sms * bps, iters = 2000;
        void* args[] = {&iters, &sink};
        cudaLaunchCooperativeKernel((void*)k_gridsync, grid, 256, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_gridsync, grid, 256, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("grid.sync grid=%d x 256: %.3f us/sync\n", grid, ms * 1e3 / iters);
    }
    {
        int iters = 100000;
        k_blocksync<<<1, 256>>>(iters, sink);
        cudaEventRecord(a);
        k_blocksync<<<1, 256>>>(iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("__syncthreads (256 thr): %.1f ns\n", ms * 1e6 / iters);
    }
    for (int grid : {1, 148, 2368}) {
        const int n = 2000;
        for (int i = 0; i < 10; ++i) k_empty<<<grid, 256>>>(sink);
        cudaEventRecord(a);
        for (int i = 0; i < n; ++i) k_empty<<<grid, 256>>>(sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("back-to-back empty launch grid=%d: %.2f us/launch\n", grid, ms * 1e3 / n);
    }
    {
        int grid = sms * 2, iters = 1;
        void* args[] = {&iters, &sink};
        const int n = 500;
        cudaEventRecord(a);
        for (int i = 0; i < n; ++i) cudaLaunchCooperativeKernel((void*)k_gridsync, grid, 256, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("back-to-back cooperative launch grid=%d (1 sync): %.2f us/launch\n", grid, ms * 1e3 / n);
    }
    {
        // launch + sync round trip
        const int n = 500;
        cudaEventRecord(a);
        for (int i = 0; i < n; ++i) {
            k_empty<<<1, 32>>>(sink);
            cudaStreamSynchronize(0);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("launch + cudaStreamSynchronize round trip: %.2f us\n", ms * 1e3 / n);
    }
    for (size_t bytes : {size_t(8) << 20, size_t(2) << 30}) {
        const size_t n = bytes / 4;
        std::vector<unsigned> h(n);
        // random cyclic permutation with 64 B stride granularity
        const size_t lines = n / 16;
        std::vector<unsigned> perm(lines);
        for (size_t i = 0; i < lines; ++i) perm[i] = (unsigned)i;
        unsigned long long s = 88172645463325252ull;
        for (size_t i = lines - 1; i > 0; --i) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            std::swap(perm[i], perm[s % (i + 1)]);
        }
        for (size_t i = 0; i < lines; ++i) h[perm[i] * 16] = perm[(i + 1) % lines] * 16;
        unsigned* d;
        cudaMalloc(&d, bytes);
        cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
        const int steps = 20000;
        k_chase<<<1, 1>>>(d, 1000, sink);
        cudaEventRecord(a);
        k_chase<<<1, 1>>>(d, steps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("dependent load latency, %zu MB footprint: %.0f ns\n", bytes >> 20, ms * 1e6 / steps);
        cudaFree(d);
    }
    return 0;
}
