// k_scan.cu -- device-wide exclusive scan (tile reduce -> tile-sum scan ->
// tile scan) built from the block scans of scan.cuh.
#include "engine.h"
#include "scan.cuh"

namespace gdp2d {

__global__ void k_tile_reduce(const u32* __restrict__ in, u32 n, u32* __restrict__ partial) {
    __shared__ u32 sh[SCAN_BLOCK / 32 + 1];
    const u32 base = blockIdx.x * (u32)SCAN_TILE;
    u32 s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        const u32 i = base + (u32)k * SCAN_BLOCK + threadIdx.x;
        if (i < n) s += in[i];
    }
    const u32 t = block_sum<SCAN_BLOCK>(s, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// Single 1024-thread block: exclusive scan of the tile sums in place (four
// sums per thread, so one pass covers 4096 tiles = 8M elements); total ->
// *d_total.
constexpr int PSCAN_BLOCK = 1024;
__global__ void __launch_bounds__(PSCAN_BLOCK) k_partial_scan(u32* __restrict__ partial, u32 ntiles,
                                                           u32* d_total) {
    __shared__ u32 sh[PSCAN_BLOCK / 32 + 1];
    u32 carry = 0;
    for (u32 base = 0; base < ntiles; base += 4 * PSCAN_BLOCK) {
        const u32 i = base + 4 * threadIdx.x;
        u32 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = i + k < ntiles ? partial[i + k] : 0u;
        const u32 sum = v[0] + v[1] + v[2] + v[3];
        u32 tot;
        u32 ex = carry + block_exclusive<PSCAN_BLOCK>(sum, sh, &tot);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (i + k < ntiles) partial[i + k] = ex;
            ex += v[k];
        }
        carry += tot;
    }
    if (threadIdx.x == 0 && d_total) *d_total = carry;
}

__global__ void k_tile_scan(const u32* __restrict__ in, u32 n, const u32* __restrict__ partial,
                            u32* __restrict__ out) {
    __shared__ u32 sh[SCAN_BLOCK / 32 + 1];
    const u32 base = blockIdx.x * (u32)SCAN_TILE;
    u32 carry = partial[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        const u32 i = base + (u32)k * SCAN_BLOCK + threadIdx.x;
        const u32 v = i < n ? in[i] : 0u;
        u32 tot;
        const u32 ex = block_exclusive<SCAN_BLOCK>(v, sh, &tot);
        if (i < n) out[i] = carry + ex;
        carry += tot;
    }
}

void scan_partials(u32* partial, u32 ntiles, u32* d_total, cudaStream_t st) {
    note_launch(), k_partial_scan<<<1, PSCAN_BLOCK, 0, st>>>(partial, ntiles, d_total);
}

void scan_exclusive(const u32* in, u32* out, u32 n, u32* d_total, ScanScratch& s,
                    cudaStream_t st) {
    const u32 tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles == 0) {
        if (d_total) cudaMemsetAsync(d_total, 0, sizeof(u32), st);
        return;
    }
    if (tiles > s.cap) {
        if (s.partial) cudaFree(s.partial);
        s.cap = tiles * 2;
        cudaMalloc(&s.partial, sizeof(u32) * s.cap);
    }
    note_launch(), k_tile_reduce<<<tiles, SCAN_BLOCK, 0, st>>>(in, n, s.partial);
    note_launch(), k_partial_scan<<<1, PSCAN_BLOCK, 0, st>>>(s.partial, tiles, d_total);
    note_launch(), k_tile_scan<<<tiles, SCAN_BLOCK, 0, st>>>(in, n, s.partial, out);
}

}  // namespace gdp2d
