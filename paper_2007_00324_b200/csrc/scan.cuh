// scan.cuh -- warp-shuffle / shared-memory block scans used by every
// work-list compaction of the engine (north_star: "warp-shuffle/shared-memory
// scans").  Block-level only; device-wide scans are composed in k_scan.cu.
#pragma once

#include "gdp2d_common.cuh"

namespace gdp2d {

// Inclusive warp scan.
__device__ __forceinline__ u32 warp_inclusive(u32 v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 n = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Exclusive block scan of one value per thread.  `sh` needs BLOCK/32 + 1
// words.  Returns the exclusive prefix; *total gets the block sum.  All
// threads of the block must call it.
template <int BLOCK>
__device__ __forceinline__ u32 block_exclusive(u32 v, u32* sh, u32* total) {
    constexpr int NW = BLOCK / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const u32 inc = warp_inclusive(v);
    if (lane == 31) sh[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        u32 w = lane < NW ? sh[lane] : 0u;
        w = warp_inclusive(w);
        if (lane < NW) sh[lane] = w;
    }
    __syncthreads();
    const u32 pre = warp ? sh[warp - 1] : 0u;
    *total = sh[NW - 1];
    __syncthreads();
    return pre + inc - v;
}

template <int BLOCK>
__device__ __forceinline__ u32 block_sum(u32 v, u32* sh) {
    constexpr int NW = BLOCK / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = __reduce_add_sync(0xFFFFFFFFu, v);
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    u32 t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < NW; ++i) t += sh[i];
    __syncthreads();
    return t;  // valid in thread 0 only
}

}  // namespace gdp2d
