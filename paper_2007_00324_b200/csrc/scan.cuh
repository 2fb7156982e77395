// scan.cuh -- warp-shuffle / shared-memory block scans used by every
// work-list compaction of the engine (north_star: "warp-shuffle/shared-memory
// scans").  Block-level only; device-wide scans are composed in k_scan.cu.
#pragma once

#include "gdp2d_common.cuh"

namespace gdp2d {

// Inclusive warp scan.
template <class T>
__device__ __forceinline__ T warp_inclusive_t(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T n = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}
__device__ __forceinline__ u32 warp_inclusive(u32 v) { return warp_inclusive_t<u32>(v); }

// Exclusive block scan of one value per thread.  `sh` needs BLOCK/32 + 1
// elements.  Returns the exclusive prefix; *total gets the block sum.  All
// threads of the block must call it.
template <int BLOCK, class T>
__device__ __forceinline__ T block_exclusive_t(T v, T* sh, T* total) {
    constexpr int NW = BLOCK / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T inc = warp_inclusive_t<T>(v);
    if (lane == 31) sh[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < NW ? sh[lane] : T(0);
        w = warp_inclusive_t<T>(w);
        if (lane < NW) sh[lane] = w;
    }
    __syncthreads();
    const T pre = warp ? sh[warp - 1] : T(0);
    *total = sh[NW - 1];
    __syncthreads();
    return pre + inc - v;
}
template <int BLOCK>
__device__ __forceinline__ u32 block_exclusive(u32 v, u32* sh, u32* total) {
    return block_exclusive_t<BLOCK, u32>(v, sh, total);
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

// Block-aggregated reservation of k slots per thread in a global work list:
// one atomicAdd per CTA (instead of one per warp, agg_reserve) on the list's
// counter, whose same-address atomics otherwise queue thousands deep at mesh
// scale.  Returns the thread's first slot.  Every thread of the block must call
// it (k may be 0).
template <int BLOCK>
__device__ __forceinline__ u32 block_reserve(u32* ctr, u32 k) {
    __shared__ u32 sh[BLOCK / 32 + 1];
    __shared__ u32 base;
    u32 tot;
    const u32 pre = block_exclusive_t<BLOCK, u32>(k, sh, &tot);
    if (threadIdx.x == 0 && tot) base = atomicAdd(ctr, tot);
    __syncthreads();
    const u32 b = base;
    __syncthreads();   // the next call's write of base must not overtake this read
    return b + pre;
}

// Block-aggregated counter add: one global atomic per CTA instead of one per
// warp (a same-address atomic per warp still serialises ~10^4 deep at mesh
// scale).  Every thread of the block must call it.
template <class T>
__device__ __forceinline__ void block_add(T* ctr, T v) {
    __shared__ T acc;
    if (threadIdx.x == 0) acc = 0;
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&acc, v);
    __syncthreads();
    if (threadIdx.x == 0 && acc) atomicAdd(ctr, acc);
    __syncthreads();   // the next call's reset must not overtake this read
}

}  // namespace gdp2d
