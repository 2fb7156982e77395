// k_collect.cu -- Line 3 of Algorithm 1: the bad-triangle / encroached-
// subsegment scan (collect, refine.hpp:226-263) fused with splitting-point
// generation (compute_splitting_points, refine.hpp:267-296).
//
// HBM-bound full scan: per triangle one coalesced uint4 (tv) + three double2
// vertex gathers; per subsegment its record + <= 2 apex gathers.  The list
// order is the reference's (subsegments by id, then triangles by id) thanks to
// a stable three-kernel compaction (flag+tile count, tile-sum scan, tile-local
// shuffle scan + scatter).  Tiebreak = list index (refine.hpp:236,248).
#include <algorithm>

#include "engine.h"
#include "gdp2d_collect.cuh"
#include "scan.cuh"

namespace gdp2d {

struct CollectRange {
    u32 nS, nT;          // element counts
    u32 tilesS, tilesT;  // tile counts
};

// Incremental mode (full == 0): an element whose dirty bit is clear keeps its
// cached verdict (eval_sub / eval_tri, gdp2d_collect.cuh).  Each thread owns
// SCAN_ITEMS (= 8) consecutive elements: one 8-byte load of the cached
// verdicts, one 8-byte store of the flags.  Order inside a tile is element
// order, so the scatter needs a single block scan per tile.
template <int MODE>
__global__ void __launch_bounds__(SCAN_BLOCK) k_collect_flags(DevMesh m, Quality q, CollectRange r,
                                                           uint8_t* __restrict__ flags,
                                                           u32* __restrict__ partial, int full,
                                                           Counters* ctr, u32* z0, u32 n0, u32* z1,
                                                           u32 n1) {
    __shared__ u32 sh[SCAN_BLOCK / 32 + 1];
    if (blockIdx.x == 0) {
        for (u32 k = threadIdx.x; k < n0; k += blockDim.x) z0[k] = 0;
        for (u32 k = threadIdx.x; k < n1; k += blockDim.x) z1[k] = 0;
    }
    const bool is_sub = blockIdx.x < r.tilesS;
    const u32 tile = is_sub ? blockIdx.x : blockIdx.x - r.tilesS;
    const u32 n = is_sub ? r.nS : r.nT;
    const u32 i0 = tile * (u32)SCAN_TILE + threadIdx.x * (u32)SCAN_ITEMS;
    u32 cnt = 0, dirty = 0;
    unsigned long long out = 0;
    if (!is_sub && !full && i0 + SCAN_ITEMS <= n) {
        // common case: eight cached verdicts in one load; dirty ones re-evaluated
        unsigned long long v = *reinterpret_cast<const unsigned long long*>(m.tflag + i0);
        if (v & 0x0202020202020202ull) {
#pragma unroll
            for (int j = 0; j < SCAN_ITEMS; ++j) {
                const uint8_t tf = (uint8_t)(v >> (8 * j));
                if (tf & 2) {
                    const uint8_t f = eval_tri(m, q, i0 + j);
                    ++dirty;
                    v = (v & ~(0xFFull << (8 * j))) | ((unsigned long long)f << (8 * j));
                }
            }
        }
        out = v & 0x0101010101010101ull;
    } else {
#pragma unroll 2
        for (int j = 0; j < SCAN_ITEMS; ++j) {
            const u32 i = i0 + j;
            if (i >= n) break;
            uint8_t f;
            if (is_sub) {
                f = eval_sub<MODE>(m, i, full, dirty);
            } else {
                const uint8_t tf = full ? 2 : m.tflag[i];
                if (tf & 2) {
                    f = eval_tri(m, q, i);
                    ++dirty;
                } else {
                    f = tf & 1;
                }
            }
            out |= (unsigned long long)f << (8 * j);
        }
    }
    *reinterpret_cast<unsigned long long*>(flags + (size_t)blockIdx.x * SCAN_TILE +
                                           threadIdx.x * SCAN_ITEMS) = out;
    cnt = __popcll(out);
    // one reduction for both: count and dirty are <= SCAN_TILE < 2^16
    const u32 t = block_sum<SCAN_BLOCK>(cnt | (dirty << 16), sh);
    if (threadIdx.x == 0) {
        partial[blockIdx.x] = t & 0xFFFFu;
        if (t >> 16) atomicAdd(&ctr->scan_dirty, t >> 16);
    }
}

__global__ void __launch_bounds__(SCAN_BLOCK) k_collect_scatter(DevMesh m, CollectRange r,
                                                             const uint8_t* __restrict__ flags,
                                                             const u32* __restrict__ partial,
                                                             DevCands c, u32 ccap,
                                                             const u32* __restrict__ d_total,
                                                             Counters* ctr) {
    __shared__ u32 sh[SCAN_BLOCK / 32 + 1];
    const bool is_sub = blockIdx.x < r.tilesS;
    const u32 tile = is_sub ? blockIdx.x : blockIdx.x - r.tilesS;
    const u32 carry = partial[blockIdx.x];
    const u32 end = blockIdx.x + 1 < r.tilesS + r.tilesT ? partial[blockIdx.x + 1] : *d_total;
    if (end == carry) return;   // no candidate in this tile (the common case in the tail)
    const u32 i0 = tile * (u32)SCAN_TILE + threadIdx.x * (u32)SCAN_ITEMS;
    const unsigned long long f8 = *reinterpret_cast<const unsigned long long*>(
        flags + (size_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS);
    u32 tot;
    u32 o = carry + block_exclusive<SCAN_BLOCK>((u32)__popcll(f8), sh, &tot);
    u32 nfb = 0;
    const int kind = is_sub ? 0 : 1;
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        if (!((f8 >> (8 * j)) & 1ull)) continue;
        if (o < ccap) nfb += write_candidate(m, c, o, kind, i0 + j);
        ++o;
    }
    warp_add_u32(&ctr->fallbacks, nfb);
}

// ---- small lists (the tail of a refinement) -------------------------------------
//
// When the previous batch had at most SMALL_LIST candidates, the flags pass
// appends the candidate elements' keys (bit 31 = triangle, then the id: the
// list order of refine.hpp:226-263, subsegments first, each by id) to a
// short unordered list instead of writing a flag per element, and ONE CTA
// sorts it and writes the records -- two launches instead of flags + scan +
// scatter over every tile of a 20M-triangle mesh.  Same list, same records.
// A list that outgrew SMALL_LIST sets the count to NONE: every filter kernel
// and the insertion kernel then skip the batch, and the host redoes it with
// the full collect.
constexpr u32 SMALL_LIST = SMALL_LIST_CAP;
constexpr int SMALL_BLOCK = 1024;

template <int MODE>
__global__ void __launch_bounds__(SCAN_BLOCK) k_collect_append(DevMesh m, Quality q, CollectRange r,
                                                            u32* __restrict__ list,
                                                            u32* __restrict__ list_n, int full,
                                                            Counters* ctr, u32* z0, u32 n0,
                                                            u32* z1, u32 n1) {
    __shared__ u32 sh[SCAN_BLOCK / 32 + 1];
    if (blockIdx.x == 0) {
        for (u32 k = threadIdx.x; k < n0; k += blockDim.x) z0[k] = 0;
        for (u32 k = threadIdx.x; k < n1; k += blockDim.x) z1[k] = 0;
    }
    const bool is_sub = blockIdx.x < r.tilesS;
    const u32 tile = is_sub ? blockIdx.x : blockIdx.x - r.tilesS;
    const u32 n = is_sub ? r.nS : r.nT;
    const u32 i0 = tile * (u32)SCAN_TILE + threadIdx.x * (u32)SCAN_ITEMS;
    u32 dirty = 0;
    unsigned long long out = 0;
    if (!is_sub && !full && i0 + SCAN_ITEMS <= n) {
        unsigned long long v = *reinterpret_cast<const unsigned long long*>(m.tflag + i0);
        if (v & 0x0202020202020202ull) {
#pragma unroll
            for (int j = 0; j < SCAN_ITEMS; ++j) {
                const uint8_t tf = (uint8_t)(v >> (8 * j));
                if (tf & 2) {
                    const uint8_t f = eval_tri(m, q, i0 + j);
                    ++dirty;
                    v = (v & ~(0xFFull << (8 * j))) | ((unsigned long long)f << (8 * j));
                }
            }
        }
        out = v & 0x0101010101010101ull;
    } else {
        for (int j = 0; j < SCAN_ITEMS; ++j) {
            const u32 i = i0 + j;
            if (i >= n) break;
            uint8_t f;
            if (is_sub) {
                f = eval_sub<MODE>(m, i, full, dirty);
            } else {
                const uint8_t tf = full ? 2 : m.tflag[i];
                if (tf & 2) {
                    f = eval_tri(m, q, i);
                    ++dirty;
                } else {
                    f = tf & 1;
                }
            }
            out |= (unsigned long long)f << (8 * j);
        }
    }
    const u32 cnt = __popcll(out);
    if (__any_sync(0xFFFFFFFFu, cnt != 0)) {
        // warp-aggregated append
        u32 pre = cnt;
        for (int d = 1; d < 32; d <<= 1) {
            const u32 y = __shfl_up_sync(0xFFFFFFFFu, pre, d);
            if ((threadIdx.x & 31) >= (u32)d) pre += y;
        }
        const u32 wtot = __shfl_sync(0xFFFFFFFFu, pre, 31);
        u32 base = 0;
        if ((threadIdx.x & 31) == 31) base = atomicAdd(list_n, wtot);
        base = __shfl_sync(0xFFFFFFFFu, base, 31) + pre - cnt;
        const u32 kbit = is_sub ? 0u : 0x80000000u;
        for (int j = 0; j < SCAN_ITEMS; ++j)
            if ((out >> (8 * j)) & 1ull) {
                if (base < SMALL_LIST) list[base] = kbit | (i0 + j);
                ++base;
            }
    }
    const u32 t = block_sum<SCAN_BLOCK>(dirty, sh);
    if (threadIdx.x == 0 && t) atomicAdd(&ctr->scan_dirty, t);
}

// One CTA: sort the appended keys (bitonic, in shared memory) and write the
// candidate records in list order.
// The sorted keys are also kept (klist): the tail loop's next collect starts
// from them, and the dirty-element list restarts (dlist_n).
__global__ void __launch_bounds__(SMALL_BLOCK) k_collect_small(DevMesh m, u32* __restrict__ list,
                                                            u32* __restrict__ list_n, DevCands c,
                                                            u32 ccap, u32* __restrict__ d_count,
                                                            Counters* ctr, u32* __restrict__ klist,
                                                            u32* __restrict__ klist_n,
                                                            u32* __restrict__ dlist_n) {
    __shared__ u32 key[SMALL_LIST];
    const u32 n = *list_n;
    if (n > SMALL_LIST || n > ccap) {
        if (threadIdx.x == 0) {
            *d_count = NONE;   // the host redoes the batch (full collect)
            *list_n = 0;
            *klist_n = NONE;
            if (dlist_n) *dlist_n = 0;
        }
        return;
    }
    u32 np = 1;
    while (np < n) np <<= 1;
    for (u32 k = threadIdx.x; k < np; k += blockDim.x) key[k] = k < n ? list[k] : NONE;
    __syncthreads();
    for (u32 size = 2; size <= np; size <<= 1)
        for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
            for (u32 k = threadIdx.x; k < np / 2; k += blockDim.x) {
                const u32 lo = 2 * k - (k & (stride - 1));
                const u32 hi = lo + stride;
                const bool up = (lo & size) == 0;
                const u32 a = key[lo], b = key[hi];
                if ((a > b) == up) {
                    key[lo] = b;
                    key[hi] = a;
                }
            }
            __syncthreads();
        }
    u32 nfb = 0;
    for (u32 o = threadIdx.x; o < n; o += blockDim.x) {
        const u32 k = key[o];
        klist[o] = k;
        nfb += write_candidate(m, c, o, k >> 31 ? 1 : 0, k & 0x7FFFFFFFu);
    }
    warp_add_u32(&ctr->fallbacks, nfb);
    if (threadIdx.x == 0) {
        *d_count = n;
        *list_n = 0;   // ready for the next batch
        *klist_n = n;
        if (dlist_n) *dlist_n = 0;
    }
}

u32 launch_collect(const DevMesh& m, const Quality& q, bool rule4, uint8_t* flags, DevCands c,
                   u32 ccap, ScanScratch& s, Counters* d_ctr, cudaStream_t st,
                   const CollectCache& cache, bool* tris_scanned, u32* d_count,
                   cudaEvent_t ev_scan0, cudaEvent_t ev_scan1, bool sync, u32* small_list,
                   u32* dlist_n) {
    u32* small_list_n = small_list ? small_list + SMALL_LIST_CAP : nullptr;
    u32* klist = small_list ? small_list + SMALL_LIST_CAP + 1 : nullptr;
    u32* klist_n = small_list ? small_list + 2 * SMALL_LIST_CAP + 1 : nullptr;
    *tris_scanned = false;
    u32 *zp0 = cache.zero[0], *zp1 = cache.zero[1];
    u32 zn0 = cache.zero_n[0], zn1 = cache.zero_n[1];
    // sync == false (rule 4 only): no host round trip -- the scatter runs
    // unconditionally and the count stays on the device (*d_count)
    if (!sync && !rule4) sync = true;
    if (!sync && small_list && small_list_n && m.nS + m.nT > 0) {
        // the previous batch was small: append + one-CTA sort (see above)
        *tris_scanned = true;
        CollectRange r;
        r.nS = m.nS;
        r.nT = m.nT;
        r.tilesS = (r.nS + SCAN_TILE - 1) / SCAN_TILE;
        r.tilesT = (r.nT + SCAN_TILE - 1) / SCAN_TILE;
        const u32 tiles = r.tilesS + r.tilesT;
        if (ev_scan0) cudaEventRecord(ev_scan0, st);
        if (q.mode == 0)
            note_launch(), k_collect_append<0><<<tiles, SCAN_BLOCK, 0, st>>>(m, q, r, small_list, small_list_n, cache.full, d_ctr, zp0, zn0, zp1, zn1);
        else
            note_launch(), k_collect_append<1><<<tiles, SCAN_BLOCK, 0, st>>>(m, q, r, small_list, small_list_n, cache.full, d_ctr, zp0, zn0, zp1, zn1);
        note_launch(), k_collect_small<<<1, SMALL_BLOCK, 0, st>>>(m, small_list, small_list_n, c, ccap, d_count, d_ctr, klist, klist_n, dlist_n);
        return NONE;
    }
    auto run = [&](bool sub, bool tri) -> u32 {
        if (tri) *tris_scanned = true;
        CollectRange r;
        r.nS = sub ? m.nS : 0;
        r.nT = tri ? m.nT : 0;
        r.tilesS = (r.nS + SCAN_TILE - 1) / SCAN_TILE;
        r.tilesT = (r.nT + SCAN_TILE - 1) / SCAN_TILE;
        const u32 tiles = r.tilesS + r.tilesT;
        if (tiles == 0) {
            if (zn0) cudaMemsetAsync(zp0, 0, 4ull * zn0, st);
            if (zn1) cudaMemsetAsync(zp1, 0, 4ull * zn1, st);
            zn0 = zn1 = 0;
            cudaMemsetAsync(d_count, 0, sizeof(u32), st);
            return 0;
        }
        if (tiles + 1 > s.cap) {
            if (s.partial) cudaFree(s.partial);
            s.cap = (tiles + 1) * 2;
            cudaMalloc(&s.partial, sizeof(u32) * s.cap);
        }
        if (ev_scan0 && sub) cudaEventRecord(ev_scan0, st);
        if (q.mode == 0)
            note_launch(), k_collect_flags<0><<<tiles, SCAN_BLOCK, 0, st>>>(m, q, r, flags, s.partial, cache.full, d_ctr, zp0, zn0, zp1, zn1);
        else
            note_launch(), k_collect_flags<1><<<tiles, SCAN_BLOCK, 0, st>>>(m, q, r, flags, s.partial, cache.full, d_ctr, zp0, zn0, zp1, zn1);
        zn0 = zn1 = 0;   // zeroed once
        if (ev_scan1 && (tri || !rule4)) cudaEventRecord(ev_scan1, st);
        scan_partials(s.partial, tiles, d_count, st);
        if (!sync) {
            note_launch(), k_collect_scatter<<<tiles, SCAN_BLOCK, 0, st>>>(m, r, flags, s.partial, c, ccap, d_count, d_ctr);
            return NONE;
        }
        u32 total = 0;
        cudaMemcpyAsync(&total, d_count, sizeof(u32), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        if (total > 0)
            note_launch(), k_collect_scatter<<<tiles, SCAN_BLOCK, 0, st>>>(m, r, flags, s.partial, c, ccap, d_count, d_ctr);
        return total;
    };
    if (rule4) return run(true, true);
    const u32 ns = run(true, false);
    if (ns > 0) return ns;
    return run(false, true);
}

// ---- batch_size_cap: keep the k highest priorities (refine.hpp:252-261) -------------
//
// The reference sorts the list by priority, keeps the first k and restores
// list order.  Here the list stays in place and the others are marked dead:
// an MSD radix select (8-bit digits, 12 passes) finds the k-th largest
// 96-bit rank (key, ~tiebreak) -- unique, since the tiebreak is the list
// index -- and a last pass keeps every candidate whose rank is at least it.
// No host round trip: the selection state lives in device memory.

struct SelState {
    unsigned long long key;   // prefix of the k-th largest rank: key part
    u32 tie;                  // ... and ~tiebreak part
    u32 k;                    // rank still to find inside the current bucket
    u32 hist[256];
};

__device__ __forceinline__ u32 sel_digit(u64 key, u32 ntie, int d) {
    return d < 8 ? (u32)(key >> (56 - 8 * d)) & 0xFFu : (ntie >> (24 - 8 * (d - 8))) & 0xFFu;
}

// true if (key, ntie) matches the selected prefix on the digits before d
__device__ __forceinline__ bool sel_match(u64 key, u32 ntie, const SelState& s, int d) {
    if (d == 0) return true;
    if (d <= 8) {
        const u64 mask = ~0ull << (64 - 8 * d);
        return (key & mask) == (s.key & mask);
    }
    if (key != s.key) return false;
    const u32 mask = ~0u << (32 - 8 * (d - 8));
    return (ntie & mask) == (s.tie & mask);
}

__global__ void __launch_bounds__(256) k_sel_hist(DevCands c, u32 n, SelState* st, int d) {
    __shared__ u32 h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const SelState s = *st;
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (!c.alive[i]) continue;
        const u64 key = c.key[i];
        const u32 ntie = ~c.tie[i];
        if (!sel_match(key, ntie, s, d)) continue;
        atomicAdd(&h[sel_digit(key, ntie, d)], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], h[threadIdx.x]);
}

// one thread: pick the bucket holding the k-th largest, extend the prefix
__global__ void k_sel_pick(SelState* st, int d) {
    u32 k = st->k, above = 0;
    int b = 255;
    for (; b > 0; --b) {
        const u32 cnt = st->hist[b];
        if (above + cnt >= k) break;
        above += cnt;
    }
    st->k = k - above;
    if (d < 8)
        st->key |= (unsigned long long)b << (56 - 8 * d);
    else
        st->tie |= (u32)b << (24 - 8 * (d - 8));
    for (int i = 0; i < 256; ++i) st->hist[i] = 0;
}

__global__ void k_sel_apply(DevCands c, u32 n, const SelState* st) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !c.alive[i]) return;
    const u64 key = c.key[i];
    const u32 ntie = ~c.tie[i];
    const bool keep = key > st->key || (key == st->key && ntie >= st->tie);
    if (!keep) c.alive[i] = 0;
}

size_t select_state_bytes() { return sizeof(SelState); }

void launch_select_topk(DevCands c, u32 n, u32 k, void* state, cudaStream_t st) {
    if (k == 0 || k >= n) return;
    SelState init{};
    init.k = k;
    SelState* s = reinterpret_cast<SelState*>(state);
    cudaMemcpyAsync(s, &init, sizeof init, cudaMemcpyHostToDevice, st);
    const u32 grid = std::min<u32>((n + 255) / 256, 148 * 8);
    for (int d = 0; d < 12; ++d) {
        note_launch(), k_sel_hist<<<grid, 256, 0, st>>>(c, n, s, d);
        note_launch(), k_sel_pick<<<1, 1, 0, st>>>(s, d);
    }
    note_launch(), k_sel_apply<<<(n + 255) / 256, 256, 0, st>>>(c, n, s);
}

// compute_splitting_points on a caller list (refine.hpp:267-296): the gdp2d_split_points
// parity entry point; the refinement fuses it into k_collect_scatter.
__global__ void k_split_points(DevMesh m, DevCands c, u32 n, Counters* ctr) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    u32 fb_count = 0;
    if (i < n) {
        uint8_t fb;
        c.pt[i] = split_point(m, c.kind[i], c.id[i], fb);
        c.fb[i] = fb;
        fb_count = fb;
    }
    warp_add_u32(&ctr->fallbacks, fb_count);
}

void launch_split_points(const DevMesh& m, DevCands c, u32 n, Counters* d_ctr, cudaStream_t st) {
    if (!n) return;
    note_launch(), k_split_points<<<(n + 255) / 256, 256, 0, st>>>(m, c, n, d_ctr);
}

}  // namespace gdp2d
