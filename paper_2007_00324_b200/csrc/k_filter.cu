// k_filter.cu -- Lines 6-7 of Algorithm 1: the per-triangle claim
// (claim_filter, refine.hpp:367-376) and the cavity-approximation filter
// (cavity_filter, refine.hpp:382-429 -> expand, expandlist.hpp:93-157).
//
// The reference's ClaimTable (refine.hpp:342-361) keeps, per triangle, the
// candidate with the maximum priority_less key (band, measure, then LOWER
// tiebreak).  On the GPU that strict total order is resolved with two atomics
// per slot, no sort: atomicMax on the 64-bit (band<<63 | bits(measure)) key,
// then atomicMin on (tiebreak<<32 | list index) among the key holders.  The
// index term reproduces the sequential first-claimer rule for exact ties.
#include "engine.h"

namespace gdp2d {

__device__ __forceinline__ u64 tie_of(const DevCands& c, u32 i) {
    return ((u64)c.tie[i] << 32) | (u64)i;
}

__global__ void k_claim_max(DevCands c, u32 n, u64* __restrict__ ckey) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && c.alive[i]) atomicMax((ull*)&ckey[c.loc[i]], (ull)c.key[i]);
}

__global__ void k_claim_tie(DevCands c, u32 n, const u64* __restrict__ ckey,
                            u64* __restrict__ ctie) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && c.alive[i]) {
        const u32 t = c.loc[i];
        if (ckey[t] == c.key[i]) atomicMin((ull*)&ctie[t], (ull)tie_of(c, i));
    }
}

__global__ void k_claim_check(DevCands c, u32 n, const u64* __restrict__ ckey,
                              const u64* __restrict__ ctie, Counters* ctr) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    u32 surv = 0;
    if (i < n && c.alive[i]) {
        const u32 t = c.loc[i];
        const bool own = ckey[t] == c.key[i] && ctie[t] == tie_of(c, i);
        if (!own) c.alive[i] = 0;
        surv = own;
    }
    warp_add_u32(&ctr->surv_claim, surv);
}

__global__ void k_claim_reset(DevCands c, u32 n, u32 nT, u64* __restrict__ ckey,
                              u64* __restrict__ ctie) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const u32 t = c.loc[i];
        if (t < nT) {
            ckey[t] = 0;
            ctie[t] = ~0ull;
        }
    }
}

void launch_claim(const DevMesh& m, DevCands c, u32 n, TriAux a, Counters* d_ctr,
                  cudaStream_t st) {
    if (!n) return;
    const u32 g = (n + 255) / 256;
    note_launch(), k_claim_max<<<g, 256, 0, st>>>(c, n, a.ckey);
    note_launch(), k_claim_tie<<<g, 256, 0, st>>>(c, n, a.ckey, a.ctie);
    note_launch(), k_claim_check<<<g, 256, 0, st>>>(c, n, a.ckey, a.ctie, d_ctr);
    note_launch(), k_claim_reset<<<g, 256, 0, st>>>(c, n, m.nT, a.ckey, a.ctie);
}

// ---- cavity ---------------------------------------------------------------------

// Per candidate: FIFO BFS of triangles whose circumcircle strictly contains
// the point (the located triangle always belongs), never crossing a
// subsegment, at most ncav+1 triangles.  Processing a FIFO queue item by item
// with emissions appended in (source, slot) order visits triangles in exactly
// the window order of expand() (expandlist.hpp:98-152), so the region -- and
// hence the claim set -- is the reference's, including when the cap binds.
__global__ void __launch_bounds__(128) k_cavity_bfs(DevMesh m, DevCands c, u32 n, u32 ncav,
                                                    int extras, u32 rs,
                                                    u32* __restrict__ regions,
                                                    u32* __restrict__ region_len,
                                                    u32* __restrict__ bfs_len,
                                                    u64* __restrict__ ckey, Counters* ctr) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    ull visits = 0;
    if (i < n) {
        u32 len = 0, blen = 0;
        if (c.alive[i]) {
            u32* reg = regions + (size_t)i * rs;
            u32 queue[1 + 3 * (MAX_CAVITY_N + 1)];
            u32 head = 0, tail = 0;
            const u32 located = c.loc[i];
            const double2 p = c.pt[i];
            const u64 key = c.key[i];
            queue[tail++] = located;
            while (head < tail && len <= ncav) {
                const u32 t = queue[head++];
                const uint4 tv = m.tv[t];
                bool pred = t == located;
                if (!pred && tv.w)
                    pred = incircle(m.xy[tv.x], m.xy[tv.y], m.xy[tv.z], p) > 0;
                if (!pred) continue;
                bool in = false;
                for (u32 k = 0; k < len; ++k) in |= reg[k] == t;
                if (in) continue;
                reg[len++] = t;
                atomicMax((ull*)&ckey[t], (ull)key);
                const uint4 tn = m.tn[t];
                const uint4 ts = m.ts[t];
                for (int e = 0; e < 3; ++e) {
                    if (comp(ts, e) != NONE) continue;
                    const u32 cc = comp(tn, e);
                    if (cc == NONE) continue;
                    const u32 nb = etri(cc);
                    bool seen = false;
                    for (u32 k = 0; k < len; ++k) seen |= reg[k] == nb;
                    if (seen) continue;
                    queue[tail++] = nb;
                }
            }
            blen = len;
            if (extras) {
                // Refine mode: the insertion also rewrites the triangle across a
                // split edge, so claim it too (SURVEY §7 hard part (i)).
                u32 far = NONE;
                if (c.kind[i] == 0) {
                    const u32 s = c.id[i];
                    const int e = seg_slot(m.ts[located], s);
                    if (e >= 0) {
                        const u32 cc = comp(m.tn[located], e);
                        if (cc != NONE) far = etri(cc);
                    }
                } else if (c.lkind[i] == 1) {
                    const u32 cc = comp(m.tn[located], c.ledge[i]);
                    if (cc != NONE) far = etri(cc);
                }
                if (far != NONE) {
                    bool in = false;
                    for (u32 k = 0; k < len; ++k) in |= reg[k] == far;
                    if (!in) {
                        reg[len++] = far;
                        atomicMax((ull*)&ckey[far], (ull)key);
                    }
                }
            }
        }
        region_len[i] = len;
        if (bfs_len) bfs_len[i] = blen;
        visits = blen;
    }
    warp_add_ull(&ctr->cavity_visits, visits);
}

__global__ void k_cavity_tie(DevCands c, u32 n, u32 rs, const u32* __restrict__ regions,
                             const u32* __restrict__ region_len, const u64* __restrict__ ckey,
                             u64* __restrict__ ctie) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const u32 len = region_len[i];
    if (!len) return;
    const u64 key = c.key[i];
    const u64 tie = tie_of(c, i);
    const u32* reg = regions + (size_t)i * rs;
    for (u32 k = 0; k < len; ++k) {
        const u32 t = reg[k];
        if (ckey[t] == key) atomicMin((ull*)&ctie[t], (ull)tie);
    }
}

__global__ void k_cavity_check(DevCands c, u32 n, u32 rs, const u32* __restrict__ regions,
                               const u32* __restrict__ region_len, const u64* __restrict__ ckey,
                               const u64* __restrict__ ctie, Counters* ctr) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    u32 surv = 0;
    if (i < n) {
        const u32 len = region_len[i];
        if (len && c.alive[i]) {
            const u64 key = c.key[i];
            const u64 tie = tie_of(c, i);
            const u32* reg = regions + (size_t)i * rs;
            bool own = true;
            for (u32 k = 0; k < len && own; ++k) {
                const u32 t = reg[k];
                own = ckey[t] == key && ctie[t] == tie;
            }
            if (!own) c.alive[i] = 0;
            surv = own;
        }
    }
    warp_add_u32(&ctr->surv_cavity, surv);
}

__global__ void k_cavity_reset(u32 n, u32 rs, const u32* __restrict__ regions,
                               const u32* __restrict__ region_len, u64* __restrict__ ckey,
                               u64* __restrict__ ctie) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const u32 len = region_len[i];
    const u32* reg = regions + (size_t)i * rs;
    for (u32 k = 0; k < len; ++k) {
        ckey[reg[k]] = 0;
        ctie[reg[k]] = ~0ull;
    }
}

void launch_cavity(const DevMesh& m, DevCands c, u32 n, u32 ncav, bool extras, TriAux a,
                   u32* regions, u32* region_len, u32* bfs_len, Counters* d_ctr,
                   cudaStream_t st) {
    if (!n) return;
    const u32 rs = ncav + 1 + MAX_CLAIM_EXTRA;
    note_launch(), k_cavity_bfs<<<(n + 127) / 128, 128, 0, st>>>(m, c, n, ncav, extras ? 1 : 0, rs, regions,
                                                   region_len, bfs_len, a.ckey, d_ctr);
    const u32 g = (n + 255) / 256;
    note_launch(), k_cavity_tie<<<g, 256, 0, st>>>(c, n, rs, regions, region_len, a.ckey, a.ctie);
    note_launch(), k_cavity_check<<<g, 256, 0, st>>>(c, n, rs, regions, region_len, a.ckey, a.ctie, d_ctr);
    note_launch(), k_cavity_reset<<<g, 256, 0, st>>>(n, rs, regions, region_len, a.ckey, a.ctie);
}

}  // namespace gdp2d
