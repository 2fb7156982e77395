// gdp2d_phases.cuh -- per-candidate bodies of Lines 5-7 of Algorithm 1, shared
// by the standalone phase kernels (parity entry points gdp2d_locate /
// gdp2d_claim / gdp2d_cavity, k_locate.cu / k_filter.cu) and the persistent
// batch kernel (k_insert.cu), so the code the parity tests check is the code
// the refinement runs.
//
//   locate_one           locate (refine.hpp:301-335) -> locate_point cdt.hpp:68-105
//   claim_*_one          ClaimTable / claim_filter (refine.hpp:342-376)
//   cavity_*_one         cavity_filter (refine.hpp:382-429) -> expand (expandlist.hpp:93-157)
//   plan_one             insert_batch phase-1 needs (refine.hpp:493-539)
//
// The reference's ClaimTable keeps, per triangle, the candidate with the
// maximum priority_less key (band, measure, then LOWER tiebreak).  On the GPU
// that strict total order is resolved with two atomics per slot, no sort:
// atomicMax on the 64-bit (band<<63 | bits(measure)) key, then atomicMin on
// (tiebreak<<32 | list index) among the key holders.  The index term
// reproduces the sequential first-claimer rule for exact ties.
#pragma once

#include "engine.h"

namespace gdp2d {

// Count of a standalone filter kernel (NArg, engine.h) and its grid-stride loop.
__device__ __forceinline__ u32 narg(const NArg& a) {
    const u32 n = a.d_n ? *a.d_n : a.n;
    return (n <= a.skip_le || n > a.cap) ? 0u : n;
}
#define GRID_STRIDE(i, n) \
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += gridDim.x * blockDim.x)

// Returns the walk steps.
__device__ __forceinline__ u32 locate_one(const DevMesh& m, const DevCands& c, u32 i) {
    if (!c.alive[i]) return 0;
    if (c.kind[i] == 0) {
        c.loc[i] = m.stri[c.id[i]];
        c.lkind[i] = 4;   // subsegment midpoint: split along the subsegment
        c.ledge[i] = -1;
        return 0;
    }
    const double2 p = c.pt[i];
    const Loc loc = locate_point(m, c.id[i], p, true);
    u32 hit = NONE;
    bool done = false;
    switch (loc.kind) {
        case 0:  // Inside
            c.loc[i] = loc.tri;
            c.lkind[i] = 0;
            c.ledge[i] = -1;
            done = true;
            break;
        case 1: {  // OnEdge
            const u32 s = has_seg(m.tv[loc.tri], loc.edge) ? comp(m.ts[loc.tri], loc.edge) : NONE;
            if (s == NONE) {
                c.loc[i] = loc.tri;
                c.lkind[i] = 1;
                c.ledge[i] = (int8_t)loc.edge;
                done = true;
            } else {
                hit = s;
            }
            break;
        }
        case 4:
            hit = loc.seg;
            break;
        default:  // OnVertex, OutsideHull
            c.alive[i] = 0;
            done = true;
            break;
    }
    if (!done) {
        // Interception: split the blocking subsegment (refine.hpp:329-334).
        c.kind[i] = 0;
        c.id[i] = hit;
        c.pt[i] = subseg_mid(m, hit);
        c.key[i] = make_key(1, subseg_len(m, hit));
        c.loc[i] = m.stri[hit];
        c.lkind[i] = 4;
        c.ledge[i] = -1;
    }
    return loc.steps;
}

__device__ __forceinline__ u64 tie_of(const DevCands& c, u32 i) {
    return ((u64)c.tie[i] << 32) | (u64)i;
}

// The claim tables: ckey and ctie of triangle t share one 16-byte record
// (TriAux: ctie = ckey + 1, both indexed by cslot(t)), so a check reads one
// sector and a reset writes one; the rewrite table's fkey / ftie likewise.
__device__ __forceinline__ size_t cslot(u32 t) { return 2ull * t; }
// the whole {key, tie} record of t: one 16-byte load / store
__device__ __forceinline__ ulonglong2 claim_rec(const u64* key_tab, u32 t) {
    return reinterpret_cast<const ulonglong2*>(key_tab)[t];
}
__device__ __forceinline__ void claim_clear(u64* key_tab, u32 t) {
    reinterpret_cast<ulonglong2*>(key_tab)[t] = make_ulonglong2(0ull, ~0ull);
}

__device__ __forceinline__ void claim_max_one(const DevCands& c, u32 i, u64* ckey) {
    if (c.alive[i]) atomicMax((ull*)&ckey[cslot(c.loc[i])], (ull)c.key[i]);
}

__device__ __forceinline__ void claim_tie_one(const DevCands& c, u32 i, const u64* ckey,
                                              u64* ctie) {
    if (c.alive[i]) {
        const u32 t = c.loc[i];
        if (ckey[cslot(t)] == c.key[i]) atomicMin((ull*)&ctie[cslot(t)], (ull)tie_of(c, i));
    }
}

// Returns 1 if the candidate owns its triangle.
__device__ __forceinline__ u32 claim_check_one(const DevCands& c, u32 i, const u64* ckey,
                                               const u64* ctie) {
    if (!c.alive[i]) return 0;
    const u32 t = c.loc[i];
    (void)ctie;
    const ulonglong2 r = claim_rec(ckey, t);
    const bool own = r.x == c.key[i] && r.y == tie_of(c, i);
    if (!own) c.alive[i] = 0;
    return own ? 1u : 0u;
}

__device__ __forceinline__ void claim_reset_one(const DevCands& c, u32 i, u32 nT, u64* ckey,
                                                u64* ctie) {
    const u32 t = c.loc[i];
    (void)ctie;
    if (t < nT) claim_clear(ckey, t);
}

__device__ __forceinline__ ull bloom_bit(u32 t) { return 1ull << ((t * 0x9E3779B1u) >> 26); }

// Per candidate: FIFO BFS of triangles whose circumcircle strictly contains
// the point (the located triangle always belongs), never crossing a
// subsegment, at most ncav+1 triangles.  Processing a FIFO queue item by item
// with emissions appended in (source, slot) order visits triangles in exactly
// the window order of expand() (expandlist.hpp:98-152), so the region -- and
// hence the claim set -- is the reference's, including when the cap binds.
// The region is exactly the reference's in both uses (extras 0: the parity
// hooks; 2: refinement, where the rewrite table rw_*_one guards the split).
// Returns the BFS region size (cavity visits).
__device__ __forceinline__ u32 cavity_bfs_one(const DevMesh& m, const DevCands& c, u32 i,
                                              u32 ncav, int extras, u32 rs, u32* regions,
                                              u32* region_len, u32* bfs_len, u64* ckey) {
    u32 len = 0, blen = 0;
    if (c.alive[i]) {
        u32* reg = regions + (size_t)i * rs;
        // the region is built in a thread-local array (L1) and written out
        // once: membership tests against global memory would cost an L2
        // round trip each
        u32 lreg[MAX_CAVITY_N + 1 + MAX_CLAIM_EXTRA];
        u32 queue[1 + 3 * (MAX_CAVITY_N + 1)];
        u32 head = 0, tail = 0;
        // 64-bit membership filter of lreg: a triangle whose bit is clear is
        // not in the region, so most membership scans of lreg are skipped
        ull bloom = 0;
        const u32 located = c.loc[i];
        const double2 p = c.pt[i];
        const u64 key = c.key[i];
        queue[tail++] = located;
        while (head < tail && len <= ncav) {
            const u32 t = queue[head++];
            // issue the record loads together (one dependent level); the
            // subsegment bits of tv.w stand in for the ts record
            const uint4 tv = m.tv[t];
            const uint4 tn = m.tn[t];
            bool pred = t == located;
            if (!pred && tv.w) pred = incircle(m.xy[tv.x], m.xy[tv.y], m.xy[tv.z], p) > 0;
            if (!pred) continue;
            const ull tb = bloom_bit(t);
            if (bloom & tb) {
                bool in = false;
                for (u32 k = 0; k < len; ++k) in |= lreg[k] == t;
                if (in) continue;
            }
            lreg[len++] = t;
            bloom |= tb;
            atomicMax((ull*)&ckey[cslot(t)], (ull)key);
            for (int e = 0; e < 3; ++e) {
                if (has_seg(tv, e)) continue;
                const u32 cc = comp(tn, e);
                if (cc == NONE) continue;
                const u32 nb = etri(cc);
                if (bloom & bloom_bit(nb)) {
                    bool seen = false;
                    for (u32 k = 0; k < len; ++k) seen |= lreg[k] == nb;
                    if (seen) continue;
                }
                queue[tail++] = nb;
            }
        }
        for (u32 k = 0; k < len; ++k) reg[k] = lreg[k];
        blen = len;
    }
    region_len[i] = len;
    if (bfs_len) bfs_len[i] = blen;
    return blen;
}

__device__ __forceinline__ void cavity_tie_one(const DevCands& c, u32 i, u32 rs,
                                               const u32* regions, const u32* region_len,
                                               const u64* ckey, u64* ctie) {
    const u32 len = region_len[i];
    if (!len) return;
    const u64 key = c.key[i];
    const u64 tie = tie_of(c, i);
    const u32* reg = regions + (size_t)i * rs;
    // the key loads first (independent, issued together), then the atomics:
    // interleaved, every load would wait behind the previous atomic
    for (u32 k0 = 0; k0 < len; k0 += 64) {
        const u32 n = min(len - k0, 64u);
        ull hold = 0;   // bit k: this candidate holds the key of reg[k0 + k]
#pragma unroll 4
        for (u32 k = 0; k < n; ++k) hold |= (ull)(ckey[cslot(reg[k0 + k])] == key) << k;
        for (u32 k = 0; k < n; ++k)
            if ((hold >> k) & 1ull) atomicMin((ull*)&ctie[cslot(reg[k0 + k])], (ull)tie);
    }
}

// Returns 1 if the candidate owns its whole region (refine.hpp:420-428).
__device__ __forceinline__ u32 cavity_check_one(const DevCands& c, u32 i, u32 rs,
                                                const u32* regions, const u32* region_len,
                                                const u64* ckey, const u64* ctie) {
    const u32 len = region_len[i];
    if (!len || !c.alive[i]) return 0;
    const u64 key = c.key[i];
    const u64 tie = tie_of(c, i);
    const u32* reg = regions + (size_t)i * rs;
    bool own = true;
    // no early exit: the loads of the whole region are issued together
#pragma unroll 4
    for (u32 k = 0; k < len; ++k) {
        const ulonglong2 r = claim_rec(ckey, reg[k]);
        own &= (r.x == key) & (r.y == tie);
    }
    if (!own) c.alive[i] = 0;
    return own ? 1u : 0u;
}

__device__ __forceinline__ void cavity_reset_one(u32 i, u32 rs, const u32* regions,
                                                 const u32* region_len, u64* ckey, u64* ctie) {
    const u32 len = region_len[i];
    const u32* reg = regions + (size_t)i * rs;
    (void)ctie;
    for (u32 k = 0; k < len; ++k) claim_clear(ckey, reg[k]);
}

// ---- isolated insertion claims (GDP2D_INSERT_ISOLATED) ------------------------
//
// Claim set = the constrained Delaunay cavity of p (BFS of triangles whose
// circumcircle strictly contains p, never crossing a subsegment, as above;
// for a subsegment midpoint also the cavity on the far side of the
// subsegment) + its one-ring (the triangles across every non-subsegment
// boundary edge).  If two survivors own disjoint claim sets, Lawson after
// their splits reaches exactly the Bowyer-Watson result of each point on its
// own cavity: every boundary edge separates p's fan from an untouched ring
// triangle whose circumcircle excludes p, so it is locally Delaunay, and no
// edge can ever join two fresh points (no dependent pair, refine.hpp:589-607).
// While scanning the boundary, a circumcenter that encroaches a splittable
// subsegment on it records the lowest such subsegment (red): the point would
// be redundant after insertion (refine.hpp:555-588), so a surviving
// candidate marks the subsegment instead of inserting (encroachment
// precedence, refine.hpp:786-804).  A cavity that reaches the cap, or a ring
// larger than the region buffer, is flagged unsafe (the batch then runs the
// rollback detection as a fallback).

__device__ __forceinline__ bool in_list(const u32* reg, u32 len, u32 t) {
    bool in = false;
    for (u32 k = 0; k < len; ++k) in |= reg[k] == t;
    return in;
}

// BFS cavity from `seed` appended to reg[len..]; returns false if capped.
// `located` always belongs (as in cavity_filter).
__device__ __forceinline__ bool cavity_bfs_into(const DevMesh& m, u32 seed, bool seed_always,
                                                double2 p, u32 ncav, u32* reg, u32& len, u32 rs) {
    u32 queue[1 + 3 * (MAX_CAVITY_N + 1)];
    u32 head = 0, tail = 0;
    const u32 start = len;
    queue[tail++] = seed;
    while (head < tail) {
        if (len - start > ncav) return false;   // cap reached with work left
        const u32 t = queue[head++];
        const uint4 tv = m.tv[t];
        bool pred = seed_always && t == seed;
        if (!pred && tv.w) pred = incircle(m.xy[tv.x], m.xy[tv.y], m.xy[tv.z], p) > 0;
        if (!pred) continue;
        if (in_list(reg, len, t)) continue;
        if (len >= rs) return false;
        reg[len++] = t;
        const uint4 tn = m.tn[t];
        const uint4 ts = load_ts(m, t, m.tv[t]);
        for (int e = 0; e < 3; ++e) {
            if (comp(ts, e) != NONE) continue;
            const u32 cc = comp(tn, e);
            if (cc == NONE) continue;
            const u32 nb = etri(cc);
            if (in_list(reg, len, nb)) continue;
            if (tail >= 1 + 3 * (MAX_CAVITY_N + 1)) return false;
            queue[tail++] = nb;
        }
    }
    return true;
}

// ring == false (GDP2D_INSERT_PRECEDENCE): the claim set is the reference's
// (cavity_bfs_one with extras); only the encroachment precedence is added and
// the rollback detection still runs for dependent pairs.
template <int MODE>
__device__ __forceinline__ u32 cavity_claims_one(const DevMesh& m, const DevCands& c, u32 i,
                                                 u32 ncav, u32 rs, u32* regions,
                                                 u32* region_len, u64* ckey, u64 depth_cap,
                                                 bool ring = true) {
    u32 len = 0, blen = 0;
    c.red[i] = NONE;
    c.unsafe[i] = 0;
    if (c.alive[i]) {
        u32* reg = regions + (size_t)i * rs;
        const u32 located = c.loc[i];
        const double2 p = c.pt[i];
        bool ok = cavity_bfs_into(m, located, true, p, ncav, reg, len, rs);
        if (!ring) {
            // reference claim set: the (possibly capped) BFS region + the far
            // side of a split edge; the precedence test reads the region's
            // subsegment edges
            blen = len;
            u32 red = NONE;
            if (c.kind[i] == 1) {
                for (u32 k = 0; k < blen; ++k) {
                    const uint4 ts = load_ts(m, reg[k], m.tv[reg[k]]);
                    for (int e = 0; e < 3; ++e) {
                        const u32 s = comp(ts, e);
                        if (s == NONE || s >= red) continue;
                        const uint2 sv = m.sv[s];
                        if (encroaches<MODE>(m.xy[sv.x], m.xy[sv.y], p) &&
                            (u64)m.sdepth[s] < depth_cap && subseg_split_ok(m, s, subseg_mid(m, s)))
                            red = s;
                    }
                }
            }
            c.red[i] = red;
            ok = false;   // take the reference fallback below (extras), no unsafe flag
        }
        if (ok && c.kind[i] == 0) {
            // subsegment midpoint: the cavity on the far side of s as well
            const u32 s = c.id[i];
            const int e = seg_slot(m.ts[located], s);
            if (e >= 0) {
                const u32 cc = comp(m.tn[located], e);
                if (cc != NONE) ok = cavity_bfs_into(m, etri(cc), true, p, ncav, reg, len, rs);
            }
        }
        blen = len;
        // one-ring across non-subsegment boundary edges; encroachment precedence
        u32 red = NONE;
        const bool is_cc = c.kind[i] == 1;
        for (u32 k = 0; k < blen && ok; ++k) {
            const u32 t = reg[k];
            const uint4 tn = m.tn[t];
            const uint4 ts = load_ts(m, t, m.tv[t]);
            for (int e = 0; e < 3; ++e) {
                const u32 s = comp(ts, e);
                if (s != NONE) {
                    if (is_cc && s < red) {
                        const uint2 sv = m.sv[s];
                        if (encroaches<MODE>(m.xy[sv.x], m.xy[sv.y], p) &&
                            (u64)m.sdepth[s] < depth_cap && subseg_split_ok(m, s, subseg_mid(m, s)))
                            red = s;
                    }
                    continue;
                }
                const u32 cc = comp(tn, e);
                if (cc == NONE) continue;
                const u32 nb = etri(cc);
                if (in_list(reg, len, nb)) continue;
                if (len >= rs) {
                    ok = false;
                    break;
                }
                reg[len++] = nb;
            }
        }
        if (ring) {
            c.red[i] = red;
            c.unsafe[i] = ok ? 0 : 1;
        }
        if (!ok) {
            // fall back to the reference claim set: the capped region (first
            // ncav + 1 triangles of the BFS); the rewrite table guards the
            // far side of a split edge
            len = min(len, ncav + 1);
            blen = len;
        }
        const u64 key = c.key[i];
        for (u32 k = 0; k < len; ++k) atomicMax((ull*)&ckey[cslot(reg[k])], (ull)key);
    }
    region_len[i] = len;
    return blen;
}

// Survivor of an isolated claim set: inserts, unless encroachment precedence
// turns it into a subsegment mark.  Returns 1 = inserts, 0 = not; *marked set
// when this candidate newly marked a subsegment; *unsafe when it inserts from
// a capped (non-isolated) claim set.
__device__ __forceinline__ u32 isolated_check_one(const DevMesh& m, const DevCands& c, u32 i,
                                                  u32 rs, const u32* regions,
                                                  const u32* region_len, const u64* ckey,
                                                  const u64* ctie, u32& marked, u32& unsafe) {
    if (!cavity_check_one(c, i, rs, regions, region_len, ckey, ctie)) return 0;
    const u32 red = c.red[i];
    if (red != NONE) {
        c.alive[i] = 0;
        if (atomicExch(&m.senc[red], 1u) == 0u) marked = 1;
        return 0;
    }
    if (c.unsafe[i]) unsafe = 1;
    return 1;
}

// ---- rewrite table -------------------------------------------------------------
//
// Two splits must never rewrite the same triangle: a circumcenter rewrites its
// located triangle (and the far side when it lies on an edge), a subsegment
// midpoint its located triangle and the triangle across the subsegment.  The
// cavity claims (the reference's, main table) do not cover the far sides, so
// every candidate also claims its rewritten triangles, with its priority, in a
// second table; a survivor must own both.  Unlike adding the far side to the
// cavity claim, this only blocks a circumcenter whose own split would touch a
// midpoint's far triangle, not one whose cavity merely reaches it (the
// reference inserts both, serially, refine.hpp:492-539).

__device__ __forceinline__ void rw_set(const DevMesh& m, const DevCands& c, u32 i, u32& t,
                                       u32& far) {
    t = c.loc[i];
    far = NONE;
    int e = -1;
    if (c.kind[i] == 0) e = seg_slot(m.ts[t], c.id[i]);
    else if (c.lkind[i] == 1) e = c.ledge[i];
    if (e >= 0) {
        const u32 cc = comp(m.tn[t], e);
        if (cc != NONE) far = etri(cc);
    }
}

__device__ __forceinline__ void rw_claim_one(const DevMesh& m, const DevCands& c, u32 i,
                                             u64* fkey) {
    u32 far = NONE;
    if (c.alive[i]) {
        u32 t;
        rw_set(m, c, i, t, far);
        atomicMax((ull*)&fkey[cslot(t)], (ull)c.key[i]);
        if (far != NONE) atomicMax((ull*)&fkey[cslot(far)], (ull)c.key[i]);
    }
    c.far[i] = far;
}

__device__ __forceinline__ void rw_tie_one(const DevCands& c, u32 i, const u64* fkey, u64* ftie) {
    if (!c.alive[i]) return;
    const u64 key = c.key[i], tie = tie_of(c, i);
    const u32 t = c.loc[i], far = c.far[i];
    if (fkey[cslot(t)] == key) atomicMin((ull*)&ftie[cslot(t)], (ull)tie);
    if (far != NONE && fkey[cslot(far)] == key) atomicMin((ull*)&ftie[cslot(far)], (ull)tie);
}

__device__ __forceinline__ bool rw_owns(const DevCands& c, u32 i, const u64* fkey,
                                        const u64* ftie) {
    const u64 key = c.key[i], tie = tie_of(c, i);
    const u32 t = c.loc[i], far = c.far[i];
    (void)ftie;
    const ulonglong2 r = claim_rec(fkey, t);
    const ulonglong2 rf = far != NONE ? claim_rec(fkey, far) : make_ulonglong2(key, tie);
    return r.x == key && r.y == tie && rf.x == key && rf.y == tie;
}

__device__ __forceinline__ void rw_reset_one(const DevCands& c, u32 i, u32 nT, u64* fkey,
                                             u64* ftie) {
    const u32 t = c.loc[i], far = c.far[i];
    (void)ftie;
    if (t < nT) claim_clear(fkey, t);
    if (far != NONE && far < nT) claim_clear(fkey, far);
}

// Needs of one surviving candidate (refine.hpp:493-539): subsegments that hit
// the depth cap or fail subsegment_split_ok are abandoned (:501-506).
// Returns 1 if the candidate was dropped.
__device__ __forceinline__ u32 plan_one(const DevMesh& m, const DevCands& c, u32 i, u64 depth_cap,
                                        u32& nv, u32& nt, u32& ns) {
    nv = nt = ns = 0;
    u32 dropped = 0;
    if (c.alive[i]) {
        if (c.kind[i] == 0) {
            const u32 s = c.id[i];
            if (!m.salive[s]) {
                dropped = 1;
            } else if ((u64)m.sdepth[s] >= depth_cap || !subseg_split_ok(m, s, c.pt[i])) {
                m.senc[s] = 0;
                dropped = 1;
            } else {
                const u32 t = c.loc[i];
                const int e = seg_slot(m.ts[t], s);
                const bool far = comp(m.tn[t], e) != NONE;
                nv = 1;
                nt = far ? 2 : 1;
                ns = 2;
            }
        } else if (c.lkind[i] == 0) {
            nv = 1;
            nt = 2;
        } else if (c.lkind[i] == 1) {
            const bool far = comp(m.tn[c.loc[i]], c.ledge[i]) != NONE;
            nv = 1;
            nt = far ? 2 : 1;
        }
        if (!nv) c.alive[i] = 0;
    }
    return dropped;
}

}  // namespace gdp2d
