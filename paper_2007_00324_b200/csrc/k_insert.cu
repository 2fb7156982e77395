// k_insert.cu -- Line 8 of Algorithm 1: parallel insertion with Flip-Flop
// (insert_batch, refine.hpp:464-610).
//
// Every mesh mutation is a LOCAL REWRITE of a set of triangles its thread
// owns exclusively (cavity claims for splits, pair claims for flips, star
// claims for removals).  A rewrite runs in two kernels:
//   phase A (owner thread): rewrite the owned triangles + allocate new ones;
//     references leaving the owned set keep the OLD outer (tri<<2|edge) and
//     are flagged pending in tn.w; every old boundary slot records where its
//     edge went in emap (TriAux::se); owned triangles are stamped with the round.
//   phase B (launch_fixup, one thread per touched triangle): a pending ref to
//     a triangle stamped this round is translated through its emap; a ref to
//     an untouched triangle stays and gets its back-pointer written (single
//     writer per edge).  vert_tri / seg_tri are recomputed as atomicMin over
//     touched triangles, so ids are deterministic run to run.
// Mirrors: split_triangle_with mesh.hpp:323-346, split_edge_with :358-401,
// split_subsegment :405-425, flip :210-258, remove_free_vertex + flop
// :261-304,442-466, lawson_fixpoint cdt.hpp:111-123.
#include <cooperative_groups.h>

#include <algorithm>

#include "gdp2d_collect.cuh"
#include "gdp2d_phases.cuh"
#include "gdp2d_rewrite.cuh"
#include "scan.cuh"

namespace cg = cooperative_groups;

// CTAs per SM the split/Lawson kernel is compiled for (register budget
// 65536 / (256 * MINB)); measured on B200, see DESIGN.md.
#ifndef GDP2D_SPLIT_MINB
#define GDP2D_SPLIT_MINB 2
#endif

namespace gdp2d {

// ---- planning + phase-1 splits ----------------------------------------------------

// One surviving candidate's phase-1 insertion (refine.hpp:492-539).
// Returns 1 = midpoint, 2 = circumcenter, 0 = nothing.
// slots (optional): the [touched, work] list slots reserved for it
// (split_appends gives the sizes).
__device__ __forceinline__ int apply_one(const DevMesh& m, const DevCands& c, u32 i, u32 batch,
                                         u32 round, const InsertBufs& b, const TriAux& x,
                                         const FreshInfo& f, const WorkLists& w, RoundCtr* rc,
                                         int seed, Counters* ctr, const u32* slots = nullptr) {
    if (!b.nv[i]) return 0;
    const u32 wv = m.nV + b.ov[i];
    const u32 nt0 = m.nT + b.ot[i];
    const double2 p = c.pt[i];
    m.xy[wv] = p;
    m.vkind[wv] = c.kind[i] == 0 ? 1 : 2;
    m.vbirth[wv] = batch;
    m.valive[wv] = 1;
    const u32 fi = b.ov[i];
    f.key[fi] = c.key[i];
    f.tie[fi] = ((u64)c.tie[i] << 32) | i;
    f.cc[fi] = c.kind[i] == 1;
    f.removed[fi] = 0;
    f.mark[fi] = 0;
    f.dirty[fi] = 0;   // becomes a detection suspect through fixup_one
    const u32 t = c.loc[i];
    if (c.kind[i] == 0) {
        const u32 s = c.id[i];
        const int e = seg_slot(m.ts[t], s);
        const uint4 tv = m.tv[t];
        const u32 bb = comp(tv, nxt(e)), ccv = comp(tv, prv(e));
        const u32 s_bw = m.nS + b.os[i], s_wc = s_bw + 1;
        const u32 par = m.sparent[s], dep = m.sdepth[s] + 1;
        m.sv[s_bw] = make_uint2(bb, wv);
        m.sv[s_wc] = make_uint2(wv, ccv);
        m.sparent[s_bw] = par;
        m.sparent[s_wc] = par;
        m.senc[s_bw] = 0;
        m.senc[s_wc] = 0;
        m.salive[s_bw] = 1;
        m.salive[s_wc] = 1;
        m.sdepth[s_bw] = dep;
        m.sdepth[s_wc] = dep;
        m.stri[s_bw] = NONE;
        m.stri[s_wc] = NONE;
        m.salive[s] = 0;
        m.senc[s] = 0;
        split_edge_A(m, x, w, t, e, wv, nt0, nt0 + 1, s_bw, s_wc, round, rc, seed, ctr, slots);
        return 1;
    }
    if (c.lkind[i] == 0) {
        split_triangle_A(m, x, w, t, wv, nt0, nt0 + 1, round, rc, seed, ctr, slots);
    } else {
        split_edge_A(m, x, w, t, c.ledge[i], wv, nt0, nt0 + 1, NONE, NONE, round, rc, seed, ctr,
                     slots);
    }
    return 2;
}

// The list appends apply_one(seed = 1) makes for candidate i: touched
// triangles and Lawson seeds (split_triangle_A / split_edge_A).
__device__ __forceinline__ void split_appends(const DevCands& c, u32 i, const InsertBufs& b,
                                              u32& nt_out, u32& nw_out) {
    nt_out = nw_out = 0;
    if (!b.nv[i]) return;
    const u32 nt = b.nt[i];   // 2: the split edge has a far side (or 1 -> 3)
    if (c.kind[i] == 0) {             // subsegment midpoint: the link edges only
        nt_out = 2 * nt;
        nw_out = 2 * nt;
    } else if (c.lkind[i] == 0) {     // 1 -> 3
        nt_out = 3;
        nw_out = 3;
    } else {                          // point on an edge: every edge of the new triangles
        nt_out = 2 * nt;
        nw_out = 6 * nt;
    }
}

// Whole Lawson fixpoint in ONE persistent cooperative launch: each round is
// test+claim | apply | post+fixup separated by grid-wide barriers (which also
// fence and invalidate L1), so the ~30 rounds of a batch cost no host round
// trips.  Per-round counters live in rcs[r] (zeroed by the host).  Stops when
// the next work list is empty or after max_rounds (the host then continues).
__global__ void __launch_bounds__(LAWSON_BLOCK) k_lawson_persistent(
    const __grid_constant__ DevMesh m, u32 round0, u32 cur0, u32 n0, u32 max_rounds,
    const __grid_constant__ TriAux x, const __grid_constant__ WorkLists w, RoundCtr* rcs,
    u32* result, Counters* ctr) {
    cg::grid_group g = cg::this_grid();
    const u32 tid = (u32)g.thread_rank(), nthr = (u32)g.size();
    u32 n = n0, cur = cur0, r = 0;
    u32 flipped = 0;
    for (; r < max_rounds && n > 0; ++r) {
        RoundCtr* rc = rcs + r;
        const u32 round = round0 + r;
        const u32* wl = w.w[cur];
        const u32 tid0 = tid - threadIdx.x;
        flip_test_waves<LAWSON_BLOCK>(m, wl, n, round, tid0, nthr, x, w, rc, ctr);
        g.sync();
        const u32 nc = min(*(volatile u32*)&rc->cand, w.cap);
        flipped += flip_apply_waves<LAWSON_BLOCK>(m, nc, round, cur ^ 1u, tid0, nthr, x, w, rc, ctr);
        g.sync();
        flip_post_waves<LAWSON_BLOCK>(nc, round, cur ^ 1u, tid0, nthr, x, w, rc, ctr);
        const u32 nt = min(*(volatile u32*)&rc->touched, w.cap);
        for (u32 i = tid; i < nt; i += nthr) fixup_one(m, round, x, w, w.touched[i], 0, 0, rc, ctr);
        g.sync();
        n = *(volatile u32*)&rc->wl_next;
        if (n > w.cap) {
            raise_err(ctr, DERR_WORKLIST_OVERFLOW, n);
            n = 0;
        }
        cur ^= 1u;
    }
    warp_add_ull(&ctr->flips, flipped);
    if (tid == 0) {
        result[0] = r;
        result[1] = cur;
        result[2] = n;
    }
}

int lawson_persistent_grid(int device) {
    static int cached[64] = {0};
    if (device >= 0 && device < 64 && cached[device]) return cached[device];
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lawson_persistent, LAWSON_BLOCK, 0);
    const int g = std::max(1, sms * std::max(1, per_sm));
    if (device >= 0 && device < 64) cached[device] = g;
    return g;
}

void launch_lawson_persistent(const DevMesh& m, u32 round0, u32 cur0, u32 n0, u32 max_rounds,
                              TriAux a, WorkLists w, RoundCtr* rcs, u32* result, Counters* d_ctr,
                              int grid, cudaStream_t st) {
    void* args[] = {(void*)&m, &round0, &cur0, &n0, &max_rounds, &a, &w, &rcs, &result, &d_ctr};
    note_launch();
    cudaLaunchCooperativeKernel((void*)k_lawson_persistent, dim3(grid), dim3(LAWSON_BLOCK), args,
                                0, st);
}

// ---- redundancy detection (refine.hpp:551-608) ----------------------------------------

// Star of v in rotation order (incident_triangles, mesh.hpp:145-171, interior
// case).  Returns the size, 0 if the fan is open or broken, or -1 if it has
// more than cap triangles (st/si are then incomplete).
__device__ __forceinline__ int walk_star(const DevMesh& m, u32 v, u32* st, int* si, int cap) {
    const u32 t0 = m.vtri[v];
    if (t0 == NONE) return 0;
    u32 cur = t0;
    int k = 0;
    do {
        // both records at once: the step's only dependent level
        const uint4 tv = m.tv[cur], tn = m.tn[cur];
        const int i = tv.x == v ? 0 : (tv.y == v ? 1 : (tv.z == v ? 2 : -1));
        if (i < 0) return 0;
        if (k >= cap) return -1;
        st[k] = cur;
        si[k] = i;
        ++k;
        const u32 c = comp(tn, nxt(i));
        if (c == NONE) return 0;
        cur = etri(c);
    } while (cur != t0);
    return k;
}

// The same rotation as a stream: fn(t, i, tv) for every star triangle (i =
// v's slot in t), nothing stored, so a vertex of any degree is handled (a
// disc bounded by an N-gon gives its centre degree N).  Returns the size, or
// 0 if the fan is open or broken (fn may have seen part of it).
static constexpr int STAR_WALK_LIMIT = 1 << 20;
template <class Fn>
__device__ __forceinline__ int stream_star(const DevMesh& m, u32 v, Fn&& fn) {
    const u32 t0 = m.vtri[v];
    if (t0 == NONE) return 0;
    u32 cur = t0;
    int k = 0;
    uint4 tv = m.tv[cur], tn = m.tn[cur];
    do {
        const int i = tv.x == v ? 0 : (tv.y == v ? 1 : (tv.z == v ? 2 : -1));
        if (i < 0 || k >= STAR_WALK_LIMIT) return 0;
        const u32 c = comp(tn, nxt(i));
        // the next step's records (both at once) are loaded before fn runs:
        // fn's own loads and stores cannot delay the walk
        const u32 nx = c == NONE ? t0 : etri(c);
        const uint4 ntv = m.tv[nx], ntn = m.tn[nx];
        fn(cur, i, tv);
        ++k;
        if (c == NONE) return 0;
        cur = nx;
        tv = ntv;
        tn = ntn;
    } while (cur != t0);
    return k;
}

__device__ __forceinline__ bool prio_gt(const FreshInfo& f, u32 a, u32 b) {
    if (f.key[a] != f.key[b]) return f.key[a] > f.key[b];
    return f.tie[a] < f.tie[b];
}

// (a) a same-batch circumcenter that encroaches a splittable subsegment of
// its star is redundant; the lowest-id such subsegment is marked.
// collect_dep != 0 (the any-higher-neighbour rule): the same star walk also
// lists the higher-priority same-batch circumcenters around v (hlist/hcnt,
// 255 = too many), so detect_b_fast needs no second walk.
template <int MODE>
__device__ __noinline__ u32 detect_a_one(const DevMesh& m, u64 depth_cap, u32 V0, u32 F, u32 j,
                                         const FreshInfo& f, Counters* ctr, int collect_dep,
                                         const WorkLists& w) {
    u32 marked = 0;
    uint8_t mark = 0;
    const u32 v = V0 + j;
    if (collect_dep) f.hcnt[j] = 0;
    if (f.cc[j] && !f.removed[j]) {
        // one streamed walk: the lowest-id splittable subsegment on an edge
        // opposite v that v encroaches, and (collect_dep) the higher-priority
        // same-batch circumcenters among the link vertices
        const double2 pv = m.xy[v];
        u32 best = NONE, cnt = 0;
        const int k = stream_star(m, v, [&](u32 t, int i, const uint4& tv) {
            if (collect_dep && cnt != 255u) {
                const u32 x = comp(tv, nxt(i));   // the star's next link vertex
                if (x >= V0 && x < V0 + F) {
                    const u32 jx = x - V0;
                    if (f.cc[jx] && f.removed[jx] != 1 && prio_gt(f, jx, j)) {
                        if (cnt == (u32)DEP_HMAX)
                            cnt = 255u;
                        else
                            f.hlist[(size_t)j * DEP_HMAX + cnt++] = jx;
                    }
                }
            }
            if (!has_seg(tv, i)) return;
            const u32 s = comp(m.ts[t], i);
            if (s >= best) return;
            const uint2 sv = m.sv[s];
            if (!encroaches<MODE>(m.xy[sv.x], m.xy[sv.y], pv)) return;
            if ((u64)m.sdepth[s] >= depth_cap) return;
            if (!subseg_split_ok(m, s, subseg_mid(m, s))) return;
            best = s;
        });
        if (collect_dep) f.hcnt[j] = (uint8_t)cnt;
        if (k == 0 && atomicCAS(&ctr->err_code, 0u, (u32)DERR_OPEN_STAR) == 0u) {
            ctr->err_info = v;
            ctr->dbg[0] = (double)m.vtri[v];
            ctr->dbg[1] = (double)m.valive[v];
            ctr->dbg[2] = (double)j;
            ctr->dbg[3] = pv.x;
            ctr->dbg[4] = pv.y;
        }
        if (best != NONE) {
            mark = 1;
            if (atomicExch(&m.senc[best], 1u) == 0u) {
                marked = 1;
                if (w.dlist) dlist_push(w, best);   // a new candidate for the tail loop
            }
        }
    }
    f.mark[j] = mark;
    return marked;
}

// (b) Delaunay-dependent pairs: a same-batch circumcenter adjacent to a
// higher-priority one (not itself redundant) is removed.
__device__ __noinline__ void detect_b_one(const DevMesh& m, u32 V0, u32 F, u32 j,
                                          const FreshInfo& f) {
    if (!f.cc[j] || f.removed[j] || f.mark[j] == 1) return;
    const u32 v = V0 + j;
    bool dep = false;
    stream_star(m, v, [&](u32, int i, const uint4& tv) {
        const u32 x = comp(tv, nxt(i));
        if (dep || x < V0 || x >= V0 + F) return;
        const u32 jx = x - V0;
        if (!f.cc[jx] || f.removed[jx] == 1 || f.mark[jx] == 1) return;
        if (prio_gt(f, jx, j)) dep = true;
    });
    if (dep) f.mark[j] = 2;
}

// (b) from the list detect_a_one collected: the first higher-priority
// neighbour that is not itself redundant makes v dependent.
__device__ __forceinline__ void detect_b_fast(const DevMesh& m, u32 V0, u32 F, u32 j,
                                              const FreshInfo& f) {
    if (!f.cc[j] || f.removed[j] || f.mark[j] == 1) return;
    const u32 cnt = f.hcnt[j];
    if (cnt == 255) {
        detect_b_one(m, V0, F, j, f);
        return;
    }
    for (u32 q = 0; q < cnt; ++q) {
        if (f.mark[f.hlist[(size_t)j * DEP_HMAX + q]] != 1) {
            f.mark[j] = 2;
            return;
        }
    }
}

// (b) with the priority-MIS rule: a same-batch circumcenter is rolled back
// iff a higher-priority neighbour that STAYS exists.  This is the smallest
// removal set leaving no two adjacent same-batch circumcenters; the
// reference's sequential sweep (refine.hpp:589-607) removes a set between it
// and the "any higher neighbour" rule of detect_b_one (a chain a > b > c loses
// b only, or b and c, depending on the triangle order of the sweep).
// Pass 1 (this function): collect the higher-priority eligible neighbours;
// no neighbour -> kept, else undecided (returned true).
__device__ __noinline__ bool detect_b_mis_one(const DevMesh& m, u32 V0, u32 F, u32 j,
                                              const FreshInfo& f) {
    if (!f.cc[j] || f.removed[j] || f.mark[j] == 1) {
        f.dstat[j] = 2;   // not a live circumcenter of this batch
        return false;
    }
    const u32 v = V0 + j;
    u32 cnt = 0;
    bool overflow = false;
    stream_star(m, v, [&](u32, int i, const uint4& tv) {
        const u32 x = comp(tv, nxt(i));
        if (x < V0 || x >= V0 + F) return;
        const u32 jx = x - V0;
        if (!f.cc[jx] || f.removed[jx] == 1 || f.mark[jx] == 1) return;
        if (prio_gt(f, jx, j)) {
            if (cnt < (u32)DEP_HMAX)
                f.hlist[(size_t)j * DEP_HMAX + cnt++] = jx;
            else
                overflow = true;
        }
    });
    f.hcnt[j] = (uint8_t)cnt;
    if (overflow) {       // cannot track them all: the conservative rule
        f.dstat[j] = 2;
        f.mark[j] = 2;
        return false;
    }
    f.dstat[j] = cnt == 0 ? 1 : 0;
    return cnt != 0;
}

// One MIS round for an undecided vertex; returns true if still undecided.
__device__ __forceinline__ bool mis_round_one(u32 j, const FreshInfo& f) {
    const u32 cnt = f.hcnt[j];
    bool all_removed = true;
    for (u32 q = 0; q < cnt; ++q) {
        const uint8_t s = f.dstat[f.hlist[(size_t)j * DEP_HMAX + q]];
        if (s == 1) {
            f.dstat[j] = 2;
            f.mark[j] = 2;
            return false;
        }
        all_removed &= s == 2;
    }
    if (all_removed) {
        f.dstat[j] = 1;
        return false;
    }
    return true;
}

// Removal list of a detection pass; returns (redundant, dependent) flags.
__device__ __forceinline__ void detect_collect_one(u32 V0, u32 j, const FreshInfo& f,
                                                   const WorkLists& w, RoundCtr* rc, u32& red,
                                                   u32& dep) {
    if (!f.removed[j] && f.mark[j]) {
        const u32 o = agg_reserve(&rc->detect, 1u);
        if (o < w.rm_cap) w.rm[0][o] = V0 + j;
        red = f.mark[j] == 1;
        dep = f.mark[j] == 2;
    }
}

// ---- parallel vertex removal (remove_free_vertex + flop, mesh.hpp:261-304,442-466) ----

// The star claims share the flips' round-tagged claim array (fown, tag
// round << 32 | ~v, atomicMax: the lowest vertex id of the round wins) and
// are never released.
__device__ __forceinline__ void rm_claim_one(const DevMesh& m, const u32* __restrict__ list, u32 i,
                                             u32 V0, u32 round, const TriAux& x,
                                             const FreshInfo& f, const WorkLists& w,
                                             Counters* ctr) {
    const u32 v = list[i];
    u32* st = w.star + (size_t)i * MAX_STAR;
    int si[MAX_STAR];
    const int k = walk_star(m, v, st, si, MAX_STAR);
    w.star_len[i] = k > 0 ? (u32)k : 0u;
    if (k < 0) {
        // Star larger than the ear-clipping buffers: keep the vertex, as the
        // reference does when remove_free_vertex returns false (mesh.hpp:462,
        // refine.hpp:580/601); it is never selected again.
        f.removed[v - V0] = 2;
        atomicAdd(&ctr->rm_kept, 1u);
        return;
    }
    if (k < 3) {
        raise_err(ctr, DERR_OPEN_STAR, v);
        w.star_len[i] = 0;
        return;
    }
    const u64 tag = flip_tag(round, v);
    for (int q = 0; q < k; ++q) atomicMax((ull*)&x.fown[st[q]], (ull)tag);
}

// Remove v by ear-clipping its link polygon: each ear is one degree-reducing
// flip of remove_free_vertex (both orient tests of mesh.hpp:223-225), the
// last three link vertices are the flop.  The k star triangles become k-2
// (ids reused in star order), the last two die.
// Lawson seeds of the rebuilt star go to seed_rc->wl_next (so successive
// removal rounds can accumulate one list for a single Lawson pass).
// What a removal leaves for the caller to append when it reserves the list
// slots itself (grid mode, block_reserve): deferred, or `created` rebuilt
// triangles (touched + their 3 * created edges as Lawson seeds).
struct RmOut {
    u32 defer;
    int created;
};

// touched slot ot (NONE: already pushed) and seed slot os of a removal's
// rebuilt star st[0..created).
__device__ __forceinline__ void rm_appends(const WorkLists& w, u32 widx, const u32* st,
                                           int created, u32 ot, u32 os, Counters* ctr) {
    if (ot != NONE)
        for (int ci = 0; ci < created; ++ci)
            if (ot + ci < w.cap) w.touched[ot + ci] = st[ci];
    const u32 ns = 3u * (u32)created;
    if (os + ns > w.cap) {
        raise_err(ctr, DERR_WORKLIST_OVERFLOW, os);
        return;
    }
    for (int ci = 0; ci < created; ++ci)
        for (int e = 0; e < 3; ++e) w.w[widx][os + 3 * ci + e] = enc(st[ci], e);
}

// N: capacity of the thread-local link arrays.  The common small star runs
// with N = 16 (a compact local frame that stays in L1); larger stars take the
// MAX_STAR instantiation (rm_apply_one dispatches on the star size).
// WARP (a round of few removals, so latency-bound): the 32 lanes of a warp
// remove ONE vertex.  Every lane holds the link polygon and does the same
// bookkeeping; the ear search tests the first 32 ears from head in parallel
// (lane l: the l-th) and takes the first that passes -- the serial order,
// so the mesh is identical -- and lane 0 alone writes.
template <int N, bool WARP>
__device__ __noinline__ u32 rm_apply_one_n(const DevMesh& m, const u32* __restrict__ list, u32 i,
                                           u32 round, u32 V0, u32 widx, u32 next_list,
                                           const TriAux& x, const FreshInfo& f,
                                           const WorkLists& w, RoundCtr* rc, Counters* ctr,
                                           RoundCtr* seed_rc, RmOut* out) {
    static_assert(!WARP || N <= 32, "warp-mode link polygons fit one alive mask");
    const u32 lane = WARP ? (threadIdx.x & 31u) : 0u;
    const bool lead = lane == 0;
    u32 done = 0;
    {
        const u32 v = list[i];
        const u32* st = w.star + (size_t)i * MAX_STAR;
        const int k = (int)w.star_len[i];
        bool own = k >= 3;
        const u64 tag = flip_tag(round, v);
        // independent loads, no early exit: the claims arrive together
#pragma unroll 8
        for (int q = 0; q < k; ++q) own &= x.fown[st[q]] == tag;
        if (k >= 3 && !own) {
            if (!lead) {
            } else if (out) {
                out->defer = 1;
            } else {
                const u32 o = agg_reserve(&rc->rm_next, 1u);
                if (o < w.rm_cap) w.rm[next_list][o] = v;
            }
        } else if (own) {
            // Link polygon, CCW: L[j] = p_j; link edge j = (L[j], L[j+1]).
            u32 L[N], R[N], SG[N], ORG[N];
            uint8_t PK[N];  // 1 = old outer ref, 2 = local (idx<<2|slot), 0 = none
            int NX[N], PV[N];
            double2 XY[N];  // link vertex coordinates, gathered once
            // records of the whole star first (independent loads), then the
            // link coordinates: two dependent levels instead of 2k
#pragma unroll 4
            for (int q = 0; q < k; ++q) {
                const u32 t = st[q];
                const uint4 tv = m.tv[t], tn = m.tn[t], ts = load_ts(m, t, tv);
                const int iv = tv.x == v ? 0 : (tv.y == v ? 1 : 2);
                L[q] = comp(tv, nxt(iv));
                R[q] = comp(tn, iv);
                PK[q] = R[q] == NONE ? 0 : 1;
                SG[q] = comp(ts, iv);
                ORG[q] = 4 * t + 1 + iv;   // word of emap slot iv in TriAux::se
                NX[q] = q + 1 == k ? 0 : q + 1;
                PV[q] = q == 0 ? k - 1 : q - 1;
            }
#pragma unroll 4
            for (int q = 0; q < k; ++q) XY[q] = m.xy[L[q]];
            // created triangles (local): vertices, refs, kinds, segs
            u32 CV[N][3];
            u32 CN[N][3];
            uint8_t CK[N][3];
            u32 CS[N][3];
            const double2 pv = m.xy[v];
            int cnt = k, head = 0, created = 0;
            bool ok = true;
            // Bind link edge `le` as slot `slot` of created triangle `ci`.
            auto bind = [&](int ci, int slot, int le) {
                const u32 tid = st[ci];
                CS[ci][slot] = SG[le];
                if (PK[le] == 2) {
                    const int oi = (int)(R[le] >> 2), os = (int)(R[le] & 3u);
                    CN[ci][slot] = enc(st[oi], os);
                    CK[ci][slot] = 0;
                    CN[oi][os] = enc(tid, slot);
                } else {
                    CN[ci][slot] = R[le];
                    CK[ci][slot] = PK[le];
                }
                if (lead && ORG[le] != NONE) x.se[ORG[le]] = enc(tid, slot);
            };
            u32 alive = N >= 32 ? ~0u : ((1u << k) - 1u);   // WARP: link positions left
            while (cnt > 3 && ok) {
                int j = head;
                bool found = false;
                if (WARP) {
                    // the first passing ear from head, 32 ears at a time: the
                    // l-th remaining position from head is the l-th set bit of
                    // the alive mask rotated to head
                    const u32 rot = head == 0 ? alive
                                              : ((alive >> head) | (alive << (k - head))) &
                                                    (k >= 32 ? ~0u : ((1u << k) - 1u));
                    for (int pass = -1; pass < 2 && !found; ++pass) {
                        bool pl = false;
                        int jl = 0;
                        if ((int)lane < cnt) {
                            const int sb = (int)__fns(rot, 0, (int)lane + 1);
                            jl = head + sb >= k ? head + sb - k : head + sb;
                            const int a = PV[jl], c = NX[jl];
                            const double2 pa = XY[a], pj = XY[jl], pc = XY[c];
                            const int side = orient2d(pa, pc, pv);
                            if (orient2d(pa, pj, pc) > 0 && (side > 0 || (pass == 1 && side == 0))) {
                                pl = true;
                                if (pass < 0)
                                    for (int q = NX[c]; q != a && pl; q = NX[q])
                                        pl = incircle(pa, pj, pc, XY[q]) <= 0;
                            }
                        }
                        const u32 bal = __ballot_sync(0xFFFFFFFFu, pl);
                        if (bal) {
                            j = __shfl_sync(0xFFFFFFFFu, jl, __ffs(bal) - 1);
                            found = true;
                        }
                    }
                    if (!found) {
                        ok = false;
                        break;
                    }
                }
                // Pass -1: a strict ear whose circumcircle holds no other
                // vertex of the remaining link polygon -- an edge of the
                // polygon's Delaunay triangulation.  Clipping only such ears
                // rebuilds the hole exactly as remove_free_vertex + Lawson on
                // the ring would (refine.hpp:442-456: the CDT around a removed
                // vertex is the polygon's), so the Lawson pass after the
                // removal round finds nothing left to flip.
                // Pass 0: a strict ear = one valid flip of remove_free_vertex.
                // Pass 1 (degenerate stars only, e.g. a point that was inserted
                // exactly on an edge): v may lie ON the new diagonal -- the
                // final hole triangulation is still valid because v leaves.
                for (int pass = -1; pass < 2 && !found && !WARP; ++pass) {
                    j = head;
                    for (int it = 0; it < cnt; ++it) {
                        const int a = PV[j], c = NX[j];
                        const double2 pa = XY[a], pj = XY[j], pc = XY[c];
                        const int side = orient2d(pa, pc, pv);
                        if (orient2d(pa, pj, pc) > 0 && (side > 0 || (pass == 1 && side == 0))) {
                            bool delaunay = true;
                            if (pass < 0) {
                                for (int q = NX[c]; q != a && delaunay; q = NX[q])
                                    delaunay = incircle(pa, pj, pc, XY[q]) <= 0;
                            }
                            if (delaunay) {
                                found = true;
                                break;
                            }
                        }
                        j = NX[j];
                    }
                }
                if (!found) {
                    ok = false;
                    break;
                }
                const int a = PV[j], c = NX[j];
                const int ci = created++;
                CV[ci][0] = L[a];
                CV[ci][1] = L[j];
                CV[ci][2] = L[c];
                bind(ci, 0, j);   // opposite L[a]: (L[j], L[c])
                bind(ci, 2, a);   // opposite L[c]: (L[a], L[j])
                CS[ci][1] = NONE; // diagonal (L[c], L[a]) -- bound later
                CN[ci][1] = NONE;
                CK[ci][1] = 0;
                // the remaining polygon's edge (L[a], L[c]) is this diagonal
                R[a] = ((u32)ci << 2) | 1u;
                PK[a] = 2;
                SG[a] = NONE;
                ORG[a] = NONE;
                NX[a] = c;
                PV[c] = a;
                if (head == j) head = c;
                alive &= ~(1u << (j & 31));
                --cnt;
            }
            if (ok) {
                const int a = head, b = NX[a], c = NX[b];
                const int ci = created++;
                CV[ci][0] = L[a];
                CV[ci][1] = L[b];
                CV[ci][2] = L[c];
                bind(ci, 0, b);
                bind(ci, 1, c);
                bind(ci, 2, a);
                ok = orient2d(XY[a], XY[b], XY[c]) > 0;
            }
            if (!lead) {
            } else if (!ok) {
                // No flippable incident edge (degenerate star): like
                // remove_free_vertex returning false (mesh.hpp:462), keep the
                // vertex; it is never selected again.
                f.removed[v - V0] = 2;
                atomicAdd(&ctr->rm_kept, 1u);
                if (w.dbg && atomicCAS(reinterpret_cast<ull*>(w.dbg), 0ull, 1ull) == 0ull) {
                    w.dbg[1] = k;
                    w.dbg[2] = pv.x;
                    w.dbg[3] = pv.y;
                    for (int q = 0; q < k; ++q) {
                        const uint4 tv = m.tv[st[q]];
                        const int iv = tv.x == v ? 0 : (tv.y == v ? 1 : 2);
                        const double2 pq = m.xy[comp(tv, nxt(iv))];
                        w.dbg[4 + 2 * q] = pq.x;
                        w.dbg[5 + 2 * q] = pq.y;
                    }
                }
            } else {
                for (int q = 0; q < k; ++q) x.se[4 * (st[q])] = round;
                for (int ci = 0; ci < created; ++ci) {
                    const u32 pend = (CK[ci][0] == 1 ? 1u : 0u) | (CK[ci][1] == 1 ? 2u : 0u) |
                                     (CK[ci][2] == 1 ? 4u : 0u);
                    write_tri(m, st[ci], CV[ci][0], CV[ci][1], CV[ci][2], CN[ci][0], CN[ci][1],
                              CN[ci][2], pend, CS[ci][0], CS[ci][1], CS[ci][2], w.vtri_from);
                }
                for (int q = created; q < k; ++q) {
                    m.tv.words(st[q])[3] = 0;   // dead (no read-modify-write)
                    m.tflag[st[q]] = 2;
                }
                m.valive[v] = 0;
                m.vtri[v] = NONE;
                f.removed[v - V0] = 1;
                if (out) {
                    out->created = created;   // the caller appends (rm_appends)
                } else {
                    push_touched(w, st, created, rc);
                    // every edge of the rebuilt hole seeds the Lawson pass: one
                    // reservation for all of them
                    const u32 ns = 3u * (u32)created;
                    rm_appends(w, widx, st, created, NONE, agg_reserve(&seed_rc->wl_next, ns),
                               ctr);
                }
                done = 1;
            }
        }
    }
    return done;
}

__device__ __forceinline__ u32 rm_apply_one(const DevMesh& m, const u32* __restrict__ list, u32 i,
                                            u32 round, u32 V0, u32 widx, u32 next_list,
                                            const TriAux& x, const FreshInfo& f,
                                            const WorkLists& w, RoundCtr* rc, Counters* ctr,
                                            RoundCtr* seed_rc, RmOut* out = nullptr) {
    if (w.star_len[i] <= 16u)
        return rm_apply_one_n<16, false>(m, list, i, round, V0, widx, next_list, x, f, w, rc, ctr,
                                         seed_rc, out);
    return rm_apply_one_n<MAX_STAR, false>(m, list, i, round, V0, widx, next_list, x, f, w, rc,
                                           ctr, seed_rc, out);
}

// Removal i by the whole calling warp (every lane calls; lane 0 returns the count).
__device__ __forceinline__ u32 rm_apply_warp(const DevMesh& m, const u32* __restrict__ list, u32 i,
                                             u32 round, u32 V0, u32 widx, u32 next_list,
                                             const TriAux& x, const FreshInfo& f,
                                             const WorkLists& w, RoundCtr* rc, Counters* ctr,
                                             RoundCtr* seed_rc) {
    if (w.star_len[i] <= 16u)
        return rm_apply_one_n<16, true>(m, list, i, round, V0, widx, next_list, x, f, w, rc, ctr,
                                        seed_rc, nullptr);
    if ((threadIdx.x & 31u) != 0u) return 0;
    return rm_apply_one_n<MAX_STAR, false>(m, list, i, round, V0, widx, next_list, x, f, w, rc,
                                           ctr, seed_rc, nullptr);
}

// =====================================================================================
// The whole insertion phase (Line 8: refine.hpp:464-610) as ONE persistent
// cooperative launch per batch: phase-1 splits, fixup, Lawson fixpoint, and
// the detect / rollback loop of phase 3 with its Lawson passes -- every
// data-dependent loop runs on the device, so a batch needs no host round
// trip between its phases.
//
// Execution contexts (Exec): grid mode (all CTAs, grid barriers) or block
// mode (CTA 0 alone, __syncthreads).  Block mode is Rule 1 of the paper
// applied to the tail: when a batch inserts only a few
// hundred points, or a Lawson work list drops below a block's worth, the
// work runs in one CTA and a barrier costs tens of nanoseconds instead of a
// grid-wide synchronisation.
//
// Per-step counters live in a ring of 4 RoundCtr; the leader zeroes the slot
// of step k+1 at the start of step k (at least one barrier separates that
// write from its first use, and no slot is read more than one step late).
// =====================================================================================

struct Exec {
    u32 tid, nthr;
    bool block;      // block mode: CTA 0 only
    RoundCtr* ring;  // step counters: global ring (grid mode) or shared memory (block mode,
                     // so the work-list atomics and the post-barrier count reads stay on-SM)
    bool cluster;    // cluster mode: the whole launch is ONE thread-block cluster
                     // (mid-size batches): barrier.cluster instead of a grid barrier
    __device__ __forceinline__ void sync() const {
        if (block)
            __syncthreads();
        else if (cluster)
            cg::this_cluster().sync();   // hardware barrier, release/acquire at cluster scope
        else
            cg::this_grid().sync();
    }
    __device__ __forceinline__ bool leader() const { return tid == 0; }
};

// Grid mode over every CTA of the launch; when the launch is one cluster
// (InsertArgs::cluster) its barriers are cluster barriers.
__device__ __forceinline__ Exec grid_exec(RoundCtr* ring, bool cluster = false) {
    cg::grid_group g = cg::this_grid();
    return Exec{(u32)g.thread_rank(), (u32)g.size(), false, ring, cluster};
}
// Block mode with its counters in shared memory: sring[5] is zeroed here
// (every thread of the CTA must call it).
__device__ __forceinline__ Exec block_exec(RoundCtr* sring) {
    if (threadIdx.x < 5) {
        RoundCtr z = {};
        sring[threadIdx.x] = z;
    }
    __syncthreads();
    return Exec{threadIdx.x, blockDim.x, true, sring, false};
}

__device__ __forceinline__ u32 vload(const u32* p) { return *(const volatile u32*)p; }

struct InsertArgs {
    DevMesh m;            // counts BEFORE this batch's insertions
    DevCands c;
    InsertBufs b;
    TriAux x;
    FreshInfo f;
    WorkLists w;
    RoundCtr* ring;       // [5]: 4-slot step ring + removal-seed accumulator, zeroed by the host
    u32* state;           // [0] status, [1] steps, [2] flip rounds, [3] removal rounds, [4..7] handoff
    Counters* ctr;
    const u32* d_C;       // candidate count (collect)
    u64 depth_cap;
    u32 batch;            // batch epoch written into vert_birth
    u32 round0;           // first stamp round of this batch
    u32 vcap, tcap, scap; // mesh capacities
    u32 small_nv;         // block mode when the batch inserts <= small_nv points
    u32 small_wl;         // Lawson switches to block mode below this many work items
    u32 rm_warp;          // removal rounds of <= rm_warp * warps run one warp per removal
    u32 max_steps;        // safety bound on barrier steps
    // Lines 5-7 (locate / claim / cavity) + the phase-1 plan and its scan
    u32 ncav, rs;         // cavity bound and region stride
    u32* regions;
    u32* region_len;
    u32* scan_part;       // [3 * grid] per-CTA chunk sums of the insertion plan
    u32 small_c;          // block mode for the whole batch when C <= small_c
    int resume;           // 1: candidates are planned, start at the capacity check
    int prefiltered;      // standalone Lines 5-7 ran (for C > small_c)
    int planned;          // ... including the phase-1 plan (b.nv / nt / ns written)
    u32 reg_cap;          // candidates the region buffers hold
    int cluster;          // the launch is one thread-block cluster (Exec::cluster)
    int isolate;          // claims: 0 reference, 1 isolated (rollback only if state[8]), 2 precedence
    int dep_mis;          // dependent pairs: 1 = priority-MIS rule, 0 = any-higher-neighbour rule
    int extras;           // refine cavity claims: 2 = the rewrite table (launch_cavity)
    unsigned long long* trace;   // GDP2D_TRACE: (globaltimer << 8 | tag) per step, or null
    u32* trace_val;              // a work count per trace entry
    u32* trace_n;
    u32 trace_cap;
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Step tags of the device trace (printed by the host under GDP2D_TRACE=1).
enum : u32 { TR_START = 1, TR_APPLY, TR_FIXUP, TR_FTEST, TR_FAPPLY, TR_FPOST, TR_DET_A, TR_DET_B,
             TR_DET_C, TR_RM_CLAIM, TR_RM_APPLY, TR_RM_POST, TR_BLOCK_IN, TR_BLOCK_OUT, TR_END,
             TR_LOCATE, TR_CLAIM, TR_CAVITY, TR_PLAN, TR_SPLIT_END, TR_RB_START };

__device__ __forceinline__ void trace(const InsertArgs& a, bool leader, u32 tag, u32 value = 0) {
    if (a.trace && leader) {
        const u32 i = atomicAdd(a.trace_n, 1u);
        if (i < a.trace_cap) {
            a.trace[i] = (globaltimer() << 8) | tag;
            a.trace_val[i] = value;
        }
    }
}

enum : u32 { INS_OK = 0, INS_GROW = 1, INS_STEPS = 2, INS_REGIONS = 3 };

__device__ __forceinline__ RoundCtr* ring_at(const Exec& ex, u32 step) {
    return ex.ring + (step & 3u);
}
__device__ __forceinline__ void ring_advance(const InsertArgs& a, const Exec& ex, u32 step) {
    (void)a;
    if (ex.leader()) {
        RoundCtr* z = ex.ring + ((step + 1u) & 3u);
        z->wl_next = z->cand = z->touched = z->rm_next = z->detect = 0;
    }
}

// Lawson rounds (test + claim | apply | post + fixup) until the work list in
// w.w[cur] (n items) is empty.  step / cur are uniform across ex.
__device__ void lawson_rounds(const InsertArgs& a, const Exec& ex, const DevMesh& m, u32& step,
                              u32& cur, u32 n, ull& flipped, u32& rounds) {
    const WorkLists& w = a.w;
    while (n > 0 && step < a.max_steps) {
        RoundCtr* rc = ring_at(ex, step);
        ring_advance(a, ex, step);
        const u32 round = a.round0 + step;
        const u32* wl = w.w[cur];
        for (u32 i = ex.tid; i < n; i += ex.nthr) flip_test_one(m, wl[i], round, a.x, w, rc, a.ctr);
        ex.sync();
        trace(a, ex.leader(), TR_FTEST, n);
        const u32 nc = min(vload(&rc->cand), w.cap);
        for (u32 i = ex.tid; i < nc; i += ex.nthr)
            flipped += flip_apply_one(m, i, round, cur ^ 1u, a.x, w, rc, a.ctr);
        ex.sync();
        trace(a, ex.leader(), TR_FAPPLY, nc);
        for (u32 i = ex.tid; i < nc; i += ex.nthr)
            flip_post_one(i, round, cur ^ 1u, a.x, w, rc, a.ctr);
        const u32 nt = min(vload(&rc->touched), w.cap);
        for (u32 i = ex.tid; i < nt; i += ex.nthr)
            fixup_one(m, round, a.x, w, w.touched[i], 0, 0, rc, a.ctr);
        ex.sync();
        trace(a, ex.leader(), TR_FPOST, nt);
        n = vload(&rc->wl_next);
        if (n > w.cap) {
            raise_err(a.ctr, DERR_WORKLIST_OVERFLOW, n);
            n = 0;
        }
        cur ^= 1u;
        ++step;
        ++rounds;
    }
}

// Lawson fixpoint from grid mode: small work lists finish in CTA 0 alone.
__device__ void lawson_fixpoint_dev(const InsertArgs& a, const Exec& ex, const DevMesh& m,
                                    u32& step, u32& cur, u32 n, ull& flipped, u32& rounds) {
    if (ex.block) {
        lawson_rounds(a, ex, m, step, cur, n, flipped, rounds);
        return;
    }
    while (n > 0 && step < a.max_steps) {
        if (n <= a.small_wl) {
            if (blockIdx.x == 0) {
                __shared__ RoundCtr hring[5];
                const Exec bx = block_exec(hring);
                trace(a, bx.leader(), TR_BLOCK_IN);
                u32 s2 = step, c2 = cur, r2 = 0;
                lawson_rounds(a, bx, m, s2, c2, n, flipped, r2);
                trace(a, bx.leader(), TR_BLOCK_OUT);
                if (threadIdx.x == 0) {
                    a.state[4] = s2;
                    a.state[5] = c2;
                    a.state[6] = r2;
                    // the grid resumes at step s2 on the global ring
                    RoundCtr z = {};
                    a.ring[s2 & 3u] = z;
                }
            }
            ex.sync();
            step = vload(&a.state[4]);
            cur = vload(&a.state[5]);
            rounds += vload(&a.state[6]);
            ex.sync();   // everyone has read the handoff before it can be reused
            return;
        }
        // one grid-wide round, then re-evaluate the list size
        RoundCtr* rc = ring_at(ex, step);
        ring_advance(a, ex, step);
        const u32 round = a.round0 + step;
        const u32* wl = a.w.w[cur];
        // waves: one list reservation per CTA (flip_*_waves, gdp2d_rewrite.cuh)
        const u32 tid0 = ex.tid - threadIdx.x;
        flip_test_waves<INSERT_BLOCK>(m, wl, n, round, tid0, ex.nthr, a.x, a.w, rc, a.ctr);
        ex.sync();
        trace(a, ex.leader(), TR_FTEST, n);
        const u32 nc = min(vload(&rc->cand), a.w.cap);
        flipped += flip_apply_waves<INSERT_BLOCK>(m, nc, round, cur ^ 1u, tid0, ex.nthr, a.x, a.w,
                                                  rc, a.ctr);
        ex.sync();
        trace(a, ex.leader(), TR_FAPPLY, nc);
        flip_post_waves<INSERT_BLOCK>(nc, round, cur ^ 1u, tid0, ex.nthr, a.x, a.w, rc, a.ctr);
        const u32 nt = min(vload(&rc->touched), a.w.cap);
        for (u32 i = ex.tid; i < nt; i += ex.nthr)
            fixup_one(m, round, a.x, a.w, a.w.touched[i], 0, 0, rc, a.ctr);
        ex.sync();
        trace(a, ex.leader(), TR_FPOST, nt);
        n = vload(&rc->wl_next);
        if (n > a.w.cap) {
            raise_err(a.ctr, DERR_WORKLIST_OVERFLOW, n);
            n = 0;
        }
        cur ^= 1u;
        ++step;
        ++rounds;
    }
}

// Lines 5-7 for the whole candidate list (tiny batches; big ones run the
// high-occupancy standalone kernels of k_locate.cu / k_filter.cu instead),
// then the phase-1 plan and its exclusive scan (three 0/1 streams packed into one u64 per
// candidate inside a CTA chunk; chunk sums cross CTAs through scan_part).
template <int MODE>
__device__ void filter(const InsertArgs& a, const Exec& ex, u32 C) {
    const DevMesh& m = a.m;
    ull steps = 0, visits = 0;
    u32 surv1 = 0, surv2 = 0;
    for (u32 i = ex.tid; i < C; i += ex.nthr) steps += locate_one(m, a.c, i);
    ex.sync();
    trace(a, ex.leader(), TR_LOCATE);
    for (u32 i = ex.tid; i < C; i += ex.nthr) claim_max_one(a.c, i, a.x.ckey);
    ex.sync();
    for (u32 i = ex.tid; i < C; i += ex.nthr) claim_tie_one(a.c, i, a.x.ckey, a.x.ctie);
    ex.sync();
    for (u32 i = ex.tid; i < C; i += ex.nthr) surv1 += claim_check_one(a.c, i, a.x.ckey, a.x.ctie);
    ex.sync();
    for (u32 i = ex.tid; i < C; i += ex.nthr) claim_reset_one(a.c, i, m.nT, a.x.ckey, a.x.ctie);
    ex.sync();
    trace(a, ex.leader(), TR_CLAIM);
    u32 marked = 0, unsafe = 0;
    const bool rw = a.isolate || a.extras >= 2;
    for (u32 i = ex.tid; i < C; i += ex.nthr) {
        visits += a.isolate
                      ? cavity_claims_one<MODE>(m, a.c, i, a.ncav, a.rs, a.regions, a.region_len,
                                                a.x.ckey, a.depth_cap, a.isolate == 1)
                      : cavity_bfs_one(m, a.c, i, a.ncav, a.extras, a.rs, a.regions, a.region_len,
                                       nullptr, a.x.ckey);
        if (rw) rw_claim_one(m, a.c, i, a.x.fkey);
    }
    ex.sync();
    for (u32 i = ex.tid; i < C; i += ex.nthr) {
        cavity_tie_one(a.c, i, a.rs, a.regions, a.region_len, a.x.ckey, a.x.ctie);
        if (rw) rw_tie_one(a.c, i, a.x.fkey, a.x.ftie);
    }
    ex.sync();
    for (u32 i = ex.tid; i < C; i += ex.nthr) {
        if (rw && a.c.alive[i] && !rw_owns(a.c, i, a.x.fkey, a.x.ftie)) {
            a.c.alive[i] = 0;
            continue;
        }
        if (a.isolate) {
            u32 mk = 0;
            surv2 += isolated_check_one(m, a.c, i, a.rs, a.regions, a.region_len, a.x.ckey,
                                        a.x.ctie, mk, unsafe);
            // a precedence mark makes a new candidate for the tail loop
            if (mk && a.w.dlist) dlist_push(a.w, a.c.red[i]);
            marked += mk;
        } else {
            surv2 += cavity_check_one(a.c, i, a.rs, a.regions, a.region_len, a.x.ckey, a.x.ctie);
        }
    }
    if (unsafe) atomicOr(&a.state[8], 1u);
    warp_add_u32(&a.ctr->marked, marked);
    ex.sync();
    for (u32 i = ex.tid; i < C; i += ex.nthr) {
        cavity_reset_one(i, a.rs, a.regions, a.region_len, a.x.ckey, a.x.ctie);
        if (rw) rw_reset_one(a.c, i, m.nT, a.x.fkey, a.x.ftie);
    }
    trace(a, ex.leader(), TR_CAVITY);
    warp_add_ull(&a.ctr->walk_steps, steps);
    warp_add_ull(&a.ctr->cavity_visits, visits);
    warp_add_u32(&a.ctr->surv_claim, surv1);
    warp_add_u32(&a.ctr->surv_cavity, surv2);
}

// planned: the standalone filter already wrote b.nv / nt / ns (and counted
// the dropped candidates); only the scan is left.
__device__ void plan_and_scan(const InsertArgs& a, const Exec& ex, u32 C, bool planned) {
    const DevMesh& m = a.m;
    u32 dropped = 0;

    // plan + chunk sums: CTA b owns candidates [b*chunk, (b+1)*chunk)
    __shared__ unsigned long long sh64[INSERT_BLOCK / 32 + 1];
    const u32 nblk = ex.block ? 1u : gridDim.x;
    const u32 b = ex.block ? 0u : blockIdx.x;
    const u32 chunk = ((C + nblk - 1) / nblk + INSERT_BLOCK - 1) / INSERT_BLOCK * INSERT_BLOCK;
    const u32 lo = min(C, b * chunk), hi = min(C, lo + chunk);
    // fields: nv (bits 0-20), far (21-41), mid (42-62); a chunk is < 2^21
    unsigned long long local = 0;
    for (u32 i = lo + threadIdx.x; i < hi; i += INSERT_BLOCK) {
        u32 nv, nt, ns;
        if (planned) {
            nv = a.b.nv[i];
            nt = a.b.nt[i];
            ns = a.b.ns[i];
        } else {
            dropped += plan_one(m, a.c, i, a.depth_cap, nv, nt, ns);
            a.b.nv[i] = nv;
            a.b.nt[i] = nt;
            a.b.ns[i] = ns;
        }
        local += (unsigned long long)nv | ((unsigned long long)(nt - nv) << 21) |
                 ((unsigned long long)(ns >> 1) << 42);
    }
    unsigned long long tot;
    block_exclusive_t<INSERT_BLOCK, unsigned long long>(local, sh64, &tot);
    if (threadIdx.x == 0) {
        a.scan_part[3 * b + 0] = (u32)(tot & 0x1FFFFF);
        a.scan_part[3 * b + 1] = (u32)((tot >> 21) & 0x1FFFFF);
        a.scan_part[3 * b + 2] = (u32)((tot >> 42) & 0x1FFFFF);
    }
    ex.sync();
    // CTA prefix = sum of the chunk sums of the CTAs before it
    u32 p0 = 0, p1 = 0, p2 = 0;
    for (u32 k = threadIdx.x; k < b; k += INSERT_BLOCK) {
        p0 += a.scan_part[3 * k];
        p1 += a.scan_part[3 * k + 1];
        p2 += a.scan_part[3 * k + 2];
    }
    __shared__ u32 shp[INSERT_BLOCK / 32 + 1];
    p0 = block_sum<INSERT_BLOCK>(p0, shp);
    p1 = block_sum<INSERT_BLOCK>(p1, shp);
    p2 = block_sum<INSERT_BLOCK>(p2, shp);
    __shared__ u32 pre[3];
    if (threadIdx.x == 0) {
        pre[0] = p0;
        pre[1] = p1;
        pre[2] = p2;
    }
    __syncthreads();
    u32 c0 = pre[0], c1 = pre[1], c2 = pre[2];
    for (u32 base = lo; base < hi; base += INSERT_BLOCK) {
        const u32 i = base + threadIdx.x;
        unsigned long long v = 0;
        if (i < hi)
            v = (unsigned long long)a.b.nv[i] | ((unsigned long long)(a.b.nt[i] - a.b.nv[i]) << 21) |
                ((unsigned long long)(a.b.ns[i] >> 1) << 42);
        unsigned long long t;
        const unsigned long long ex64 = block_exclusive_t<INSERT_BLOCK, unsigned long long>(v, sh64, &t);
        if (i < hi) {
            const u32 e0 = (u32)(ex64 & 0x1FFFFF), e1 = (u32)((ex64 >> 21) & 0x1FFFFF),
                      e2 = (u32)((ex64 >> 42) & 0x1FFFFF);
            a.b.ov[i] = c0 + e0;
            a.b.ot[i] = c0 + e0 + c1 + e1;
            a.b.os[i] = 2u * (c2 + e2);
        }
        c0 += (u32)(t & 0x1FFFFF);
        c1 += (u32)((t >> 21) & 0x1FFFFF);
        c2 += (u32)((t >> 42) & 0x1FFFFF);
    }
    if (b == nblk - 1 && threadIdx.x == 0) {
        a.b.totals[0] = c0;
        a.b.totals[1] = c0 + c1;
        a.b.totals[2] = 2u * c2;
    }
    warp_add_u32(&a.ctr->dropped, dropped);
    ex.sync();
    trace(a, ex.leader(), TR_PLAN);
}

// Phase 1 (splits) + the Lawson fixpoint.  step / flip_rounds / flips are
// left in state[] for the rollback kernel.
__device__ void split_and_flip(const InsertArgs& a, const Exec& ex, u32 nv, u32 nt, u32 ns) {
    const u32 C = vload(a.d_C);
    const WorkLists& w = a.w;
    DevMesh m = a.m;   // pre-insertion counts: new ids are m.nV + offset, ...
    u32 step = 0, cur = 0, flip_rounds = 0;
    ull flipped = 0;
    u32 mid = 0, cc = 0;
    RoundCtr* rc = ring_at(ex, step);
    ring_advance(a, ex, step);
    {
        const u32 round = a.round0 + step;
        if (ex.block) {
            for (u32 i = ex.tid; i < C; i += ex.nthr) {
                const int r = apply_one(m, a.c, i, a.batch, round, a.b, a.x, a.f, w, rc, 1, a.ctr);
                mid += r == 1;
                cc += r == 2;
            }
        } else {
            // waves: one touched / seed reservation per CTA (block_reserve)
            for (u32 base = ex.tid - threadIdx.x; base < C; base += ex.nthr) {
                const u32 i = base + threadIdx.x;
                u32 ntc = 0, nwc = 0;
                if (i < C) split_appends(a.c, i, a.b, ntc, nwc);
                u32 slots[2];
                slots[0] = block_reserve<INSERT_BLOCK>(&rc->touched, ntc);
                slots[1] = block_reserve<INSERT_BLOCK>(&rc->wl_next, nwc);
                if (i < C) {
                    const int r = apply_one(m, a.c, i, a.batch, round, a.b, a.x, a.f, w, rc, 1,
                                            a.ctr, slots);
                    mid += r == 1;
                    cc += r == 2;
                }
            }
        }
        m.nV += nv;
        m.nT += nt;
        m.nS += ns;
        ex.sync();
        trace(a, ex.leader(), TR_APPLY);
        const u32 ntouch = min(vload(&rc->touched), w.cap);
        for (u32 i = ex.tid; i < ntouch; i += ex.nthr)
            fixup_one(m, round, a.x, w, w.touched[i], 0, 0, rc, a.ctr);
        ex.sync();
        trace(a, ex.leader(), TR_FIXUP);
    }
    const u32 n = vload(&rc->wl_next);
    ++step;
    lawson_fixpoint_dev(a, ex, m, step, cur, n, flipped, flip_rounds);
    warp_add_u32(&a.ctr->ins_mid, mid);
    warp_add_u32(&a.ctr->ins_cc, cc);
    warp_add_ull(&a.ctr->flips, flipped);
    {
        // flips of this kernel alone (roofline split of the two launches)
        u32 f32 = (u32)flipped;
        f32 = __reduce_add_sync(0xFFFFFFFFu, f32);
        if ((threadIdx.x & 31) == 0 && f32) atomicAdd(&a.state[7], f32);
    }
    if (ex.leader()) {
        a.state[0] = step >= a.max_steps ? INS_STEPS : INS_OK;
        a.state[1] = step;
        a.state[2] = flip_rounds;
        a.state[3] = 0;
    }
    trace(a, ex.leader(), TR_SPLIT_END);
}

// Phase 3 (refine.hpp:551-608): detection + parallel rollback to fixpoint,
// each removal round followed by its Lawson pass.
template <int MODE>
__device__ void rollback_loop(const InsertArgs& a, const Exec& ex, u32 nv, u32 nt, u32 ns) {
    const WorkLists& w = a.w;
    DevMesh m = a.m;
    m.nV += nv;
    m.nT += nt;
    m.nS += ns;
    u32 step = vload(&a.state[1]), cur = 0, flip_rounds = 0, rm_rounds = 0;
    ull flipped = 0;
    u32 marked = 0, red = 0, dep = 0, done = 0;
    const u32 V0 = a.m.nV, F = nv;
    if (ex.leader()) {   // the split kernel may have run on a different ring
        RoundCtr z = {};
        ex.ring[step & 3u] = z;
    }
    ex.sync();   // every thread has read state[1] before the leader rewrites it
    // Detection passes evaluate only suspects (f.dirty, set by fixup_one when
    // a rewritten triangle makes a fresh circumcenter the apex of a
    // subsegment or puts two of them on one triangle).  A vertex that is not
    // re-suspected keeps its verdict: its star did not change in a way that
    // could make it redundant or dependent (a neighbour turning redundant only
    // removes a reason to be dependent, and removed neighbours rewrite it).
    // dirty: 1 = suspect, 2 = evaluated in this pass, 0 = clean.
    RoundCtr* seed_rc = ex.ring + 4;   // Lawson seeds of all removal rounds of a pass
    for (u32 pass = 0; step < a.max_steps; ++pass) {
        RoundCtr* rc = ring_at(ex, step);
        ring_advance(a, ex, step);
        if (ex.leader()) seed_rc->wl_next = 0;   // visible after the barriers below
        for (u32 j = ex.tid; j < F; j += ex.nthr) {
            if (a.f.dirty[j] == 0) continue;   // not a suspect since the last pass
            a.f.dirty[j] = 2;
            marked += detect_a_one<MODE>(m, a.depth_cap, V0, F, j, a.f, a.ctr, !a.dep_mis, w);
        }
        ex.sync();
        trace(a, ex.leader(), TR_DET_A);
        if (!a.dep_mis) {
            for (u32 j = ex.tid; j < F; j += ex.nthr) {
                if (a.f.dirty[j] != 2) continue;
                a.f.dirty[j] = 0;
                detect_b_fast(m, V0, F, j, a.f);
            }
            ex.sync();
        } else {
            // undecided vertices go to w.rm[1] (free until the removal rounds)
            for (u32 j = ex.tid; j < F; j += ex.nthr) {
                if (a.f.dirty[j] != 2) continue;
                a.f.dirty[j] = 0;
                if (detect_b_mis_one(m, V0, F, j, a.f)) {
                    const u32 o = agg_reserve(&rc->cand, 1u);
                    if (o < w.rm_cap) w.rm[1][o] = j;
                }
            }
            ex.sync();
            u32 nu = min(vload(&rc->cand), w.rm_cap);
            ++step;   // the detect slot is used up: MIS rounds take fresh ring slots
            // rounds alternate between rm[1] and w.touched (both >= F entries)
            u32* lists[2] = {w.rm[1], w.touched};
            u32 lc = 0;
            for (u32 r = 0; nu > 0 && r < 4096; ++r) {
                RoundCtr* rr = ring_at(ex, step);
                ring_advance(a, ex, step);
                ++step;
                for (u32 i = ex.tid; i < nu; i += ex.nthr) {
                    const u32 j = lists[lc][i];
                    if (mis_round_one(j, a.f)) {
                        const u32 o = agg_reserve(&rr->cand, 1u);
                        lists[lc ^ 1u][o] = j;
                    }
                }
                ex.sync();
                const u32 nn = vload(&rr->cand);
                if (nn == nu) {
                    // no progress (cannot happen for a strict priority order):
                    // fall back to removing the rest
                    for (u32 i = ex.tid; i < nn; i += ex.nthr) {
                        const u32 j = lists[lc ^ 1u][i];
                        a.f.dstat[j] = 2;
                        a.f.mark[j] = 2;
                    }
                    ex.sync();
                    break;
                }
                nu = nn;
                lc ^= 1u;
            }
            rc = ring_at(ex, step);
            ring_advance(a, ex, step);
            if (ex.leader()) seed_rc->wl_next = 0;
            ex.sync();
        }
        trace(a, ex.leader(), TR_DET_B);
        for (u32 j = ex.tid; j < F; j += ex.nthr) {
            u32 r1 = 0, r2 = 0;
            detect_collect_one(V0, j, a.f, w, rc, r1, r2);
            red += r1;
            dep += r2;
        }
        ex.sync();
        trace(a, ex.leader(), TR_DET_C);
        u32 nrm = min(vload(&rc->detect), w.rm_cap);
        ++step;
        if (nrm == 0) break;
        // Removal rounds until every listed vertex is gone (or kept): each
        // round removes the vertices whose stars it owns; the rebuilt stars'
        // edges accumulate in ONE Lawson list (seed_rc), flipped once after
        // the last round -- a removal only needs a valid triangulation, not
        // a Delaunay one, so intermediate Lawson passes are unnecessary.
        u32 rcur = 0;
        while (nrm > 0 && step < a.max_steps) {
            rc = ring_at(ex, step);
            ring_advance(a, ex, step);
            const u32 round = a.round0 + step;
            const u32* list = w.rm[rcur];
            for (u32 i = ex.tid; i < nrm; i += ex.nthr) rm_claim_one(m, list, i, V0, round, a.x, a.f, w, a.ctr);
            ex.sync();
            trace(a, ex.leader(), TR_RM_CLAIM, nrm);
            if (nrm <= a.rm_warp * (ex.nthr >> 5)) {
                // few removals: one warp each (latency), direct list appends
                for (u32 wi = ex.tid >> 5; wi < nrm; wi += ex.nthr >> 5)
                    done += rm_apply_warp(m, list, wi, round, V0, 0, rcur ^ 1u, a.x, a.f, w, rc,
                                          a.ctr, seed_rc);
            } else if (ex.block) {
                for (u32 i = ex.tid; i < nrm; i += ex.nthr)
                    done += rm_apply_one(m, list, i, round, V0, 0, rcur ^ 1u, a.x, a.f, w, rc,
                                         a.ctr, seed_rc);
            } else {
                // waves: one reservation per CTA for each list (block_reserve)
                for (u32 base = ex.tid - threadIdx.x; base < nrm; base += ex.nthr) {
                    const u32 i = base + threadIdx.x;
                    RmOut ro{0u, 0};
                    if (i < nrm)
                        done += rm_apply_one(m, list, i, round, V0, 0, rcur ^ 1u, a.x, a.f, w, rc,
                                             a.ctr, seed_rc, &ro);
                    const u32 od = block_reserve<ROLLBACK_BLOCK>(&rc->rm_next, ro.defer);
                    const u32 ot = block_reserve<ROLLBACK_BLOCK>(&rc->touched, (u32)ro.created);
                    const u32 os =
                        block_reserve<ROLLBACK_BLOCK>(&seed_rc->wl_next, 3u * (u32)ro.created);
                    if (ro.defer && od < w.rm_cap) w.rm[rcur ^ 1u][od] = list[i];
                    if (ro.created)
                        rm_appends(w, 0, w.star + (size_t)i * MAX_STAR, ro.created, ot, os,
                                   a.ctr);
                }
            }
            ex.sync();
            trace(a, ex.leader(), TR_RM_APPLY);
            const u32 ntouch = min(vload(&rc->touched), w.cap);
            for (u32 i = ex.tid; i < ntouch; i += ex.nthr)
                fixup_one(m, round, a.x, w, w.touched[i], 0, 0, rc, a.ctr);
            ex.sync();
            trace(a, ex.leader(), TR_RM_POST);
            nrm = min(vload(&rc->rm_next), w.rm_cap);
            ++step;
            ++rm_rounds;
            rcur ^= 1u;
        }
        const u32 nl = min(vload(&seed_rc->wl_next), w.cap);
        ex.sync();   // everyone has read the seed count before the next pass resets it
        cur = 0;
        lawson_fixpoint_dev(a, ex, m, step, cur, nl, flipped, flip_rounds);
    }
    warp_add_u32(&a.ctr->marked, marked);
    warp_add_u32(&a.ctr->rm_red, red);
    warp_add_u32(&a.ctr->rm_dep, dep);
    warp_add_u32(&a.ctr->rm_done, done);
    warp_add_ull(&a.ctr->flips, flipped);
    trace(a, ex.leader(), TR_END);
    if (ex.leader()) {
        if (step >= a.max_steps) a.state[0] = INS_STEPS;
        a.state[1] = step;
        a.state[2] += flip_rounds;
        a.state[3] = rm_rounds;
    }
}

__device__ __forceinline__ bool fits_and_status(const InsertArgs& a, u32 nv, u32 nt, u32 ns) {
    const bool fits = (u64)a.m.nV + nv <= a.vcap && (u64)a.m.nT + nt <= a.tcap &&
                      (u64)a.m.nS + ns <= a.scap && nv <= a.f.cap && nv <= a.w.rm_cap &&
                      12ull * nv <= a.w.cap;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    if (!fits && lead) {
        a.state[0] = INS_GROW;
        a.state[1] = 0;
    }
    if (fits && nv == 0 && lead) a.state[0] = a.state[1] = a.state[2] = a.state[3] = 0;
    return fits && nv > 0;
}

// Kernel 1 of a batch after collect: [Lines 5-7 when the batch is small] +
// the phase-1 plan + splits + Lawson.  Block mode (CTA 0 alone) when the
// candidate list is small -- the long tail of the refinement (Rule 1).
template <int MODE>
__global__ void __launch_bounds__(INSERT_BLOCK, GDP2D_SPLIT_MINB) k_batch_split(const __grid_constant__ InsertArgs a) {
    // start stamp (state words 10-11): the host splits the kernel pair's
    // event-timed span at the rollback kernel's stamp, so no event record sits
    // between the two launches
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *reinterpret_cast<unsigned long long*>(a.state + 10) = globaltimer();
    const u32 C = vload(a.d_C);
    if (C > a.reg_cap) {   // uniform: the host grows the regions and redoes the batch
        if (blockIdx.x == 0 && threadIdx.x == 0) a.state[0] = INS_REGIONS;
        return;
    }
    const bool block = C <= a.small_c;
    if (block && blockIdx.x != 0) return;
    __shared__ RoundCtr sring[5];
    const Exec ex = block ? block_exec(sring) : grid_exec(a.ring, a.cluster != 0);
    if (!a.resume) {
        trace(a, ex.leader(), TR_START);
        const bool here = block || !a.prefiltered;   // Lines 5-7 in this kernel
        if (here) filter<MODE>(a, ex, C);
        plan_and_scan(a, ex, C, !here && a.planned);
    }
    const u32 nv = vload(&a.b.totals[0]), nt = vload(&a.b.totals[1]), ns = vload(&a.b.totals[2]);
    if (!fits_and_status(a, nv, nt, ns)) return;   // uniform
    split_and_flip(a, ex, nv, nt, ns);
}

// Kernel 2: phase 3 rollback (skipped when kernel 1 asked for growth).
template <int MODE>
__global__ void __launch_bounds__(ROLLBACK_BLOCK) k_batch_rollback(const __grid_constant__ InsertArgs a) {
    if (blockIdx.x == 0 && threadIdx.x == 0)   // start stamp (state words 12-13)
        *reinterpret_cast<unsigned long long*>(a.state + 12) = globaltimer();
    if (vload(&a.state[0]) != INS_OK) return;
    // isolated insertions cannot create redundant or dependent points: the
    // detection runs only when some survivor came from a capped claim set
    if (a.isolate == 1 && vload(&a.state[8]) == 0) return;
    const u32 nv = vload(&a.b.totals[0]), nt = vload(&a.b.totals[1]), ns = vload(&a.b.totals[2]);
    if (nv == 0) return;
    const bool block = nv <= a.small_c;
    if (block && blockIdx.x != 0) return;
    __shared__ RoundCtr sring[5];
    const Exec ex = block ? block_exec(sring) : grid_exec(a.ring, a.cluster != 0);
    trace(a, ex.leader(), TR_RB_START);
    rollback_loop<MODE>(a, ex, nv, nt, ns);
}

// =====================================================================================
// The device-resident tail loop: the long run of small batches at the end of a
// refinement (Rule 1 / Rule 4 of PAPER.md:104-116 taken to the batch loop) in
// ONE single-CTA launch.  Each iteration is one batch of refine.hpp:658-708:
//   collect   incremental, and the list is the one a full scan would make:
//             every element whose verdict can have changed since the last
//             collect is in klist (the last list: still bad unless rewritten)
//             or in the dirty list (rewritten triangles, the subsegments on
//             them, newly marked subsegments).  Their union is sorted, each
//             element re-evaluated through the dirty-bit cache (eval_sub /
//             eval_tri) and the bad ones written as records in key order
//             (subsegments, then triangles, each by id; tiebreak = index).
//   Lines 5-8 the block-mode batch code of k_batch_split / k_batch_rollback.
// The loop leaves to the host when the list outgrows small_c (BIG), a batch
// does not fit the buffers (GROW, nothing written), a device error, the
// iteration budget, or the refinement ends (DONE: C == 0, or nothing
// retained and nothing marked, refine.hpp:706).
// =====================================================================================

template <int MODE>
__global__ void __launch_bounds__(INSERT_BLOCK, 1) k_tail_loop(const __grid_constant__ InsertArgs a0,
                                                            const __grid_constant__ TailArgs t) {
    __shared__ u32 key[SMALL_LIST_CAP];
    __shared__ u32 sh[INSERT_BLOCK / 32 + 1];
    __shared__ u32 s_n;
    __shared__ RoundCtr sring[5];
    InsertArgs a = a0;   // per-batch counts / epoch / stamp round (every thread the same)
    u32 b = 0, exitr = TAIL_CAP, lastC = 0;
    for (; b < t.max_batches; ++b) {
        const unsigned long long t0 = globaltimer();
        // ---- incremental collect ----
        const u32 nk = vload(t.klist_n), nd = vload(a.w.dlist_n);
        if (nk > SMALL_LIST_CAP || nd > a.w.dlist_cap || nk + nd > SMALL_LIST_CAP) {
            exitr = TAIL_NOKEYS;   // nothing consumed: the host collects from scratch
            break;
        }
        const u32 n = nk + nd;
        u32 np = 1;
        while (np < n) np <<= 1;
        for (u32 k = threadIdx.x; k < np; k += blockDim.x)
            key[k] = k < nk ? t.klist[k] : (k < n ? a.w.dlist[k - nk] : NONE);
        __syncthreads();
        for (u32 size = 2; size <= np; size <<= 1)
            for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
                for (u32 k = threadIdx.x; k < np / 2; k += blockDim.x) {
                    const u32 lo = 2 * k - (k & (stride - 1)), hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const u32 x = key[lo], y = key[hi];
                    if ((x > y) == up) {
                        key[lo] = y;
                        key[hi] = x;
                    }
                }
                __syncthreads();
            }
        // unique keys, verdicts through the dirty-bit cache, order-preserving
        // compaction: chunks of blockDim keys, one block scan each
        u32 C = 0, dirty = 0, nfb = 0;
        for (u32 base = 0; base < n; base += blockDim.x) {
            const u32 k = base + threadIdx.x;
            u32 bad = 0, kk = NONE;
            if (k < n) {
                kk = key[k];
                if (kk != NONE && (k == 0 || key[k - 1] != kk)) {
                    const u32 id = kk & 0x7FFFFFFFu;
                    if (kk >> 31) {
                        const uint8_t tf = a.m.tflag[id];
                        if (tf & 2) {
                            bad = eval_tri(a.m, t.q, id);
                            ++dirty;
                        } else {
                            bad = tf & 1;
                        }
                    } else {
                        bad = eval_sub<MODE>(a.m, id, 0, dirty);
                    }
                }
            }
            u32 tot;
            const u32 o = C + block_exclusive<INSERT_BLOCK>(bad, sh, &tot);
            __syncthreads();   // every thread has read key[] of this chunk
            if (bad) {
                t.klist[o] = kk;
                nfb += write_candidate(a.m, a.c, o, kk >> 31 ? 1 : 0, kk & 0x7FFFFFFFu);
            }
            C += tot;
        }
        warp_add_u32(&a.ctr->fallbacks, nfb);
        {
            const u32 d = block_sum<INSERT_BLOCK>(dirty, sh);
            if (threadIdx.x == 0) {
                a.ctr->scan_dirty += d;
                *t.klist_n = C;
                *a.w.dlist_n = 0;
                *const_cast<u32*>(a.d_C) = C;
                for (int k = 0; k < 10; ++k) a.state[k] = 0;
            }
        }
        __syncthreads();
        lastC = C;
        if (C == 0) {
            exitr = TAIL_DONE;
            break;
        }
        if (C > a.small_c || C > a.reg_cap) {
            exitr = TAIL_BIG;   // the host runs this list's batch on the grid kernels
            break;
        }
        const unsigned long long t1 = globaltimer();
        // ---- Lines 5-8 (block mode) ----
        const Exec ex = block_exec(sring);
        filter<MODE>(a, ex, C);
        plan_and_scan(a, ex, C, false);
        const u32 nv = vload(&a.b.totals[0]), nt = vload(&a.b.totals[1]),
                  ns = vload(&a.b.totals[2]);
        if (nv > 0) {
            if (!fits_and_status(a, nv, nt, ns)) {
                exitr = TAIL_GROW;   // nothing written; the host grows and redoes it
                break;
            }
            split_and_flip(a, ex, nv, nt, ns);
            __syncthreads();
            if (vload(&a.state[0]) == INS_OK && !(a.isolate == 1 && vload(&a.state[8]) == 0))
                rollback_loop<MODE>(a, ex, nv, nt, ns);
        } else {
            fits_and_status(a, 0, 0, 0);   // status words zero
        }
        __syncthreads();
        const unsigned long long t2 = globaltimer();
        // ---- the batch's record; the next batch's counts ----
        const u32 steps = vload(&a.state[1]);
        if (threadIdx.x == 0) {
            TailRec& r = t.rec[b];
            r.attempted = C;
            r.nv = nv;
            r.nt = nt;
            r.ns = ns;
            r.steps = steps;
            r.flip_rounds = vload(&a.state[2]);
            r.rm_rounds = vload(&a.state[3]);
            r.dirty = 0;
            r.t0 = t0;
            r.t1 = t1;
            r.t2 = t2;
            // word by word past L1: the counters were bumped by L2 atomics
            const volatile u32* src = reinterpret_cast<const volatile u32*>(a.ctr);
            u32* dst = reinterpret_cast<u32*>(&r.ctr);
            for (u32 k = 0; k < sizeof(Counters) / 4; ++k) dst[k] = src[k];
        }
        __syncthreads();
        const Counters& h = t.rec[b].ctr;
        const u32 err = vload(&a.ctr->err_code);
        const u32 st0 = vload(&a.state[0]);
        const u32 ins = h.ins_mid + h.ins_cc, rmd = h.rm_done, marked = h.marked;
        __syncthreads();   // everyone has read the record before the counters reset
        if (threadIdx.x == 0) {
            Counters z = {};
            *a.ctr = z;
        }
        if (err != 0 || (nv > 0 && st0 != INS_OK)) {
            exitr = TAIL_ERR;
            ++b;
            break;
        }
        a.m.nV += nv;
        a.m.nT += nt;
        a.m.nS += ns;
        a.batch += 1;
        a.round0 += nv > 0 ? steps + 1 : 1;
        a.w.fresh_v0 = a.m.nV;
        a.w.vtri_from = a.m.nV;
        if (ins - min(ins, rmd) == 0 && marked == 0) {
            exitr = TAIL_DONE;
            ++b;
            break;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        t.out[0] = exitr;
        t.out[1] = b;
        t.out[2] = a.m.nV;
        t.out[3] = a.m.nT;
        t.out[4] = a.m.nS;
        t.out[5] = a.round0;
        t.out[6] = lastC;
    }
}

template <class K0, class K1>
static int coop_grid(K0 k0, K1 k1, int device, int block = INSERT_BLOCK) {
    int sms = 0, per0 = 0, per1 = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per0, k0, block, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, k1, block, 0);
    return std::max(1, sms * std::max(1, std::min(per0, per1)));
}

int insert_persistent_grid(int device) {
    return coop_grid(k_batch_split<0>, k_batch_split<1>, device);
}
int rollback_persistent_grid(int device) {
    return coop_grid(k_batch_rollback<0>, k_batch_rollback<1>, device, ROLLBACK_BLOCK);
}

static InsertArgs make_args(const InsertLaunch& L) {
    InsertArgs a;
    a.m = L.m;
    a.c = L.c;
    a.b = L.b;
    a.x = L.x;
    a.f = L.f;
    a.w = L.w;
    a.ring = L.ring;
    a.state = L.state;
    a.ctr = L.ctr;
    a.d_C = L.d_C;
    a.depth_cap = L.depth_cap;
    a.batch = L.batch;
    a.round0 = L.round0;
    a.vcap = L.vcap;
    a.tcap = L.tcap;
    a.scap = L.scap;
    a.small_nv = L.small_nv;
    a.small_wl = L.small_wl;
    a.rm_warp = L.rm_warp;
    a.max_steps = L.max_steps;
    a.ncav = L.ncav;
    a.rs = L.rs;
    a.regions = L.regions;
    a.region_len = L.region_len;
    a.scan_part = L.scan_part;
    a.small_c = L.small_c;
    a.resume = L.resume;
    a.prefiltered = L.prefiltered;
    a.planned = L.planned;
    a.reg_cap = L.reg_cap;
    a.cluster = L.cluster;
    a.isolate = L.isolate;
    a.dep_mis = L.dep_mis;
    a.extras = L.extras;
    a.trace = L.trace;
    a.trace_val = L.trace_val;
    a.trace_n = L.trace_n;
    a.trace_cap = L.trace_cap;
    return a;
}

void launch_tail_loop(const InsertLaunch& L, const TailArgs& t, int mode, cudaStream_t st) {
    const InsertArgs a = make_args(L);
    note_launch();
    if (mode)
        k_tail_loop<1><<<1, INSERT_BLOCK, 0, st>>>(a, t);
    else
        k_tail_loop<0><<<1, INSERT_BLOCK, 0, st>>>(a, t);
}

// Cluster launch: the grid is ONE cluster of `grid` CTAs (non-portable sizes
// up to 16 are enabled once per kernel), no cooperative attribute -- the
// kernels' barriers are then barrier.cluster (Exec::cluster).
static cudaError_t launch_as_cluster(const void* fn, int grid, int block, void** args,
                                     cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = grid;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

static const void* split_fn(int mode) {
    return mode ? (const void*)k_batch_split<1> : (const void*)k_batch_split<0>;
}
static const void* rollback_fn(int mode) {
    return mode ? (const void*)k_batch_rollback<1> : (const void*)k_batch_rollback<0>;
}

int insert_cluster_size(int device, int want) {
    // largest cluster <= want that both persistent kernels can place (0 = none)
    static int cached[64][17];
    if (want < 2) return 0;
    want = std::min(want, 16);
    if (device >= 0 && device < 64 && cached[device][want]) return cached[device][want] - 1;
    int got = 0;
    for (int cs = want; cs >= 2 && !got; cs /= 2) {
        bool ok = true;
        for (int mode = 0; mode < 2 && ok; ++mode)
            for (int k = 0; k < 2 && ok; ++k) {
                const void* fn = k ? rollback_fn(mode) : split_fn(mode);
                if (cs > 8 &&
                    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                        cudaSuccess) {
                    ok = false;
                    break;
                }
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(cs);
                cfg.blockDim = dim3(k ? ROLLBACK_BLOCK : INSERT_BLOCK);
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cs;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int n = 0;
                if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n < 1) ok = false;
            }
        if (ok) got = cs;
    }
    cudaGetLastError();
    if (device >= 0 && device < 64) cached[device][want] = got + 1;
    return got;
}

void launch_insert_persistent(const InsertLaunch& L, int mode, int grid, int grid2, cudaStream_t st,
                              cudaEvent_t between, int which) {
    InsertArgs a = make_args(L);
    void* args[] = {&a};
    if (which & 1) {
        note_launch();
        if (L.cluster)
            launch_as_cluster(split_fn(mode), grid, INSERT_BLOCK, args, st);
        else
            cudaLaunchCooperativeKernel(split_fn(mode), dim3(grid), dim3(INSERT_BLOCK), args, 0, st);
    }
    if (between) cudaEventRecord(between, st);
    if (which & 2) {
        note_launch();
        if (L.cluster)
            launch_as_cluster(rollback_fn(mode), grid2, ROLLBACK_BLOCK, args, st);
        else
            cudaLaunchCooperativeKernel(rollback_fn(mode), dim3(grid2), dim3(ROLLBACK_BLOCK), args,
                                        0, st);
    }
}

}  // namespace gdp2d
