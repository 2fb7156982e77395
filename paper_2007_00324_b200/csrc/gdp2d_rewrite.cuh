// gdp2d_rewrite.cuh -- the local rewrite protocol shared by every kernel that
// changes the mesh (refinement splits, Lawson flips, the device CDT builder).
//
// Phase A: the owner of a claimed region rewrites its triangles in place
// (write_tri), marks the edges whose far side is outside the region as
// pending (tn.w bits) and records, per old edge slot, where that edge now
// lives (emap) together with stamp[t] = round -- one 16-byte record per
// triangle, TriAux::se = {stamp, emap[0..2]}.  Phase B (fixup_one, after a
// barrier): each rewritten triangle resolves its pending edges -- a far side
// rewritten in the same round is followed through its emap, any other far
// side gets its back-pointer written.  Regions of one round must be disjoint;
// adjacent regions are fine.
#pragma once

#include "engine.h"
#include "gdp2d_geom.cuh"
#include "scan.cuh"

namespace gdp2d {

// ---- shared phase-A helpers ----------------------------------------------------

// vfrom: vert_tri is invalidated only for corner ids >= vfrom (WorkLists::vtri_from)
__device__ __forceinline__ void write_tri(const DevMesh& m, u32 t, u32 a, u32 b, u32 c, u32 n0,
                                          u32 n1, u32 n2, u32 pend, u32 s0, u32 s1, u32 s2,
                                          u32 vfrom = 0) {
    const u32 fl = tri_flags(s0, s1, s2);
    m.tv[t] = make_uint4(a, b, c, fl);
    m.tn[t] = make_uint4(n0, n1, n2, pend);
    // ts is read only behind the tv.w subsegment bits (load_ts / has_seg)
    if (fl != 1u) m.ts[t] = make_uint4(s0, s1, s2, 0u);
    m.tflag[t] = 2;
    if (a >= vfrom) m.vtri[a] = NONE;
    if (b >= vfrom) m.vtri[b] = NONE;
    if (c >= vfrom) m.vtri[c] = NONE;
    if (s0 != NONE) m.stri[s0] = NONE, m.sflag[s0] = 2;
    if (s1 != NONE) m.stri[s1] = NONE, m.sflag[s1] = 2;
    if (s2 != NONE) m.stri[s2] = NONE, m.sflag[s2] = 2;
}

// slot: a slot reserved beforehand (block_reserve), or NONE to reserve here
__device__ __forceinline__ void push_touched(const WorkLists& w, const u32* ts, int k,
                                             RoundCtr* rc = nullptr, u32 slot = NONE) {
    const u32 o = slot != NONE ? slot : agg_reserve(&(rc ? rc : w.rc)->touched, (u32)k);
    for (int j = 0; j < k; ++j)
        if (o + j < w.cap) w.touched[o + j] = ts[j];
}

__device__ __forceinline__ void push_work(const WorkLists& w, u32 widx, const u32* codes, int k,
                                          Counters* ctr, RoundCtr* rc = nullptr, u32 slot = NONE) {
    const u32 o = slot != NONE ? slot : agg_reserve(&(rc ? rc : w.rc)->wl_next, (u32)k);
    if (o + k > w.cap) {
        raise_err(ctr, DERR_WORKLIST_OVERFLOW, o);
        return;
    }
    for (int j = 0; j < k; ++j) w.w[widx][o + j] = codes[j];
}

// split_triangle_with (mesh.hpp:323-346): t := (a,b,w), t1 := (b,c,w), t2 := (c,a,w).
// seed != 0: push the three link edges (opposite wv) as Lawson seeds.  The
// spokes (wv, a) need no test: an empty circle through wv and a exists inside
// the old circumcircle, so they are Delaunay edges (Lawson insertion); the
// flips that later change a spoke's quad push it again (flip_apply_one).
// slots (optional): [touched, work] slots reserved by the caller (block_reserve)
static __device__ void split_triangle_A(const DevMesh& m, const TriAux& x, const WorkLists& w, u32 t,
                                 u32 wv, u32 t1, u32 t2, u32 round, RoundCtr* rc = nullptr,
                                 int seed = 0, Counters* ctr = nullptr,
                                 const u32* slots = nullptr) {
    const uint4 ov = m.tv[t], on = m.tn[t], os = load_ts(m, t, ov);
    x.se[4 * t] = round;
    write_tri(m, t, ov.x, ov.y, wv, enc(t1, 1), enc(t2, 0), on.z, 4u, NONE, NONE, os.z, w.vtri_from);
    write_tri(m, t1, ov.y, ov.z, wv, enc(t2, 1), enc(t, 0), on.x, 4u, NONE, NONE, os.x, w.vtri_from);
    write_tri(m, t2, ov.z, ov.x, wv, enc(t, 1), enc(t1, 0), on.y, 4u, NONE, NONE, os.y, w.vtri_from);
    x.se[4 * t + 1 + 0] = enc(t1, 2);
    x.se[4 * t + 1 + 1] = enc(t2, 2);
    x.se[4 * t + 1 + 2] = enc(t, 2);
    m.vtri[wv] = NONE;
    const u32 tl[3] = {t, t1, t2};
    push_touched(w, tl, 3, rc, slots ? slots[0] : NONE);
    if (seed) {
        const u32 codes[3] = {enc(t, 2), enc(t1, 2), enc(t2, 2)};
        push_work(w, 0, codes, 3, ctr, rc, slots ? slots[1] : NONE);
    }
}

// split_edge_with (mesh.hpp:358-401) on edge e of t; new t2 (and u2 when the
// edge has a far side).  s_bw / s_wc are the child subsegments or NONE.
// seed != 0: push every edge of the new triangles (a point on an edge gets no
// empty-circle guarantee for the edge halves).
static __device__ void split_edge_A(const DevMesh& m, const TriAux& x, const WorkLists& w, u32 t, int e,
                             u32 wv, u32 t2, u32 u2, u32 s_bw, u32 s_wc, u32 round,
                             RoundCtr* rc = nullptr, int seed = 0, Counters* ctr = nullptr,
                             const u32* slots = nullptr) {
    const uint4 ov = m.tv[t], on = m.tn[t], os = load_ts(m, t, ov);
    const u32 a = comp(ov, e), b = comp(ov, nxt(e)), c = comp(ov, prv(e));
    const u32 uc = comp(on, e);
    x.se[4 * t] = round;
    if (uc == NONE) {
        // t := (a,b,w) {-, t2, n_prev}, t2 := (a,w,c) {-, n_next, t}
        write_tri(m, t, a, b, wv, NONE, enc(t2, 2), comp(on, prv(e)), 4u, s_bw, NONE,
                  comp(os, prv(e)), w.vtri_from);
        write_tri(m, t2, a, wv, c, NONE, comp(on, nxt(e)), enc(t, 1), 2u, s_wc,
                  comp(os, nxt(e)), NONE, w.vtri_from);
        x.se[4 * t + 1 + nxt(e)] = enc(t2, 1);
        x.se[4 * t + 1 + prv(e)] = enc(t, 2);
        x.se[4 * t + 1 + e] = NONE;
        m.vtri[wv] = NONE;
        const u32 tl[2] = {t, t2};
        push_touched(w, tl, 2, rc, slots ? slots[0] : NONE);
        if (seed && s_bw != NONE) {
            const u32 codes[2] = {enc(t, 2), enc(t2, 1)};
            push_work(w, 0, codes, 2, ctr, rc, slots ? slots[1] : NONE);
        } else if (seed) {
            const u32 codes[6] = {enc(t, 0), enc(t, 1), enc(t, 2), enc(t2, 0), enc(t2, 1),
                                  enc(t2, 2)};
            push_work(w, 0, codes, 6, ctr, rc, slots ? slots[1] : NONE);
        }
        return;
    }
    const u32 u = etri(uc);
    const int f = eidx(uc);
    const uint4 uv = m.tv[u], un = m.tn[u], us = load_ts(m, u, uv);
    const u32 d = comp(uv, f);
    x.se[4 * u] = round;
    // t := (a,b,w) {u2, t2, n_ab}; t2 := (a,w,c) {u, n_ca, t}
    write_tri(m, t, a, b, wv, enc(u2, 0), enc(t2, 2), comp(on, prv(e)), 4u, s_bw, NONE,
              comp(os, prv(e)), w.vtri_from);
    write_tri(m, t2, a, wv, c, enc(u, 0), comp(on, nxt(e)), enc(t, 1), 2u, s_wc,
              comp(os, nxt(e)), NONE, w.vtri_from);
    // u := (d,c,w) {t2, u2, n_dc}; u2 := (d,w,b) {t, n_bd, u}
    write_tri(m, u, d, c, wv, enc(t2, 0), enc(u2, 2), comp(un, prv(f)), 4u, s_wc, NONE,
              comp(us, prv(f)), w.vtri_from);
    write_tri(m, u2, d, wv, b, enc(t, 0), comp(un, nxt(f)), enc(u, 1), 2u, s_bw,
              comp(us, nxt(f)), NONE, w.vtri_from);
    x.se[4 * t + 1 + nxt(e)] = enc(t2, 1);
    x.se[4 * t + 1 + prv(e)] = enc(t, 2);
    x.se[4 * t + 1 + e] = NONE;
    x.se[4 * u + 1 + prv(f)] = enc(u, 2);
    x.se[4 * u + 1 + nxt(f)] = enc(u2, 1);
    x.se[4 * u + 1 + f] = NONE;
    m.vtri[wv] = NONE;
    const u32 tl[4] = {t, t2, u, u2};
    push_touched(w, tl, 4, rc, slots ? slots[0] : NONE);
    if (seed && s_bw != NONE) {
        // subsegment midpoint: the halves are constrained and the spokes
        // (w,a), (w,d) are constrained-Delaunay (a circle through a and w
        // inside the empty circumcircle of (a,b,c)); only the link edges
        const u32 codes[4] = {enc(t, 2), enc(t2, 1), enc(u, 2), enc(u2, 1)};
        push_work(w, 0, codes, 4, ctr, rc, slots ? slots[1] : NONE);
    } else if (seed) {
        const u32 codes[12] = {enc(t, 0), enc(t, 1), enc(t, 2), enc(t2, 0), enc(t2, 1),
                               enc(t2, 2), enc(u, 0), enc(u, 1), enc(u, 2), enc(u2, 0),
                               enc(u2, 1), enc(u2, 2)};
        push_work(w, 0, codes, 12, ctr, rc, slots ? slots[1] : NONE);
    }
}

// ---- the tail loop's dirty-element list (WorkLists::dlist) ---------------------------

__device__ __forceinline__ void dlist_push(const WorkLists& w, u32 key) {
    const u32 o = atomicAdd(w.dlist_n, 1u);
    if (o < w.dlist_cap) w.dlist[o] = key;
}

// ---- phase B ------------------------------------------------------------------------

__device__ __forceinline__ void fixup_one(const DevMesh& m, u32 round, const TriAux& x,
                                          const WorkLists& w, u32 t, int seed, u32 widx,
                                          RoundCtr* rc, Counters* ctr) {
    uint4 tn = m.tn[t];
    const uint4 tv = m.tv[t];
    if (!tv.w) return;
    const uint4 ts = load_ts(m, t, tv);
    const u32 pend = tn.w;
    // each far side's {stamp, emap[3]} record in one 16-byte load, all three
    // issued together before any store (a store between them would order
    // each load behind it)
    u32 sx[3], em[3];
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        const u32 r = comp(tn, e);
        uint4 se = make_uint4(0u, NONE, NONE, NONE);
        if (((pend >> e) & 1u) && r != NONE) se = reinterpret_cast<const uint4*>(x.se)[etri(r)];
        sx[e] = se.x;
        const int k = r != NONE ? eidx(r) : 0;   // emap slot k is word 1 + k
        em[e] = k == 0 ? se.y : (k == 1 ? se.z : se.w);
    }
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        if (!((pend >> e) & 1u)) continue;
        const u32 r = comp(tn, e);
        if (r == NONE) continue;
        if (sx[e] == round) {
            set_comp(tn, e, em[e]);
        } else {
            m.tn.words(etri(r))[eidx(r)] = enc(t, e);
        }
    }
    tn.w = 0;
    m.tn[t] = tn;
    if (w.dlist) {   // the tail loop re-evaluates what a rewrite touched
        dlist_push(w, 0x80000000u | t);
        if (ts.x != NONE) dlist_push(w, ts.x);
        if (ts.y != NONE) dlist_push(w, ts.y);
        if (ts.z != NONE) dlist_push(w, ts.z);
    }
    if (tv.x >= w.vtri_from) atomicMin(&m.vtri[tv.x], t);
    if (tv.y >= w.vtri_from) atomicMin(&m.vtri[tv.y], t);
    if (tv.z >= w.vtri_from) atomicMin(&m.vtri[tv.z], t);
    if (w.vdirty) {
        // Suspects for the redundancy detection (refine.hpp:551-608): a
        // same-batch circumcenter can only be redundant as the apex of a
        // subsegment, or dependent next to another same-batch circumcenter --
        // both visible on one triangle, and every triangle around a fresh
        // vertex passes through a fixup.  Only suspects are evaluated.
        const u32 j0 = tv.x - w.fresh_v0, j1 = tv.y - w.fresh_v0, j2 = tv.z - w.fresh_v0;
        const bool c0 = j0 < w.fresh_n && w.fresh_cc[j0];
        const bool c1 = j1 < w.fresh_n && w.fresh_cc[j1];
        const bool c2 = j2 < w.fresh_n && w.fresh_cc[j2];
        const bool pair = (int)c0 + (int)c1 + (int)c2 >= 2;
        if (c0 && (pair || ts.x != NONE)) w.vdirty[j0] = 1;
        if (c1 && (pair || ts.y != NONE)) w.vdirty[j1] = 1;
        if (c2 && (pair || ts.z != NONE)) w.vdirty[j2] = 1;
    }
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        const u32 s = comp(ts, e);
        if (s == NONE) continue;
        const u32 r = comp(tn, e);
        const u32 other = r == NONE ? NONE : etri(r);
        atomicMin(&m.stri[s], min(t, other));
    }
    if (seed) {
        const u32 codes[3] = {enc(t, 0), enc(t, 1), enc(t, 2)};
        push_work(w, widx, codes, 3, ctr, rc);
    }
}

// ---- Lawson flip rounds (lawson_fixpoint cdt.hpp:111-123) -----------------------------

// Test one work item (is_non_delaunay_edge mesh.hpp:430-437) on its canonical
// side (lower triangle id) and claim both triangles with the edge code as key:
// the minimum key wins, so a round's flip set is deterministic.  The claim is
// round-tagged, fown = max over (round << 32 | ~key): a later round's claim
// beats any stale one, so the claims are never reset.
// The test itself: true for a flip candidate (claims made), with its key
// (canonical side) and the far side's code.
__device__ __forceinline__ u64 flip_tag(u32 round, u32 key) {
    return ((u64)round << 32) | (u64)(~key);
}

__device__ __forceinline__ bool flip_test_eval(const DevMesh& m, u32 code, u32 round,
                                               const TriAux& x, u32& key_out, u32& uc_out) {
    u32 t = etri(code);
    int e = eidx(code);
    if (t >= m.nT) return false;
    // record loads issued together: the dependent chain is t's record ->
    // the neighbour's corners -> the four coordinates
    const uint4 tv0 = m.tv[t], tn0 = m.tn[t];
    if (!tv0.w) return false;
    const u32 c = comp(tn0, e);
    if (c == NONE || has_seg(tv0, e)) return false;
    u32 u = etri(c);
    int f = eidx(c);
    const uint4 tvu = m.tv[u];
    uint4 tv = tv0;
    u32 d = comp(tvu, f);
    if (u < t) {   // test on the canonical (lower id) side
        d = comp(tv0, e);
        tv = tvu;
        const u32 tt = t;
        const int ee = e;
        t = u;
        e = f;
        u = tt;
        f = ee;
    }
    if (incircle(m.xy[tv.x], m.xy[tv.y], m.xy[tv.z], m.xy[d]) <= 0) return false;
    const u32 key = enc(t, e);
    const u64 tag = flip_tag(round, key);
    atomicMax((ull*)&x.fown[t], (ull)tag);
    atomicMax((ull*)&x.fown[u], (ull)tag);
    key_out = key;
    uc_out = enc(u, f);
    return true;
}

__device__ __forceinline__ void flip_cand_store(const WorkLists& w, u32 o, u32 key, u32 uc,
                                                Counters* ctr) {
    if (o < w.cap) {
        w.fc[o] = key;
        w.fu[o] = uc;
    } else {
        raise_err(ctr, DERR_WORKLIST_OVERFLOW, o);
    }
}

__device__ __forceinline__ void flip_test_one(const DevMesh& m, u32 code, u32 round,
                                              const TriAux& x, const WorkLists& w, RoundCtr* rc,
                                              Counters* ctr) {
    u32 key, uc;
    if (!flip_test_eval(m, code, round, x, key, uc)) return;
    flip_cand_store(w, agg_reserve(&rc->cand, 1u), key, uc, ctr);
}

// flip (mesh.hpp:210-258) as a phase-A rewrite: t := (a,b,d), u := (a,d,c).
// Everything but the two list appends (the rewritten pair -> touched, its four
// outer edges -> the next work list); returns true when it flipped (t_out,
// u_out = the pair).
__device__ __forceinline__ bool flip_apply_core(const DevMesh& m, u32 i, u32 round,
                                                const TriAux& x, const WorkLists& w,
                                                Counters* ctr, u32& t_out, u32& u_out) {
    const u32 key = w.fc[i], uc = w.fu[i];
    const u32 t = etri(key), u = etri(uc);
    const int e = eidx(key), f = eidx(uc);
    // the pair's records are loaded together with the claims; a duplicate
    // work item (same key, all "win") that loses the stamp exchange below
    // discards them, and the winner's reads precede any write to the pair
    const u64 ot = x.fown[t], ou = x.fown[u];
    const uint4 tv = m.tv[t], tn = m.tn[t];
    const uint4 uv = m.tv[u], un = m.tn[u];
    const u64 tag = flip_tag(round, key);
    const bool won = ot == tag && ou == tag;
    w.fwin[i] = won;
    // exactly one duplicate performs the flip
    if (!won || atomicExch(&x.se[4 * t], round) == round) return false;
    const u32 a = comp(tv, e), b = comp(tv, nxt(e)), c = comp(tv, prv(e));
    const u32 d = comp(uv, f);
    const double2 pa = m.xy[a], pb = m.xy[b], pc = m.xy[c], pd = m.xy[d];
    const uint4 ts = load_ts(m, t, tv), us = load_ts(m, u, uv);
    x.se[4 * u] = round;
    if (orient2d(pa, pb, pd) <= 0 || orient2d(pa, pd, pc) <= 0) {
        if (atomicCAS(&ctr->err_code, 0u, (u32)DERR_NONCONVEX_FLIP) == 0u) {
            ctr->err_info = t;
            ctr->dbg[0] = pa.x; ctr->dbg[1] = pa.y; ctr->dbg[2] = pb.x; ctr->dbg[3] = pb.y;
            ctr->dbg[4] = pc.x; ctr->dbg[5] = pc.y; ctr->dbg[6] = pd.x; ctr->dbg[7] = pd.y;
        }
        return false;
    }
    write_tri(m, t, a, b, d, comp(un, nxt(f)), enc(u, 2), comp(tn, prv(e)), 5u,
              comp(us, nxt(f)), NONE, comp(ts, prv(e)), w.vtri_from);
    write_tri(m, u, a, d, c, comp(un, prv(f)), comp(tn, nxt(e)), enc(t, 1), 3u,
              comp(us, prv(f)), comp(ts, nxt(e)), NONE, w.vtri_from);
    x.se[4 * t + 1 + nxt(e)] = enc(u, 1);
    x.se[4 * t + 1 + prv(e)] = enc(t, 2);
    x.se[4 * t + 1 + e] = NONE;
    x.se[4 * u + 1 + nxt(f)] = enc(t, 0);
    x.se[4 * u + 1 + prv(f)] = enc(u, 0);
    x.se[4 * u + 1 + f] = NONE;
    t_out = t;
    u_out = u;
    return true;
}

// The appends of a flip at reserved slots: touched [ot, ot+2), work [ow, ow+4).
__device__ __forceinline__ void flip_appends(const WorkLists& w, u32 widx, u32 t, u32 u, u32 ot,
                                             u32 ow, Counters* ctr) {
    if (ot + 2 <= w.cap) {
        w.touched[ot] = t;
        w.touched[ot + 1] = u;
    }
    if (ow + 4 > w.cap) {
        raise_err(ctr, DERR_WORKLIST_OVERFLOW, ow);
        return;
    }
    w.w[widx][ow] = enc(t, 0);
    w.w[widx][ow + 1] = enc(t, 2);
    w.w[widx][ow + 2] = enc(u, 0);
    w.w[widx][ow + 3] = enc(u, 1);
}

__device__ __forceinline__ u32 flip_apply_one(const DevMesh& m, u32 i, u32 round, u32 widx,
                                              const TriAux& x, const WorkLists& w, RoundCtr* rc,
                                              Counters* ctr) {
    u32 t, u;
    if (!flip_apply_core(m, i, round, x, w, ctr, t, u)) return 0;
    const u32 tl[2] = {t, u};
    push_touched(w, tl, 2, rc);
    const u32 codes[4] = {enc(t, 0), enc(t, 2), enc(u, 0), enc(u, 1)};
    push_work(w, widx, codes, 4, ctr, rc);
    return 1;
}

// A loser whose triangles were both left untouched retries (returns its key
// to re-queue, or NONE).  The claims need no release (round-tagged).
__device__ __forceinline__ u32 flip_post_core(u32 i, u32 round, const TriAux& x,
                                              const WorkLists& w) {
    const u32 key = w.fc[i], uc = w.fu[i];
    const u32 t = etri(key), u = etri(uc);
    return (!w.fwin[i] && x.se[4 * t] != round && x.se[4 * u] != round) ? key : NONE;
}

__device__ __forceinline__ void flip_post_one(u32 i, u32 round, u32 widx, const TriAux& x,
                                              const WorkLists& w, RoundCtr* rc, Counters* ctr) {
    const u32 key = flip_post_core(i, round, x, w);
    if (key != NONE) {
        const u32 codes[1] = {key};
        push_work(w, widx, codes, 1, ctr, rc);
    }
}

// ---- grid-wide Lawson phases in waves --------------------------------------------
//
// The grid-mode rounds (refinement, device CDT, the parity hook) process their
// lists in waves of one item per thread, and every wave reserves the slots it
// appends with ONE atomic per CTA (block_reserve) instead of one per warp:
// the list counters are single addresses, and their same-address atomics
// queue thousands deep at mesh scale.  tid0 = the CTA's first grid thread,
// nthr = grid threads.  Every thread of every CTA calls these.

template <int BLOCK>
__device__ __forceinline__ void flip_test_waves(const DevMesh& m, const u32* wl, u32 n, u32 round,
                                                u32 tid0, u32 nthr, const TriAux& x,
                                                const WorkLists& w, RoundCtr* rc, Counters* ctr) {
    for (u32 base = tid0; base < n; base += nthr) {
        const u32 i = base + threadIdx.x;
        u32 key = 0, uc = 0;
        const bool cand = i < n && flip_test_eval(m, wl[i], round, x, key, uc);
        const u32 o = block_reserve<BLOCK>(&rc->cand, cand ? 1u : 0u);
        if (cand) flip_cand_store(w, o, key, uc, ctr);
    }
}

template <int BLOCK>
__device__ __forceinline__ u32 flip_apply_waves(const DevMesh& m, u32 nc, u32 round, u32 widx,
                                                u32 tid0, u32 nthr, const TriAux& x,
                                                const WorkLists& w, RoundCtr* rc, Counters* ctr) {
    u32 flipped = 0;
    for (u32 base = tid0; base < nc; base += nthr) {
        const u32 i = base + threadIdx.x;
        u32 t = 0, u = 0;
        const bool fl = i < nc && flip_apply_core(m, i, round, x, w, ctr, t, u);
        const u32 ot = block_reserve<BLOCK>(&rc->touched, fl ? 2u : 0u);
        const u32 ow = block_reserve<BLOCK>(&rc->wl_next, fl ? 4u : 0u);
        if (fl) flip_appends(w, widx, t, u, ot, ow, ctr);
        flipped += fl;
    }
    return flipped;
}

template <int BLOCK>
__device__ __forceinline__ void flip_post_waves(u32 nc, u32 round, u32 widx, u32 tid0, u32 nthr,
                                                const TriAux& x, const WorkLists& w,
                                                RoundCtr* rc, Counters* ctr) {
    for (u32 base = tid0; base < nc; base += nthr) {
        const u32 i = base + threadIdx.x;
        const u32 key = i < nc ? flip_post_core(i, round, x, w) : NONE;
        const u32 o = block_reserve<BLOCK>(&rc->wl_next, key != NONE ? 1u : 0u);
        if (key != NONE) {
            if (o < w.cap)
                w.w[widx][o] = key;
            else
                raise_err(ctr, DERR_WORKLIST_OVERFLOW, o);
        }
    }
}

}  // namespace gdp2d
