// k_cdt.cu -- Line 1 of Algorithm 1 on the device: the initial constrained
// Delaunay triangulation of a PSLG (build_cdt, cdt.hpp:483 =
// build_delaunay :198-250 + recover_segments :371-445 + lawson_fixpoint_all).
//
// The reference inserts points one at a time (walk, split, Lawson queue) and
// then recovers each segment by flipping the edges its pipe crosses.  Here:
//
//  1. Delaunay (k_cdt_delaunay, ONE persistent cooperative launch): all N
//     points start inside a super triangle (vertices N..N+2).  Each insertion
//     round every triangle that still contains points picks the one nearest
//     its circumcentre (u64 atomicMin of (distance, index), warp-aggregated
//     over lanes of the same triangle), the winners split 1->3 (or 2->4 on an
//     edge) through the shared local-rewrite protocol (gdp2d_rewrite.cuh)
//     with new triangle ids from a prefix sum over point index (so ids are
//     deterministic), the parallel Lawson rounds restore Delaunayhood, and
//     every point whose triangle was rewritten re-walks (a visibility walk,
//     which terminates on a Delaunay triangulation) from its old slot --
//     flips and splits keep slots, so the walk is a few steps.
//  2. Segment recovery (k_cdt_recover, one cooperative launch): each piece
//     (a segment, or part of one split at a collinear vertex exactly as
//     recover_chain :371-389 does) finds its edge in the star of its first
//     endpoint, or walks its pipe (collect_pipe :300-369) and claims the
//     pipe's triangles (atomicMin of the piece id).  A piece owning its whole
//     pipe re-triangulates it in private scratch with the reference's
//     crossing-edge flip queue (:391-432) -- every flip stays inside the pipe
//     -- and writes it back as one region rewrite.  Pipes of one round are
//     disjoint, so the pieces of a round run in parallel; the lowest id always
//     owns its pipe, so every round makes progress.
//  3. The super triangle's fan is cut away (every hull edge is an input
//     segment after close_hull, cdt.hpp:447), the constrained Lawson fixpoint
//     runs from the rewritten pipes, and the mesh is compacted (engine.cu).
//
// The CDT of a PSLG in general position is unique, so the result equals the
// reference's as a set of triangles (tests/test_gpu_cdt.py); ids differ.
#include <cooperative_groups.h>

#include <algorithm>

#include "gdp2d_rewrite.cuh"
#include "scan.cuh"

namespace cg = cooperative_groups;

#ifndef GDP2D_CDT_MINB
#define GDP2D_CDT_MINB 2   // CTAs per SM the Delaunay kernel is compiled for
#endif

namespace gdp2d {

namespace {

__device__ __forceinline__ u32 vld(const u32* p) { return *(const volatile u32*)p; }

__device__ __forceinline__ RoundCtr* ring_slot(const CdtArgs& a, u32 step) {
    return a.ring + (step & 3u);
}
// Zero the NEXT step's counters (read only after the barrier that ends this step).
__device__ __forceinline__ void ring_next(const CdtArgs& a, u32 step, bool leader) {
    if (leader) {
        RoundCtr* z = a.ring + ((step + 1u) & 3u);
        z->wl_next = z->cand = z->touched = z->rm_next = z->detect = 0;
        z->pad[0] = z->pad[1] = z->pad[2] = 0;
    }
}

static constexpr u32 PT_DEFER = 0xFFFFFFFDu;   // point of a later insertion level

__device__ __forceinline__ bool has_super(const uint4& tv, u32 N) {
    return tv.x >= N || tv.y >= N || tv.z >= N;
}

// ---- 1. Delaunay ----------------------------------------------------------------

// Pick key of point i in triangle t: squared distance to t's circumcentre (as
// an order-preserving float), then the index.
__device__ __forceinline__ u64 pick_key(const DevMesh& m, u32 t, u32 i, double2 p) {
    const uint4 tv = m.tv[t];
    bool ok;
    const double2 cc = circumcenter(m.xy[tv.x], m.xy[tv.y], m.xy[tv.z], ok);
    float f = ok ? (float)sqdist(p, cc) : 0.0f;
    if (!(f >= 0.0f)) f = 0.0f;
    return ((u64)__float_as_uint(f) << 32) | i;
}

// Visibility walk from t to p (terminates: the triangulation is Delaunay).
// 0 inside, 1 on edge *edge, 2 on a vertex (duplicate point), 3 failure.
__device__ __noinline__ int cdt_walk(const DevMesh& m, u32& t, double2 p, int& edge) {
    for (u32 it = 0; it < (1u << 22); ++it) {
        const uint4 tv = m.tv[t];
        const double2 a = m.xy[tv.x], b = m.xy[tv.y], c = m.xy[tv.z];
        int exit_e = -1;
        const int o0 = orient2d(b, c, p);
        int o1 = 1, o2 = 1;
        if (o0 < 0) {
            exit_e = 0;
        } else {
            o1 = orient2d(c, a, p);
            if (o1 < 0) {
                exit_e = 1;
            } else {
                o2 = orient2d(a, b, p);
                if (o2 < 0) exit_e = 2;
            }
        }
        if (exit_e >= 0) {
            const u32 r = comp(m.tn[t], exit_e);
            if (r == NONE) return 3;
            t = etri(r);
            continue;
        }
        const int z = (o0 == 0) + (o1 == 0) + (o2 == 0);
        if (z == 0) {
            edge = -1;
            return 0;
        }
        if (z == 1) {
            edge = o0 == 0 ? 0 : (o1 == 0 ? 1 : 2);
            return 1;
        }
        return 2;
    }
    return 3;
}

// (Re)locate point i starting from triangle t; sets ptri / pedge / pother / pkey.
__device__ __forceinline__ void relocate(const CdtArgs& a, u32 i, u32 t) {
    const double2 p = a.m.xy[i];
    int e = -1;
    const int r = cdt_walk(a.m, t, p, e);
    if (r >= 2) {
        raise_err(a.ctr, r == 2 ? DERR_DUPLICATE : DERR_CDT, i);
        a.ptri[i] = NONE;
        return;
    }
    a.ptri[i] = t;
    a.pedge[i] = (int8_t)e;
    a.pother[i] = e >= 0 ? etri(comp(a.m.tn[t], e)) : NONE;
    a.pkey[i] = pick_key(a.m, t, i, p);
}

}  // namespace

// state[]: CDT_ST_ROUNDS insertion rounds, CDT_ST_FLIP_ROUNDS, CDT_ST_STEPS,
// [0] = triangles in use at the end.
__global__ void __launch_bounds__(CDT_BLOCK, GDP2D_CDT_MINB) k_cdt_delaunay(const __grid_constant__ CdtArgs a) {
    cg::grid_group g = cg::this_grid();
    const u32 tid = (u32)g.thread_rank(), nthr = (u32)g.size();
    const u32 lane = threadIdx.x & 31u;
    const bool leader = tid == 0;
    const DevMesh& m = a.m;
    const u32 N = a.N;
    __shared__ u32 sh[CDT_BLOCK / 32 + 1];
    __shared__ u32 bc[2];

    // Insertion levels (biased randomised insertion order): the points with
    // i % stride == 0 first, then stride / 32, ... 1.  A level's points start
    // their walk at the triangle of the previous level's point (i / stride) *
    // stride -- a neighbour for spatially sorted input -- so the early rounds,
    // where every point would re-walk after every round, run on a sample.
    u32 stride = a.stride0;
    for (u32 i = tid; i < N; i += nthr) {
        if (i % stride == 0)
            relocate(a, i, 0);   // the super triangle
        else
            a.ptri[i] = PT_DEFER;
    }
    const u32 nblk = gridDim.x, b = blockIdx.x;
    const u32 chunk = ((N + nblk - 1) / nblk + CDT_BLOCK - 1) / CDT_BLOCK * CDT_BLOCK;
    const u32 lo = min(N, b * chunk), hi = min(N, lo + chunk);
    u32 step = 0, nT = 1, remaining = (N + stride - 1) / stride, rounds = 0, flip_rounds = 0;
    ull flipped = 0;
    ring_next(a, step + 3u, leader);   // slot of step 0
    g.sync();
    // Loop conditions are read from counters after a barrier, so they are
    // uniform over the grid; a device error never changes control flow (the
    // failing point / piece is dropped and the host raises the error).
    while (remaining > 0 && rounds < (1u << 16)) {
        // A: every occupied triangle keeps its minimum key
        for (u32 base = tid - lane; base < N; base += nthr) {
            const u32 i = base + lane;
            u32 t = NONE;
            u64 key = ~0ull;
            if (i < N) {
                t = a.ptri[i];
                if (t < PT_DEFER)
                    key = a.pkey[i];
                else
                    t = NONE;
            }
            const u32 grp = __match_any_sync(0xFFFFFFFFu, t);
            const u32 khi = (u32)(key >> 32);
            const u32 hmin = __reduce_min_sync(grp, khi);
            const u32 lmin = __reduce_min_sync(grp, khi == hmin ? (u32)key : 0xFFFFFFFFu);
            if (t != NONE) {
                const u64 k = ((u64)hmin << 32) | lmin;
                if ((int)lane == __ffs(grp) - 1 && a.tkey[t] > k) atomicMin((ull*)&a.tkey[t], (ull)k);
                const u32 u = a.pother[i];
                if (u != NONE) atomicMin((ull*)&a.tkey[u], (ull)key);
            }
        }
        g.sync();
        // B: winners (own their triangle, and the far one for an on-edge point)
        u32 cnt = 0;
        for (u32 i = lo + threadIdx.x; i < hi; i += CDT_BLOCK) {
            const u32 t = a.ptri[i];
            uint8_t win = 0;
            if (t < PT_DEFER) {
                const u64 key = a.pkey[i];
                const u32 u = a.pother[i];
                win = a.tkey[t] == key && (u == NONE || a.tkey[u] == key);
            }
            a.pwin[i] = win;
            cnt += win;
        }
        cnt = block_sum<CDT_BLOCK>(cnt, sh);
        if (threadIdx.x == 0) a.part[b] = cnt;
        g.sync();
        // C: prefix over the chunk sums, split the winners in index order
        u32 pre = 0, tot = 0;
        for (u32 k = threadIdx.x; k < nblk; k += CDT_BLOCK) {
            const u32 v = a.part[k];
            tot += v;
            if (k < b) pre += v;
        }
        pre = block_sum<CDT_BLOCK>(pre, sh);
        if (threadIdx.x == 0) bc[0] = pre;
        tot = block_sum<CDT_BLOCK>(tot, sh);
        if (threadIdx.x == 0) bc[1] = tot;
        __syncthreads();
        pre = bc[0];
        tot = bc[1];
        RoundCtr* rc = ring_slot(a, step);
        ring_next(a, step, leader);
        const u32 R = a.round0 + step;
        u32 c0 = pre;
        for (u32 base = lo; base < hi; base += CDT_BLOCK) {
            const u32 i = base + threadIdx.x;
            const u32 wv = i < hi ? a.pwin[i] : 0u;
            u32 bsum;
            const u32 ex = block_exclusive<CDT_BLOCK>(wv, sh, &bsum);
            if (i < hi) {
                const u32 t = a.ptri[i];
                if (t < PT_DEFER) {
                    const u32 u = a.pother[i];
                    if (wv) {
                        const u32 t1 = nT + 2u * (c0 + ex);
                        const int e = a.pedge[i];
                        if (e < 0)
                            split_triangle_A(m, a.x, a.w, t, i, t1, t1 + 1, R, rc, 1, a.ctr);
                        else
                            split_edge_A(m, a.x, a.w, t, e, i, t1, t1 + 1, NONE, NONE, R, rc, 1,
                                         a.ctr);
                        a.ptri[i] = NONE;
                    }
                    a.tkey[t] = ~0ull;
                    if (u != NONE) a.tkey[u] = ~0ull;
                }
            }
            c0 += bsum;
        }
        nT += 2u * tot;
        g.sync();
        if (tot == 0) {   // cannot happen: the minimum key always wins
            raise_err(a.ctr, DERR_CDT, remaining);
            break;
        }
        // D: phase B of the splits
        {
            const u32 nt = min(vld(&rc->touched), a.w.cap);
            for (u32 i = tid; i < nt; i += nthr) fixup_one(m, R, a.x, a.w, a.w.touched[i], 0, 0, rc, a.ctr);
        }
        g.sync();
        u32 n = vld(&rc->wl_next), cur = 0;
        ++step;
        // E: Lawson rounds (lawson_fixpoint, cdt.hpp:111-123)
        while (n > 0) {
            if (n > a.w.cap) {
                raise_err(a.ctr, DERR_WORKLIST_OVERFLOW, n);
                break;
            }
            RoundCtr* fr = ring_slot(a, step);
            ring_next(a, step, leader);
            const u32 round = a.round0 + step;
            const u32* wl = a.w.w[cur];
            const u32 tid0 = tid - threadIdx.x;   // waves (flip_*_waves)
            flip_test_waves<CDT_BLOCK>(m, wl, n, round, tid0, nthr, a.x, a.w, fr, a.ctr);
            g.sync();
            const u32 nc = min(vld(&fr->cand), a.w.cap);
            flipped += flip_apply_waves<CDT_BLOCK>(m, nc, round, cur ^ 1u, tid0, nthr, a.x, a.w, fr,
                                                   a.ctr);
            g.sync();
            flip_post_waves<CDT_BLOCK>(nc, round, cur ^ 1u, tid0, nthr, a.x, a.w, fr, a.ctr);
            const u32 nt = min(vld(&fr->touched), a.w.cap);
            for (u32 i = tid; i < nt; i += nthr) fixup_one(m, round, a.x, a.w, a.w.touched[i], 0, 0, fr, a.ctr);
            g.sync();
            n = vld(&fr->wl_next);
            cur ^= 1u;
            ++step;
            ++flip_rounds;
        }
        // F: points of rewritten triangles re-walk
        RoundCtr* lr = ring_slot(a, step);
        ring_next(a, step, leader);
        u32 left = 0;
        for (u32 i = tid; i < N; i += nthr) {
            const u32 t = a.ptri[i];
            if (t >= PT_DEFER) continue;
            ++left;
            if (a.x.se[4 * t] >= R) relocate(a, i, t);
        }
        block_add(&lr->detect, left);
        g.sync();
        remaining = vld(&lr->detect);
        ++step;
        ++rounds;
        if (remaining == 0 && stride > 1) {
            // next level: walk from the previous level's anchor point
            const u32 s2 = stride > 32 ? stride / 32 : 1;
            RoundCtr* ar = ring_slot(a, step);
            ring_next(a, step, leader);
            u32 act = 0;
            for (u32 i = tid; i < N; i += nthr) {
                if (i % s2 != 0 || a.ptri[i] != PT_DEFER) continue;
                const u32 t0 = m.vtri[(i / stride) * stride];
                relocate(a, i, t0 == NONE ? 0u : t0);
                ++act;
            }
            block_add(&ar->detect, act);
            g.sync();
            remaining = vld(&ar->detect);
            ++step;
            stride = s2;
        }
    }
    warp_add_ull(&a.ctr->flips, flipped);
    if (leader) {
        a.state[0] = nT;
        a.state[CDT_ST_ROUNDS] = rounds;
        a.state[CDT_ST_FLIP_ROUNDS] = flip_rounds;
        a.state[CDT_ST_STEPS] = step;
    }
}

// ---- 2. segment recovery --------------------------------------------------------

namespace {

// strictly_between (cdt.hpp:291-295): p on the open segment (u,w), given collinear.
__device__ __forceinline__ bool strictly_between(double2 u, double2 w, double2 p) {
    if (peq(p, u) || peq(p, w)) return false;
    return dot2(sub2(w, u), sub2(p, u)) > 0.0 && dot2(sub2(u, w), sub2(p, w)) > 0.0;
}

// proper_cross (cdt.hpp:286-290)
__device__ __forceinline__ bool proper_cross(double2 a, double2 b, double2 c, double2 d) {
    const int o1 = orient2d(a, b, c), o2 = orient2d(a, b, d);
    const int o3 = orient2d(c, d, a), o4 = orient2d(c, d, b);
    return o1 * o2 < 0 && o3 * o4 < 0;
}

enum : int { PIPE_FOUND = 0, PIPE_PIPE = 1, PIPE_SPLIT = 2, PIPE_ERR = 3 };

// Star of u (collect_pipe's exit-wedge search, cdt.hpp:306-327; find_edge
// :256-271).  FOUND: (t, e) is the edge (u, w).  SPLIT: info = the vertex
// strictly inside (u, w).  PIPE: (t, e) is the first crossed edge, opposite u.
__device__ int pipe_start(const DevMesh& m, u32 u, u32 w, u32& t_out, int& e_out, u32& info) {
    const double2 pu = m.xy[u], pw = m.xy[w];
    const u32 t0 = m.vtri[u];
    if (t0 == NONE) return PIPE_ERR;
    u32 t = t0;
    for (u32 guard = 0; guard < (1u << 16); ++guard) {
        const uint4 tv = m.tv[t];
        const int i = tv.x == u ? 0 : (tv.y == u ? 1 : 2);
        const u32 b = comp(tv, nxt(i)), c = comp(tv, prv(i));
        if (b == w) {
            t_out = t;
            e_out = prv(i);
            return PIPE_FOUND;
        }
        if (c == w) {
            t_out = t;
            e_out = nxt(i);
            return PIPE_FOUND;
        }
        const double2 pb = m.xy[b], pc = m.xy[c];
        const int ob = orient2d(pu, pw, pb), oc = orient2d(pu, pw, pc);
        if (ob == 0 && strictly_between(pu, pw, pb)) {
            info = b;
            return PIPE_SPLIT;
        }
        if (oc == 0 && strictly_between(pu, pw, pc)) {
            info = c;
            return PIPE_SPLIT;
        }
        if (ob < 0 && oc > 0) {
            t_out = t;
            e_out = i;
            return PIPE_PIPE;
        }
        // next triangle around u: across the edge (u, b), opposite c
        const u32 r = comp(m.tn[t], prv(i));
        if (r == NONE) return PIPE_ERR;   // open star: cannot happen inside the super triangle
        t = etri(r);
        if (t == t0) break;
    }
    return PIPE_ERR;
}

// Walk the pipe of (u, w) from its first crossed edge; writes the pipe's
// triangles to out[0..len) when out != null.  Returns PIPE_PIPE, PIPE_SPLIT
// (info = collinear vertex) or PIPE_ERR (info = DERR_*).
__device__ int pipe_walk(const DevMesh& m, u32 u, u32 w, u32 t, int e, u32* out, u32& len,
                         u32& info) {
    const double2 pu = m.xy[u], pw = m.xy[w];
    const uint4 tv0 = m.tv[t];
    u32 x = comp(tv0, prv(e)), y = comp(tv0, nxt(e));   // x on the + side, y on the - side
    len = 0;
    for (u32 guard = 0; guard < (1u << 26); ++guard) {
        if (out) out[len] = t;
        ++len;
        if (has_seg(m.tv[t], e)) {
            info = DERR_SEG_CROSS;
            return PIPE_ERR;
        }
        const u32 r = comp(m.tn[t], e);
        if (r == NONE) {
            info = DERR_CDT;
            return PIPE_ERR;
        }
        const u32 tn = etri(r);
        const int f = eidx(r);
        const uint4 tv = m.tv[tn];
        const u32 d = comp(tv, f);
        if (d == w) {
            if (out) out[len] = tn;
            ++len;
            return PIPE_PIPE;
        }
        const double2 pd = m.xy[d];
        const int od = orient2d(pu, pw, pd);
        if (od == 0) {
            if (strictly_between(pu, pw, pd)) {
                info = d;
                return PIPE_SPLIT;
            }
            info = DERR_SEG_VERTEX;
            return PIPE_ERR;
        }
        // exit through (d, y) when d is on the + side (opposite x), else (x, d)
        const u32 opp = od > 0 ? x : y;
        const int ne = tv.x == opp ? 0 : (tv.y == opp ? 1 : 2);
        if (od > 0)
            x = d;
        else
            y = d;
        t = tn;
        e = ne;
    }
    info = DERR_CDT;
    return PIPE_ERR;
}

__device__ __forceinline__ bool lbit(const CdtLocal& L, int e) { return (L.n.w >> e) & 1u; }

// Find the local edge {x, y} with a local far side.
__device__ bool lfind(const CdtLocal* L, u32 len, u32 x, u32 y, u32& j, int& e) {
    for (u32 k = 0; k < len; ++k) {
        const uint4 v = L[k].v;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const u32 p0 = comp(v, nxt(q)), p1 = comp(v, prv(q));
            if (((p0 == x && p1 == y) || (p0 == y && p1 == x)) && lbit(L[k], q)) {
                j = k;
                e = q;
                return true;
            }
        }
    }
    return false;
}

__device__ __forceinline__ void lset(CdtLocal& T, int e, u32 n, bool local, u32 s, u32 o) {
    set_comp(T.n, e, n);
    T.n.w = local ? (T.n.w | (1u << e)) : (T.n.w & ~(1u << e));
    set_comp(T.s, e, s);
    set_comp(T.o, e, o);
}

// flip (mesh.hpp:210-258) on local records: j := (a,b,d), j2 := (a,d,c).
__device__ void lflip(CdtLocal* L, u32 j, int e) {
    const CdtLocal T = L[j];
    const u32 r = comp(T.n, e);
    const u32 j2 = etri(r);
    const int f = eidx(r);
    const CdtLocal U = L[j2];
    const u32 a = comp(T.v, e), b = comp(T.v, nxt(e)), c = comp(T.v, prv(e));
    const u32 d = comp(U.v, f);
    CdtLocal NT, NU;
    NT.v = make_uint4(a, b, d, 0u);
    NU.v = make_uint4(a, d, c, 0u);
    NT.n.w = NU.n.w = 0;
    // j: edge 0 (b,d) from u's nxt(f); edge 1 (d,a) the diagonal; edge 2 (a,b) from t's prv(e)
    lset(NT, 0, comp(U.n, nxt(f)), lbit(U, nxt(f)), comp(U.s, nxt(f)), comp(U.o, nxt(f)));
    lset(NT, 1, enc(j2, 2), true, NONE, NONE);
    lset(NT, 2, comp(T.n, prv(e)), lbit(T, prv(e)), comp(T.s, prv(e)), comp(T.o, prv(e)));
    // j2: edge 0 (d,c) from u's prv(f); edge 1 (c,a) from t's nxt(e); edge 2 the diagonal
    lset(NU, 0, comp(U.n, prv(f)), lbit(U, prv(f)), comp(U.s, prv(f)), comp(U.o, prv(f)));
    lset(NU, 1, comp(T.n, nxt(e)), lbit(T, nxt(e)), comp(T.s, nxt(e)), comp(T.o, nxt(e)));
    lset(NU, 2, enc(j, 1), true, NONE, NONE);
    L[j] = NT;
    L[j2] = NU;
    // back-pointers of local neighbours whose edge moved
    const auto relink = [&](const CdtLocal& X, int q, u32 to) {
        if (lbit(X, q)) {
            const u32 rr = comp(X.n, q);
            set_comp(L[etri(rr)].n, eidx(rr), to);
        }
    };
    relink(NT, 0, enc(j, 0));
    relink(NT, 2, enc(j, 2));
    relink(NU, 0, enc(j2, 0));
    relink(NU, 1, enc(j2, 1));
}

// Re-triangulate one owned pipe (recover_chain's flip loop, cdt.hpp:391-432)
// and write it back as a region rewrite.  Returns false on failure (raised).
__device__ bool recover_pipe(const CdtArgs& a, u32 p, const u32* gid, u32 len, u32 R,
                             RoundCtr* rc) {
    const DevMesh& m = a.m;
    const uint2 seg = a.pc[p];
    const double2 pa = m.xy[seg.x], pb = m.xy[seg.y];
    const u32 base = agg_reserve(&rc->pad[0], len);
    if (base + len > a.pool_cap) {
        raise_err(a.ctr, DERR_WORKLIST_OVERFLOW, base + len);
        return false;
    }
    CdtLocal* L = a.pool + base;
    uint2* Q = a.queue + base;
    // local copy; neighbours inside the pipe become local references
    for (u32 j = 0; j < len; ++j) {
        const u32 g = gid[j];
        CdtLocal T;
        T.v = m.tv[g];
        T.s = load_ts(m, g, T.v);
        T.v.w = 0;
        const uint4 tn = m.tn[g];
        T.n = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const u32 r = comp(tn, e);
            u32 loc = NONE;
            if (r != NONE) {
                const u32 X = etri(r);
                if (j > 0 && gid[j - 1] == X) {
                    loc = j - 1;
                } else if (j + 1 < len && gid[j + 1] == X) {
                    loc = j + 1;
                } else {
                    for (u32 k = 0; k < len; ++k)
                        if (gid[k] == X) {
                            loc = k;
                            break;
                        }
                }
            }
            if (loc != NONE) {
                set_comp(T.n, e, enc(loc, eidx(r)));
                T.n.w |= 1u << e;
                set_comp(T.o, e, NONE);
            } else {
                set_comp(T.n, e, r);
                set_comp(T.o, e, enc(g, e));
            }
        }
        L[j] = T;
    }
    // the crossed edges, in pipe order
    const u32 k = len - 1;
    for (u32 j = 0; j < k; ++j) {
        int e = -1;
#pragma unroll
        for (int q = 0; q < 3; ++q)
            if (lbit(L[j], q) && etri(comp(L[j].n, q)) == j + 1) e = q;
        Q[j] = make_uint2(comp(L[j].v, nxt(e)), comp(L[j].v, prv(e)));
    }
    u32 qh = 0, qn = k;
    const u64 cap = 100000ull + 16ull * k * k;
    for (u64 guard = 0; qn > 0; ++guard) {
        if (guard > cap) {
            raise_err(a.ctr, DERR_CDT, p);
            return false;
        }
        const uint2 xy = Q[qh];
        qh = qh + 1 == k ? 0 : qh + 1;
        --qn;
        u32 j;
        int e;
        if (!lfind(L, len, xy.x, xy.y, j, e)) continue;
        if (!proper_cross(pa, pb, m.xy[xy.x], m.xy[xy.y])) continue;
        if (comp(L[j].s, e) != NONE) {
            raise_err(a.ctr, DERR_SEG_CROSS, p);
            return false;
        }
        const u32 r = comp(L[j].n, e);
        const u32 j2 = etri(r);
        const int f = eidx(r);
        const u32 va = comp(L[j].v, e), vb = comp(L[j].v, nxt(e)), vc = comp(L[j].v, prv(e));
        const u32 vd = comp(L[j2].v, f);
        const double2 xa = m.xy[va], xb = m.xy[vb], xc = m.xy[vc], xd = m.xy[vd];
        if (orient2d(xa, xb, xd) <= 0 || orient2d(xa, xd, xc) <= 0) {
            // not convex yet: retry after its neighbours are flipped
            u32 qt = qh + qn;
            if (qt >= k) qt -= k;
            Q[qt] = xy;
            ++qn;
            continue;
        }
        lflip(L, j, e);
        if (proper_cross(pa, pb, xa, xd)) {
            u32 qt = qh + qn;
            if (qt >= k) qt -= k;
            Q[qt] = make_uint2(va, vd);
            ++qn;
        }
    }
    // flag the recovered edge on both sides
    u32 j;
    int e;
    if (!lfind(L, len, seg.x, seg.y, j, e)) {
        raise_err(a.ctr, DERR_CDT, p);
        return false;
    }
    set_comp(L[j].s, e, p);
    {
        const u32 r = comp(L[j].n, e);
        set_comp(L[etri(r)].s, eidx(r), p);
    }
    // write back: one region rewrite (phase A); outer edges pending
    for (u32 q = 0; q < len; ++q) {
        const CdtLocal& T = L[q];
        const u32 g = gid[q];
        u32 nn[3], pend = 0;
#pragma unroll
        for (int e2 = 0; e2 < 3; ++e2) {
            const u32 r = comp(T.n, e2);
            if (lbit(T, e2)) {
                nn[e2] = enc(gid[etri(r)], eidx(r));
            } else {
                nn[e2] = r;
                if (r != NONE) pend |= 1u << e2;
                const u32 o = comp(T.o, e2);
                a.x.se[4 * (etri(o)) + 1 + eidx(o)] = enc(g, e2);
            }
        }
        a.x.se[4 * g] = R;
        write_tri(m, g, T.v.x, T.v.y, T.v.z, nn[0], nn[1], nn[2], pend, T.s.x, T.s.y, T.s.z);
    }
    {
        const u32 o = agg_reserve(&rc->touched, len);
        for (u32 q = 0; q < len; ++q)
            if (o + q < a.w.cap) a.w.touched[o + q] = gid[q];
        const u32 so = atomicAdd(&a.state[CDT_ST_SEEDS], 3u * len);
        for (u32 q = 0; q < len; ++q)
            for (int e2 = 0; e2 < 3; ++e2)
                if (so + 3 * q + e2 < a.seed_cap) a.seeds[so + 3 * q + e2] = enc(gid[q], e2);
        if (so + 3 * len > a.seed_cap) raise_err(a.ctr, DERR_WORKLIST_OVERFLOW, so + 3 * len);
    }
    return true;
}

}  // namespace

// Pieces of plist[0][0..n0).  state[CDT_ST_NPIECES] = pieces allocated.
__global__ void __launch_bounds__(CDT_BLOCK) k_cdt_recover(const __grid_constant__ CdtArgs a, u32 n0) {
    cg::grid_group g = cg::this_grid();
    const u32 tid = (u32)g.thread_rank(), nthr = (u32)g.size();
    const bool leader = tid == 0;
    const DevMesh& m = a.m;
    u32* tsw = reinterpret_cast<u32*>(m.ts);
    u32 n = n0, cur = 0, step = 0, rounds = 0;
    u32 found = 0, pipes = 0, splits = 0, pmax = 0;
    ring_next(a, step + 3u, leader);
    // rewrites do not store the ts record of a triangle without subsegments
    // (write_tri): make every such record NONE before edges get flagged
    for (u32 t = tid; t < m.nT; t += nthr)
        if (!any_seg(m.tv[t])) m.ts[t] = make_uint4(NONE, NONE, NONE, 0u);
    g.sync();
    while (n > 0 && rounds < (1u << 16)) {
        RoundCtr* rc = ring_slot(a, step);
        ring_next(a, step, leader);
        const u32 R = a.round0 + step;
        const u32* list = a.plist[cur];
        u32* next = a.plist[cur ^ 1u];
        // A: find the edge, split at a collinear vertex, or claim the pipe
        for (u32 j = tid; j < n; j += nthr) {
            const u32 p = list[j];
            const uint2 s = a.pc[p];
            u32 t = NONE, info = 0, len = 0;
            int e = -1;
            int r = pipe_start(m, s.x, s.y, t, e, info);
            if (r == PIPE_PIPE) r = pipe_walk(m, s.x, s.y, t, e, nullptr, len, info);
            if (r == PIPE_FOUND) {
                // flag_edge (cdt.hpp:273-284); the lower piece keeps a shared edge
                const u32 far = comp(m.tn[t], e);
                atomicMin(&tsw[4 * (size_t)t + e], p);
                atomicOr(&m.tv.words(t)[3], 2u << e);   // the tv.w subsegment bit
                if (far != NONE) {
                    atomicMin(&tsw[4 * (size_t)etri(far) + eidx(far)], p);
                    atomicOr(&m.tv.words(etri(far))[3], 2u << eidx(far));
                }
                a.plen[p] = 0;
                ++found;
            } else if (r == PIPE_SPLIT) {
                // recover_chain (cdt.hpp:386-389): (u, c) then (c, w)
                const u32 q = atomicAdd(&a.state[CDT_ST_NPIECES], 2u);
                if (q + 2 > a.pcap) {
                    raise_err(a.ctr, DERR_WORKLIST_OVERFLOW, q + 2);
                    continue;
                }
                const u32 par = a.ppar[p];
                a.pc[q] = make_uint2(s.x, info);
                a.pc[q + 1] = make_uint2(info, s.y);
                a.ppar[q] = par;
                a.ppar[q + 1] = par;
                a.plen[q] = a.plen[q + 1] = NONE;
                a.plen[p] = NONE;   // retired
                const u32 o = agg_reserve(&rc->rm_next, 2u);
                next[o] = q;
                next[o + 1] = q + 1;
                ++splits;
            } else if (r == PIPE_PIPE) {
                const u32 o = agg_reserve(&rc->cand, len);
                if (o + len > a.claim_cap) {
                    raise_err(a.ctr, DERR_WORKLIST_OVERFLOW, o + len);
                    continue;
                }
                u32 l2 = 0;
                pipe_walk(m, s.x, s.y, t, e, a.claims + o, l2, info);
                for (u32 k = 0; k < len; ++k) atomicMin(&a.x.owner[a.claims[o + k]], p);
                a.poff[p] = o;
                a.plen[p] = len;
                pmax = max(pmax, len);
            } else {
                raise_err(a.ctr, info >= DERR_DUPLICATE && info <= DERR_SEG_VERTEX ? info : DERR_CDT, p);
            }
        }
        g.sync();
        // B: a piece owning its whole pipe re-triangulates it
        for (u32 j = tid; j < n; j += nthr) {
            const u32 p = list[j];
            const u32 len = a.plen[p];
            if (len == 0 || len == NONE) continue;
            const u32* gid = a.claims + a.poff[p];
            bool own = true;
            for (u32 k = 0; k < len && own; ++k) own = a.x.owner[gid[k]] == p;
            if (own) {
                if (recover_pipe(a, p, gid, len, R, rc)) ++pipes;
            } else {
                const u32 o = agg_reserve(&rc->rm_next, 1u);
                next[o] = p;
            }
        }
        g.sync();
        // C: phase B of the rewrites; release the claims
        {
            const u32 nt = min(vld(&rc->touched), a.w.cap);
            for (u32 i = tid; i < nt; i += nthr) fixup_one(m, R, a.x, a.w, a.w.touched[i], 0, 0, rc, a.ctr);
            const u32 nc = min(vld(&rc->cand), a.claim_cap);
            for (u32 i = tid; i < nc; i += nthr) a.x.owner[a.claims[i]] = NONE;
        }
        g.sync();
        n = vld(&rc->rm_next);
        cur ^= 1u;
        ++step;
        ++rounds;
    }
    block_add(&a.state[CDT_ST_FOUND], found);
    block_add(&a.state[CDT_ST_PIPES], pipes);
    block_add(&a.state[CDT_ST_SPLITS], splits);
    pmax = __reduce_max_sync(0xFFFFFFFFu, pmax);
    if ((threadIdx.x & 31) == 0) atomicMax(&a.state[CDT_ST_PIPE_MAX], pmax);
    if (leader) {
        a.state[CDT_ST_RECOVER_ROUNDS] = rounds;
        a.state[12] = step;
    }
}

// ---- 3. super triangle removal, compaction -----------------------------------

// pass 0: real triangles drop their links to the super triangle's fan
// pass 1: the fan dies
__global__ void k_cdt_strip(DevMesh m, u32 N, int pass) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m.nT) return;
    const uint4 tv = m.tv[t];
    if (!tv.w) return;
    if (pass == 1) {
        if (has_super(tv, N)) {
            m.tv[t].w = 0;
            m.tflag[t] = 2;
        }
        return;
    }
    if (has_super(tv, N)) return;
    uint4 tn = m.tn[t];
    bool ch = false;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        const u32 r = comp(tn, e);
        if (r != NONE && has_super(m.tv[etri(r)], N)) {
            set_comp(tn, e, NONE);
            ch = true;
        }
    }
    if (ch) m.tn[t] = tn;
}

__global__ void k_cdt_bbox(const double2* __restrict__ xy, u32 n, ull* out, Counters* ctr) {
    // order-preserving u64 images of doubles: min x, min y, max x, max y
    const auto key = [](double d) {
        const ull b = (ull)__double_as_longlong(d);
        return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    };
    ull k0 = ~0ull, k1 = ~0ull, k2 = 0, k3 = 0;
    bool bad = false;
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double2 p = xy[i];
        if (!isfinite(p.x) || !isfinite(p.y)) {
            bad = true;
            continue;
        }
        const ull kx = key(p.x), ky = key(p.y);
        k0 = min(k0, kx);
        k1 = min(k1, ky);
        k2 = max(k2, kx);
        k3 = max(k3, ky);
    }
    for (int o = 16; o > 0; o >>= 1) {
        k0 = min(k0, __shfl_down_sync(0xFFFFFFFFu, k0, o));
        k1 = min(k1, __shfl_down_sync(0xFFFFFFFFu, k1, o));
        k2 = max(k2, __shfl_down_sync(0xFFFFFFFFu, k2, o));
        k3 = max(k3, __shfl_down_sync(0xFFFFFFFFu, k3, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&out[0], k0);
        atomicMin(&out[1], k1);
        atomicMax(&out[2], k2);
        atomicMax(&out[3], k3);
    }
    if (bad) raise_err(ctr, DERR_NONFINITE, 0);
}

__global__ void k_alive_flags(DevMesh m, u32* flags) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m.nT) flags[t] = m.tv[t].w != 0;
}

// plive[p] = 1 for every piece that owns a flagged edge
__global__ void k_cdt_piece_live(DevMesh m, u32* plive) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m.nT) return;
    const uint4 tv = m.tv[t];
    if (!tv.w) return;
    const uint4 ts = load_ts(m, t, tv);
    if (ts.x != NONE) plive[ts.x] = 1;
    if (ts.y != NONE) plive[ts.y] = 1;
    if (ts.z != NONE) plive[ts.z] = 1;
}

__global__ void k_cdt_compact_tris(DevMesh s, DevMesh d, const u32* __restrict__ newid,
                                   const u32* __restrict__ pmap) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s.nT) return;
    const uint4 tv = s.tv[t];
    if (!tv.w) return;
    const u32 nt = newid[t];
    const uint4 tn = s.tn[t], ts = load_ts(s, t, tv);
    const auto mapn = [&](u32 r) { return r == NONE ? NONE : enc(newid[etri(r)], eidx(r)); };
    const auto maps = [&](u32 p) { return p == NONE ? NONE : pmap[p]; };
    const uint4 sn = make_uint4(maps(ts.x), maps(ts.y), maps(ts.z), 0u);
    d.tv[nt] = make_uint4(tv.x, tv.y, tv.z, tri_flags(sn.x, sn.y, sn.z));
    d.tn[nt] = make_uint4(mapn(tn.x), mapn(tn.y), mapn(tn.z), 0u);
    d.ts[nt] = sn;
    d.tflag[nt] = 2;
    atomicMin(&d.vtri[tv.x], nt);
    atomicMin(&d.vtri[tv.y], nt);
    atomicMin(&d.vtri[tv.z], nt);
    if (sn.x != NONE) atomicMin(&d.stri[sn.x], nt);
    if (sn.y != NONE) atomicMin(&d.stri[sn.y], nt);
    if (sn.z != NONE) atomicMin(&d.stri[sn.z], nt);
}

__global__ void k_cdt_compact_verts(DevMesh s, DevMesh d, u32 N) {
    const u32 v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= N) return;
    d.xy[v] = s.xy[v];
    d.vkind[v] = 0;
    d.vbirth[v] = 0;
    d.valive[v] = 1;
    d.vtri[v] = NONE;
}

__global__ void k_cdt_compact_segs(DevMesh d, const uint2* __restrict__ pc,
                                   const u32* __restrict__ ppar, const u32* __restrict__ pmap,
                                   u32 np) {
    const u32 p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= np) return;
    const u32 s = pmap[p];
    if (s == NONE) return;
    d.sv[s] = pc[p];
    d.sparent[s] = ppar[p];
    d.senc[s] = 0;
    d.salive[s] = 1;
    d.stri[s] = NONE;
    d.sdepth[s] = 0;
    d.sflag[s] = 2;
}

__global__ void k_cdt_pmap(const u32* __restrict__ plive, const u32* __restrict__ pre, u32* pmap,
                           u32 n) {
    const u32 p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) pmap[p] = plive[p] ? pre[p] : NONE;
}

// ---- launchers -------------------------------------------------------------------

int cdt_grid(int device, int which) {
    static int cached[64][2] = {};
    if (device >= 0 && device < 64 && cached[device][which]) return cached[device][which];
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, which ? (const void*)k_cdt_recover : (const void*)k_cdt_delaunay, CDT_BLOCK, 0);
    const int g = std::max(1, sms * std::max(1, per_sm));
    if (device >= 0 && device < 64) cached[device][which] = g;
    return g;
}

void launch_cdt_delaunay(const CdtArgs& a, int grid, cudaStream_t st) {
    void* args[] = {(void*)&a};
    note_launch();
    cudaLaunchCooperativeKernel((void*)k_cdt_delaunay, dim3(grid), dim3(CDT_BLOCK), args, 0, st);
}

void launch_cdt_recover(const CdtArgs& a, u32 n_pieces, int grid, cudaStream_t st) {
    void* args[] = {(void*)&a, &n_pieces};
    note_launch();
    cudaLaunchCooperativeKernel((void*)k_cdt_recover, dim3(grid), dim3(CDT_BLOCK), args, 0, st);
}

void launch_cdt_strip(const DevMesh& m, u32 N, cudaStream_t st) {
    if (!m.nT) return;
    const u32 g = (m.nT + 255) / 256;
    note_launch(), k_cdt_strip<<<g, 256, 0, st>>>(m, N, 0);
    note_launch(), k_cdt_strip<<<g, 256, 0, st>>>(m, N, 1);
}

void launch_cdt_bbox(const double2* xy, u32 n, ull* out4, Counters* ctr, cudaStream_t st) {
    const ull init[4] = {~0ull, ~0ull, 0ull, 0ull};
    cudaMemcpyAsync(out4, init, sizeof init, cudaMemcpyHostToDevice, st);
    const u32 g = std::min<u32>(1184, (n + 255) / 256 + 1);
    note_launch(), k_cdt_bbox<<<g, 256, 0, st>>>(xy, n, out4, ctr);
}

void launch_cdt_pmap(const u32* plive, const u32* pre, u32* pmap, u32 n, cudaStream_t st) {
    if (n) note_launch(), k_cdt_pmap<<<(n + 255) / 256, 256, 0, st>>>(plive, pre, pmap, n);
}

void launch_alive_flags(const DevMesh& m, u32* flags, cudaStream_t st) {
    if (!m.nT) return;
    note_launch(), k_alive_flags<<<(m.nT + 255) / 256, 256, 0, st>>>(m, flags);
}

void launch_cdt_piece_live(const DevMesh& m, u32* plive, cudaStream_t st) {
    if (!m.nT) return;
    note_launch(), k_cdt_piece_live<<<(m.nT + 255) / 256, 256, 0, st>>>(m, plive);
}

void launch_cdt_compact(const DevMesh& src, DevMesh dst, u32 N, const u32* newid,
                        const uint2* pc, const u32* ppar, const u32* pmap, u32 npieces,
                        cudaStream_t st) {
    if (N) note_launch(), k_cdt_compact_verts<<<(N + 255) / 256, 256, 0, st>>>(src, dst, N);
    if (npieces)
        note_launch(), k_cdt_compact_segs<<<(npieces + 255) / 256, 256, 0, st>>>(dst, pc, ppar, pmap, npieces);
    if (src.nT) note_launch(), k_cdt_compact_tris<<<(src.nT + 255) / 256, 256, 0, st>>>(src, dst, newid, pmap);
}

}  // namespace gdp2d
