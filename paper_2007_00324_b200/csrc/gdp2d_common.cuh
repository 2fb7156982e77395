// gdp2d_common.cuh -- device-side mesh layout, adjacency encoding and shared
// helpers of the B200 gDP2d engine.
//
// HBM layout (structure of arrays, one mesh per GPU, pre-allocated with
// headroom and grown by the host between batches):
//   double2 xy[V]                       vertex coordinates (16 B, one LDG.128)
//   TriRec  tr[T] = {tv, tn}            one 32-byte record per triangle, so the
//                                       corners and the neighbours that nearly every
//                                       step reads together share one DRAM burst:
//   uint4   tv[T] = {v0, v1, v2, flags} triangle corners   (reference Triangle::v);
//                                       flags = 0 dead, else bit 0 (alive) | bit 1+e
//                                       when edge e carries a subsegment, so the hot
//                                       paths read ts only for the few triangles
//                                       that have one
//   uint4   tn[T] = {n0, n1, n2, pend}  neighbours encoded (tri << 2) | edge so the
//                                       far side's edge slot is known without the
//                                       index_of_neighbor scan of mesh.hpp:107
//   uint4   ts[T] = {s0, s1, s2, -}     subsegment carried by edge i (or NONE)
//   uint2   sv[S], sparent[S], senc[S], salive[S], stri[S], sdepth[S]
// Edge i of a triangle is opposite corner i: (v[i+1], v[i+2]) (mesh.hpp:115).
#pragma once

#include <cooperative_groups.h>
#include <cooperative_groups/scan.h>
#include <cstdint>
#include <cuda_runtime.h>

namespace gdp2d {

typedef uint32_t u32;
typedef uint64_t u64;
typedef unsigned long long ull;

static constexpr u32 NONE = 0xFFFFFFFFu;
static constexpr u32 PENDING = 0xFFFFFFFEu;
static constexpr int MAX_CAVITY_N = 64;     // cavity_n upper bound (region <= n+1)
static constexpr int MAX_STAR = 96;         // vertex degree bound for removal
static constexpr int MAX_CLAIM_EXTRA = 2;   // extra claimed triangles per candidate

__host__ __device__ __forceinline__ u32 enc(u32 t, int e) { return (t << 2) | (u32)e; }
__host__ __device__ __forceinline__ u32 etri(u32 c) { return c >> 2; }
__host__ __device__ __forceinline__ int eidx(u32 c) { return (int)(c & 3u); }
__host__ __device__ __forceinline__ int nxt(int i) { return i == 2 ? 0 : i + 1; }
__host__ __device__ __forceinline__ int prv(int i) { return i == 0 ? 2 : i - 1; }

__device__ __forceinline__ u32 comp(const uint4& q, int i) {
    return i == 0 ? q.x : (i == 1 ? q.y : q.z);
}
__device__ __forceinline__ void set_comp(uint4& q, int i, u32 v) {
    if (i == 0) q.x = v; else if (i == 1) q.y = v; else q.z = v;
}

// tv.w of an alive triangle whose edges carry subsegments s0, s1, s2 (or NONE)
__host__ __device__ __forceinline__ u32 tri_flags(u32 s0, u32 s1, u32 s2) {
    return 1u | (s0 != NONE ? 2u : 0u) | (s1 != NONE ? 4u : 0u) | (s2 != NONE ? 8u : 0u);
}
// edge e of the triangle whose corners record is tv carries a subsegment
__device__ __forceinline__ bool has_seg(const uint4& tv, int e) { return (tv.w >> (1 + e)) & 1u; }
__device__ __forceinline__ bool any_seg(const uint4& tv) { return (tv.w & 14u) != 0u; }

// tv / tn are views into the triangle records tr: element t at p[2 t].
struct TriRec {
    uint4 v, n;
};
struct RecField {
    uint4* p;
    __host__ __device__ __forceinline__ uint4& operator[](size_t t) const { return p[2 * t]; }
    __host__ __device__ __forceinline__ u32* words(size_t t) const {
        return reinterpret_cast<u32*>(p + 2 * t);
    }
};

struct DevMesh {
    double2* xy;
    uint8_t* vkind;
    u32* vbirth;
    uint8_t* valive;
    u32* vtri;
    TriRec* tr;
    RecField tv;     // = {&tr->v}
    RecField tn;     // = {&tr->n}
    uint4* ts;
    uint2* sv;
    u32* sparent;
    u32* senc;       // encroached flag (u32 so it can be set atomically)
    uint8_t* salive;
    u32* stri;
    u32* sdepth;
    // collect cache: bit0 = cached verdict (is_bad_triangle && resolvable /
    // geometric encroachment), bit1 = dirty.  Every triangle rewrite
    // (write_tri) and kill sets 2 on the triangle and on its subsegments, so
    // the Line-3 scan re-evaluates exactly the elements whose inputs changed.
    uint8_t* tflag;
    uint8_t* sflag;
    u32 nV, nT, nS;
};

// re-point the tv / tn views after tr was (re)allocated
__host__ __forceinline__ void bind_tris(DevMesh& m) {
    m.tv.p = m.tr ? &m.tr->v : nullptr;
    m.tn.p = m.tr ? &m.tr->n : nullptr;
}

// ts[t] for a triangle whose corners record tv is already loaded: the load is
// skipped (all NONE) when no edge carries a subsegment -- most triangles.
// Every reader of ts goes through the bits: a rewrite that leaves a triangle
// without subsegments does not store its ts record, so ts[t] is stale then.
__device__ __forceinline__ uint4 load_ts(const DevMesh& m, u32 t, const uint4& tv) {
    return any_seg(tv) ? m.ts[t] : make_uint4(NONE, NONE, NONE, 0u);
}

// Candidate list (SplitCandidate, refine.hpp:71) as structure of arrays.
struct DevCands {
    double2* pt;
    u64* key;       // (band << 63) | bits(measure): order-preserving for measure >= 0
    u32* id;
    u32* tie;       // PriorityKey::tiebreak
    u32* loc;       // located triangle
    uint8_t* kind;  // 0 Subseg, 1 Tri
    uint8_t* alive;
    uint8_t* lkind; // Location kind found by the walk (GDP2D_LOC_*)
    int8_t* ledge;  // edge for OnEdge
    uint8_t* fb;    // circumcenter fallback used
    u32* red;       // isolated insertion: lowest splittable subsegment the point would encroach
    uint8_t* unsafe;// isolated insertion: cavity hit the cap (not provably isolated)
    u32* far;       // far side of this candidate's split edge (rewrite table), or NONE
};

// Per-batch device counters (zeroed at the start of each batch).
struct Counters {
    u32 ncand;
    u32 nsub;
    u32 surv_claim;
    u32 surv_cavity;
    ull walk_steps;
    ull cavity_visits;
    u32 ins_mid, ins_cc;
    u32 rm_red, rm_dep;
    u32 dropped, marked;
    u32 nops;           // insertion ops scheduled
    u32 flip_rounds;
    ull flips;
    u32 rm_rounds;
    u32 rm_done;
    u32 err_code;
    u32 err_info;
    u32 fallbacks;
    u32 rm_kept;        // removals abandoned (degenerate star)
    u32 scan_dirty;     // triangles re-evaluated by the collect scan
    double dbg[8];      // coordinates attached to the first device error
};

// Per-round work-list counters (zeroed by the host before every round).
struct RoundCtr {
    u32 wl_next;   // entries appended to the next Lawson work list
    u32 cand;      // flip candidates of this round
    u32 touched;   // triangles rewritten this round
    u32 rm_next;   // removals deferred to the next round
    u32 detect;    // removals found by a detection pass
    u32 pad[3];
};

// Error codes raised on the device (copied into gdp2d_last_error()).
enum DevErr : u32 {
    DERR_NONE = 0,
    DERR_NONCONVEX_FLIP = 1,
    DERR_STAR_TOO_LARGE = 2,
    DERR_NO_EAR = 3,
    DERR_WORKLIST_OVERFLOW = 4,
    DERR_OPEN_STAR = 5,
    DERR_STALE = 6,
    DERR_WALK = 7,
    DERR_DUPLICATE = 8,     // CDT: two input points coincide
    DERR_SEG_CROSS = 9,     // CDT: input segments cross
    DERR_CDT = 10,          // CDT: walk / recovery did not converge
    DERR_NONFINITE = 11,    // CDT: non-finite coordinate
    DERR_SEG_VERTEX = 12,   // CDT: a segment passes through a vertex at its end (degenerate pipe)
};

__device__ __forceinline__ void raise_err(Counters* c, u32 code, u32 info) {
    if (atomicCAS(&c->err_code, 0u, code) == 0u) c->err_info = info;
}

__device__ __forceinline__ u64 make_key(int band, double measure) {
    return ((u64)band << 63) | ((u64)__double_as_longlong(measure) & 0x7FFFFFFFFFFFFFFFull);
}

// Warp-aggregated reservation of k slots on a shared append counter: the
// lanes that are converged at the call site scan their k, ONE lane issues the
// atomicAdd and broadcasts the base.  Work lists are appended by every thread
// of a grid; a same-address atomic per thread serialises in one L2 slice
// (hundreds of microseconds per round at mesh scale), one per warp does not.
__device__ __forceinline__ u32 agg_reserve(u32* ctr, u32 k) {
    namespace cg = cooperative_groups;
    cg::coalesced_group g = cg::coalesced_threads();
    const u32 pre = cg::exclusive_scan(g, k);
    u32 base = 0;
    const u32 last = g.num_threads() - 1;
    if (g.thread_rank() == last) base = atomicAdd(ctr, pre + k);
    base = g.shfl(base, last);
    return base + pre;
}

// Warp-aggregated atomic add on a 64-bit counter.  Must be called by all 32
// lanes of the warp (kernels never return early before calling it).
__device__ __forceinline__ void warp_add_ull(ull* ctr, ull v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(ctr, v);
}
__device__ __forceinline__ void warp_add_u32(u32* ctr, u32 v) {
    v = __reduce_add_sync(0xFFFFFFFFu, v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(ctr, v);
}

}  // namespace gdp2d
