// engine.h -- internal host-side declarations shared by the engine's
// translation units (kernel launchers + context).  Not part of the C ABI.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "gdp2d.h"
#include "gdp2d_common.cuh"
#include "gdp2d_geom.cuh"

namespace gdp2d {

// Process-wide count of engine kernel launches (reported by bench.py as
// gpu_launches; every <<<>>> in the engine goes through note_launch()).
unsigned long long& launch_counter();
inline void note_launch() { __atomic_add_fetch(&launch_counter(), 1ull, __ATOMIC_RELAXED); }

constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;

struct ScanScratch {
    u32* partial = nullptr;   // per-tile sums
    u32 cap = 0;              // tiles
};

// Exclusive scan of n u32 values; writes total to *d_total (device) if given.
void scan_exclusive(const u32* in, u32* out, u32 n, u32* d_total, ScanScratch& s,
                    cudaStream_t st);

// In-place exclusive scan of per-tile sums (single block).
void scan_partials(u32* partial, u32 ntiles, u32* d_total, cudaStream_t st);

// Per-triangle scratch (claims, stamps, edge maps).
struct TriAux {
    // claim key (band|measure) and tie (tiebreak << 32 | list index) of
    // triangle t at ckey[cslot(t)] / ctie[cslot(t)]: one allocation of 2T
    // words, ctie = ckey + 1 (interleaved 16-byte records)
    u64* ckey = nullptr;
    u64* ctie = nullptr;
    u32* owner = nullptr;    // device-CDT pipe claim
    u64* fown = nullptr;     // flip / removal claim: max (round << 32 | ~key), never reset
    // one 16-byte record per triangle: se[4t] = stamp (round in which the
    // triangle was rewritten), se[4t + 1 + k] = emap (old edge slot k -> new
    // tri<<2|edge); fixup reads a far side's stamp and emap in one load
    u32* se = nullptr;
    // rewrite table: every candidate claims the triangles its split REWRITES
    // (located, + the far side of a split edge); see gdp2d_phases.cuh
    u64* fkey = nullptr;     // interleaved like ckey / ctie: ftie = fkey + 1, cslot(t)
    u64* ftie = nullptr;
};

struct CollectBufs {
    uint8_t* flags = nullptr;
    u32 flags_cap = 0;
};

// ---- launchers -----------------------------------------------------------------

// collect + fused compute_splitting_points (refine.hpp:226-296).  Returns the
// candidate count (synchronises).  If rule4 == false and subsegment
// candidates exist, triangles are skipped (refine.hpp:239); *tris_scanned
// then stays false and the caller must not advance the incremental cache
// (the cached per-triangle flags were not refreshed; with the dirty-bit
// cache this only matters for the full flag).
struct CollectCache {
    int full = 1;                 // 1 = recompute every element (ignore the dirty bits)
    // words the first CTA of the scan zeroes for the insertion kernels that
    // follow (step ring + status words): saves the per-batch memsets
    u32* zero[2] = {nullptr, nullptr};
    u32 zero_n[2] = {0, 0};
};
u32 launch_collect(const DevMesh& m, const Quality& q, bool rule4, uint8_t* flags, DevCands c,
                   u32 ccap, ScanScratch& s, Counters* d_ctr, cudaStream_t st,
                   const CollectCache& cache, bool* tris_scanned, u32* d_count,
                   cudaEvent_t ev_scan0 = nullptr,
                   cudaEvent_t ev_scan1 = nullptr, bool sync = true,
                   u32* small_list = nullptr, u32* dlist_n = nullptr);
// small_list (SMALL_LIST_WORDS: append keys [CAP], their count, the sorted
// keys of the list made (klist) [CAP], klist's count): the no-round-trip
// collect of a small list (k_collect_append + k_collect_small, k_collect.cu);
// *d_count = NONE when the list outgrew it.  dlist_n: the tail loop's
// dirty-element count, restarted by every small-list collect.
constexpr u32 SMALL_LIST_CAP = 4096;
constexpr u32 SMALL_LIST_WORDS = 2 * SMALL_LIST_CAP + 2;
constexpr u32 DLIST_CAP = 1u << 16;
void launch_split_points(const DevMesh& m, DevCands c, u32 n, Counters* d_ctr, cudaStream_t st);
// batch_size_cap (refine.hpp:252-261): keep the k highest-priority alive
// candidates of the list (others marked dead), device-side radix select.
size_t select_state_bytes();
u32 cavity_resident_candidates(int device);
void launch_select_topk(DevCands c, u32 n, u32 k, void* state, cudaStream_t st);
// Item count of a standalone filter kernel: a host value, or the device count
// written by collect (no host round trip).  Kernels loop grid-stride over
// [0, n) and do nothing when n <= skip_le or n > cap (region capacity).
struct NArg {
    u32 n = 0;
    const u32* d_n = nullptr;
    u32 skip_le = 0;
    u32 cap = 0xFFFFFFFFu;
    u32 grid_n = 0;   // items the launch grid is sized for (grid-stride covers the rest)
    static NArg host(u32 n) { NArg a; a.n = n; a.grid_n = n; return a; }
};
void launch_locate(const DevMesh& m, DevCands c, NArg n, Counters* d_ctr, cudaStream_t st);
inline void launch_locate(const DevMesh& m, DevCands c, u32 n, Counters* d_ctr, cudaStream_t st) {
    launch_locate(m, c, NArg::host(n), d_ctr, st);
}
void launch_claim(const DevMesh& m, DevCands c, NArg n, TriAux a, Counters* d_ctr,
                  cudaStream_t st);
inline void launch_claim(const DevMesh& m, DevCands c, u32 n, TriAux a, Counters* d_ctr,
                         cudaStream_t st) {
    launch_claim(m, c, NArg::host(n), a, d_ctr, st);
}
struct InsertBufs {
    u32* nv = nullptr;  // per-candidate needs / offsets
    u32* nt = nullptr;
    u32* ns = nullptr;
    u32* ov = nullptr;
    u32* ot = nullptr;
    u32* os = nullptr;
    u32* totals = nullptr;   // device [3]
    u32 cap = 0;
};

// Cavity filter (refine.hpp:382-429).  extras: 0 parity (the reference's
// claims only), 2 refinement: the rewrite table also guards each split
// (rw_*_one, gdp2d_phases.cuh).
// plan != null: the survivors' phase-1 plan (plan_one) is written to
// plan->nv / nt / ns by the last filter kernel (InsertLaunch::planned).
void launch_cavity(const DevMesh& m, DevCands c, NArg n, u32 ncav, int extras, TriAux a,
                   u32* regions, u32* region_len, u32* bfs_len, Counters* d_ctr,
                   cudaStream_t st, const InsertBufs* plan = nullptr, u64 depth_cap = 0);
inline void launch_cavity(const DevMesh& m, DevCands c, u32 n, u32 ncav, int extras, TriAux a,
                          u32* regions, u32* region_len, u32* bfs_len, Counters* d_ctr,
                          cudaStream_t st) {
    launch_cavity(m, c, NArg::host(n), ncav, extras, a, regions, region_len, bfs_len, d_ctr, st);
}

// Isolated-insertion claims (cavity + one-ring + encroachment precedence);
// regions stride rs = isolated_stride(ncav); *unsafe_flag |= 1 when a survivor
// inserts from a capped claim set.
inline u32 isolated_stride(u32 ncav) { return 4 * (ncav + 1) + 8; }
void launch_cavity_isolated(const DevMesh& m, DevCands c, NArg n, u32 ncav, u32 rs, int mode,
                            u64 depth_cap, bool ring, TriAux a, u32* regions, u32* region_len,
                            u32* unsafe_flag, Counters* d_ctr, cudaStream_t st);

// ---- insertion ---------------------------------------------------------------------


struct FreshInfo {
    u64* key = nullptr;
    u64* tie = nullptr;
    uint8_t* cc = nullptr;
    uint8_t* removed = nullptr;
    uint8_t* mark = nullptr;
    uint8_t* dirty = nullptr;   // star rewritten since the last detection pass
    // dependent-pair resolution by priority (MIS rule, see k_insert.cu)
    uint8_t* dstat = nullptr;   // 0 undecided, 1 kept, 2 removed
    uint8_t* hcnt = nullptr;    // higher-priority same-batch circumcenter neighbours
    u32* hlist = nullptr;       // [cap * DEP_HMAX]
    u32 cap = 0;
};
constexpr int DEP_HMAX = 16;

struct WorkLists {
    u32* w[2] = {nullptr, nullptr};   // Lawson edge codes
    u32* fc = nullptr;                // flip candidates: key
    u32* fu = nullptr;                // flip candidates: neighbour code
    u32* touched = nullptr;
    uint8_t* fwin = nullptr;          // flip candidate won its claims
    u32* rm[2] = {nullptr, nullptr};  // pending removals
    u32* star = nullptr;              // removal stars (MAX_STAR each)
    u32* star_len = nullptr;
    u32 cap = 0;                      // capacity of w / fc / touched
    u32 rm_cap = 0;
    RoundCtr* rc = nullptr;           // device round counters
    double* dbg = nullptr;            // debug dump: [0]=flag, [1]=k, [2..3]=v, then link xy
    // fresh-vertex dirty marking by fixup (persistent insertion kernel only):
    // a rewritten triangle flags its corners in [fresh_v0, fresh_v0 + fresh_n)
    uint8_t* vdirty = nullptr;
    const uint8_t* fresh_cc = nullptr;   // FreshInfo::cc
    u32 fresh_v0 = 0, fresh_n = 0;
    // vert_tri is maintained for vertex ids >= vtri_from only (0 = every
    // vertex).  A refinement batch reads vert_tri of its own fresh vertices
    // alone (detection and removal stars), so it passes its first fresh id and
    // refine_loop rebuilds the whole array once at the end (launch_vtri_rebuild).
    u32 vtri_from = 0;
    // dirty-element list of the device-resident tail loop (k_tail_loop): every
    // rewritten triangle, the subsegments on it and every newly marked
    // subsegment, as collect keys (bit 31 = triangle | id); null = off
    u32* dlist = nullptr;
    u32* dlist_n = nullptr;
    u32 dlist_cap = 0;
};

// The whole Lawson fixpoint as one persistent cooperative kernel (see
// k_insert.cu).  result[0..2] = rounds run, list buffer holding the remaining
// work, remaining work count.
constexpr int LAWSON_BLOCK = 256;
int lawson_persistent_grid(int device);
void launch_lawson_persistent(const DevMesh& m, u32 round0, u32 cur0, u32 n0, u32 max_rounds,
                              TriAux a, WorkLists w, RoundCtr* rcs, u32* result, Counters* d_ctr,
                              int grid, cudaStream_t st);
// The whole insertion phase of a batch (phase 1 splits, Lawson, detect +
// rollback loops) as one persistent cooperative launch (k_insert.cu).
#ifndef GDP2D_INSERT_BLOCK
#define GDP2D_INSERT_BLOCK 256
#endif
constexpr int INSERT_BLOCK = GDP2D_INSERT_BLOCK;
constexpr int ROLLBACK_BLOCK = 256;   // the rollback kernel's frame needs the 255-register budget
struct InsertLaunch {
    DevMesh m;            // counts before the batch
    DevCands c;
    InsertBufs b;
    TriAux x;
    FreshInfo f;
    WorkLists w;
    RoundCtr* ring;       // [5] zeroed before the launch
    u32* state;           // [8] status / steps / flip rounds / removal rounds / handoff
    Counters* ctr;
    const u32* d_C;
    u64 depth_cap;
    u32 batch, round0;
    u32 vcap, tcap, scap;
    u32 small_nv, small_wl, max_steps;
    u32 rm_warp;
    u32 ncav = 32, rs = 35;
    u32* regions = nullptr;
    u32* region_len = nullptr;
    u32* scan_part = nullptr;   // [3 * grid]
    u32 small_c = 0;
    int resume = 0;
    int prefiltered = 0;        // standalone Lines 5-7 kernels ran (they skip C <= small_c)
    int planned = 0;            // ... and made the phase-1 plan (launch_cavity's plan)
    u32 reg_cap = 0xFFFFFFFFu;  // candidates the region buffers hold (INS_REGIONS beyond)
    int cluster = 0;            // launch both kernels as ONE cluster of `grid` CTAs
    int isolate = 1;            // claims: 0 reference cavity, 1 isolated (ring), 2 precedence
    int dep_mis = 0;            // dependent pairs by the priority-MIS rule
    int extras = 2;             // cavity extras mode (see launch_cavity)
    unsigned long long* trace = nullptr;   // device step trace (GDP2D_TRACE=1)
    u32* trace_val = nullptr;
    u32* trace_n = nullptr;
    u32 trace_cap = 0;
};
int insert_persistent_grid(int device);
int rollback_persistent_grid(int device);
// Largest cluster size <= want (a power of two, <= 16) the persistent kernels can
// be launched with as one thread-block cluster; 0 if none.
int insert_cluster_size(int device, int want);
// The device-resident tail loop (k_tail_loop, k_insert.cu): consecutive small
// batches (C <= small_c) run back to back in ONE single-CTA launch -- an
// incremental collect over the previous candidate keys and the elements the
// previous batch dirtied (klist + WorkLists::dlist), Lines 5-7, the splits,
// Lawson, detection and rollback -- with one host readback at the end.
struct TailRec {            // one batch of the loop, for the host's RunReport
    u32 attempted, nv, nt, ns;
    u32 steps, flip_rounds, rm_rounds, dirty;
    unsigned long long t0, t1, t2;   // globaltimer: batch start, collect end, batch end
    Counters ctr;
};
enum : u32 { TAIL_DONE = 0, TAIL_BIG = 1, TAIL_GROW = 2, TAIL_CAP = 3, TAIL_ERR = 4,
             TAIL_NOKEYS = 5 };
struct TailArgs {
    TailRec* rec;           // [max_batches]
    u32 max_batches;
    u32* klist;             // [SMALL_LIST_CAP] sorted keys of the last collect's list
    u32* klist_n;           // their count (NONE = not valid)
    Quality q;
    u32* out;               // [8]: exit reason, batches, nV, nT, nS, next round0, last C
};
void launch_tail_loop(const InsertLaunch& L, const TailArgs& t, int mode, cudaStream_t st);

// Kernel 1 (plan + splits + Lawson, with Lines 5-7 unless L.prefiltered) then
// kernel 2 (detect + rollback loop), both cooperative, no host sync between.
// which: bit 0 = kernel 1, bit 1 = kernel 2, launched in that order.
void launch_insert_persistent(const InsertLaunch& L, int mode, int grid, int grid2,
                              cudaStream_t st, cudaEvent_t between = nullptr, int which = 3);

// Quality summary (refine.hpp:614-645).
struct QualitySummary {
    double total_area, bad_area, min_angle, max_edge;
    ull bad, alive_v, steiner;
};
QualitySummary launch_quality(const DevMesh& m, const Quality& q, void* scratch,
                              cudaStream_t st);

// Device validators (k_verify.cu): structure, local CDT, quality, conformity
// against the input segments (in_sv = the pristine mesh's subsegments).
struct VerifySummary {
    u32 structure_failure, structure_tri;
    ull cdt_violations, bad_triangles, conformity_failures;
    double min_angle_deg;
    double mean_min_angle_deg;
    ull min_angle_hist[GDP2D_HIST_BINS];
    size_t scratch_needed;   // nonzero: scratch too small, nothing run
};
VerifySummary launch_verify(const DevMesh& m, const Quality& q, const uint2* in_sv, u32 nIn,
                            void* scratch, size_t scratch_bytes, u32* d_val, cudaStream_t st);

// Compacted node/ele export (k_verify.cu).
void launch_export(const DevMesh& m, u32* fv, u32* ov, u32* ft, u32* ot, double2* xy,
                   uint8_t* marker, u32* tri, u32* totals, ScanScratch& s, cudaStream_t st);

// Debug structural validator (out: 4 u32 device words).
void launch_validate(const DevMesh& m, u32* out, cudaStream_t st);
// vert_tri of every vertex = its lowest alive incident triangle (k_misc.cu).
void launch_vtri_rebuild(const DevMesh& m, cudaStream_t st);

// Line 1 on the device (k_cdt.cu): Delaunay triangulation of the input
// points inside a super triangle (vertices N..N+2), then segment recovery by
// pipe flips, removal of the super triangle and a constrained Lawson pass.
struct CdtLocal {          // one triangle of a pipe being re-triangulated
    uint4 v;               // corners (w unused)
    uint4 n;               // neighbours: local (j<<2|e) where bit e of n.w is set, else global code
    uint4 s;               // subsegment (piece id) per edge
    uint4 o;               // original (tri<<2|edge) of an outer edge (emap key)
};
struct CdtArgs {
    DevMesh m;             // work mesh; nT = triangle capacity (2N+1)
    u32 N;                 // input points (vertices 0..N-1)
    u32 stride0;           // first insertion level: points i % stride0 == 0
    TriAux x;
    WorkLists w;           // vdirty = null
    RoundCtr* ring;        // [4]
    u32* state;            // [16], see k_cdt.cu
    Counters* ctr;
    u32 round0;
    // points
    u32* ptri;             // containing triangle, NONE once inserted
    int8_t* pedge;         // -1 inside, else the edge the point lies on
    u32* pother;           // far triangle claimed by an on-edge point
    u64* pkey;             // pick key (distance to the circumcircle centre, index)
    uint8_t* pwin;
    u64* tkey;             // per-triangle pick slot (~0 when free)
    u32* part;             // [grid] chunk sums
    // segment recovery: pieces are (sub)segments still to be recovered
    uint2* pc;             // piece endpoints
    u32* ppar;             // input segment the piece belongs to
    u32* plist[2];         // active piece lists
    u32* poff;             // claim-log offset of the piece's pipe
    u32* plen;             // pipe length (triangles)
    u32* claims;           // claim log (pipe triangles)
    u32* seeds;            // Lawson seeds (edge codes) of re-triangulated pipes
    CdtLocal* pool;        // per-pipe scratch (pipes of a round are disjoint)
    uint2* queue;          // per-pipe crossing-edge ring
    u32 pcap, claim_cap, seed_cap, pool_cap;
};
constexpr int CDT_BLOCK = 256;
enum : u32 { CDT_ST_ROUNDS = 1, CDT_ST_FLIP_ROUNDS = 2, CDT_ST_STEPS = 3, CDT_ST_RECOVER_ROUNDS = 4,
             CDT_ST_NPIECES = 5, CDT_ST_FOUND = 6, CDT_ST_PIPES = 7, CDT_ST_SPLITS = 8,
             CDT_ST_SEEDS = 9, CDT_ST_POOL = 10, CDT_ST_PIPE_MAX = 11 };
int cdt_grid(int device, int which);
void launch_cdt_delaunay(const CdtArgs& a, int grid, cudaStream_t st);
void launch_cdt_recover(const CdtArgs& a, u32 n_pieces, int grid, cudaStream_t st);
// super-triangle removal: unlink (pass 0) then kill (pass 1)
void launch_cdt_strip(const DevMesh& m, u32 N, cudaStream_t st);
void launch_cdt_bbox(const double2* xy, u32 n, ull* out4, Counters* ctr, cudaStream_t st);
// compaction of the work mesh into dst (alive triangles renumbered, pieces
// mapped through pmap), vertex/subsegment records rebuilt
void launch_cdt_piece_live(const DevMesh& m, u32* plive, cudaStream_t st);
void launch_cdt_compact(const DevMesh& src, DevMesh dst, u32 N, const u32* newid,
                        const uint2* pc, const u32* ppar, const u32* pmap, u32 npieces,
                        cudaStream_t st);
void launch_alive_flags(const DevMesh& m, u32* flags, cudaStream_t st);
void launch_cdt_pmap(const u32* plive, const u32* pre, u32* pmap, u32 n, cudaStream_t st);

// Upload helpers.
void launch_encode_neighbors(DevMesh m, const u32* plain_n, cudaStream_t st);
void launch_decode_neighbors(const DevMesh& m, u32* plain_n, cudaStream_t st);

// Predicate batches.
void launch_predicates(int kind, const double* pts, u32 n, const Quality& q, int8_t* out,
                       cudaStream_t st);
void launch_circumcenters(const double* pts, u32 n, double* out, uint8_t* ok,
                          cudaStream_t st);

}  // namespace gdp2d
