/*
 * gdp2d.h -- C ABI of the B200-native gDP2d constrained-Delaunay refinement
 * engine (libgdp2d.so).  Plain pointers and sizes only; no CUDA or torch types.
 *
 * The boundary replaces the header-only C++ entry point
 *     RunReport cdtref::refine(Mesh&, const QualityCriteria&, const EngineConfig&)
 *     (/root/reference/proj/include/cdtref/refine.hpp:651)
 * and, for bit-exact parity testing, its phase functions
 *     collect                 (refine.hpp:226)
 *     compute_splitting_points(refine.hpp:267)
 *     locate                  (refine.hpp:301)
 *     claim_filter            (refine.hpp:367)
 *     cavity_filter           (refine.hpp:382)
 *     lawson_fixpoint         (cdt.hpp:111)
 * plus the predicates of predicates.hpp:63-185 and is_bad_triangle
 * (refine.hpp:192).  The reference has no ABI (it is header-only and inline);
 * INTEGRATION.md shows the C++ shim (include/gdp2d_cdtref.hpp) that re-exposes
 * the exact cdtref::refine signature on top of these entry points.
 *
 * Mesh exchange format: the reference's Mesh (mesh.hpp:43-75) flattened to
 * structure-of-arrays with IDENTICAL ids and vertex rotations:
 *   tri_v[3t+i]  = triangles[t].v[i]
 *   tri_n[3t+i]  = triangles[t].nbr[i]   (plain TriId, kNone = 0xFFFFFFFF)
 *   tri_seg[3t+i]= triangles[t].seg[i]
 * Dead slots are kept (alive = 0); ids are never recycled (as in the reference).
 *
 * Threading: one call = one device + one stream, blocking.  Distinct host
 * threads may drive distinct devices (one context each).  gdp2d_last_error()
 * is thread-local.
 */
#ifndef GDP2D_H
#define GDP2D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GDP2D_NONE    0xFFFFFFFFu /* cdtref::kNone    (mesh.hpp:23) */
#define GDP2D_PENDING 0xFFFFFFFEu /* cdtref::kPending (mesh.hpp:24) */

/* Status codes.  0 = success. */
enum {
    GDP2D_OK = 0,
    GDP2D_EINVAL = 1,     /* bad argument / malformed mesh view            */
    GDP2D_ECUDA = 2,      /* CUDA runtime error                            */
    GDP2D_ENODEVICE = 3,  /* no usable sm_100 device                       */
    GDP2D_ECAPACITY = 4,  /* device work-list / stack capacity exceeded    */
    GDP2D_EMESH = 5,      /* structural failure inside a mesh mutation     */
    GDP2D_EINTERNAL = 6,
    GDP2D_ECDT = 7        /* PSLG cannot be triangulated (CdtError, cdt.hpp:20):
                             duplicate points, all collinear, crossing segments,
                             non-finite coordinates                        */
};

/* VertexKind (mesh.hpp:26) */
enum { GDP2D_VK_INPUT = 0, GDP2D_VK_MIDPOINT = 1, GDP2D_VK_CIRCUMCENTER = 2 };
/* RefineMode (refine.hpp:28) */
enum { GDP2D_RUPPERT = 0, GDP2D_CHEW = 1 };
/* SplitCandidate::Kind (refine.hpp:72) */
enum { GDP2D_CAND_SUBSEG = 0, GDP2D_CAND_TRI = 1 };
/* PriorityKey::Band (refine.hpp:58) */
enum { GDP2D_BAND_CIRCUMCENTER = 0, GDP2D_BAND_MIDPOINT = 1 };
/* Location::Kind (cdt.hpp:31) */
enum { GDP2D_LOC_INSIDE = 0, GDP2D_LOC_ONEDGE = 1, GDP2D_LOC_ONVERTEX = 2,
       GDP2D_LOC_OUTSIDE = 3, GDP2D_LOC_INTERCEPTED = 4 };

/* Read-only host mesh (the reference Mesh, SoA). */
typedef struct gdp2d_mesh_view {
    uint32_t n_vertices, n_triangles, n_subsegments, batch_epoch;
    const double*   xy;             /* [2V] x,y interleaved                   */
    const uint8_t*  vert_kind;      /* [V]  VertexKind                        */
    const uint32_t* vert_birth;     /* [V]  birth_batch                       */
    const uint8_t*  vert_alive;     /* [V]                                    */
    const uint32_t* vert_tri;       /* [V]  some alive incident triangle      */
    const uint32_t* tri_v;          /* [3T]                                   */
    const uint32_t* tri_n;          /* [3T] nbr[i] opposite v[i]              */
    const uint32_t* tri_seg;        /* [3T] subsegment on edge i or NONE      */
    const uint8_t*  tri_alive;      /* [T]                                    */
    const uint32_t* seg_v;          /* [2S]                                   */
    const uint32_t* seg_parent;     /* [S]  input segment index               */
    const uint8_t*  seg_encroached; /* [S]  sticky flag                       */
    const uint8_t*  seg_alive;      /* [S]                                    */
    const uint32_t* seg_tri;        /* [S]  some triangle carrying s          */
} gdp2d_mesh_view;

/* Library-owned host mesh (output of refine / download).  Release with
 * gdp2d_free().  Same layout as gdp2d_mesh_view. */
typedef struct gdp2d_mesh_buf {
    uint32_t n_vertices, n_triangles, n_subsegments, batch_epoch;
    double*   xy;
    uint8_t*  vert_kind;
    uint32_t* vert_birth;
    uint8_t*  vert_alive;
    uint32_t* vert_tri;
    uint32_t* tri_v;
    uint32_t* tri_n;
    uint32_t* tri_seg;
    uint8_t*  tri_alive;
    uint32_t* seg_v;
    uint32_t* seg_parent;
    uint8_t*  seg_encroached;
    uint8_t*  seg_alive;
    uint32_t* seg_tri;
} gdp2d_mesh_buf;

/* QualityCriteria (refine.hpp:31) + EngineConfig (refine.hpp:37) + RuleFlags
 * (ruleskit.hpp:24).  cos2_theta MUST be computed on the host exactly as
 * is_bad_triangle does (refine.hpp:195-196): c = std::cos(theta*pi/180); c*c.
 * gdp2d_params_init() does that. */
typedef struct gdp2d_params {
    double   theta_deg;
    double   cos2_theta;
    double   ell;                    /* +inf = no edge bound                    */
    uint32_t mode;                   /* GDP2D_RUPPERT / GDP2D_CHEW              */
    uint32_t cavity_n;               /* 32                                      */
    uint32_t rule1_compaction_threshold; /* 1024: below it work lists are not compacted */
    uint32_t rule2_filtering_enabled;    /* cavity filter on/off               */
    uint32_t rule4_unified_collection;   /* subsegs + triangles in one batch   */
    uint32_t little_batch_sizing;    /* GPU: Little's-law batch sizing from the
                                        measured concurrency / latency of the
                                        previous batches (1 = on, the default)  */
    uint32_t insert_mode;            /* GDP2D_INSERT_* (see below)               */
    uint32_t reserved0;
    uint64_t iteration_cap;          /* 10000                                   */
    uint64_t split_depth_cap;        /* 64                                      */
    uint64_t batch_size_cap;         /* 0 = unlimited; keep highest priorities  */
} gdp2d_params;

/* Insertion policy of a batch (gdp2d_params.insert_mode).
 * ROLLBACK: the reference's insert_batch (refine.hpp:464-610): every cavity
 *   survivor is inserted, then redundant (encroaching) and dependent
 *   same-batch circumcenters are rolled back by vertex removal.
 * ISOLATED: a survivor also owns the one-ring of its cavity (both sides of a
 *   split subsegment), so inserted points cannot interact: no dependent pair
 *   can form and no rollback is needed.  A circumcenter that would encroach a
 *   splittable subsegment on its cavity boundary is not inserted and the
 *   subsegment is marked instead (encroachment precedence, the classic rule of
 *   refine.hpp:786-804).  Cavities that hit the cavity_n cap fall back to the
 *   rollback detection for that batch. */
/* PRECEDENCE: the reference's claim sets and rollback, plus the encroachment
 *   precedence test on each survivor's cavity boundary (an encroaching
 *   circumcenter marks its subsegment instead of being inserted and rolled
 *   back). */
enum { GDP2D_INSERT_ISOLATED = 0, GDP2D_INSERT_ROLLBACK = 1, GDP2D_INSERT_PRECEDENCE = 2 };

/* Phase order of the per-batch timers (refine.hpp:671-701). */
enum { GDP2D_PH_COLLECT = 0, GDP2D_PH_SPLIT_POINTS = 1, GDP2D_PH_LOCATE = 2,
       GDP2D_PH_CLAIM = 3, GDP2D_PH_CAVITY = 4, GDP2D_PH_INSERT = 5, GDP2D_NPHASES = 6 };

/* BatchMetrics (ruleskit.hpp:32) + device counters used by the roofline. */
typedef struct gdp2d_batch_metrics {
    uint32_t batch_index;
    uint32_t attempted;          /* candidates entering the batch            */
    uint32_t concurrency;        /* retained insertions (useful work, C)     */
    uint32_t removals_kept;      /* redundant points whose star had no ear   */
    double   latency;            /* seconds (sum of phases, L)               */
    double   throughput;         /* C / L                                    */
    double   waste_fraction;     /* 1 - useful/attempted                     */
    double   phase_seconds[GDP2D_NPHASES];
    /* alive counts at the start of the batch */
    uint64_t tris_alive, verts_alive, subsegs_alive;
    /* work counters */
    uint64_t walk_steps, cavity_visits;
    uint32_t survivors_claim, survivors_cavity;
    uint32_t inserted_midpoints, inserted_circumcenters;
    uint32_t removed_redundant, removed_dependent;
    uint32_t dropped, marked_encroached;
    uint64_t flips;              /* Lawson + degree-reduction flips           */
    uint32_t flip_rounds, removal_rounds;
} gdp2d_batch_metrics;

/* RunReport (ruleskit.hpp:42). batches: caller-provided array of
 * batches_capacity entries (may be NULL); n_batches is always the true count. */
typedef struct gdp2d_report {
    gdp2d_batch_metrics* batches;
    uint32_t batches_capacity;
    uint32_t n_batches;
    uint64_t output_points;
    uint64_t steiner_points;
    uint64_t bad_triangles;
    double   bad_area_percent;
    double   min_angle_deg;
    double   max_edge;
    double   wall_seconds;       /* refine loop only (refine.hpp:653,710)     */
    int32_t  iteration_cap_hit;
    int32_t  pad0;
    /* totals over all batches */
    uint64_t total_candidates, total_walk_steps, total_cavity_visits;
    uint64_t total_inserted, total_flips, total_removed;
    uint64_t sum_tris_alive, sum_verts_alive, sum_subsegs_alive;
    double   device_seconds;     /* CUDA-event time of the device loop        */
    /* roofline instrumentation of the Line-3 full scan (collect flags kernel):
     * CUDA-event time summed over its launches and its algorithmic bytes
     * (16 B per triangle slot + 16 B per vertex + 48 B per subsegment). */
    double   scan_seconds;
    uint64_t scan_bytes;
    uint64_t scan_launches;
    uint64_t kernel_launches;    /* engine kernels launched by this call      */
    /* roofline instrumentation of the persistent batch kernels (k_batch_split:
     * plan + splits + Lawson; k_batch_rollback: detection + rollback + Lawson):
     * CUDA-event time summed over launches and algorithmic bytes
     * (32 B/candidate planned + 128 B/insertion + 128 B/flip; 64 B/fresh vertex
     * detected + 128 B/flip + 128 B/removal). */
    double   split_seconds;
    uint64_t split_bytes;
    uint64_t split_launches;
    double   rollback_seconds;
    uint64_t rollback_bytes;
    uint64_t rollback_launches;
    /* gdp2d_refine only: H2D of the input + refine loop + D2H of the output,
     * timed once the device context exists (0 from gdp2d_ctx_refine). */
    double   e2e_seconds;
} gdp2d_report;

/* SplitCandidate (refine.hpp:71) in exchange form. */
typedef struct gdp2d_candidate {
    double   x, y;               /* splitting point                          */
    double   measure;            /* PriorityKey::measure                      */
    uint32_t id;                 /* SubsegId or TriId                         */
    uint32_t tiebreak;           /* PriorityKey::tiebreak (list index)        */
    uint32_t located;            /* TriId or GDP2D_PENDING                    */
    uint8_t  kind;               /* GDP2D_CAND_*                              */
    uint8_t  band;               /* GDP2D_BAND_*                              */
    uint8_t  alive;
    uint8_t  fallback;           /* circumcenter fell back to longest edge   */
} gdp2d_candidate;

/* ---- whole-run entry point ------------------------------------------------ */

/* Fill p with the reference defaults (QualityCriteria{theta, ell, mode},
 * EngineConfig{}) and the host-computed cos^2(theta). */
void gdp2d_params_init(gdp2d_params* p, double theta_deg, double ell, uint32_t mode);

/* Refine `in` on `device`; writes the refined mesh into *out (library-owned
 * host buffers) and the run report into *r.  Timed scope (r->wall_seconds)
 * covers H2D of the input, every batch and D2H of the result.  The device
 * context (HBM buffers, stream) is cached per device and reused by later
 * calls; concurrent calls on the same device are serialised. */
int gdp2d_refine(const gdp2d_mesh_view* in, gdp2d_mesh_buf* out, const gdp2d_params* p,
                 gdp2d_report* r, int device);

/* Array-of-structures records: the reference's own element vectors
 * (cdtref::Vertex / Triangle / Subsegment, mesh.hpp:43-62) described by byte
 * size and field offsets, so the drop-in refine (include/gdp2d_cdtref.hpp)
 * hands the caller's vectors over as they are -- no host pack / unpack, no
 * library-owned output buffers.  Fields: vertex pos (2 x f64), kind (u8),
 * birth (u32), alive (u8); triangle v[3], nbr[3], seg[3] (u32), alive (u8);
 * subsegment v[2], parent (u32), encroached (u8), alive (u8). */
typedef struct gdp2d_aos_layout {
    uint32_t vert_size, vert_pos, vert_kind, vert_birth, vert_alive;
    uint32_t tri_size, tri_v, tri_nbr, tri_seg, tri_alive;
    uint32_t seg_size, seg_v, seg_parent, seg_encroached, seg_alive;
} gdp2d_aos_layout;

enum { GDP2D_AOS_VERTS = 0, GDP2D_AOS_TRIS = 1, GDP2D_AOS_SEGS = 2, GDP2D_AOS_VERT_TRI = 3,
       GDP2D_AOS_SEG_TRI = 4 };

/* A caller-owned AoS mesh, refined in place.  After the refinement the
 * library calls resize(user, what, n) once per array (GDP2D_AOS_*) with its
 * output length; the callback sizes the caller's array and returns its
 * (possibly moved) base, which the library overwrites with n records.
 * batch_epoch is updated on return. */
typedef struct gdp2d_aos_mesh {
    uint32_t n_vertices, n_triangles, n_subsegments, batch_epoch;
    const void* verts;
    const void* tris;
    const void* segs;
    const uint32_t* vert_tri;
    const uint32_t* seg_tri;
    void* (*resize)(void* user, int what, uint64_t n);
    void* user;
} gdp2d_aos_mesh;

/* gdp2d_refine on AoS records (replaces cdtref::refine, refine.hpp:651, for
 * callers that hold a cdtref::Mesh): records are converted on the device. */
int gdp2d_refine_aos(const gdp2d_aos_layout* layout, gdp2d_aos_mesh* mesh,
                     const gdp2d_params* p, gdp2d_report* r, int device);

/* Create the cached context of `device` and run one tiny CDT build +
 * refinement on it, so CUDA context creation and kernel loading (~1-2 s in a
 * fresh process) are paid here.  Meant to run on a helper thread while the
 * caller reads its input; later gdp2d_refine / gdp2d_build_cdt calls on the
 * device wait for it (they share the context's lock).  No reference
 * counterpart (the CPU reference has no device to prepare). */
int gdp2d_warmup(int device);

void gdp2d_free(gdp2d_mesh_buf* out);
const char* gdp2d_last_error(void);
const char* gdp2d_version(void);
/* sizeof() of the exchange structs, for binding-layout checks:
 * 0 mesh_view, 1 mesh_buf, 2 params, 3 batch_metrics, 4 report, 5 candidate,
 * 6 validation, 7 node_ele, 8 cdt_report, 9 aos_layout, 10 aos_mesh */
size_t gdp2d_struct_size(int which);
/* Process-wide count of engine kernel launches so far (all devices). */
uint64_t gdp2d_kernel_launches(void);

/* ---- device-resident context (bench / replicas / parity) ------------------- */

typedef struct gdp2d_ctx gdp2d_ctx;

int  gdp2d_ctx_create(gdp2d_ctx** ctx, int device);
void gdp2d_ctx_destroy(gdp2d_ctx* ctx);
/* Upload a mesh into the context's pristine copy and working mesh. */
int  gdp2d_ctx_upload(gdp2d_ctx* ctx, const gdp2d_mesh_view* in);
/* Restore the working mesh from the pristine copy (device-to-device). */
int  gdp2d_ctx_reset(gdp2d_ctx* ctx);
/* Refine the working mesh in place (device-resident input and output). */
int  gdp2d_ctx_refine(gdp2d_ctx* ctx, const gdp2d_params* p, gdp2d_report* r);
int  gdp2d_ctx_download(gdp2d_ctx* ctx, gdp2d_mesh_buf* out);
/* Current working-mesh sizes (slots, including dead ones). */
int  gdp2d_ctx_sizes(gdp2d_ctx* ctx, uint32_t* n_vertices, uint32_t* n_triangles,
                     uint32_t* n_subsegments);
/* Download into CALLER-allocated arrays sized from gdp2d_ctx_sizes(); the
 * pointers in *dst are used as given (nothing is allocated or freed). */
int  gdp2d_ctx_download_to(gdp2d_ctx* ctx, gdp2d_mesh_buf* dst);
/* Page-locked host memory (cudaHostAlloc, portable) for meshes that are
 * uploaded / downloaded repeatedly: H2D/D2H at full PCIe/C2C rate. */
void* gdp2d_pinned_alloc(size_t bytes);
void  gdp2d_pinned_free(void* p);
/* Release the per-device contexts that gdp2d_refine() keeps cached. */
void gdp2d_release_cached(void);
/* Bytes of device memory held by the context. */
uint64_t gdp2d_ctx_device_bytes(gdp2d_ctx* ctx);

/* ---- device validators (k_verify.cu) ------------------- */

/* Histogram of per-triangle minimum angles: bin k counts alive triangles whose
 * smallest corner angle (min_angle_degrees' formula, verify.hpp:186-200) lies
 * in [k, k+1) * GDP2D_HIST_BIN_DEG degrees; the last bin takes the rest. */
#define GDP2D_HIST_BINS 120
#define GDP2D_HIST_BIN_DEG 0.5

/* What the reference validates on the host (mesh.hpp:505-557,
 * verify.hpp:92-200) computed on the device for the working mesh: */
typedef struct gdp2d_validation {
    uint32_t structure_failure;    /* 0 = check_structure passes, else a code  */
    uint32_t structure_tri;        /* first failing triangle                   */
    uint64_t cdt_violations;       /* interior non-subsegment edges failing the
                                      exact local Delaunay test                 */
    uint64_t bad_triangles;        /* is_bad_triangle && triangle_resolvable    */
    uint64_t conformity_failures;  /* 0 = every input segment exactly covered   */
    double   min_angle_deg;
    double   mean_min_angle_deg;   /* mean over alive triangles of their min angle */
    uint64_t min_angle_hist[GDP2D_HIST_BINS];
} gdp2d_validation;

/* Validate the working mesh against p's quality criteria and the uploaded
 * input's segments (the pristine mesh's subsegments). */
int gdp2d_ctx_validate(gdp2d_ctx* ctx, const gdp2d_params* p, gdp2d_validation* out);

/* ---- compacted export ----------------------------------- */

/* write_node_ele (pslg_io.hpp:294-319) data, compacted on the device: alive
 * vertices renumbered densely in id order (xy + marker 1 = input, 0 =
 * Steiner), alive triangles in id order as dense vertex triples.  Caller
 * allocates xy[2V], marker[V], tri[3T] with V, T from gdp2d_ctx_sizes (upper
 * bounds); n_nodes / n_tris return the counts.  Moves ~17 B per alive vertex
 * + 12 B per alive triangle instead of the whole slot-preserving mesh. */
typedef struct gdp2d_node_ele {
    uint32_t n_nodes, n_tris;
    double*  xy;
    uint8_t* marker;
    uint32_t* tri;
} gdp2d_node_ele;

int gdp2d_ctx_export(gdp2d_ctx* ctx, gdp2d_node_ele* out);

/* ---- Line 1 on the device: initial constrained Delaunay triangulation ----
 * Replaces build_cdt(const Pslg&) (cdt.hpp:483 = build_delaunay :198 +
 * recover_segments :437 + lawson_fixpoint_all).  Input: the PSLG after
 * close_hull (cdt.hpp:447; read_poly/to_pslg already apply it): n points
 * xy[2n] and m segments seg[2m] (vertex indices).  The result becomes the
 * context's input mesh (as gdp2d_ctx_upload would), so gdp2d_ctx_refine /
 * gdp2d_ctx_download follow directly.  Vertex i = points[i]; subsegment s
 * belongs to segment sparent[s] (s = segment index unless a segment passes
 * through a vertex, which splits it exactly as recover_chain does).  Triangle
 * ids differ from the reference's; the triangle SET equals it for PSLGs in
 * general position (the CDT is unique).  Errors: GDP2D_ECDT. */
typedef struct gdp2d_cdt_report {
    uint32_t struct_size;
    uint32_t n_triangles;        /* alive triangles of the CDT            */
    uint32_t n_subsegments;
    uint32_t insert_rounds;      /* parallel insertion rounds             */
    uint32_t flip_rounds;        /* Lawson rounds during insertion        */
    uint32_t recover_rounds;     /* segment recovery rounds               */
    uint32_t segments_present;   /* pieces already edges of the DT        */
    uint32_t pipes_recovered;    /* pieces recovered by pipe flips        */
    uint32_t collinear_splits;   /* pieces split at a vertex on them      */
    uint32_t max_pipe;           /* longest pipe (triangles)              */
    uint32_t final_flip_rounds;  /* constrained Lawson after recovery     */
    uint32_t reserved;
    uint64_t flips;              /* all Lawson flips                      */
    double seconds;              /* device time, upload to compacted mesh */
    double delaunay_seconds, recover_seconds, finish_seconds;
} gdp2d_cdt_report;

int gdp2d_ctx_build_cdt(gdp2d_ctx* ctx, const double* xy, uint32_t n_points,
                        const uint32_t* seg, uint32_t n_segments, gdp2d_cdt_report* rep);
/* One-shot form: build on `device` and download into *out (free with
 * gdp2d_free). */
int gdp2d_build_cdt(const double* xy, uint32_t n_points, const uint32_t* seg,
                    uint32_t n_segments, gdp2d_mesh_buf* out, gdp2d_cdt_report* rep,
                    int device);

/* ---- per-phase parity entry points (operate on the working mesh) ----------- */

/* collect + compute_splitting_points: writes up to cap candidates in the
 * reference's list order; *n = true count.  Returns GDP2D_ECAPACITY if cap is
 * too small (nothing written beyond cap). */
int gdp2d_collect(gdp2d_ctx* ctx, const gdp2d_params* p, gdp2d_candidate* out,
                  uint32_t cap, uint32_t* n);
/* compute_splitting_points on a caller list (ids/kinds given). */
int gdp2d_split_points(gdp2d_ctx* ctx, gdp2d_candidate* c, uint32_t n);
/* locate (refine.hpp:301): in/out on the list. */
int gdp2d_locate(gdp2d_ctx* ctx, gdp2d_candidate* c, uint32_t n);
/* claim_filter (refine.hpp:367): in/out (alive). */
int gdp2d_claim(gdp2d_ctx* ctx, gdp2d_candidate* c, uint32_t n);
/* cavity_filter (refine.hpp:382) with bound n_cav; optional regions out
 * (regions[i*(n_cav+1) ...], region_len[i]) may be NULL. */
int gdp2d_cavity(gdp2d_ctx* ctx, gdp2d_candidate* c, uint32_t n, uint32_t n_cav,
                 uint32_t* regions, uint32_t* region_len);
/* lawson_fixpoint (cdt.hpp:111) seeded with (tri, edge) pairs. */
int gdp2d_flip_fixpoint(gdp2d_ctx* ctx, const uint32_t* seed_tri, const uint8_t* seed_edge,
                        uint32_t n, uint64_t* flips);

/* ---- predicate batches (predicates.hpp, refine.hpp:192) -------------------- */

enum { GDP2D_PRED_ORIENT2D = 0,      /* pts: a,b,c          -> {-1,0,1}   */
       GDP2D_PRED_INCIRCLE = 1,      /* pts: a,b,c,d        -> {-1,0,1}   */
       GDP2D_PRED_DIAMETRIC = 2,     /* pts: sa,sb,p        -> {0,1}      */
       GDP2D_PRED_LENS = 3,          /* pts: sa,sb,p        -> {0,1}      */
       GDP2D_PRED_BAD_TRIANGLE = 4 };/* pts: a,b,c          -> {0,1} (uses p) */
/* pts holds n records of 2*arity doubles; out gets n int8 results. */
int gdp2d_predicates_batch(int device, int kind, const double* pts, uint32_t n,
                           const gdp2d_params* p, int8_t* out);
/* circumcenter (predicates.hpp:172): pts = n*(a,b,c); out = n*(x,y); ok = n. */
int gdp2d_circumcenter_batch(int device, const double* pts, uint32_t n, double* out,
                             uint8_t* ok);

#ifdef __cplusplus
}
#endif

#endif /* GDP2D_H */
