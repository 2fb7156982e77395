// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" wrapper that compiles the UNMODIFIED reference headers
// from /root/reference/proj/include (no source is copied into this repo) into
// oracle/_ref/libcdtref_ref.so, so the parity tests, smoke() and bench.py's
// cpu_baseline / --impl reference legs can call the reference itself:
//   cdtref::refine            refine.hpp:651
//   cdtref::collect           refine.hpp:226
//   compute_splitting_points  refine.hpp:267
//   locate                    refine.hpp:301
//   claim_filter              refine.hpp:367
//   cavity_filter             refine.hpp:382
//   insert_batch              refine.hpp:464
//   lawson_fixpoint           cdt.hpp:111
//   build_cdt / close_hull    cdt.hpp:483 / cdt.hpp:447
//   validators                mesh.hpp:505-557, verify.hpp:92-200
//   predicates                predicates.hpp:63-185, refine.hpp:192
//   min-angle histogram       verify.hpp:186-200 / refine.hpp:625-632 (per triangle)
// The SURVEY 8(d) synthetic PSLG generator (paper_2007_00324_b200/csrc/host/
// pslg_gen.cpp, plain host code) is compiled into this library as well, so the
// CPU reference legs build their input without loading any product library.
// Mesh exchange uses the gdp2d_mesh_view SoA layout of include/gdp2d.h.
// Build: oracle/Makefile (g++ -std=c++20 -O3 -DNDEBUG -ffp-contract=off).

#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "cdtref/cdt.hpp"
#include "cdtref/mesh.hpp"
#include "cdtref/predicates.hpp"
#include "cdtref/pslg_io.hpp"
#include "cdtref/refine.hpp"
#include "cdtref/verify.hpp"
#include "gdp2d.h"

using namespace cdtref;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return 1;
}

Mesh from_view(const gdp2d_mesh_view* v) {
    Mesh m;
    m.batch_epoch = v->batch_epoch;
    m.vertices.resize(v->n_vertices);
    m.vert_tri.resize(v->n_vertices);
    for (uint32_t i = 0; i < v->n_vertices; ++i) {
        m.vertices[i].pos = {v->xy[2 * i], v->xy[2 * i + 1]};
        m.vertices[i].kind = static_cast<VertexKind>(v->vert_kind[i]);
        m.vertices[i].birth_batch = v->vert_birth[i];
        m.vertices[i].alive = v->vert_alive[i] != 0;
        m.vert_tri[i] = v->vert_tri[i];
    }
    m.triangles.resize(v->n_triangles);
    for (uint32_t t = 0; t < v->n_triangles; ++t) {
        for (int i = 0; i < 3; ++i) {
            m.triangles[t].v[i] = v->tri_v[3 * t + i];
            m.triangles[t].nbr[i] = v->tri_n[3 * t + i];
            m.triangles[t].seg[i] = v->tri_seg[3 * t + i];
        }
        m.triangles[t].alive = v->tri_alive[t] != 0;
    }
    m.subsegments.resize(v->n_subsegments);
    m.seg_tri.resize(v->n_subsegments);
    for (uint32_t s = 0; s < v->n_subsegments; ++s) {
        m.subsegments[s].v = {v->seg_v[2 * s], v->seg_v[2 * s + 1]};
        m.subsegments[s].parent = v->seg_parent[s];
        m.subsegments[s].encroached = v->seg_encroached[s] != 0;
        m.subsegments[s].alive = v->seg_alive[s] != 0;
        m.seg_tri[s] = v->seg_tri[s];
    }
    return m;
}

template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

void to_buf(const Mesh& m, gdp2d_mesh_buf* b) {
    const uint32_t V = static_cast<uint32_t>(m.vertices.size());
    const uint32_t T = static_cast<uint32_t>(m.triangles.size());
    const uint32_t S = static_cast<uint32_t>(m.subsegments.size());
    b->n_vertices = V;
    b->n_triangles = T;
    b->n_subsegments = S;
    b->batch_epoch = m.batch_epoch;
    std::vector<double> xy(2 * V);
    std::vector<uint8_t> vk(V), va(V);
    std::vector<uint32_t> vb(V);
    for (uint32_t i = 0; i < V; ++i) {
        xy[2 * i] = m.vertices[i].pos.x;
        xy[2 * i + 1] = m.vertices[i].pos.y;
        vk[i] = static_cast<uint8_t>(m.vertices[i].kind);
        va[i] = m.vertices[i].alive;
        vb[i] = m.vertices[i].birth_batch;
    }
    std::vector<uint32_t> tv(3 * T), tn(3 * T), ts(3 * T);
    std::vector<uint8_t> ta(T);
    for (uint32_t t = 0; t < T; ++t) {
        for (int i = 0; i < 3; ++i) {
            tv[3 * t + i] = m.triangles[t].v[i];
            tn[3 * t + i] = m.triangles[t].nbr[i];
            ts[3 * t + i] = m.triangles[t].seg[i];
        }
        ta[t] = m.triangles[t].alive;
    }
    std::vector<uint32_t> sv(2 * S), sp(S);
    std::vector<uint8_t> se(S), sa(S);
    for (uint32_t s = 0; s < S; ++s) {
        sv[2 * s] = m.subsegments[s].v[0];
        sv[2 * s + 1] = m.subsegments[s].v[1];
        sp[s] = m.subsegments[s].parent;
        se[s] = m.subsegments[s].encroached;
        sa[s] = m.subsegments[s].alive;
    }
    b->xy = dup(xy);
    b->vert_kind = dup(vk);
    b->vert_birth = dup(vb);
    b->vert_alive = dup(va);
    b->vert_tri = dup(m.vert_tri);
    b->tri_v = dup(tv);
    b->tri_n = dup(tn);
    b->tri_seg = dup(ts);
    b->tri_alive = dup(ta);
    b->seg_v = dup(sv);
    b->seg_parent = dup(sp);
    b->seg_encroached = dup(se);
    b->seg_alive = dup(sa);
    b->seg_tri = dup(m.seg_tri);
}

QualityCriteria quality(const gdp2d_params* p) {
    return {p->theta_deg, p->ell, p->mode == GDP2D_CHEW ? RefineMode::Chew : RefineMode::Ruppert};
}

EngineConfig engine(const gdp2d_params* p, unsigned executors) {
    EngineConfig c;
    c.execution = executors > 1 ? ExecutionMode::Parallel : ExecutionMode::Sequential;
    c.executor_count = executors > 1 ? executors : 1;
    c.cavity_n = p->cavity_n;
    c.rules.rule1_compaction_threshold = p->rule1_compaction_threshold;
    c.rules.rule2_filtering_enabled = p->rule2_filtering_enabled != 0;
    c.rules.rule4_unified_collection = p->rule4_unified_collection != 0;
    c.iteration_cap = p->iteration_cap;
    c.split_depth_cap = p->split_depth_cap;
    c.batch_size_cap = p->batch_size_cap;
    return c;
}

SplitCandidate to_ref(const gdp2d_candidate& c) {
    SplitCandidate s;
    s.kind = c.kind == GDP2D_CAND_SUBSEG ? SplitCandidate::Kind::Subseg : SplitCandidate::Kind::Tri;
    s.id = c.id;
    s.point = {c.x, c.y};
    s.priority.band = c.band == GDP2D_BAND_MIDPOINT ? PriorityKey::Band::Midpoint
                                                     : PriorityKey::Band::Circumcenter;
    s.priority.measure = c.measure;
    s.priority.tiebreak = c.tiebreak;
    s.located = c.located;
    s.alive = c.alive != 0;
    return s;
}

gdp2d_candidate from_ref(const SplitCandidate& s, uint8_t fallback = 0) {
    gdp2d_candidate c{};
    c.x = s.point.x;
    c.y = s.point.y;
    c.measure = s.priority.measure;
    c.id = s.id;
    c.tiebreak = s.priority.tiebreak;
    c.located = s.located;
    c.kind = s.kind == SplitCandidate::Kind::Subseg ? GDP2D_CAND_SUBSEG : GDP2D_CAND_TRI;
    c.band = s.priority.band == PriorityKey::Band::Midpoint ? GDP2D_BAND_MIDPOINT
                                                            : GDP2D_BAND_CIRCUMCENTER;
    c.alive = s.alive;
    c.fallback = fallback;
    return c;
}

std::vector<SplitCandidate> list_in(const gdp2d_candidate* c, uint32_t n) {
    std::vector<SplitCandidate> l(n);
    for (uint32_t i = 0; i < n; ++i) l[i] = to_ref(c[i]);
    return l;
}

void list_out(const std::vector<SplitCandidate>& l, gdp2d_candidate* c) {
    for (std::size_t i = 0; i < l.size(); ++i) {
        const uint8_t fb = c[i].fallback;
        c[i] = from_ref(l[i], fb);
    }
}

void fill_report(const RunReport& rep, gdp2d_report* r) {
    r->n_batches = static_cast<uint32_t>(rep.batches.size());
    r->output_points = rep.output_points;
    r->steiner_points = rep.steiner_points;
    r->bad_triangles = rep.bad_triangles;
    r->bad_area_percent = rep.bad_area_percent;
    r->min_angle_deg = rep.min_angle_deg;
    r->max_edge = rep.max_edge;
    r->wall_seconds = rep.wall_seconds;
    r->iteration_cap_hit = rep.iteration_cap_hit;
    static const char* names[GDP2D_NPHASES] = {"collect", "split_points", "locate",
                                               "claim",   "cavity",       "insert"};
    uint64_t total = 0;
    for (std::size_t i = 0; i < rep.batches.size(); ++i) {
        total += rep.batches[i].attempted;
        if (!r->batches || i >= r->batches_capacity) continue;
        gdp2d_batch_metrics& b = r->batches[i];
        std::memset(&b, 0, sizeof b);
        b.batch_index = static_cast<uint32_t>(rep.batches[i].batch_index);
        b.attempted = static_cast<uint32_t>(rep.batches[i].attempted);
        b.concurrency = static_cast<uint32_t>(rep.batches[i].concurrency);
        b.latency = rep.batches[i].latency;
        b.throughput = rep.batches[i].throughput;
        b.waste_fraction = rep.batches[i].waste_fraction;
        for (int k = 0; k < GDP2D_NPHASES; ++k) {
            auto it = rep.batches[i].phase_breakdown.find(names[k]);
            if (it != rep.batches[i].phase_breakdown.end()) b.phase_seconds[k] = it->second;
        }
    }
    r->total_candidates = total;
}

}  // namespace

extern "C" {

typedef struct ref_mesh ref_mesh;  // opaque: a cdtref::Mesh

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_mesh_free(ref_mesh* h) { delete reinterpret_cast<Mesh*>(h); }

ref_mesh* ref_mesh_clone(const ref_mesh* h) {
    return reinterpret_cast<ref_mesh*>(new Mesh(*reinterpret_cast<const Mesh*>(h)));
}

ref_mesh* ref_mesh_from_view(const gdp2d_mesh_view* v) {
    try {
        return reinterpret_cast<ref_mesh*>(new Mesh(from_view(v)));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_mesh_to_buf(const ref_mesh* h, gdp2d_mesh_buf* b) {
    to_buf(*reinterpret_cast<const Mesh*>(h), b);
}

void ref_buf_free(gdp2d_mesh_buf* b) {
    void* ptrs[] = {b->xy,      b->vert_kind, b->vert_birth, b->vert_alive, b->vert_tri,
                    b->tri_v,   b->tri_n,     b->tri_seg,    b->tri_alive,  b->seg_v,
                    b->seg_parent, b->seg_encroached, b->seg_alive, b->seg_tri};
    for (void* p : ptrs) std::free(p);
    std::memset(b, 0, sizeof *b);
}

// close_hull (cdt.hpp:447): returns the number of segments after closing;
// out_segs must hold 2*(m + n) entries.
uint32_t ref_close_hull(const double* xy, uint32_t n, const uint32_t* segs, uint32_t m,
                        uint32_t* out_segs) {
    Pslg g;
    g.points.resize(n);
    for (uint32_t i = 0; i < n; ++i) g.points[i] = {xy[2 * i], xy[2 * i + 1]};
    for (uint32_t i = 0; i < m; ++i) g.segments.emplace_back(segs[2 * i], segs[2 * i + 1]);
    g = close_hull(std::move(g));
    for (std::size_t i = 0; i < g.segments.size(); ++i) {
        out_segs[2 * i] = g.segments[i].first;
        out_segs[2 * i + 1] = g.segments[i].second;
    }
    return static_cast<uint32_t>(g.segments.size());
}

// build_cdt (cdt.hpp:483) of the PSLG exactly as given (caller closes the hull).
ref_mesh* ref_build_cdt(const double* xy, uint32_t n, const uint32_t* segs, uint32_t m) {
    try {
        Pslg g;
        g.points.resize(n);
        for (uint32_t i = 0; i < n; ++i) g.points[i] = {xy[2 * i], xy[2 * i + 1]};
        for (uint32_t i = 0; i < m; ++i) g.segments.emplace_back(segs[2 * i], segs[2 * i + 1]);
        return reinterpret_cast<ref_mesh*>(new Mesh(build_cdt(g)));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// build_delaunay (cdt.hpp:198), no segments.
ref_mesh* ref_build_delaunay(const double* xy, uint32_t n) {
    try {
        std::vector<Point2> pts(n);
        for (uint32_t i = 0; i < n; ++i) pts[i] = {xy[2 * i], xy[2 * i + 1]};
        return reinterpret_cast<ref_mesh*>(new Mesh(build_delaunay(pts)));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_mesh_sizes(const ref_mesh* h, uint32_t* V, uint32_t* T, uint32_t* S) {
    const Mesh& m = *reinterpret_cast<const Mesh*>(h);
    *V = static_cast<uint32_t>(m.vertices.size());
    *T = static_cast<uint32_t>(m.triangles.size());
    *S = static_cast<uint32_t>(m.subsegments.size());
}

// refine (refine.hpp:651); executors > 1 selects ExecutionMode::Parallel.
int ref_refine(ref_mesh* h, const gdp2d_params* p, gdp2d_report* r, unsigned executors) {
    try {
        const RunReport rep = refine(*reinterpret_cast<Mesh*>(h), quality(p), engine(p, executors));
        fill_report(rep, r);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// refine_ruppert_sequential (refine.hpp:724): Steiner-count yardstick.
int ref_refine_sequential(ref_mesh* h, const gdp2d_params* p, gdp2d_report* r) {
    try {
        const RunReport rep =
            refine_ruppert_sequential(*reinterpret_cast<Mesh*>(h), quality(p), engine(p, 1));
        fill_report(rep, r);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Histogram of per-triangle minimum angles, in degrees, with the corner angle
// formula of min_angle_degrees (verify.hpp:186-200): bin k counts alive
// triangles whose min angle lies in [k*bin_deg, (k+1)*bin_deg); the last bin
// also takes everything above.  *sum gets the sum of the min angles.
uint64_t ref_min_angle_hist(const ref_mesh* h, double bin_deg, uint32_t nbins, uint64_t* hist,
                            double* sum) {
    const Mesh& m = *reinterpret_cast<const Mesh*>(h);
    std::memset(hist, 0, sizeof(uint64_t) * nbins);
    double s = 0.0;
    uint64_t n = 0;
    for (const Triangle& t : m.triangles) {
        if (!t.alive) continue;
        double best = 180.0;
        for (int i = 0; i < 3; ++i) {
            const Point2& p = m.pos(t.v[i]);
            const Point2 u = m.pos(t.v[Mesh::next(i)]) - p;
            const Point2 v = m.pos(t.v[Mesh::prev(i)]) - p;
            best = std::min(best, std::atan2(std::abs(cross(u, v)), dot(u, v)) * 180.0 /
                                      3.14159265358979323846);
        }
        uint32_t k = static_cast<uint32_t>(best / bin_deg);
        if (k >= nbins) k = nbins - 1;
        ++hist[k];
        s += best;
        ++n;
    }
    *sum = s;
    return n;
}

// quality_report (refine.hpp:716)
void ref_quality(const ref_mesh* h, const gdp2d_params* p, gdp2d_report* r) {
    const RunReport rep = quality_report(*reinterpret_cast<const Mesh*>(h), quality(p));
    fill_report(rep, r);
}

// collect (refine.hpp:226) followed by compute_splitting_points (:267).
int ref_collect(const ref_mesh* h, const gdp2d_params* p, gdp2d_candidate* out, uint32_t cap,
                uint32_t* n, uint32_t* fallbacks) {
    try {
        const Mesh& m = *reinterpret_cast<const Mesh*>(h);
        std::vector<SplitCandidate> l = collect(m, quality(p), engine(p, 1));
        *fallbacks = static_cast<uint32_t>(compute_splitting_points(m, l));
        *n = static_cast<uint32_t>(l.size());
        for (std::size_t i = 0; i < l.size() && i < cap; ++i) out[i] = from_ref(l[i]);
        return l.size() > cap ? 2 : 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_split_points(const ref_mesh* h, gdp2d_candidate* c, uint32_t n, uint32_t* fallbacks) {
    try {
        std::vector<SplitCandidate> l = list_in(c, n);
        *fallbacks = static_cast<uint32_t>(
            compute_splitting_points(*reinterpret_cast<const Mesh*>(h), l));
        list_out(l, c);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_locate(const ref_mesh* h, gdp2d_candidate* c, uint32_t n) {
    try {
        std::vector<SplitCandidate> l = list_in(c, n);
        for (auto& x : l) locate(*reinterpret_cast<const Mesh*>(h), x);
        list_out(l, c);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_claim(const ref_mesh* h, gdp2d_candidate* c, uint32_t n) {
    try {
        std::vector<SplitCandidate> l = list_in(c, n);
        claim_filter(*reinterpret_cast<const Mesh*>(h), l);
        list_out(l, c);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_cavity(const ref_mesh* h, gdp2d_candidate* c, uint32_t n, uint32_t n_cav) {
    try {
        std::vector<SplitCandidate> l = list_in(c, n);
        cavity_filter(*reinterpret_cast<const Mesh*>(h), l, n_cav, CompactionPolicy{});
        list_out(l, c);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// insert_batch (refine.hpp:464) on a prepared list; outcome = 7 counters.
int ref_insert_batch(ref_mesh* h, gdp2d_candidate* c, uint32_t n, const gdp2d_params* p,
                     uint64_t* outcome) {
    try {
        Mesh& m = *reinterpret_cast<Mesh*>(h);
        std::vector<SplitCandidate> l = list_in(c, n);
        std::vector<std::uint32_t> depth(m.subsegments.size(), 0);
        const BatchOutcome o = insert_batch(m, l, quality(p), engine(p, 1), depth);
        outcome[0] = o.inserted_midpoints;
        outcome[1] = o.inserted_circumcenters;
        outcome[2] = o.removed_redundant;
        outcome[3] = o.removed_dependent;
        outcome[4] = o.dropped;
        outcome[5] = o.marked_encroached;
        outcome[6] = o.retained();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Phase 1 of insert_batch (refine.hpp:492-539) WITHOUT the Lawson pass:
// splits only, using the reference's own mesh primitives (split_subsegment
// mesh.hpp:405, split_triangle :307, split_edge :351), so the flip-fixpoint
// primitive can be compared on identical ids.  Returns the fresh vertex ids.
int ref_split_only(ref_mesh* h, gdp2d_candidate* c, uint32_t n, uint32_t* fresh,
                   uint32_t* n_fresh) {
    try {
        Mesh& m = *reinterpret_cast<Mesh*>(h);
        std::vector<SplitCandidate> l = list_in(c, n);
        std::vector<std::size_t> order;
        for (std::size_t i = 0; i < l.size(); ++i)
            if (l[i].alive) order.push_back(i);
        std::sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
            return priority_less(l[b].priority, l[a].priority);
        });
        const std::uint32_t batch = ++m.batch_epoch;
        uint32_t k = 0;
        for (std::size_t i : order) {
            SplitCandidate& x = l[i];
            if (x.kind == SplitCandidate::Kind::Subseg) {
                if (!m.subsegments[x.id].alive) continue;
                fresh[k++] = m.split_subsegment(x.id, x.point, batch);
            } else {
                const Location loc = locate_point(m, x.located, x.point, true);
                if (loc.kind == Location::Kind::Inside)
                    fresh[k++] = m.split_triangle(loc.tri, x.point,
                                                  VertexKind::SteinerCircumcenter, batch);
                else if (loc.kind == Location::Kind::OnEdge &&
                         m.triangles[loc.tri].seg[loc.edge] == kNone)
                    fresh[k++] = m.split_edge(loc.tri, loc.edge, x.point,
                                              VertexKind::SteinerCircumcenter, batch);
            }
        }
        *n_fresh = k;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// incident_triangles (mesh.hpp:145) of v.
uint32_t ref_incident(const ref_mesh* h, uint32_t v, uint32_t* out, uint32_t cap) {
    const auto tris = reinterpret_cast<const Mesh*>(h)->incident_triangles(v);
    for (std::size_t i = 0; i < tris.size() && i < cap; ++i) out[i] = tris[i];
    return static_cast<uint32_t>(tris.size());
}

// lawson_fixpoint (cdt.hpp:111) seeded with (t, e) pairs.
int ref_lawson(ref_mesh* h, const uint32_t* t, const uint8_t* e, uint32_t n) {
    try {
        std::deque<std::pair<TriId, int>> work;
        for (uint32_t i = 0; i < n; ++i) work.emplace_back(t[i], e[i]);
        lawson_fixpoint(*reinterpret_cast<Mesh*>(h), std::move(work));
        return 0;
    } catch (const std::exception& e2) {
        return fail(e2);
    }
}

// ---- validators -------------------------------------------------------------

int ref_check_structure(const ref_mesh* h) {
    try {
        reinterpret_cast<const Mesh*>(h)->check_structure();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_euler_holds(const ref_mesh* h) { return reinterpret_cast<const Mesh*>(h)->euler_holds(); }

int ref_conformity_ok(const ref_mesh* h, const double* xy, uint32_t n, const uint32_t* segs,
                      uint32_t m) {
    Pslg g;
    g.points.resize(n);
    for (uint32_t i = 0; i < n; ++i) g.points[i] = {xy[2 * i], xy[2 * i + 1]};
    for (uint32_t i = 0; i < m; ++i) g.segments.emplace_back(segs[2 * i], segs[2 * i + 1]);
    try {
        return conformity_ok(*reinterpret_cast<const Mesh*>(h), g) ? 1 : 0;
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

uint64_t ref_cdt_violations(const ref_mesh* h, uint64_t cap) {
    return constrained_delaunay_violations(*reinterpret_cast<const Mesh*>(h), cap);
}

uint64_t ref_delaunay_violations(const ref_mesh* h, uint64_t cap) {
    return delaunay_violations(*reinterpret_cast<const Mesh*>(h), cap);
}

uint64_t ref_count_bad(const ref_mesh* h, const gdp2d_params* p) {
    const Mesh& m = *reinterpret_cast<const Mesh*>(h);
    const QualityCriteria q = quality(p);
    uint64_t n = 0;
    for (TriId t = 0; t < m.triangles.size(); ++t)
        if (m.triangles[t].alive && is_bad_triangle(m, t, q)) ++n;
    return n;
}

// Canonical triangle set: for each alive triangle, its vertex ids rotated so
// the smallest comes first (orientation kept); out holds 3 per triangle.
uint32_t ref_canonical_triangles(const ref_mesh* h, uint32_t* out) {
    const Mesh& m = *reinterpret_cast<const Mesh*>(h);
    uint32_t k = 0;
    for (const Triangle& t : m.triangles) {
        if (!t.alive) continue;
        int i = 0;
        if (t.v[1] < t.v[i]) i = 1;
        if (t.v[2] < t.v[i]) i = 2;
        out[3 * k] = t.v[i];
        out[3 * k + 1] = t.v[(i + 1) % 3];
        out[3 * k + 2] = t.v[(i + 2) % 3];
        ++k;
    }
    return k;
}

// write_node_ele (pslg_io.hpp:294): sizes first (out==NULL), then copy.
uint64_t ref_write_node_ele(const ref_mesh* h, char* node, uint64_t node_cap, char* ele,
                            uint64_t ele_cap, uint64_t* ele_len) {
    const NodeEle ne = write_node_ele(*reinterpret_cast<const Mesh*>(h));
    *ele_len = ne.ele.size();
    if (node && node_cap >= ne.node.size()) std::memcpy(node, ne.node.data(), ne.node.size());
    if (ele && ele_cap >= ne.ele.size()) std::memcpy(ele, ne.ele.data(), ne.ele.size());
    return ne.node.size();
}

// ---- predicates ---------------------------------------------------------------

void ref_predicates_batch(int kind, const double* pts, uint32_t n, const gdp2d_params* p,
                          int8_t* out) {
    auto P = [&](uint32_t rec, int arity, int k) {
        return Point2{pts[(static_cast<std::size_t>(rec) * arity + k) * 2],
                      pts[(static_cast<std::size_t>(rec) * arity + k) * 2 + 1]};
    };
    for (uint32_t i = 0; i < n; ++i) {
        switch (kind) {
            case GDP2D_PRED_ORIENT2D:
                out[i] = static_cast<int8_t>(orient2d(P(i, 3, 0), P(i, 3, 1), P(i, 3, 2)));
                break;
            case GDP2D_PRED_INCIRCLE:
                out[i] = static_cast<int8_t>(
                    incircle(P(i, 4, 0), P(i, 4, 1), P(i, 4, 2), P(i, 4, 3)));
                break;
            case GDP2D_PRED_DIAMETRIC:
                out[i] = in_diametric_circle(P(i, 3, 0), P(i, 3, 1), P(i, 3, 2));
                break;
            case GDP2D_PRED_LENS:
                out[i] = in_diametral_lens(P(i, 3, 0), P(i, 3, 1), P(i, 3, 2));
                break;
            case GDP2D_PRED_BAD_TRIANGLE: {
                Mesh m;
                for (int k = 0; k < 3; ++k) m.add_vertex(P(i, 3, k), VertexKind::Input, 0);
                m.add_triangle(0, 1, 2);
                out[i] = is_bad_triangle(m, 0, quality(p));
                break;
            }
            default:
                out[i] = -128;
        }
    }
}

void ref_circumcenter_batch(const double* pts, uint32_t n, double* out, uint8_t* ok) {
    for (uint32_t i = 0; i < n; ++i) {
        const double* q = pts + 6 * static_cast<std::size_t>(i);
        const auto cc = circumcenter({q[0], q[1]}, {q[2], q[3]}, {q[4], q[5]});
        out[2 * i] = cc.center.x;
        out[2 * i + 1] = cc.center.y;
        ok[i] = cc.well_conditioned;
    }
}

}  // extern "C"
