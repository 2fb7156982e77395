/*
 * gdp2d_cdtref.hpp -- drop-in C++ shim: the reference's refine entry point
 *
 *     RunReport cdtref::refine(Mesh&, const QualityCriteria&, const EngineConfig&)
 *     (/root/reference/proj/include/cdtref/refine.hpp:651)
 *
 * re-exposed with the SAME signature on top of the C ABI of gdp2d.h, so an
 * existing caller (tools/cdtref.cpp:175, tests/unit/test_refine.cpp:374, ...)
 * switches by including this header and writing gdp2d::refine instead of
 * cdtref::refine.  The caller keeps the reference's own Mesh, PSLG/mesh I/O
 * (pslg_io.hpp) and Line-1 build_cdt (cdt.hpp:483): this header hands the
 * Mesh's element vectors (mesh.hpp:43-75) to gdp2d_refine_aos as they are --
 * the records are converted on the device, so there is no host pack / unpack
 * -- runs the whole refinement loop on the GPU (libgdp2d.so) and writes the
 * result back into the same vectors.
 *
 * Include AFTER the reference headers ("cdtref/refine.hpp"); link -lgdp2d.
 *
 * Semantics kept from the reference:
 *   - the mesh is mutated in place; ids of surviving input elements are kept,
 *     dead slots stay (alive = false), new vertices carry kind
 *     SteinerMidpoint / SteinerCircumcenter and birth_batch, batch_epoch is
 *     bumped once per batch (refine.hpp:468);
 *   - RunReport is filled exactly like refine.hpp:651-713 (per-batch
 *     BatchMetrics with the six phase names of refine.hpp:671-701,
 *     iteration_cap_hit, and the quality summary of refine.hpp:614-645);
 *   - cfg.execution / executor_count / seed are accepted and ignored (the GPU
 *     is the executor), as rule3_gamma / rule5 are ignored by the reference;
 *   - on an error the mesh's element vectors are left unspecified (the
 *     reference leaves a partially refined mesh behind a MeshError too);
 *   - errors: a device structural failure throws cdtref::MeshError
 *     (MeshErrc::StaleHandle), capacity / CUDA / argument failures throw
 *     std::runtime_error carrying gdp2d_last_error().  There is no CPU
 *     fallback: without an sm_100 device the call throws.
 */
#ifndef GDP2D_CDTREF_HPP
#define GDP2D_CDTREF_HPP

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstddef>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "gdp2d.h"

#ifdef __linux__
#include <sys/mman.h>
#endif

namespace gdp2d {

namespace detail {

// Transparent-huge-page hint for [p, p + bytes) (the 2 MB pages inside it):
// the first touch of a multi-GB mesh array then faults 2 MB pages.
inline void hint_huge(const void* p, size_t bytes) {
#if defined(__linux__) && defined(MADV_HUGEPAGE)
    constexpr uintptr_t kHuge = uintptr_t(2) << 20;
    const uintptr_t lo = (reinterpret_cast<uintptr_t>(p) + kHuge - 1) & ~(kHuge - 1);
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(p) + bytes) & ~(kHuge - 1);
    if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
#else
    (void)p;
    (void)bytes;
#endif
}

// Uninitialised host array (no value-initialisation pass: the parallel fill
// below is its first touch, so page faults spread over the host cores).
template <class T>
inline std::unique_ptr<T[]> raw_array(size_t n) {
    std::unique_ptr<T[]> a(new T[n ? n : 1]);
    hint_huge(a.get(), sizeof(T) * n);
    return a;
}

// Size a vector to n elements whose contents are about to be overwritten
// wholesale: beyond its capacity a fresh (huge-page hinted) buffer replaces
// it instead of reallocating and copying the old elements.
template <class V>
inline void resize_for_overwrite(V& v, size_t n) {
    if (n > v.capacity()) {
        V fresh;
        fresh.reserve(n);
        hint_huge(fresh.data(), sizeof(typename V::value_type) * n);
        fresh.resize(n);
        v.swap(fresh);
    } else {
        v.resize(n);
    }
}

// The AoS <-> SoA conversion of a multi-million-element mesh is host work on
// the drop-in path: split it over the host cores (contiguous blocks, so the
// result is identical to a serial loop).
template <class F>
inline void parallel_for(size_t n, F&& f) {
    const unsigned hw = std::thread::hardware_concurrency();
    const size_t parts = std::min<size_t>(hw ? hw : 1, std::max<size_t>(1, n / 65536));
    if (parts <= 1) {
        for (size_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    for (size_t p = 0; p < parts; ++p)
        th.emplace_back([&, p] {
            const size_t lo = n * p / parts, hi = n * (p + 1) / parts;
            for (size_t i = lo; i < hi; ++i) f(i);
        });
    for (auto& t : th) t.join();
}

inline const char* const kPhaseNames[GDP2D_NPHASES] = {"collect", "split_points", "locate",
                                                       "claim", "cavity", "insert"};

inline gdp2d_params make_params(const cdtref::QualityCriteria& q,
                                const cdtref::EngineConfig& cfg) {
    gdp2d_params p;
    // host-computed cos^2(theta), exactly as is_bad_triangle (refine.hpp:195-196)
    gdp2d_params_init(&p, q.theta, q.ell,
                      q.mode == cdtref::RefineMode::Chew ? GDP2D_CHEW : GDP2D_RUPPERT);
    p.cavity_n = static_cast<uint32_t>(cfg.cavity_n);
    p.rule1_compaction_threshold = static_cast<uint32_t>(cfg.rules.rule1_compaction_threshold);
    p.rule2_filtering_enabled = cfg.rules.rule2_filtering_enabled ? 1u : 0u;
    p.rule4_unified_collection = cfg.rules.rule4_unified_collection ? 1u : 0u;
    p.iteration_cap = cfg.iteration_cap;
    p.split_depth_cap = cfg.split_depth_cap;
    p.batch_size_cap = cfg.batch_size_cap;
    return p;
}

// AoS Mesh -> SoA staging owned by the caller's stack frame.
struct Packed {
    std::unique_ptr<double[]> xy;
    std::unique_ptr<uint8_t[]> vkind, valive, talive, senc, salive;
    std::unique_ptr<uint32_t[]> vbirth, tv, tn, ts, sv, sparent;
    gdp2d_mesh_view view{};

    explicit Packed(const cdtref::Mesh& m) {
        const size_t V = m.vertices.size(), T = m.triangles.size(), S = m.subsegments.size();
        xy = raw_array<double>(2 * V);
        vkind = raw_array<uint8_t>(V);
        valive = raw_array<uint8_t>(V);
        vbirth = raw_array<uint32_t>(V);
        parallel_for(V, [&](size_t i) {
            const cdtref::Vertex& v = m.vertices[i];
            xy[2 * i] = v.pos.x;
            xy[2 * i + 1] = v.pos.y;
            vkind[i] = static_cast<uint8_t>(v.kind);
            vbirth[i] = v.birth_batch;
            valive[i] = v.alive ? 1 : 0;
        });
        tv = raw_array<uint32_t>(3 * T);
        tn = raw_array<uint32_t>(3 * T);
        ts = raw_array<uint32_t>(3 * T);
        talive = raw_array<uint8_t>(T);
        parallel_for(T, [&](size_t t) {
            const cdtref::Triangle& tr = m.triangles[t];
            for (int i = 0; i < 3; ++i) {
                tv[3 * t + i] = tr.v[i];
                tn[3 * t + i] = tr.nbr[i];
                ts[3 * t + i] = tr.seg[i];
            }
            talive[t] = tr.alive ? 1 : 0;
        });
        sv = raw_array<uint32_t>(2 * S);
        sparent = raw_array<uint32_t>(S);
        senc = raw_array<uint8_t>(S);
        salive = raw_array<uint8_t>(S);
        parallel_for(S, [&](size_t s) {
            const cdtref::Subsegment& sg = m.subsegments[s];
            sv[2 * s] = sg.v[0];
            sv[2 * s + 1] = sg.v[1];
            sparent[s] = sg.parent;
            senc[s] = sg.encroached ? 1 : 0;
            salive[s] = sg.alive ? 1 : 0;
        });
        view.n_vertices = static_cast<uint32_t>(V);
        view.n_triangles = static_cast<uint32_t>(T);
        view.n_subsegments = static_cast<uint32_t>(S);
        view.batch_epoch = m.batch_epoch;
        view.xy = xy.get();
        view.vert_kind = vkind.get();
        view.vert_birth = vbirth.get();
        view.vert_alive = valive.get();
        view.vert_tri = m.vert_tri.data();
        view.tri_v = tv.get();
        view.tri_n = tn.get();
        view.tri_seg = ts.get();
        view.tri_alive = talive.get();
        view.seg_v = sv.get();
        view.seg_parent = sparent.get();
        view.seg_encroached = senc.get();
        view.seg_alive = salive.get();
        view.seg_tri = m.seg_tri.data();
    }
};

// SoA result -> the caller's Mesh, in place (ids preserved).
inline void unpack(const gdp2d_mesh_buf& b, cdtref::Mesh& m) {
    const size_t V = b.n_vertices, T = b.n_triangles, S = b.n_subsegments;
    resize_for_overwrite(m.vertices, V);
    m.vert_tri.assign(b.vert_tri, b.vert_tri + V);
    parallel_for(V, [&](size_t i) {
        cdtref::Vertex& v = m.vertices[i];
        v.pos = cdtref::Point2{b.xy[2 * i], b.xy[2 * i + 1]};
        v.kind = static_cast<cdtref::VertexKind>(b.vert_kind[i]);
        v.birth_batch = b.vert_birth[i];
        v.alive = b.vert_alive[i] != 0;
    });
    resize_for_overwrite(m.triangles, T);
    parallel_for(T, [&](size_t t) {
        cdtref::Triangle& tr = m.triangles[t];
        for (int i = 0; i < 3; ++i) {
            tr.v[i] = b.tri_v[3 * t + i];
            tr.nbr[i] = b.tri_n[3 * t + i];
            tr.seg[i] = b.tri_seg[3 * t + i];
        }
        tr.alive = b.tri_alive[t] != 0;
    });
    resize_for_overwrite(m.subsegments, S);
    m.seg_tri.assign(b.seg_tri, b.seg_tri + S);
    parallel_for(S, [&](size_t s) {
        cdtref::Subsegment& sg = m.subsegments[s];
        sg.v = {b.seg_v[2 * s], b.seg_v[2 * s + 1]};
        sg.parent = b.seg_parent[s];
        sg.encroached = b.seg_encroached[s] != 0;
        sg.alive = b.seg_alive[s] != 0;
    });
    m.batch_epoch = b.batch_epoch;
}

// Expected output/input size ratio of a refinement: ~2x at radius-edge
// sqrt(2), ~5x at 30 degrees (BASELINE configs 2-4).  Only a hint: a larger
// output just grows again when the library asks for the output vectors.
inline double growth_hint(const cdtref::QualityCriteria& q) {
    return q.theta >= 28.0 ? 5.5 : q.theta >= 24.0 ? 3.5 : 2.2;
}

inline void throw_status(int rc) {
    const std::string what = std::string("gdp2d_refine: ") + gdp2d_last_error();
    if (rc == GDP2D_EMESH) throw cdtref::MeshError(cdtref::MeshErrc::StaleHandle, what);
    throw std::runtime_error(what);
}

}  // namespace detail

namespace detail {

// The reference's records as gdp2d_refine_aos sees them.
inline gdp2d_aos_layout aos_layout() {
    gdp2d_aos_layout L;
    L.vert_size = sizeof(cdtref::Vertex);
    L.vert_pos = offsetof(cdtref::Vertex, pos);
    L.vert_kind = offsetof(cdtref::Vertex, kind);
    L.vert_birth = offsetof(cdtref::Vertex, birth_batch);
    L.vert_alive = offsetof(cdtref::Vertex, alive);
    L.tri_size = sizeof(cdtref::Triangle);
    L.tri_v = offsetof(cdtref::Triangle, v);
    L.tri_nbr = offsetof(cdtref::Triangle, nbr);
    L.tri_seg = offsetof(cdtref::Triangle, seg);
    L.tri_alive = offsetof(cdtref::Triangle, alive);
    L.seg_size = sizeof(cdtref::Subsegment);
    L.seg_v = offsetof(cdtref::Subsegment, v);
    L.seg_parent = offsetof(cdtref::Subsegment, parent);
    L.seg_encroached = offsetof(cdtref::Subsegment, encroached);
    L.seg_alive = offsetof(cdtref::Subsegment, alive);
    return L;
}
static_assert(sizeof(cdtref::VertexKind) == 1 && sizeof(bool) == 1 &&
                  sizeof(cdtref::Point2) == 16 && sizeof(cdtref::TriId) == 4 &&
                  sizeof(cdtref::SubsegId) == 4 && sizeof(cdtref::VertexId) == 4,
              "gdp2d_aos_layout field widths");

// The output vectors, built on a host thread while the device refines:
// std::vector's value-initialisation of a multi-GB tail is serial, and the
// fresh buffers are swapped in only when the library asks for them (the
// caller's input vectors are being read by the upload until then).
struct OutVectors {
    cdtref::Mesh& m;
    double g;
    std::vector<cdtref::Vertex> verts;
    std::vector<cdtref::Triangle> tris;
    std::vector<cdtref::Subsegment> segs;
    std::vector<cdtref::TriId> vtri, stri;
    std::thread th[3];
    OutVectors(cdtref::Mesh& mesh, double growth) : m(mesh), g(growth) {
        auto make = [this](auto* v, size_t n0) {
            const size_t n = static_cast<size_t>(static_cast<double>(n0) * g);
            v->reserve(n + n / 8);   // room to grow a little without a copy
            hint_huge(v->data(), sizeof(typename std::decay_t<decltype(*v)>::value_type) * v->capacity());
            v->resize(n);
        };
        const size_t V = m.vertices.size(), T = m.triangles.size(), S = m.subsegments.size();
        // one thread per big vector (the triangle records dominate)
        th[0] = std::thread([=] { make(&tris, T); });
        th[1] = std::thread([=] {
            make(&verts, V);
            make(&vtri, V);
        });
        th[2] = std::thread([=] {
            make(&segs, S);
            make(&stri, S);
        });
    }
    void join() {
        for (auto& t : th)
            if (t.joinable()) t.join();
    }
    ~OutVectors() { join(); }
    template <class V>
    static void* take(V& dst, V& fresh, size_t n) {
        if (n <= fresh.capacity()) {
            dst.swap(fresh);
            dst.resize(n);
        } else {
            resize_for_overwrite(dst, n);
        }
        return dst.data();
    }
    // gdp2d_aos_mesh::resize
    static void* resize(void* user, int what, uint64_t n) {
        OutVectors& o = *static_cast<OutVectors*>(user);
        // wait only for the thread that builds the requested vector
        std::thread& t = o.th[what == GDP2D_AOS_TRIS ? 0 : (what == GDP2D_AOS_VERTS || what == GDP2D_AOS_VERT_TRI) ? 1 : 2];
        if (t.joinable()) t.join();
        switch (what) {
            case GDP2D_AOS_VERTS: return take(o.m.vertices, o.verts, n);
            case GDP2D_AOS_TRIS: return take(o.m.triangles, o.tris, n);
            case GDP2D_AOS_SEGS: return take(o.m.subsegments, o.segs, n);
            case GDP2D_AOS_VERT_TRI: return take(o.m.vert_tri, o.vtri, n);
            case GDP2D_AOS_SEG_TRI: return take(o.m.seg_tri, o.stri, n);
            default: return nullptr;
        }
    }
};

}  // namespace detail

// Drop-in for cdtref::refine (refine.hpp:651).  `device` selects the GPU
// (one call = one device + one stream, blocking; distinct host threads may
// drive distinct devices).
inline cdtref::RunReport refine(cdtref::Mesh& m, const cdtref::QualityCriteria& q,
                                const cdtref::EngineConfig& cfg, int device = 0) {
    const gdp2d_params p = detail::make_params(q, cfg);
    const gdp2d_aos_layout L = detail::aos_layout();
    std::vector<gdp2d_batch_metrics> bm(cfg.iteration_cap < 100000 ? cfg.iteration_cap + 1 : 100001);
    gdp2d_report r{};
    r.batches = bm.data();
    r.batches_capacity = static_cast<uint32_t>(bm.size());
    int rc;
    {
        detail::OutVectors out(m, detail::growth_hint(q));
        gdp2d_aos_mesh a{};
        a.n_vertices = static_cast<uint32_t>(m.vertices.size());
        a.n_triangles = static_cast<uint32_t>(m.triangles.size());
        a.n_subsegments = static_cast<uint32_t>(m.subsegments.size());
        a.batch_epoch = m.batch_epoch;
        a.verts = m.vertices.data();
        a.tris = m.triangles.data();
        a.segs = m.subsegments.data();
        a.vert_tri = m.vert_tri.data();
        a.seg_tri = m.seg_tri.data();
        a.resize = &detail::OutVectors::resize;
        a.user = &out;
        rc = gdp2d_refine_aos(&L, &a, &p, &r, device);
        if (rc == GDP2D_OK) m.batch_epoch = a.batch_epoch;
    }
    if (rc != GDP2D_OK) detail::throw_status(rc);

    cdtref::RunReport rep;
    const uint32_t nb = r.n_batches < r.batches_capacity ? r.n_batches : r.batches_capacity;
    for (uint32_t i = 0; i < nb; ++i) {
        std::map<std::string, double> phases;
        for (int k = 0; k < GDP2D_NPHASES; ++k) {
            // the reference records "cavity" only when rule 2 is on (refine.hpp:688)
            if (k == GDP2D_PH_CAVITY && !cfg.rules.rule2_filtering_enabled) continue;
            phases[detail::kPhaseNames[k]] = bm[i].phase_seconds[k];
        }
        rep.batches.push_back(cdtref::record_batch(bm[i].batch_index, std::move(phases),
                                                   bm[i].attempted, bm[i].concurrency));
    }
    rep.output_points = r.output_points;
    rep.steiner_points = r.steiner_points;
    rep.bad_triangles = r.bad_triangles;
    rep.bad_area_percent = r.bad_area_percent;
    rep.min_angle_deg = r.min_angle_deg;
    rep.max_edge = r.max_edge;
    rep.wall_seconds = r.wall_seconds;
    rep.iteration_cap_hit = r.iteration_cap_hit != 0;
    return rep;
}

// Drop-in for cdtref::build_cdt (cdt.hpp:483) on the GPU (gdp2d_build_cdt).
// Same Pslg in (hull already closed by read_poly / to_pslg), a fresh Mesh out
// whose vertex i is g.points[i]; the triangle set equals the reference's for
// PSLGs in general position (ids differ).  Throws cdtref::CdtError where the
// reference does (duplicate points, all collinear, crossing segments).
inline cdtref::Mesh build_cdt(const cdtref::Pslg& g, int device = 0) {
    std::vector<double> xy(2 * g.points.size());
    for (size_t i = 0; i < g.points.size(); ++i) {
        xy[2 * i] = g.points[i].x;
        xy[2 * i + 1] = g.points[i].y;
    }
    std::vector<uint32_t> seg(2 * g.segments.size());
    for (size_t i = 0; i < g.segments.size(); ++i) {
        seg[2 * i] = g.segments[i].first;
        seg[2 * i + 1] = g.segments[i].second;
    }
    gdp2d_mesh_buf out{};
    gdp2d_cdt_report rep{};
    const int rc = gdp2d_build_cdt(xy.data(), static_cast<uint32_t>(g.points.size()), seg.data(),
                                   static_cast<uint32_t>(g.segments.size()), &out, &rep, device);
    if (rc == GDP2D_ECDT) throw cdtref::CdtError(std::string("gdp2d_build_cdt: ") + gdp2d_last_error());
    if (rc != GDP2D_OK) detail::throw_status(rc);
    cdtref::Mesh m;
    detail::unpack(out, m);
    gdp2d_free(&out);
    return m;
}

}  // namespace gdp2d

#endif  // GDP2D_CDTREF_HPP
