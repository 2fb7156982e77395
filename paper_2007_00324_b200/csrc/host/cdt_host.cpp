// cdt_host.cpp -- the host side that north_star keeps from the reference:
// PSLG / mesh I/O and the untimed Line-1 CDT construction, compiled from the
// unmodified headers under /root/reference/proj/include (nothing is copied).
//   read_poly / to_pslg   pslg_io.hpp:196-272 (duplicate + crossing checks, close_hull)
//   close_hull            cdt.hpp:447
//   build_cdt             cdt.hpp:483 (Line 1; PAPER.md:508 excludes it from timing)
//   write_node_ele        pslg_io.hpp:294
// The refinement itself (Lines 2-9) never runs here: it is libgdp2d.so, reached
// through the drop-in shim (include/gdp2d_cdtref.hpp) by gdp2d_host_time_dropin.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>
#include <thread>
#include <algorithm>

#include "cdtref/cdt.hpp"
#include "cdtref/mesh.hpp"
#include "cdtref/pslg_io.hpp"
#include "cdtref/refine.hpp"
#include "gdp2d.h"
#include "gdp2d_cdtref.hpp"

using namespace cdtref;

namespace {

thread_local std::string g_err;

template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

void mesh_to_buf(const Mesh& m, gdp2d_mesh_buf* b) {
    const uint32_t V = (uint32_t)m.vertices.size(), T = (uint32_t)m.triangles.size(),
                   S = (uint32_t)m.subsegments.size();
    b->n_vertices = V;
    b->n_triangles = T;
    b->n_subsegments = S;
    b->batch_epoch = m.batch_epoch;
    std::vector<double> xy(2 * (size_t)V);
    std::vector<uint8_t> vk(V), va(V);
    std::vector<uint32_t> vb(V);
    for (uint32_t i = 0; i < V; ++i) {
        xy[2 * i] = m.vertices[i].pos.x;
        xy[2 * i + 1] = m.vertices[i].pos.y;
        vk[i] = (uint8_t)m.vertices[i].kind;
        va[i] = m.vertices[i].alive;
        vb[i] = m.vertices[i].birth_batch;
    }
    std::vector<uint32_t> tv(3 * (size_t)T), tn(3 * (size_t)T), ts(3 * (size_t)T);
    std::vector<uint8_t> ta(T);
    for (uint32_t t = 0; t < T; ++t) {
        for (int i = 0; i < 3; ++i) {
            tv[3 * t + i] = m.triangles[t].v[i];
            tn[3 * t + i] = m.triangles[t].nbr[i];
            ts[3 * t + i] = m.triangles[t].seg[i];
        }
        ta[t] = m.triangles[t].alive;
    }
    std::vector<uint32_t> sv(2 * (size_t)S), sp(S);
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

Mesh view_to_mesh(const gdp2d_mesh_view* v) {
    Mesh m;
    m.batch_epoch = v->batch_epoch;
    m.vertices.resize(v->n_vertices);
    m.vert_tri.assign(v->vert_tri, v->vert_tri + v->n_vertices);
    for (uint32_t i = 0; i < v->n_vertices; ++i) {
        m.vertices[i].pos = {v->xy[2 * i], v->xy[2 * i + 1]};
        m.vertices[i].kind = static_cast<VertexKind>(v->vert_kind[i]);
        m.vertices[i].birth_batch = v->vert_birth[i];
        m.vertices[i].alive = v->vert_alive[i] != 0;
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
    m.seg_tri.assign(v->seg_tri, v->seg_tri + v->n_subsegments);
    for (uint32_t s = 0; s < v->n_subsegments; ++s) {
        m.subsegments[s].v = {v->seg_v[2 * s], v->seg_v[2 * s + 1]};
        m.subsegments[s].parent = v->seg_parent[s];
        m.subsegments[s].encroached = v->seg_encroached[s] != 0;
        m.subsegments[s].alive = v->seg_alive[s] != 0;
    }
    return m;
}

}  // namespace

extern "C" {

const char* gdp2d_host_last_error(void) { return g_err.c_str(); }

// PSLG -> (optionally close_hull) -> check_crossings -> build_cdt -> SoA.
// *segs_out receives the final segment list (2 * *m_out, malloc'd).
int gdp2d_host_build_cdt(const double* xy, uint32_t n, const uint32_t* segs, uint32_t m,
                         int close, gdp2d_mesh_buf* out, uint32_t** segs_out, uint32_t* m_out) {
    try {
        Pslg g;
        g.points.resize(n);
        for (uint32_t i = 0; i < n; ++i) g.points[i] = {xy[2 * i], xy[2 * i + 1]};
        for (uint32_t i = 0; i < m; ++i) g.segments.emplace_back(segs[2 * i], segs[2 * i + 1]);
        if (close) g = close_hull(std::move(g));
        detail::check_crossings(g);
        const Mesh mesh = build_cdt(g);
        mesh_to_buf(mesh, out);
        if (segs_out && m_out) {
            *m_out = (uint32_t)g.segments.size();
            *segs_out = static_cast<uint32_t*>(std::malloc(8 * (g.segments.size() + 1)));
            for (size_t i = 0; i < g.segments.size(); ++i) {
                (*segs_out)[2 * i] = g.segments[i].first;
                (*segs_out)[2 * i + 1] = g.segments[i].second;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// close_hull (cdt.hpp:447) [+ check_crossings]: the segment list the device
// CDT builder (gdp2d_ctx_build_cdt) takes.
int gdp2d_host_close_hull(const double* xy, uint32_t n, const uint32_t* segs, uint32_t m,
                          int check, uint32_t** segs_out, uint32_t* m_out) {
    try {
        Pslg g;
        g.points.resize(n);
        for (uint32_t i = 0; i < n; ++i) g.points[i] = {xy[2 * i], xy[2 * i + 1]};
        for (uint32_t i = 0; i < m; ++i) g.segments.emplace_back(segs[2 * i], segs[2 * i + 1]);
        g = close_hull(std::move(g));
        if (check) detail::check_crossings(g);
        *m_out = (uint32_t)g.segments.size();
        *segs_out = static_cast<uint32_t*>(std::malloc(8 * (g.segments.size() + 1)));
        for (size_t i = 0; i < g.segments.size(); ++i) {
            (*segs_out)[2 * i] = g.segments[i].first;
            (*segs_out)[2 * i + 1] = g.segments[i].second;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// read_poly (pslg_io.hpp:272): text -> closed PSLG.
int gdp2d_host_read_poly(const char* text, double** xy, uint32_t* n, uint32_t** segs,
                         uint32_t* m) {
    try {
        const Pslg g = read_poly(text);
        *n = (uint32_t)g.points.size();
        *m = (uint32_t)g.segments.size();
        *xy = static_cast<double*>(std::malloc(16 * (g.points.size() + 1)));
        *segs = static_cast<uint32_t*>(std::malloc(8 * (g.segments.size() + 1)));
        for (size_t i = 0; i < g.points.size(); ++i) {
            (*xy)[2 * i] = g.points[i].x;
            (*xy)[2 * i + 1] = g.points[i].y;
        }
        for (size_t i = 0; i < g.segments.size(); ++i) {
            (*segs)[2 * i] = g.segments[i].first;
            (*segs)[2 * i + 1] = g.segments[i].second;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// write_node_ele (pslg_io.hpp:294) of a refined mesh.
int gdp2d_host_write_node_ele(const gdp2d_mesh_view* v, char** node, char** ele) {
    try {
        const Mesh mesh = view_to_mesh(v);
        const NodeEle ne = write_node_ele(mesh);
        *node = static_cast<char*>(std::malloc(ne.node.size() + 1));
        *ele = static_cast<char*>(std::malloc(ne.ele.size() + 1));
        std::memcpy(*node, ne.node.c_str(), ne.node.size() + 1);
        std::memcpy(*ele, ne.ele.c_str(), ne.ele.size() + 1);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// write_node_ele's text (pslg_io.hpp:294-319) from an already compacted mesh
// (gdp2d_ctx_export): same header lines, same shortest round-trip doubles
// (detail::shortest -> std::to_chars), same row numbering.
int gdp2d_host_format_node_ele(uint32_t n_nodes, const double* xy, const uint8_t* marker,
                               uint32_t n_tris, const uint32_t* tri, char** node, char** ele) {
    try {
        // Text of write_node_ele (pslg_io.hpp:294-319), formatted in parallel:
        // each thread renders a contiguous block of lines, the blocks are
        // concatenated in order (byte-identical to the serial loop).
        unsigned nthr = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        if (const char* e = std::getenv("GDP2D_IO_THREADS")) nthr = std::max(1, std::atoi(e));
        auto render = [&](uint32_t n, size_t per_line, auto&& line) {
            const uint32_t parts = (uint32_t)std::min<uint64_t>(nthr, std::max<uint32_t>(1, n / 4096));
            std::vector<std::string> blk(parts);
            std::vector<std::thread> th;
            for (uint32_t p = 0; p < parts; ++p) {
                th.emplace_back([&, p] {
                    const uint32_t lo = (uint32_t)((uint64_t)n * p / parts);
                    const uint32_t hi = (uint32_t)((uint64_t)n * (p + 1) / parts);
                    std::string& out = blk[p];
                    out.reserve(per_line * (hi - lo));
                    for (uint32_t i = lo; i < hi; ++i) line(out, i);
                });
            }
            for (auto& t : th) t.join();
            return blk;
        };
        const auto node_blocks = render(n_nodes, 48, [&](std::string& o, uint32_t i) {
            o += std::to_string(i);
            o += ' ';
            o += cdtref::detail::shortest(xy[2 * i]);
            o += ' ';
            o += cdtref::detail::shortest(xy[2 * i + 1]);
            o += marker[i] ? " 1\n" : " 0\n";
        });
        const auto ele_blocks = render(n_tris, 32, [&](std::string& o, uint32_t t) {
            o += std::to_string(t);
            for (int k = 0; k < 3; ++k) {
                o += ' ';
                o += std::to_string(tri[3ull * t + k]);
            }
            o += '\n';
        });
        auto join = [](const std::string& head, const std::vector<std::string>& blocks) {
            size_t len = head.size();
            for (const auto& b : blocks) len += b.size();
            char* out = static_cast<char*>(std::malloc(len + 1));
            size_t o = 0;
            std::memcpy(out, head.data(), head.size());
            o += head.size();
            for (const auto& b : blocks) {
                std::memcpy(out + o, b.data(), b.size());
                o += b.size();
            }
            out[o] = 0;
            return out;
        };
        *node = join(std::to_string(n_nodes) + " 2 0 1\n", node_blocks);
        *ele = join(std::to_string(n_tris) + " 3 0\n", ele_blocks);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void gdp2d_host_free_buf(gdp2d_mesh_buf* b) {
    void* ptrs[] = {b->xy,      b->vert_kind, b->vert_birth, b->vert_alive, b->vert_tri,
                    b->tri_v,   b->tri_n,     b->tri_seg,    b->tri_alive,  b->seg_v,
                    b->seg_parent, b->seg_encroached, b->seg_alive, b->seg_tri};
    for (void* p : ptrs) std::free(p);
    std::memset(b, 0, sizeof *b);
}

// One drop-in call, for parity tests: the reference Mesh built from *in,
// refined by gdp2d::refine (include/gdp2d_cdtref.hpp, gdp2d_refine_aos) and
// returned as an SoA buffer (gdp2d_host_free_buf).
int gdp2d_host_dropin_refine(const gdp2d_mesh_view* in, double theta_deg, int device,
                             gdp2d_mesh_buf* out, uint64_t* steiner) {
    try {
        Mesh m = view_to_mesh(in);
        QualityCriteria q;
        q.theta = theta_deg;
        const RunReport rep = gdp2d::refine(m, q, EngineConfig{}, device);
        *steiner = rep.steiner_points;
        mesh_to_buf(m, out);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// The drop-in caller's path, timed: gdp2d::refine(cdtref::Mesh&, q, cfg)
// (include/gdp2d_cdtref.hpp) on the reference's own AoS Mesh in pageable
// memory -- its element vectors go to gdp2d_refine_aos as they are (H2D,
// device record conversion, device loop, D2H back into the vectors) --
// exactly what a cdtref caller gets after swapping the namespace.  The
// reference Mesh is built from *in once; each of `steps` calls refines a
// fresh copy of it (the copy is untimed).  Writes the summed call time and
// the last call's Steiner count.  parts (optional, 4 doubles): summed seconds
// of a further `steps` calls split by the library's own clocks -- transfers
// (gdp2d_report e2e_seconds minus the loop: H2D, record conversion, D2H, and
// any wait for the output vectors), the refinement loop (wall_seconds), the
// shim around the library call, and 0.
int gdp2d_host_time_dropin(const gdp2d_mesh_view* in, double theta_deg, int steps, int device,
                           double* seconds, uint64_t* steiner, double* parts) {
    try {
        const Mesh base = view_to_mesh(in);
        QualityCriteria q;
        q.theta = theta_deg;
        const EngineConfig cfg{};
        double total = 0.0;
        for (int i = 0; i < steps; ++i) {
            Mesh m = base;
            const auto t0 = std::chrono::steady_clock::now();
            const RunReport rep = gdp2d::refine(m, q, cfg, device);
            total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            *steiner = rep.steiner_points;
        }
        *seconds = total;
        if (parts) {
            using clk = std::chrono::steady_clock;
            for (int k = 0; k < 4; ++k) parts[k] = 0.0;
            for (int i = 0; i < steps; ++i) {
                Mesh m = base;
                const gdp2d_params p = gdp2d::detail::make_params(q, cfg);
                const gdp2d_aos_layout L = gdp2d::detail::aos_layout();
                std::vector<gdp2d_batch_metrics> bm(cfg.iteration_cap + 1);
                gdp2d_report r{};
                r.batches = bm.data();
                r.batches_capacity = (uint32_t)bm.size();
                const auto t0 = clk::now();
                int rc;
                {
                    gdp2d::detail::OutVectors out(m, gdp2d::detail::growth_hint(q));
                    gdp2d_aos_mesh a{};
                    a.n_vertices = (uint32_t)m.vertices.size();
                    a.n_triangles = (uint32_t)m.triangles.size();
                    a.n_subsegments = (uint32_t)m.subsegments.size();
                    a.batch_epoch = m.batch_epoch;
                    a.verts = m.vertices.data();
                    a.tris = m.triangles.data();
                    a.segs = m.subsegments.data();
                    a.vert_tri = m.vert_tri.data();
                    a.seg_tri = m.seg_tri.data();
                    a.resize = &gdp2d::detail::OutVectors::resize;
                    a.user = &out;
                    rc = gdp2d_refine_aos(&L, &a, &p, &r, device);
                }
                if (rc != GDP2D_OK) throw std::runtime_error(gdp2d_last_error());
                const double call = std::chrono::duration<double>(clk::now() - t0).count();
                parts[0] += r.e2e_seconds - r.wall_seconds;
                parts[1] += r.wall_seconds;
                parts[2] += call - r.e2e_seconds;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
