// gdp2d_cli.cpp -- the reference CLI's run_one (tools/cdtref.cpp:151-199)
// with the ONE change a maintainer makes to adopt the GPU engine:
// cdtref::refine (refine.hpp:651) -> gdp2d::refine (include/gdp2d_cdtref.hpp).
// Everything around it is the reference's own host code, compiled from the
// unmodified headers: read_poly (pslg_io.hpp:272), build_cdt (cdt.hpp:483,
// Line 1, untimed), conformity_ok (verify.hpp:147), write_node_ele
// (pslg_io.hpp:294).  Exit codes follow cdtref.cpp: 0 ok, 2 input error,
// 3 cap hit / verification failure, 4 engine error.
//
//   gdp2d_cli input.poly [--theta DEG] [--ell L] [--chew] [--out PREFIX] [--device D]
//             [--device-cdt]   (Line 1 via gdp2d::build_cdt instead of cdtref::build_cdt)
//             [--device-io]    (the mesh stays on the device --
//                               device validators instead of the host checks, the
//                               compaction of write_node_ele on the device and the
//                               text rendered on all host cores; same bytes)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <thread>
#include <sstream>
#include <limits>
#include <stdexcept>
#include <string>

#include "cdtref/cdt.hpp"
#include "cdtref/pslg_io.hpp"
#include "cdtref/refine.hpp"
#include "cdtref/verify.hpp"
#include "gdp2d_cdtref.hpp"

// libgdp2d_host.so: write_node_ele's text from compacted arrays, multi-threaded
extern "C" int gdp2d_host_format_node_ele(uint32_t n_nodes, const double* xy,
                                          const uint8_t* marker, uint32_t n_tris,
                                          const uint32_t* tri, char** node, char** ele);

namespace {

// --device-io: Lines 1-9 in one device context, the output compacted on the
// device (gdp2d_ctx_export) and validated there (gdp2d_ctx_validate).
int run_device_io(const cdtref::Pslg& g, const cdtref::QualityCriteria& q,
                  const cdtref::EngineConfig& cfg, int device, bool device_cdt,
                  const std::string& prefix) {
    gdp2d_ctx* ctx = nullptr;
    if (gdp2d_ctx_create(&ctx, device) != GDP2D_OK) {
        std::fprintf(stderr, "engine error: %s\n", gdp2d_last_error());
        return 4;
    }
    struct Guard {
        gdp2d_ctx* c;
        ~Guard() { gdp2d_ctx_destroy(c); }
    } guard{ctx};
    if (device_cdt) {
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
        gdp2d_cdt_report cr{};
        const int rc = gdp2d_ctx_build_cdt(ctx, xy.data(), (uint32_t)g.points.size(), seg.data(),
                                           (uint32_t)g.segments.size(), &cr);
        if (rc != GDP2D_OK) {
            std::fprintf(stderr, "%s error: %s\n", rc == GDP2D_ECDT ? "input" : "engine",
                         gdp2d_last_error());
            return rc == GDP2D_ECDT ? 2 : 4;
        }
    } else {
        cdtref::Mesh m;
        try {
            m = cdtref::build_cdt(g);
        } catch (const std::exception& e) {
            std::fprintf(stderr, "input error: %s\n", e.what());
            return 2;
        }
        gdp2d::detail::Packed in(m);
        if (gdp2d_ctx_upload(ctx, &in.view) != GDP2D_OK) {
            std::fprintf(stderr, "engine error: %s\n", gdp2d_last_error());
            return 4;
        }
    }
    const gdp2d_params p = gdp2d::detail::make_params(q, cfg);
    std::vector<gdp2d_batch_metrics> bm(100001);
    gdp2d_report r{};
    r.batches = bm.data();
    r.batches_capacity = (uint32_t)bm.size();
    if (gdp2d_ctx_refine(ctx, &p, &r) != GDP2D_OK) {
        std::fprintf(stderr, "engine error: %s\n", gdp2d_last_error());
        return 4;
    }
    int rc = r.iteration_cap_hit ? 3 : 0;
    gdp2d_validation v{};
    if (gdp2d_ctx_validate(ctx, &p, &v) != GDP2D_OK) {
        std::fprintf(stderr, "engine error: %s\n", gdp2d_last_error());
        return 4;
    }
    if (rc == 0 && (v.structure_failure || v.conformity_failures)) {
        std::fprintf(stderr, "post-run verification failed: structure %u, conformity %llu\n",
                     v.structure_failure, (unsigned long long)v.conformity_failures);
        rc = 3;
    }
    uint32_t nv = 0, nt = 0, ns = 0;
    gdp2d_ctx_sizes(ctx, &nv, &nt, &ns);
    std::vector<double> xy(2ull * nv);
    std::vector<uint8_t> marker(nv);
    std::vector<uint32_t> tri(3ull * nt);
    gdp2d_node_ele ne{};
    ne.xy = xy.data();
    ne.marker = marker.data();
    ne.tri = tri.data();
    if (gdp2d_ctx_export(ctx, &ne) != GDP2D_OK) {
        std::fprintf(stderr, "engine error: %s\n", gdp2d_last_error());
        return 4;
    }
    char *node = nullptr, *ele = nullptr;
    if (gdp2d_host_format_node_ele(ne.n_nodes, xy.data(), marker.data(), ne.n_tris, tri.data(),
                                   &node, &ele) != 0) {
        std::fprintf(stderr, "output error\n");
        return 4;
    }
    std::ofstream(prefix + ".node") << node;
    std::ofstream(prefix + ".ele") << ele;
    std::free(node);
    std::free(ele);
    std::printf("batches=%u output_points=%llu steiner_points=%llu bad_triangles=%llu "
                "min_angle_deg=%.6f wall_seconds=%.6f exit=%d\n",
                r.n_batches, (unsigned long long)r.output_points,
                (unsigned long long)r.steiner_points, (unsigned long long)r.bad_triangles,
                r.min_angle_deg, r.wall_seconds, rc);
    return rc;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s input.poly [--theta DEG] [--ell L] [--chew] "
                             "[--out PREFIX] [--device D] [--device-cdt] [--device-io]\n", argv[0]);
        return 2;
    }
    std::string input = argv[1], prefix;
    cdtref::QualityCriteria q;
    cdtref::EngineConfig cfg;
    int device = 0;
    bool device_cdt = false;   // --device-cdt: Line 1 on the GPU too (gdp2d::build_cdt)
    bool device_io = false;    // --device-io: validate + compact on the device
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> const char* {
            if (i + 1 >= argc) throw std::invalid_argument("flag " + a + " needs a value");
            return argv[++i];
        };
        try {
        if (a == "--theta") q.theta = std::atof(val());
        else if (a == "--ell") {
            // 0 (or negative) = unbounded, as the reference CLI (tools/cdtref.cpp:85)
            const double v = std::atof(val());
            q.ell = v > 0.0 ? v : std::numeric_limits<double>::infinity();
        }
        else if (a == "--chew") q.mode = cdtref::RefineMode::Chew;
        else if (a == "--out") prefix = val();
        else if (a == "--device") device = std::atoi(val());
        else if (a == "--device-cdt") device_cdt = true;
        else if (a == "--device-io") device_io = true;
        else {
            std::fprintf(stderr, "unknown flag %s\n", a.c_str());
            return 2;
        }
        } catch (const std::invalid_argument& e) {
            std::fprintf(stderr, "%s\n", e.what());
            return 2;
        }
    }
    // CUDA context creation and kernel loading overlap the input parsing and
    // the host CDT (gdp2d_refine / build_cdt wait on the context's lock)
    std::thread warm([device] { gdp2d_warmup(device); });
    struct Join {
        std::thread& t;
        ~Join() { t.join(); }
    } join{warm};
    std::ifstream in(input);
    if (!in) {
        std::fprintf(stderr, "cannot open %s\n", input.c_str());
        return 2;
    }
    std::stringstream buf;
    buf << in.rdbuf();
    cdtref::Pslg g;
    cdtref::Mesh m;
    try {
        g = cdtref::read_poly(buf.str());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "input error: %s\n", e.what());
        return 2;
    }
    if (prefix.empty()) {
        prefix = input;
        const size_t dot = prefix.rfind('.');
        if (dot != std::string::npos) prefix.resize(dot);
    }
    if (device_io) return run_device_io(g, q, cfg, device, device_cdt, prefix);
    try {
        // Line 1 on the host (as the reference), or on the GPU with --device-cdt
        m = device_cdt ? gdp2d::build_cdt(g, device) : cdtref::build_cdt(g);
    } catch (const cdtref::CdtError& e) {
        std::fprintf(stderr, "input error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s error: %s\n", device_cdt ? "engine" : "input", e.what());
        return device_cdt ? 4 : 2;
    }
    cdtref::RunReport rep;
    try {
        rep = gdp2d::refine(m, q, cfg, device);   // was: cdtref::refine(m, q, cfg)
    } catch (const std::exception& e) {
        std::fprintf(stderr, "engine error: %s\n", e.what());
        return 4;
    }
    int rc = 0;
    if (rep.iteration_cap_hit) rc = 3;
    if (rc == 0 && !cdtref::conformity_ok(m, g)) {
        std::fprintf(stderr, "post-run verification failed: not conforming to the PSLG\n");
        rc = 3;
    }
    if (rc == 0) {
        try {
            m.check_structure();
        } catch (const std::exception& e) {
            std::fprintf(stderr, "post-run verification failed: %s\n", e.what());
            rc = 3;
        }
    }
    if (prefix.empty()) {
        prefix = input;
        const size_t dot = prefix.rfind('.');
        if (dot != std::string::npos) prefix.resize(dot);
    }
    const cdtref::NodeEle ne = cdtref::write_node_ele(m);
    std::ofstream(prefix + ".node") << ne.node;
    std::ofstream(prefix + ".ele") << ne.ele;
    std::printf("batches=%zu output_points=%zu steiner_points=%zu bad_triangles=%zu "
                "min_angle_deg=%.6f wall_seconds=%.6f exit=%d\n",
                rep.batches.size(), rep.output_points, rep.steiner_points, rep.bad_triangles,
                rep.min_angle_deg, rep.wall_seconds, rc);
    return rc;
}
