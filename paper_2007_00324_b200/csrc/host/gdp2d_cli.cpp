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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "cdtref/cdt.hpp"
#include "cdtref/pslg_io.hpp"
#include "cdtref/refine.hpp"
#include "cdtref/verify.hpp"
#include "gdp2d_cdtref.hpp"

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s input.poly [--theta DEG] [--ell L] [--chew] "
                             "[--out PREFIX] [--device D] [--device-cdt]\n", argv[0]);
        return 2;
    }
    std::string input = argv[1], prefix;
    cdtref::QualityCriteria q;
    cdtref::EngineConfig cfg;
    int device = 0;
    bool device_cdt = false;   // --device-cdt: Line 1 on the GPU too (gdp2d::build_cdt)
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> const char* { return i + 1 < argc ? argv[++i] : "0"; };
        if (a == "--theta") q.theta = std::atof(val());
        else if (a == "--ell") q.ell = std::atof(val());
        else if (a == "--chew") q.mode = cdtref::RefineMode::Chew;
        else if (a == "--out") prefix = val();
        else if (a == "--device") device = std::atoi(val());
        else if (a == "--device-cdt") device_cdt = true;
        else {
            std::fprintf(stderr, "unknown flag %s\n", a.c_str());
            return 2;
        }
    }
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
