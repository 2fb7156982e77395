// pslg_gen.cpp -- the synthetic PSLG generator of SURVEY §8(d), shared by the
// GPU runs, the CPU reference runs and the tests (host code, no reference
// headers needed).
//
//  * points: the 4 pinned corners of the unit square plus N-4 distinct points
//    in the open square; uniform U(0,1)^2, or 64 Gaussian clusters (centres
//    U(0.1,0.9)^2, sigma 0.03, rejection outside the square); mt19937_64.
//  * points are sorted by a 16-bit-per-axis Morton key (stable), so the
//    reference's incremental build_delaunay walk stays O(1) per point.
//  * segments: M vertex-disjoint segments, each joining a random unused
//    interior point to one of its 8 nearest unused interior neighbours; a
//    candidate is rejected if it crosses or touches another segment or comes
//    within delta = 0.1/sqrt(N) of any other input point or segment.
//  The hull (the square) is closed afterwards by cdtref::close_hull.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <random>
#include <unordered_set>
#include <vector>

namespace {

struct P2 {
    double x, y;
};

inline uint32_t spread16(uint32_t v) {
    v &= 0xFFFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}

inline uint32_t morton(const P2& p) {
    const auto q = [](double c) {
        const double s = std::floor(std::clamp(c, 0.0, 1.0) * 65535.0);
        return static_cast<uint32_t>(s);
    };
    return spread16(q(p.x)) | (spread16(q(p.y)) << 1);
}

inline double cross(P2 a, P2 b, P2 c) { return (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x); }

inline double dist_point_seg(P2 p, P2 a, P2 b) {
    const double abx = b.x - a.x, aby = b.y - a.y;
    const double l2 = abx * abx + aby * aby;
    double t = l2 > 0 ? ((p.x - a.x) * abx + (p.y - a.y) * aby) / l2 : 0.0;
    t = std::clamp(t, 0.0, 1.0);
    const double dx = a.x + t * abx - p.x, dy = a.y + t * aby - p.y;
    return std::sqrt(dx * dx + dy * dy);
}

inline bool segs_intersect(P2 a, P2 b, P2 c, P2 d) {
    const double d1 = cross(a, b, c), d2 = cross(a, b, d), d3 = cross(c, d, a), d4 = cross(c, d, b);
    if (((d1 > 0 && d2 < 0) || (d1 < 0 && d2 > 0)) && ((d3 > 0 && d4 < 0) || (d3 < 0 && d4 > 0)))
        return true;
    return false;  // touching cases are excluded by the clearance test
}

struct Grid {
    int side;
    std::vector<std::vector<uint32_t>> pts, segs;
    explicit Grid(int s) : side(s), pts((size_t)s * s), segs((size_t)s * s) {}
    int cell(double c) const { return std::min(side - 1, std::max(0, (int)(c * side))); }
};

}  // namespace

extern "C" {

// Generates the PSLG (without the hull segments).  Returns 0 on success.
// *xy (2n doubles) and *segs (2*(*m_out) u32) are malloc'd; free with
// gdp2d_host_free.  dist: 0 uniform, 1 gaussian.
int gdp2d_host_generate(uint64_t n, uint32_t m_req, int dist, uint64_t seed, double** xy,
                        uint32_t** segs, uint32_t* m_out) {
    if (n < 4 || !xy || !segs || !m_out) return 1;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    std::vector<P2> pts;
    pts.reserve(n);
    pts.push_back({0, 0});
    pts.push_back({1, 0});
    pts.push_back({1, 1});
    pts.push_back({0, 1});
    struct H {
        size_t operator()(const std::pair<uint64_t, uint64_t>& k) const {
            return std::hash<uint64_t>()(k.first * 0x9E3779B97F4A7C15ull ^ k.second);
        }
    };
    std::unordered_set<std::pair<uint64_t, uint64_t>, H> seen;
    seen.reserve(n * 2);
    auto key = [](const P2& p) {
        uint64_t a, b;
        std::memcpy(&a, &p.x, 8);
        std::memcpy(&b, &p.y, 8);
        return std::make_pair(a, b);
    };
    for (const P2& p : pts) seen.insert(key(p));
    std::vector<P2> centres;
    if (dist == 1) {
        std::uniform_real_distribution<double> cu(0.1, 0.9);
        for (int i = 0; i < 64; ++i) centres.push_back({cu(rng), cu(rng)});
    }
    std::normal_distribution<double> gauss(0.0, 0.03);
    std::uniform_int_distribution<int> pick(0, 63);
    while (pts.size() < n) {
        P2 p;
        if (dist == 1) {
            const P2 c = centres[pick(rng)];
            p = {c.x + gauss(rng), c.y + gauss(rng)};
        } else {
            p = {uni(rng), uni(rng)};
        }
        if (!(p.x > 0.0 && p.x < 1.0 && p.y > 0.0 && p.y < 1.0)) continue;
        if (!seen.insert(key(p)).second) continue;
        pts.push_back(p);
    }
    // Morton order (stable: generation order breaks key ties).
    std::vector<uint32_t> order(n);
    for (uint32_t i = 0; i < n; ++i) order[i] = i;
    std::vector<uint32_t> mk(n);
    for (uint32_t i = 0; i < n; ++i) mk[i] = morton(pts[i]);
    std::stable_sort(order.begin(), order.end(),
                     [&](uint32_t a, uint32_t b) { return mk[a] < mk[b]; });
    std::vector<P2> sorted(n);
    for (uint32_t i = 0; i < n; ++i) sorted[i] = pts[order[i]];
    pts.swap(sorted);

    // Segments.
    const double delta = 0.1 / std::sqrt((double)n);
    const int side = std::max(1, (int)std::sqrt((double)n / 2.0));
    Grid g(side);
    std::vector<uint8_t> corner(n, 0), used(n, 0);
    for (uint32_t i = 0; i < n; ++i) {
        const P2& p = pts[i];
        if ((p.x == 0 || p.x == 1) && (p.y == 0 || p.y == 1)) corner[i] = 1;
        g.pts[(size_t)g.cell(p.y) * side + g.cell(p.x)].push_back(i);
    }
    std::vector<std::pair<uint32_t, uint32_t>> out;
    out.reserve(m_req);
    std::uniform_int_distribution<uint64_t> any(0, n - 1);
    std::uniform_int_distribution<int> k8(0, 7);
    const uint64_t max_attempts = 40ull * m_req + 1000;
    std::vector<std::pair<double, uint32_t>> nn;
    for (uint64_t att = 0; att < max_attempts && out.size() < m_req; ++att) {
        const uint32_t a = (uint32_t)any(rng);
        if (corner[a] || used[a]) continue;
        const P2 pa = pts[a];
        // 8 nearest unused interior neighbours (ring search on the grid).
        nn.clear();
        const int cx = g.cell(pa.x), cy = g.cell(pa.y);
        for (int r = 1; r <= side && nn.size() < 64; ++r) {
            nn.clear();
            for (int yy = std::max(0, cy - r); yy <= std::min(side - 1, cy + r); ++yy)
                for (int xx = std::max(0, cx - r); xx <= std::min(side - 1, cx + r); ++xx)
                    for (uint32_t q : g.pts[(size_t)yy * side + xx]) {
                        if (q == a || corner[q] || used[q]) continue;
                        const double dx = pts[q].x - pa.x, dy = pts[q].y - pa.y;
                        nn.push_back({dx * dx + dy * dy, q});
                    }
            if (nn.size() >= 8) {
                // the ring radius must cover the 8th distance
                std::partial_sort(nn.begin(), nn.begin() + 8, nn.end());
                const double reach = (double)r / side;
                if (nn[7].first <= reach * reach) break;
            }
        }
        if (nn.empty()) continue;
        const size_t kk = std::min<size_t>(8, nn.size());
        std::partial_sort(nn.begin(), nn.begin() + kk, nn.end());
        const uint32_t b = nn[(size_t)k8(rng) % kk].second;
        const P2 pb = pts[b];
        // clearance + crossing tests against nearby points and segments
        const double x0 = std::min(pa.x, pb.x) - delta, x1 = std::max(pa.x, pb.x) + delta;
        const double y0 = std::min(pa.y, pb.y) - delta, y1 = std::max(pa.y, pb.y) + delta;
        const int gx0 = g.cell(x0), gx1 = g.cell(x1), gy0 = g.cell(y0), gy1 = g.cell(y1);
        bool ok = true;
        for (int yy = gy0; yy <= gy1 && ok; ++yy)
            for (int xx = gx0; xx <= gx1 && ok; ++xx) {
                for (uint32_t q : g.pts[(size_t)yy * side + xx]) {
                    if (q == a || q == b) continue;
                    if (dist_point_seg(pts[q], pa, pb) <= delta) {
                        ok = false;
                        break;
                    }
                }
                if (!ok) break;
                for (uint32_t si : g.segs[(size_t)yy * side + xx]) {
                    const P2 c = pts[out[si].first], d = pts[out[si].second];
                    if (segs_intersect(pa, pb, c, d) || dist_point_seg(pa, c, d) <= delta ||
                        dist_point_seg(pb, c, d) <= delta) {
                        ok = false;
                        break;
                    }
                }
            }
        if (!ok) continue;
        const uint32_t si = (uint32_t)out.size();
        out.push_back({a, b});
        used[a] = used[b] = 1;
        const double sx0 = std::min(pa.x, pb.x) - delta, sx1 = std::max(pa.x, pb.x) + delta;
        const double sy0 = std::min(pa.y, pb.y) - delta, sy1 = std::max(pa.y, pb.y) + delta;
        for (int yy = g.cell(sy0); yy <= g.cell(sy1); ++yy)
            for (int xx = g.cell(sx0); xx <= g.cell(sx1); ++xx)
                g.segs[(size_t)yy * side + xx].push_back(si);
    }
    *xy = static_cast<double*>(std::malloc(sizeof(double) * 2 * n));
    for (uint64_t i = 0; i < n; ++i) {
        (*xy)[2 * i] = pts[i].x;
        (*xy)[2 * i + 1] = pts[i].y;
    }
    *segs = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * 2 * (out.size() + 1)));
    for (size_t i = 0; i < out.size(); ++i) {
        (*segs)[2 * i] = out[i].first;
        (*segs)[2 * i + 1] = out[i].second;
    }
    *m_out = (uint32_t)out.size();
    return 0;
}

void gdp2d_host_free(void* p) { std::free(p); }

}  // extern "C"
