// gdp2d_geom.cuh -- mesh-level device helpers (reads only).  Each mirrors the
// reference function cited beside it, on the encoded SoA layout.
#pragma once

#include "gdp2d_common.cuh"
#include "gdp2d_predicates.cuh"

namespace gdp2d {

struct Quality {
    double cos2;   // host std::cos(theta)^2 (refine.hpp:195-196)
    double ell;    // +inf = none
    int mode;      // 0 Ruppert, 1 Chew
};

__device__ __forceinline__ double2 P(const DevMesh& m, u32 v) { return m.xy[v]; }
__device__ __forceinline__ bool tri_alive(const DevMesh& m, u32 t) { return m.tv[t].w != 0; }

// is_bad_triangle (refine.hpp:192-206); c2 from the host.
__device__ __forceinline__ bool is_bad_pts(double2 a, double2 b, double2 c, const Quality& q) {
    const double2 p3[3] = {a, b, c};
    const bool ell_finite = isfinite(q.ell);
    const double ell2 = q.ell * q.ell;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double2 p = p3[i];
        const double2 u = sub2(p3[nxt(i)], p);
        const double2 v = sub2(p3[prv(i)], p);
        if (ell_finite && dot2(u, u) > ell2) return true;
        const double d = dot2(u, v);
        if (d > 0.0 && d * d > q.cos2 * dot2(u, u) * dot2(v, v)) return true;
    }
    return false;
}

// triangle_resolvable (refine.hpp:169-178)
__device__ __forceinline__ bool resolvable_pts(double2 a, double2 b, double2 c) {
    const double2 p3[3] = {a, b, c};
    double mag = 0.0, len2 = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        mag = fmax(mag, fmax(fabs(p3[i].x), fabs(p3[i].y)));
        len2 = fmax(len2, sqdist(p3[i], p3[nxt(i)]));
    }
    const double fl = mag * 1e-12;
    return len2 > fl * fl;
}

// detail::triangle_area (refine.hpp:116-119)
__device__ __forceinline__ double area_pts(double2 a, double2 b, double2 c) {
    return 0.5 * fabs(cross2(sub2(b, a), sub2(c, a)));
}

// detail::point_encroaches (refine.hpp:180-185)
template <int MODE>
__device__ __forceinline__ bool encroaches(double2 sa, double2 sb, double2 p) {
    if (MODE == 0) return in_diametric_circle(sa, sb, p);
    return in_diametral_lens(sa, sb, p);
}

// Slot of subsegment s on triangle t, or -1.
__device__ __forceinline__ int seg_slot(const uint4& ts, u32 s) {
    return ts.x == s ? 0 : (ts.y == s ? 1 : (ts.z == s ? 2 : -1));
}

// detail::subsegment_apexes (refine.hpp:126-137)
__device__ __forceinline__ void subseg_apexes(const DevMesh& m, u32 s, u32& a0, u32& a1) {
    a0 = NONE;
    a1 = NONE;
    const u32 t = m.stri[s];
    const int e = seg_slot(m.ts[t], s);
    if (e < 0) return;
    a0 = comp(m.tv[t], e);
    const u32 c = comp(m.tn[t], e);
    if (c != NONE) a1 = comp(m.tv[etri(c)], eidx(c));
}

// is_encroached without pending points (refine.hpp:210-221)
template <int MODE>
__device__ __forceinline__ bool is_encroached(const DevMesh& m, u32 s) {
    u32 a0, a1;
    subseg_apexes(m, s, a0, a1);
    const uint2 sv = m.sv[s];
    const double2 sa = P(m, sv.x), sb = P(m, sv.y);
    if (a0 != NONE && encroaches<MODE>(sa, sb, P(m, a0))) return true;
    if (a1 != NONE && encroaches<MODE>(sa, sb, P(m, a1))) return true;
    return false;
}

// detail::subsegment_split_ok (refine.hpp:143-164)
__device__ __forceinline__ bool side_ok(const DevMesh& m, u32 t, u32 s, double2 p) {
    if (t == NONE) return true;
    const int e = seg_slot(m.ts[t], s);
    if (e < 0) return true;
    const uint4 tv = m.tv[t];
    const double2 a = P(m, comp(tv, e));
    const double2 x = P(m, comp(tv, nxt(e)));
    const double2 y = P(m, comp(tv, prv(e)));
    return orient2d(x, p, a) > 0 && orient2d(p, y, a) > 0;
}

__device__ __forceinline__ bool subseg_split_ok(const DevMesh& m, u32 s, double2 p) {
    const uint2 sv = m.sv[s];
    if (peq(p, P(m, sv.x)) || peq(p, P(m, sv.y))) return false;
    const u32 t = m.stri[s];
    u32 u = NONE;
    const uint4 ts = m.ts[t];
    const uint4 tn = m.tn[t];
#pragma unroll
    for (int e = 0; e < 3; ++e)
        if (comp(ts, e) == s) u = comp(tn, e) == NONE ? NONE : etri(comp(tn, e));
    return side_ok(m, t, s, p) && side_ok(m, u, s, p);
}

__device__ __forceinline__ double2 subseg_mid(const DevMesh& m, u32 s) {
    const uint2 sv = m.sv[s];
    return midpoint2(P(m, sv.x), P(m, sv.y));
}

__device__ __forceinline__ double subseg_len(const DevMesh& m, u32 s) {
    const uint2 sv = m.sv[s];
    return sqrt(sqdist(P(m, sv.x), P(m, sv.y)));
}

// ---- point location (cdt.hpp:41-105) -------------------------------------------

struct Loc {
    int kind;    // GDP2D_LOC_*
    u32 tri;
    int edge;
    u32 seg;
    u32 steps;
};

// detail::classify_in_triangle (cdt.hpp:41-60)
__device__ __forceinline__ Loc classify(const DevMesh& m, u32 t, double2 p) {
    const uint4 tv = m.tv[t];
    const double2 v3[3] = {P(m, tv.x), P(m, tv.y), P(m, tv.z)};
    int zero_edge = -1, zero_count = 0;
    for (int e = 0; e < 3; ++e) {
        const int o = orient2d(v3[nxt(e)], v3[prv(e)], p);
        if (o < 0) return Loc{3 /*Outside*/, t, e, NONE, 0};
        if (o == 0) {
            zero_edge = e;
            ++zero_count;
        }
    }
    if (zero_count == 0) return Loc{0 /*Inside*/, t, -1, NONE, 0};
    if (zero_count == 1) return Loc{1 /*OnEdge*/, t, zero_edge, NONE, 0};
    return Loc{2 /*OnVertex*/, t, -1, NONE, 0};
}

// locate_point (cdt.hpp:68-105) with intercept_subsegments.
__device__ __forceinline__ Loc locate_point(const DevMesh& m, u32 start, double2 p,
                                            bool intercept) {
    u32 cur = start, prev = NONE;
    const ull cap = 8ull + 2ull * (ull)m.nT;
    for (ull step = 0; step < cap; ++step) {
        const uint4 tv = m.tv[cur];
        const uint4 tn = m.tn[cur];
        const double2 v3[3] = {P(m, tv.x), P(m, tv.y), P(m, tv.z)};
        int exit_edge = -1;
        for (int e = 0; e < 3; ++e) {
            const u32 c = comp(tn, e);
            const u32 nb = c == NONE ? NONE : etri(c);
            if (nb == prev && prev != NONE) continue;
            if (orient2d(v3[nxt(e)], v3[prv(e)], p) < 0) {
                exit_edge = e;
                break;
            }
        }
        if (exit_edge < 0) {
            Loc loc = classify(m, cur, p);
            loc.steps = (u32)step;
            if (loc.kind != 3) return loc;
            exit_edge = loc.edge;
        }
        if (intercept && has_seg(tv, exit_edge))
            return Loc{4 /*Intercepted*/, cur, exit_edge, comp(m.ts[cur], exit_edge), (u32)step};
        const u32 c = comp(tn, exit_edge);
        if (c == NONE) return Loc{3, cur, exit_edge, NONE, (u32)step};
        prev = cur;
        cur = etri(c);
    }
    // Exhaustive fallback (cdt.hpp:98-104).
    for (u32 t = 0; t < m.nT; ++t) {
        if (!tri_alive(m, t)) continue;
        Loc loc = classify(m, t, p);
        if (loc.kind != 3) {
            loc.steps = (u32)cap;
            return loc;
        }
    }
    return Loc{3, cur, 0, NONE, (u32)cap};
}

}  // namespace gdp2d
