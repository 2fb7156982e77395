// gdp2d_collect.cuh -- the per-element pieces of Line 3 (collect,
// refine.hpp:226-263) and Line 5 (compute_splitting_points, :267-296) shared by
// the scan kernels (k_collect.cu) and the device-resident tail loop
// (k_insert.cu): an element's verdict with the dirty-bit cache, and one
// candidate record.
#pragma once

#include "engine.h"

namespace gdp2d {

// With the dirty-bit cache (full == 0) an element whose dirty bit is clear
// keeps its cached verdict -- its corners (and, for a subsegment, both
// adjacent triangles and hence its apexes) are unchanged since the last scan --
// so it costs one byte instead of the 64 B record + corner gathers.  Only the
// sticky encroached flag is read for every subsegment.
template <int MODE>
__device__ __forceinline__ uint8_t eval_sub(const DevMesh& m, u32 i, int full, u32& dirty) {
    if (!m.salive[i]) return 0;
    const uint8_t sf = full ? 2 : m.sflag[i];
    bool enc;
    if (sf & 2) {
        enc = is_encroached<MODE>(m, i);
        m.sflag[i] = enc ? 1 : 0;
        ++dirty;
    } else {
        enc = sf & 1;
    }
    return (m.senc[i] || enc) ? 1 : 0;
}

__device__ __forceinline__ uint8_t eval_tri(const DevMesh& m, const Quality& q, u32 i) {
    uint8_t f = 0;
    const uint4 tv = m.tv[i];
    if (tv.w) {
        const double2 a = m.xy[tv.x], b = m.xy[tv.y], c = m.xy[tv.z];
        if (is_bad_pts(a, b, c, q) && resolvable_pts(a, b, c)) f = 1;
    }
    m.tflag[i] = f;
    return f;
}

// compute_splitting_points for one candidate (refine.hpp:269-294).
__device__ __forceinline__ double2 split_point(const DevMesh& m, int kind, u32 id, uint8_t& fb) {
    fb = 0;
    if (kind == 0) return subseg_mid(m, id);
    const uint4 tv = m.tv[id];
    const double2 v3[3] = {m.xy[tv.x], m.xy[tv.y], m.xy[tv.z]};
    bool ok;
    const double2 cc = circumcenter(v3[0], v3[1], v3[2], ok);
    if (ok && isfinite(cc.x) && isfinite(cc.y)) return cc;
    fb = 1;
    int best = 0;
    double best_len = -1.0;
    for (int e = 0; e < 3; ++e) {
        const double len = sqdist(v3[nxt(e)], v3[prv(e)]);
        if (len > best_len) {
            best_len = len;
            best = e;
        }
    }
    return midpoint2(v3[nxt(best)], v3[prv(best)]);
}

// One candidate record (refine.hpp:236-248 + compute_splitting_points):
// list position o, element i of kind 0 (subsegment) / 1 (triangle).
__device__ __forceinline__ u32 write_candidate(const DevMesh& m, const DevCands& c, u32 o,
                                               int kind, u32 i) {
    uint8_t fb;
    c.pt[o] = split_point(m, kind, i, fb);
    double measure;
    if (kind == 0) {
        measure = subseg_len(m, i);
    } else {
        const uint4 tv = m.tv[i];
        measure = area_pts(m.xy[tv.x], m.xy[tv.y], m.xy[tv.z]);
    }
    c.key[o] = make_key(kind == 0 ? 1 : 0, measure);
    c.id[o] = i;
    c.tie[o] = o;
    c.loc[o] = PENDING;
    c.kind[o] = (uint8_t)kind;
    c.alive[o] = 1;
    c.lkind[o] = 0;
    c.ledge[o] = -1;
    c.fb[o] = fb;
    return fb;
}

}  // namespace gdp2d
