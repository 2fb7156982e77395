// k_misc.cu -- adjacency encode/decode for the exchange format, predicate
// batches (parity entry points) and the final quality summary
// (fill_quality_summary, refine.hpp:614-645).
#include <cstring>

#include "engine.h"

namespace gdp2d {

// Plain TriId neighbours (mesh.hpp:52) -> (tri<<2)|edge: the far slot is the
// one whose edge has the same endpoints reversed (falls back to the first
// slot pointing back, as index_of_neighbor mesh.hpp:107 would).
__global__ void k_encode_nbrs(DevMesh m, const u32* __restrict__ plain) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m.nT) return;
    const uint4 tv = m.tv[t];
    uint4 out = make_uint4(NONE, NONE, NONE, 0u);
    for (int e = 0; e < 3; ++e) {
        const u32 u = plain[3 * t + e];
        if (u == NONE) continue;
        const u32 x = comp(tv, nxt(e)), y = comp(tv, prv(e));
        const uint4 uv = m.tv[u];
        int f = -1;
        for (int g = 0; g < 3; ++g)
            if (comp(uv, nxt(g)) == y && comp(uv, prv(g)) == x) f = g;
        if (f < 0)
            for (int g = 2; g >= 0; --g)
                if (plain[3 * u + g] == t) f = g;
        if (f < 0) f = 0;
        set_comp(out, e, enc(u, f));
    }
    m.tn[t] = out;
}

__global__ void k_decode_nbrs(DevMesh m, u32* __restrict__ plain) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m.nT) return;
    const uint4 tn = m.tn[t];
    for (int e = 0; e < 3; ++e) {
        const u32 c = comp(tn, e);
        plain[3 * t + e] = c == NONE ? NONE : etri(c);
    }
}

void launch_encode_neighbors(DevMesh m, const u32* plain_n, cudaStream_t st) {
    if (!m.nT) return;
    note_launch(), k_encode_nbrs<<<(m.nT + 255) / 256, 256, 0, st>>>(m, plain_n);
}

void launch_decode_neighbors(const DevMesh& m, u32* plain_n, cudaStream_t st) {
    if (!m.nT) return;
    note_launch(), k_decode_nbrs<<<(m.nT + 255) / 256, 256, 0, st>>>(m, plain_n);
}

// ---- predicate batches ------------------------------------------------------------

template <int KIND>
__global__ void k_predicates(const double2* __restrict__ pts, u32 n, Quality q,
                             int8_t* __restrict__ out) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (KIND == 0) {
        const double2* r = pts + 3 * (size_t)i;
        out[i] = (int8_t)orient2d(r[0], r[1], r[2]);
    } else if (KIND == 1) {
        const double2* r = pts + 4 * (size_t)i;
        out[i] = (int8_t)incircle(r[0], r[1], r[2], r[3]);
    } else if (KIND == 2) {
        const double2* r = pts + 3 * (size_t)i;
        out[i] = in_diametric_circle(r[0], r[1], r[2]);
    } else if (KIND == 3) {
        const double2* r = pts + 3 * (size_t)i;
        out[i] = in_diametral_lens(r[0], r[1], r[2]);
    } else {
        const double2* r = pts + 3 * (size_t)i;
        out[i] = is_bad_pts(r[0], r[1], r[2], q);
    }
}

void launch_predicates(int kind, const double* pts, u32 n, const Quality& q, int8_t* out,
                       cudaStream_t st) {
    if (!n) return;
    const u32 g = (n + 127) / 128;
    const double2* p = reinterpret_cast<const double2*>(pts);
    switch (kind) {
        case 0: note_launch(), k_predicates<0><<<g, 128, 0, st>>>(p, n, q, out); break;
        case 1: note_launch(), k_predicates<1><<<g, 128, 0, st>>>(p, n, q, out); break;
        case 2: note_launch(), k_predicates<2><<<g, 128, 0, st>>>(p, n, q, out); break;
        case 3: note_launch(), k_predicates<3><<<g, 128, 0, st>>>(p, n, q, out); break;
        default: note_launch(), k_predicates<4><<<g, 128, 0, st>>>(p, n, q, out); break;
    }
}

__global__ void k_circumcenters(const double2* __restrict__ pts, u32 n, double2* __restrict__ out,
                                uint8_t* __restrict__ ok) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool k;
    out[i] = circumcenter(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], k);
    ok[i] = k;
}

void launch_circumcenters(const double* pts, u32 n, double* out, uint8_t* ok, cudaStream_t st) {
    if (!n) return;
    note_launch(), k_circumcenters<<<(n + 255) / 256, 256, 0, st>>>(reinterpret_cast<const double2*>(pts), n,
                                                     reinterpret_cast<double2*>(out), ok);
}

// ---- quality summary ---------------------------------------------------------------

struct QAcc {
    double total_area, bad_area;
    ull min_angle_bits, max_edge_bits;
    ull bad, alive_v, steiner;
};

__global__ void k_quality_tris(DevMesh m, Quality q, QAcc* acc) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    double area = 0.0, bad_area = 0.0, min_ang = 180.0, max_edge = 0.0;
    ull bad = 0;
    if (t < m.nT) {
        const uint4 tv = m.tv[t];
        if (tv.w) {
            const double2 p3[3] = {m.xy[tv.x], m.xy[tv.y], m.xy[tv.z]};
            area = area_pts(p3[0], p3[1], p3[2]);
            if (is_bad_pts(p3[0], p3[1], p3[2], q)) {
                bad = 1;
                bad_area = area;
            }
            for (int i = 0; i < 3; ++i) {
                const double2 u = sub2(p3[nxt(i)], p3[i]);
                const double2 v = sub2(p3[prv(i)], p3[i]);
                min_ang = fmin(min_ang, atan2(fabs(cross2(u, v)), dot2(u, v)) * 180.0 /
                                            3.14159265358979323846);
                max_edge = fmax(max_edge, sqrt(dot2(u, u)));
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        area += __shfl_down_sync(0xFFFFFFFFu, area, o);
        bad_area += __shfl_down_sync(0xFFFFFFFFu, bad_area, o);
        min_ang = fmin(min_ang, __shfl_down_sync(0xFFFFFFFFu, min_ang, o));
        max_edge = fmax(max_edge, __shfl_down_sync(0xFFFFFFFFu, max_edge, o));
        bad += __shfl_down_sync(0xFFFFFFFFu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&acc->total_area, area);
        if (bad_area != 0.0) atomicAdd(&acc->bad_area, bad_area);
        atomicMin(&acc->min_angle_bits, (ull)__double_as_longlong(min_ang));
        atomicMax(&acc->max_edge_bits, (ull)__double_as_longlong(max_edge));
        if (bad) atomicAdd(&acc->bad, bad);
    }
}

__global__ void k_quality_verts(DevMesh m, QAcc* acc) {
    const u32 v = blockIdx.x * blockDim.x + threadIdx.x;
    u32 alive = 0, steiner = 0;
    if (v < m.nV && m.valive[v]) {
        alive = 1;
        steiner = m.vkind[v] != 0;
    }
    alive = __reduce_add_sync(0xFFFFFFFFu, alive);
    steiner = __reduce_add_sync(0xFFFFFFFFu, steiner);
    if ((threadIdx.x & 31) == 0) {
        if (alive) atomicAdd(&acc->alive_v, (ull)alive);
        if (steiner) atomicAdd(&acc->steiner, (ull)steiner);
    }
}

static double bits_to_double(ull b) {
    double d;
    memcpy(&d, &b, sizeof d);
    return d;
}

QualitySummary launch_quality(const DevMesh& m, const Quality& q, void* scratch,
                              cudaStream_t st) {
    QAcc h{};
    h.min_angle_bits = (ull)0x4066800000000000ull;  // 180.0
    h.max_edge_bits = 0;
    QAcc* d = reinterpret_cast<QAcc*>(scratch);
    cudaMemcpyAsync(d, &h, sizeof h, cudaMemcpyHostToDevice, st);
    if (m.nT) note_launch(), k_quality_tris<<<(m.nT + 255) / 256, 256, 0, st>>>(m, q, d);
    if (m.nV) note_launch(), k_quality_verts<<<(m.nV + 255) / 256, 256, 0, st>>>(m, d);
    cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    QualitySummary s;
    s.total_area = h.total_area;
    s.bad_area = h.bad_area;
    s.min_angle = bits_to_double(h.min_angle_bits);
    s.max_edge = bits_to_double(h.max_edge_bits);
    s.bad = h.bad;
    s.alive_v = h.alive_v;
    s.steiner = h.steiner;
    return s;
}

}  // namespace gdp2d

namespace gdp2d {

// Debug validator (GDP2D_CHECK=1, gdp2d_ctx_validate): the structural checks of
// Mesh::check_structure (mesh.hpp:505-551) on the device.  out[0] = first
// failure code, out[1] = triangle, out[2] = edge.
__global__ void k_validate(DevMesh m, u32* out) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m.nT) return;
    const uint4 tv = m.tv[t];
    if (!tv.w) return;
    auto fail = [&](u32 code, int e) {
        if (atomicCAS(&out[0], 0u, code) == 0u) {
            out[1] = t;
            out[2] = (u32)e;
        }
    };
    if (tv.x >= m.nV || tv.y >= m.nV || tv.z >= m.nV) return fail(1, -1);
    if (orient2d(m.xy[tv.x], m.xy[tv.y], m.xy[tv.z]) <= 0) return fail(2, -1);
    const uint4 tn = m.tn[t], ts = load_ts(m, t, tv);
    if (tn.w) return fail(3, -1);
    for (int e = 0; e < 3; ++e)   // the subsegment bits of tv.w match the ts record
        if (has_seg(tv, e) != (comp(ts, e) != NONE)) return fail(14, e);
    for (int e = 0; e < 3; ++e) {
        const u32 c = comp(tn, e);
        if (c == NONE) continue;
        const u32 u = etri(c);
        const int f = eidx(c);
        if (u >= m.nT || f > 2) return fail(4, e);
        const uint4 uv = m.tv[u];
        if (!uv.w) return fail(5, e);
        if (comp(m.tn[u], f) != enc(t, e)) return fail(6, e);
        if (comp(uv, nxt(f)) != comp(tv, prv(e)) || comp(uv, prv(f)) != comp(tv, nxt(e)))
            return fail(7, e);
        if (comp(load_ts(m, u, uv), f) != comp(ts, e)) return fail(8, e);
    }
    for (int e = 0; e < 3; ++e) {
        const u32 s = comp(ts, e);
        if (s == NONE) continue;
        if (s >= m.nS || !m.salive[s]) return fail(9, e);
        const uint2 sv = m.sv[s];
        const u32 x = comp(tv, nxt(e)), y = comp(tv, prv(e));
        if (!((sv.x == x && sv.y == y) || (sv.x == y && sv.y == x))) return fail(10, e);
        const u32 st = m.stri[s];
        if (st == NONE || st >= m.nT || seg_slot(load_ts(m, st, m.tv[st]), s) < 0)
            return fail(11, e);
    }
    for (int i = 0; i < 3; ++i) {
        const u32 v = comp(tv, i);
        const u32 vt = m.vtri[v];
        if (vt == NONE || vt >= m.nT || !m.tv[vt].w) return fail(12, i);
        const uint4 w = m.tv[vt];
        if (w.x != v && w.y != v && w.z != v) return fail(13, i);
    }
}

void launch_validate(const DevMesh& m, u32* out, cudaStream_t st) {
    cudaMemsetAsync(out, 0, 4 * sizeof(u32), st);
    if (m.nT) note_launch(), k_validate<<<(m.nT + 255) / 256, 256, 0, st>>>(m, out);
}

// vert_tri rebuilt from scratch: the lowest alive incident triangle id of every
// vertex (Mesh::vert_tri, mesh.hpp:73; refinement batches maintain it only for
// their fresh vertices, WorkLists::vtri_from).
__global__ void k_vtri_min(DevMesh m) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m.nT) return;
    const uint4 tv = m.tv[t];
    if (!tv.w) return;
    atomicMin(&m.vtri[tv.x], t);
    atomicMin(&m.vtri[tv.y], t);
    atomicMin(&m.vtri[tv.z], t);
}

void launch_vtri_rebuild(const DevMesh& m, cudaStream_t st) {
    if (m.nV) cudaMemsetAsync(m.vtri, 0xFF, 4ull * m.nV, st);
    if (m.nT) note_launch(), k_vtri_min<<<(m.nT + 255) / 256, 256, 0, st>>>(m);
}

}  // namespace gdp2d
