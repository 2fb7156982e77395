// k_verify.cu -- device-side validators for refined meshes (SURVEY §8(f)
// row 2): what the reference checks on the host with verify.hpp:92-200 and
// mesh.hpp:505-557, as data-parallel passes that finish in milliseconds on
// 10M-vertex outputs (the reference's brute-force CDT check is capped at
// 1e5 vertices, cdtref.cpp:115).
//
//   structure     Mesh::check_structure (mesh.hpp:505-551): k_validate
//   local CDT     every interior non-subsegment edge passes incircle <= 0
//                 (exact) -- for a valid triangulation equivalent to the
//                 global constrained-Delaunay property
//   quality       is_bad_triangle && triangle_resolvable (refine.hpp:169-206)
//                 count + min angle + the histogram of per-triangle minimum
//                 angles (GDP2D_HIST_BINS bins of GDP2D_HIST_BIN_DEG degrees,
//                 corner formula of min_angle_degrees, verify.hpp:186-200)
//                 and their mean (fixed-point sum, so it is deterministic)
//   conformity    conformity_ok (verify.hpp:147-183): every alive subsegment
//                 is a mesh edge carrying it (structure), its parent is an
//                 input segment, its interior endpoints lie on the parent
//                 segment (|cross| <= 1e-9 |ab|^2, the reference's
//                 tolerance), and per input segment the alive children form
//                 one chain: parent endpoints have degree 1, every other
//                 child endpoint degree 2 within that parent, and the child
//                 lengths sum to the parent's length (relative 1e-9).
#include "engine.h"
#include "scan.cuh"

namespace gdp2d {

struct VerifyAcc {
    unsigned long long cdt_violations;
    unsigned long long bad;
    unsigned long long conformity_failures;
    unsigned long long min_angle_bits;   // double bits, atomicMin on non-negative values
    unsigned long long angle_sum_fx;     // sum of per-triangle min angles * 2^kAngleFx
    unsigned long long hist[GDP2D_HIST_BINS];
};

constexpr int kAngleFx = 30;

__global__ void k_verify_tris(DevMesh m, Quality q, VerifyAcc* acc) {
    __shared__ u32 hist[GDP2D_HIST_BINS];
    for (u32 i = threadIdx.x; i < GDP2D_HIST_BINS; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    ull viol = 0, bad = 0, angle_fx = 0;
    double min_ang = 180.0;
    if (t < m.nT) {
        const uint4 tv = m.tv[t];
        if (tv.w) {
            const double2 p3[3] = {m.xy[tv.x], m.xy[tv.y], m.xy[tv.z]};
            if (is_bad_pts(p3[0], p3[1], p3[2], q) && resolvable_pts(p3[0], p3[1], p3[2])) bad = 1;
            for (int i = 0; i < 3; ++i) {
                const double2 u = sub2(p3[nxt(i)], p3[i]);
                const double2 v = sub2(p3[prv(i)], p3[i]);
                min_ang = fmin(min_ang, atan2(fabs(cross2(u, v)), dot2(u, v)) * 180.0 /
                                            3.14159265358979323846);
            }
            u32 bin = (u32)(min_ang / GDP2D_HIST_BIN_DEG);
            if (bin >= GDP2D_HIST_BINS) bin = GDP2D_HIST_BINS - 1;
            atomicAdd(&hist[bin], 1u);
            angle_fx = (ull)__double2ll_rn(ldexp(min_ang, kAngleFx));
            const uint4 tn = m.tn[t];
            for (int e = 0; e < 3; ++e) {
                const u32 c = comp(tn, e);
                if (c == NONE || has_seg(tv, e)) continue;
                const u32 u = etri(c);
                if (u < t) continue;   // each interior edge once
                const u32 d = comp(m.tv[u], eidx(c));
                if (incircle(p3[0], p3[1], p3[2], m.xy[d]) > 0) ++viol;
            }
        }
    }
    block_add<ull>(&acc->cdt_violations, viol);
    block_add<ull>(&acc->bad, bad);
    block_add<ull>(&acc->angle_sum_fx, angle_fx);
    for (u32 i = threadIdx.x; i < GDP2D_HIST_BINS; i += blockDim.x)
        if (hist[i]) atomicAdd(&acc->hist[i], (ull)hist[i]);
    for (int o = 16; o > 0; o >>= 1) min_ang = fmin(min_ang, __shfl_down_sync(0xFFFFFFFFu, min_ang, o));
    if ((threadIdx.x & 31) == 0 && min_ang < 180.0)
        atomicMin(&acc->min_angle_bits, (ull)__double_as_longlong(min_ang));
}

// Input segments = the pristine mesh's alive subsegments (parent index = id).
__global__ void k_verify_segs(DevMesh m, const uint2* __restrict__ in_sv, u32 nIn,
                              u32* __restrict__ deg, double* __restrict__ len_sum,
                              VerifyAcc* acc) {
    const u32 s = blockIdx.x * blockDim.x + threadIdx.x;
    ull fail = 0;
    if (s < m.nS && m.salive[s]) {
        const u32 p = m.sparent[s];
        if (p >= nIn) {
            fail = 1;
        } else {
            const uint2 sv = m.sv[s];
            const uint2 ab = in_sv[p];
            const double2 a = m.xy[ab.x], b = m.xy[ab.y];
            const double2 d = sub2(b, a);
            const double dd = dot2(d, d);
            const u32 ends[2] = {sv.x, sv.y};
            for (int k = 0; k < 2; ++k) {
                const u32 v = ends[k];
                if (v == ab.x || v == ab.y) continue;
                const double off = fabs(cross2(d, sub2(m.xy[v], a)));
                if (off > 1e-9 * dd) fail = 1;
                atomicAdd(&deg[v], 1u);
            }
            atomicAdd(&len_sum[p], sqrt(sqdist(m.xy[sv.x], m.xy[sv.y])));
            if (sv.x == ab.x || sv.y == ab.x) atomicAdd(&deg[ab.x], 1u << 16);
            if (sv.x == ab.y || sv.y == ab.y) atomicAdd(&deg[ab.y], 1u << 16);
        }
    }
    block_add<ull>(&acc->conformity_failures, fail);
}

// Chain check: interior child endpoints have degree 2, parent endpoints
// exactly one child per incident input segment; lengths add up.
__global__ void k_verify_chain(DevMesh m, const uint2* __restrict__ in_sv, u32 nIn,
                               const u32* __restrict__ in_deg, const u32* __restrict__ deg,
                               const double* __restrict__ len_sum, VerifyAcc* acc) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    ull fail = 0;
    if (i < m.nV) {
        const u32 dg = deg[i];
        const u32 interior = dg & 0xFFFFu, endpoint = dg >> 16;
        if (interior != 0 && interior != 2) fail = 1;
        if (endpoint != in_deg[i]) fail = 1;
    }
    if (i < nIn) {
        const uint2 ab = in_sv[i];
        const double L = sqrt(sqdist(m.xy[ab.x], m.xy[ab.y]));
        if (fabs(len_sum[i] - L) > 1e-9 * L) fail = 1;
    }
    block_add<ull>(&acc->conformity_failures, fail);
}

// in_deg[v] = number of input segments ending at v
__global__ void k_input_degree(const uint2* __restrict__ in_sv, u32 nIn, u32* __restrict__ in_deg) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nIn) {
        atomicAdd(&in_deg[in_sv[i].x], 1u);
        atomicAdd(&in_deg[in_sv[i].y], 1u);
    }
}

VerifySummary launch_verify(const DevMesh& m, const Quality& q, const uint2* in_sv, u32 nIn,
                            void* scratch, size_t scratch_bytes, u32* d_val,
                            cudaStream_t st) {
    VerifySummary out{};
    // scratch: acc | deg[V] | in_deg[V] | len_sum[nIn]
    const size_t need = sizeof(VerifyAcc) + 8ull * m.nV + 8ull * nIn + 16;
    if (scratch_bytes < need) {
        out.scratch_needed = need;
        return out;
    }
    char* base = static_cast<char*>(scratch);
    VerifyAcc* acc = reinterpret_cast<VerifyAcc*>(base);
    u32* deg = reinterpret_cast<u32*>(base + sizeof(VerifyAcc));
    u32* in_deg = deg + m.nV;
    double* len_sum = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(in_deg + m.nV) + 15) & ~uintptr_t(15));
    VerifyAcc init{};
    init.min_angle_bits = (ull)0x4066800000000000ull;   // 180.0
    cudaMemcpyAsync(acc, &init, sizeof init, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(deg, 0, 8ull * m.nV, st);   // deg + in_deg
    cudaMemsetAsync(len_sum, 0, 8ull * nIn, st);
    launch_validate(m, d_val, st);
    if (m.nT) note_launch(), k_verify_tris<<<(m.nT + 255) / 256, 256, 0, st>>>(m, q, acc);
    if (nIn) note_launch(), k_input_degree<<<(nIn + 255) / 256, 256, 0, st>>>(in_sv, nIn, in_deg);
    if (m.nS) note_launch(), k_verify_segs<<<(m.nS + 255) / 256, 256, 0, st>>>(m, in_sv, nIn, deg, len_sum, acc);
    const u32 nc = m.nV > nIn ? m.nV : nIn;
    if (nc) note_launch(), k_verify_chain<<<(nc + 255) / 256, 256, 0, st>>>(m, in_sv, nIn, in_deg, deg, len_sum, acc);
    VerifyAcc h;
    u32 sv[4];
    cudaMemcpyAsync(&h, acc, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(sv, d_val, sizeof sv, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    out.structure_failure = sv[0];
    out.structure_tri = sv[1];
    out.cdt_violations = h.cdt_violations;
    out.bad_triangles = h.bad;
    out.conformity_failures = h.conformity_failures;
    double ma;
    memcpy(&ma, &h.min_angle_bits, sizeof ma);
    out.min_angle_deg = ma;
    ull n_alive = 0;
    for (int i = 0; i < GDP2D_HIST_BINS; ++i) {
        out.min_angle_hist[i] = h.hist[i];
        n_alive += h.hist[i];
    }
    out.mean_min_angle_deg = n_alive ? ldexp((double)h.angle_sum_fx, -kAngleFx) / n_alive : 0.0;
    return out;
}

// ---- compacted export (write_node_ele, pslg_io.hpp:294-319) ---------------------

__global__ void k_alive_flags(DevMesh m, u32* __restrict__ fv, u32* __restrict__ ft) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m.nV) fv[i] = m.valive[i] ? 1u : 0u;
    if (i < m.nT) ft[i] = m.tv[i].w ? 1u : 0u;
}

__global__ void k_emit_nodes(DevMesh m, const u32* __restrict__ ov, double2* __restrict__ xy,
                             uint8_t* __restrict__ marker) {
    const u32 v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= m.nV || !m.valive[v]) return;
    const u32 o = ov[v];
    xy[o] = m.xy[v];
    marker[o] = m.vkind[v] == 0 ? 1 : 0;
}

__global__ void k_emit_tris(DevMesh m, const u32* __restrict__ ov, const u32* __restrict__ ot,
                            u32* __restrict__ tri) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m.nT) return;
    const uint4 tv = m.tv[t];
    if (!tv.w) return;
    const u32 o = ot[t];
    tri[3 * (size_t)o] = ov[tv.x];
    tri[3 * (size_t)o + 1] = ov[tv.y];
    tri[3 * (size_t)o + 2] = ov[tv.z];
}

// scratch: fv[V] ov[V] ft[T] ot[T] | out xy[2V] marker[V] tri[3T] | totals
void launch_export(const DevMesh& m, u32* fv, u32* ov, u32* ft, u32* ot, double2* xy,
                   uint8_t* marker, u32* tri, u32* totals, ScanScratch& s, cudaStream_t st) {
    const u32 n = m.nV > m.nT ? m.nV : m.nT;
    if (n) note_launch(), k_alive_flags<<<(n + 255) / 256, 256, 0, st>>>(m, fv, ft);
    scan_exclusive(fv, ov, m.nV, totals + 0, s, st);
    scan_exclusive(ft, ot, m.nT, totals + 1, s, st);
    if (m.nV) note_launch(), k_emit_nodes<<<(m.nV + 255) / 256, 256, 0, st>>>(m, ov, xy, marker);
    if (m.nT) note_launch(), k_emit_tris<<<(m.nT + 255) / 256, 256, 0, st>>>(m, ov, ot, tri);
}

}  // namespace gdp2d
