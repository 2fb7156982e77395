// engine.cu -- the device-resident refinement loop (refine, refine.hpp:651-713)
// and the C ABI of include/gdp2d.h.
//
// One context = one device + one stream.  The working mesh lives in HBM with
// headroom; the host only reads a handful of counters per batch / round to
// size the next launch (and to grow buffers between batches).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <mutex>
#include <string>
#include <vector>
#include <thread>

#include <sys/mman.h>

#include "engine.h"
#include "gdp2d.h"
#include "scan.cuh"

using namespace gdp2d;

unsigned long long& gdp2d::launch_counter() {
    static unsigned long long n = 0;
    return n;
}

namespace {

thread_local std::string g_err;

struct CudaError {
    std::string what;
};

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess)                                                       \
            throw CudaError{std::string(#x) + ": " + cudaGetErrorString(e_)};        \
    } while (0)

struct Fail {
    int code;
    std::string what;
};

template <class T>
void dalloc(T*& p, size_t n) {
    p = nullptr;
    if (n == 0) n = 1;
    CK(cudaMalloc(&p, sizeof(T) * n));
}
template <class T>
void dfree(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

// Grow a device array to n elements, preserving the first keep elements.
template <class T>
void dgrow(T*& p, size_t keep, size_t n, cudaStream_t st) {
    T* q = nullptr;
    dalloc(q, n);
    if (p && keep) CK(cudaMemcpyAsync(q, p, sizeof(T) * keep, cudaMemcpyDeviceToDevice, st));
    if (p) {
        CK(cudaStreamSynchronize(st));
        cudaFree(p);
    }
    p = q;
}

struct MeshStore {
    DevMesh m{};
    u32 vcap = 0, tcap = 0, scap = 0;
};

void mesh_free(MeshStore& s) {
    DevMesh& m = s.m;
    dfree(m.xy); dfree(m.vkind); dfree(m.vbirth); dfree(m.valive); dfree(m.vtri);
    dfree(m.tr); dfree(m.ts);
    bind_tris(m);
    dfree(m.sv); dfree(m.sparent); dfree(m.senc); dfree(m.salive); dfree(m.stri); dfree(m.sdepth);
    dfree(m.tflag); dfree(m.sflag);
    s.vcap = s.tcap = s.scap = 0;
}

void mesh_reserve(MeshStore& s, u32 V, u32 T, u32 S, cudaStream_t st) {
    DevMesh& m = s.m;
    if (V > s.vcap) {
        dgrow(m.xy, m.nV, V, st);
        dgrow(m.vkind, m.nV, V, st);
        dgrow(m.vbirth, m.nV, V, st);
        dgrow(m.valive, m.nV, V, st);
        dgrow(m.vtri, m.nV, V, st);
        s.vcap = V;
    }
    if (T > s.tcap) {
        dgrow(m.tr, m.nT, T, st);
        bind_tris(m);
        dgrow(m.ts, m.nT, T, st);
        dgrow(m.tflag, m.nT, T, st);
        s.tcap = T;
    }
    if (S > s.scap) {
        dgrow(m.sv, m.nS, S, st);
        dgrow(m.sparent, m.nS, S, st);
        dgrow(m.senc, m.nS, S, st);
        dgrow(m.salive, m.nS, S, st);
        dgrow(m.stri, m.nS, S, st);
        dgrow(m.sdepth, m.nS, S, st);
        dgrow(m.sflag, m.nS, S, st);
        s.scap = S;
    }
}

void mesh_copy(MeshStore& dst, const MeshStore& src, cudaStream_t st) {
    const DevMesh& a = src.m;
    DevMesh& b = dst.m;
    mesh_reserve(dst, a.nV, a.nT, a.nS, st);
    auto cp = [&](void* d, const void* s, size_t bytes) {
        if (bytes) CK(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, st));
    };
    cp(b.xy, a.xy, sizeof(double2) * a.nV);
    cp(b.vkind, a.vkind, a.nV);
    cp(b.vbirth, a.vbirth, 4ull * a.nV);
    cp(b.valive, a.valive, a.nV);
    cp(b.vtri, a.vtri, 4ull * a.nV);
    cp(b.tr, a.tr, sizeof(TriRec) * a.nT);
    cp(b.ts, a.ts, sizeof(uint4) * a.nT);
    cp(b.sv, a.sv, sizeof(uint2) * a.nS);
    cp(b.sparent, a.sparent, 4ull * a.nS);
    cp(b.senc, a.senc, 4ull * a.nS);
    cp(b.salive, a.salive, a.nS);
    cp(b.stri, a.stri, 4ull * a.nS);
    cp(b.sdepth, a.sdepth, 4ull * a.nS);
    b.nV = a.nV;
    b.nT = a.nT;
    b.nS = a.nS;
}

__global__ void k_pack_tris(DevMesh m, const u32* __restrict__ tv3, const u32* __restrict__ ts3,
                            const uint8_t* __restrict__ alive) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m.nT) return;
    m.tv[t] = make_uint4(tv3[3 * t], tv3[3 * t + 1], tv3[3 * t + 2],
                         alive[t] ? tri_flags(ts3[3 * t], ts3[3 * t + 1], ts3[3 * t + 2]) : 0u);
    m.ts[t] = make_uint4(ts3[3 * t], ts3[3 * t + 1], ts3[3 * t + 2], 0u);
}

__global__ void k_unpack_tris(DevMesh m, u32* __restrict__ tv3, u32* __restrict__ ts3,
                              uint8_t* __restrict__ alive) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m.nT) return;
    const uint4 tv = m.tv[t], ts = load_ts(m, t, tv);
    tv3[3 * t] = tv.x;
    tv3[3 * t + 1] = tv.y;
    tv3[3 * t + 2] = tv.z;
    alive[t] = tv.w ? 1 : 0;
    ts3[3 * t] = ts.x;
    ts3[3 * t + 1] = ts.y;
    ts3[3 * t + 2] = ts.z;
}

__global__ void k_u8_to_u32(const uint8_t* __restrict__ a, u32* __restrict__ b, u32 n) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}
__global__ void k_u32_to_u8(const u32* __restrict__ a, uint8_t* __restrict__ b, u32 n) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i] ? 1 : 0;
}

// ---- AoS records (gdp2d_refine_aos): the caller's element vectors as bytes ----
// Field offsets come from gdp2d_aos_layout (checked on the host: natural
// alignment, inside the record).
template <class T>
__device__ __forceinline__ T& fld(uint8_t* rec, u32 off) {
    return *reinterpret_cast<T*>(rec + off);
}
template <class T>
__device__ __forceinline__ T fldc(const uint8_t* rec, u32 off) {
    return *reinterpret_cast<const T*>(rec + off);
}

__global__ void k_aos_verts_in(const uint8_t* __restrict__ in, const __grid_constant__ gdp2d_aos_layout L,
                               DevMesh m, u32 V) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    const uint8_t* r = in + (size_t)i * L.vert_size;
    m.xy[i] = make_double2(fldc<double>(r, L.vert_pos), fldc<double>(r, L.vert_pos + 8));
    m.vkind[i] = r[L.vert_kind];
    m.vbirth[i] = fldc<u32>(r, L.vert_birth);
    m.valive[i] = r[L.vert_alive] ? 1 : 0;
}

__global__ void k_aos_tris_in(const uint8_t* __restrict__ in, const __grid_constant__ gdp2d_aos_layout L,
                              u32* __restrict__ tv3, u32* __restrict__ ts3, u32* __restrict__ tn3,
                              uint8_t* __restrict__ alive, u32 T) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    const uint8_t* r = in + (size_t)t * L.tri_size;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        tv3[3 * t + k] = fldc<u32>(r, L.tri_v + 4 * k);
        tn3[3 * t + k] = fldc<u32>(r, L.tri_nbr + 4 * k);
        ts3[3 * t + k] = fldc<u32>(r, L.tri_seg + 4 * k);
    }
    alive[t] = r[L.tri_alive] ? 1 : 0;
}

__global__ void k_aos_segs_in(const uint8_t* __restrict__ in, const __grid_constant__ gdp2d_aos_layout L,
                              DevMesh m, u32 S) {
    const u32 s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const uint8_t* r = in + (size_t)s * L.seg_size;
    m.sv[s] = make_uint2(fldc<u32>(r, L.seg_v), fldc<u32>(r, L.seg_v + 4));
    m.sparent[s] = fldc<u32>(r, L.seg_parent);
    m.senc[s] = r[L.seg_encroached] ? 1u : 0u;
    m.salive[s] = r[L.seg_alive] ? 1 : 0;
    m.sdepth[s] = 0;
}

__global__ void k_aos_verts_out(DevMesh m, const __grid_constant__ gdp2d_aos_layout L,
                                uint8_t* __restrict__ out, u32 V) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    uint8_t* r = out + (size_t)i * L.vert_size;
    const double2 p = m.xy[i];
    fld<double>(r, L.vert_pos) = p.x;
    fld<double>(r, L.vert_pos + 8) = p.y;
    r[L.vert_kind] = m.vkind[i];
    fld<u32>(r, L.vert_birth) = m.vbirth[i];
    r[L.vert_alive] = m.valive[i] ? 1 : 0;
}

__global__ void k_aos_tris_out(const u32* __restrict__ tv3, const u32* __restrict__ ts3,
                               const u32* __restrict__ tn3, const uint8_t* __restrict__ alive,
                               const __grid_constant__ gdp2d_aos_layout L, uint8_t* __restrict__ out,
                               u32 T) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    uint8_t* r = out + (size_t)t * L.tri_size;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        fld<u32>(r, L.tri_v + 4 * k) = tv3[3 * t + k];
        fld<u32>(r, L.tri_nbr + 4 * k) = tn3[3 * t + k];
        fld<u32>(r, L.tri_seg + 4 * k) = ts3[3 * t + k];
    }
    r[L.tri_alive] = alive[t];
}

__global__ void k_aos_segs_out(DevMesh m, const __grid_constant__ gdp2d_aos_layout L,
                               uint8_t* __restrict__ out, u32 S) {
    const u32 s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    uint8_t* r = out + (size_t)s * L.seg_size;
    const uint2 sv = m.sv[s];
    fld<u32>(r, L.seg_v) = sv.x;
    fld<u32>(r, L.seg_v + 4) = sv.y;
    fld<u32>(r, L.seg_parent) = m.sparent[s];
    r[L.seg_encroached] = m.senc[s] ? 1 : 0;
    r[L.seg_alive] = m.salive[s] ? 1 : 0;
}

__global__ void k_fill_u64(u64* p, u64 v, size_t n) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

u32 grid(size_t n, u32 b = 256) { return (u32)((n + b - 1) / b); }

__global__ void k_count_alive(DevMesh m, ull* cnt) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    const ull v = i < m.nV && m.valive[i];
    const ull t = i < m.nT && m.tv[i].w;
    const ull s = i < m.nS && m.salive[i];
    block_add<ull>(&cnt[0], v);
    block_add<ull>(&cnt[1], t);
    block_add<ull>(&cnt[2], s);
}

Quality make_quality(const gdp2d_params* p) {
    Quality q;
    q.cos2 = p->cos2_theta;
    q.ell = p->ell;
    q.mode = p->mode == GDP2D_CHEW ? 1 : 0;
    return q;
}

const char* dev_err_name(u32 c) {
    switch (c) {
        case DERR_NONCONVEX_FLIP: return "non-convex flip of a non-Delaunay edge";
        case DERR_STAR_TOO_LARGE: return "vertex star exceeds MAX_STAR";
        case DERR_NO_EAR: return "no removable ear in a vertex star";
        case DERR_WORKLIST_OVERFLOW: return "device work list overflow";
        case DERR_OPEN_STAR: return "open star around a free vertex";
        case DERR_STALE: return "stale handle";
        case DERR_WALK: return "walk failure";
        case DERR_DUPLICATE: return "duplicate point";
        case DERR_SEG_CROSS: return "input segments cross";
        case DERR_CDT: return "CDT construction did not converge";
        case DERR_NONFINITE: return "non-finite coordinate";
        case DERR_SEG_VERTEX: return "degenerate pipe vertex";
        default: return "unknown device error";
    }
}

}  // namespace

// GDP2D_TRACE=1: CUDA events between the launches of every batch plus the
// device step trace of the persistent insertion kernel, printed to stderr.
struct Tracer {
    bool on = false;
    cudaEvent_t ev[48] = {};
    const char* name[48] = {};
    int n = 0;
    unsigned long long* d_trace = nullptr;
    u32* d_trace_val = nullptr;
    u32* d_trace_n = nullptr;
    bool rounds = false;   // GDP2D_TRACE=2: also print every Lawson round
    static constexpr u32 kCap = 1u << 16;
    void init() {
        for (auto& e : ev) cudaEventCreate(&e);
        cudaMalloc(&d_trace, sizeof(unsigned long long) * kCap);
        cudaMalloc(&d_trace_val, sizeof(u32) * kCap);
        cudaMalloc(&d_trace_n, sizeof(u32));
    }
    void release() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (d_trace) cudaFree(d_trace);
        if (d_trace_val) cudaFree(d_trace_val);
        if (d_trace_n) cudaFree(d_trace_n);
    }
    void mark(const char* what, cudaStream_t st) {
        if (!on || n >= 48) return;
        name[n] = what;
        cudaEventRecord(ev[n++], st);
    }
    void flush(u32 batch, cudaStream_t st) {
        if (!on) return;
        cudaStreamSynchronize(st);
        fprintf(stderr, "[trace] batch %u host:", batch);
        for (int i = 1; i < n; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, " %s=%.1f", name[i], ms * 1e3f);
        }
        fprintf(stderr, " (us)\n");
        n = 0;
        u32 cnt = 0;
        cudaMemcpy(&cnt, d_trace_n, sizeof cnt, cudaMemcpyDeviceToHost);
        cnt = std::min(cnt, kCap);
        if (cnt > 1) {
            std::vector<unsigned long long> t(cnt);
            std::vector<u32> val(cnt);
            cudaMemcpy(t.data(), d_trace, sizeof(unsigned long long) * cnt, cudaMemcpyDeviceToHost);
            cudaMemcpy(val.data(), d_trace_val, sizeof(u32) * cnt, cudaMemcpyDeviceToHost);
            static const char* tags[] = {"?", "start", "apply", "fixup", "ftest", "fapply", "fpost",
                                         "detA", "detB", "detC", "rmclaim", "rmapply", "rmpost",
                                         "blkin", "blkout", "end", "locate", "claim", "cavity",
                                         "plan", "splitend", "rbstart"};
            constexpr u32 NT = sizeof(tags) / sizeof(tags[0]);
            double sum[NT] = {0};
            int cntt[NT] = {0};
            for (u32 i = 1; i < cnt; ++i) {
                const u32 tag = (u32)(t[i] & 0xFF);
                const double dt = double((t[i] >> 8) - (t[i - 1] >> 8)) * 1e-3;
                if (tag < NT) {
                    sum[tag] += dt;
                    cntt[tag]++;
                }
            }
            fprintf(stderr, "[trace] batch %u device:", batch);
            for (u32 k = 2; k < NT; ++k)
                if (cntt[k]) fprintf(stderr, " %s=%.1f/%d", tags[k], sum[k], cntt[k]);
            fprintf(stderr, " total=%.1f (us/steps)\n",
                    double((t[cnt - 1] >> 8) - (t[0] >> 8)) * 1e-3);
            if (rounds) {
                fprintf(stderr, "[trace] batch %u steps:", batch);
                for (u32 i = 1; i < cnt; ++i) {
                    const u32 tag = (u32)(t[i] & 0xFF);
                    const double dt = double((t[i] >> 8) - (t[i - 1] >> 8)) * 1e-3;
                    fprintf(stderr, " %s:%u:%.1f", tag < NT ? tags[tag] : "?", val[i], dt);
                }
                fprintf(stderr, "\n");
            }
        }
    }
};

constexpr size_t kStatusWords = 20 + (sizeof(Counters) + 3) / 4;
static_assert(sizeof(Counters) % 8 == 0, "Counters follows word 20 (8-byte aligned)");

// Little's-law batch sizing (PAPER.md:94 and Rules 1-2, :104-137; the
// throughput of ruleskit.hpp:55-58 little_throughput as record_batch
// :128-142 measures it per batch; the cap policy of refine.hpp:252-261).
// Every finished batch is one measurement: attempted A, concurrency U (the
// retained insertions -- the useful work) and latency L (its device time),
// throughput T = U / L.  The size of the next batch follows from them:
//   * low workload -- C at most the measured occupancy of the filter kernels
//     (`resident` candidates in flight, cudaOccupancy*): never capped (Rule 1);
//   * high workload: A* = the attempted size of the best measured throughput.
//     If a batch that attempted MORE than A* achieved LESS throughput, the
//     measurements say oversubscription costs more than it yields (Rule 2):
//     a larger batch is cut to A* (highest priorities kept, as the reference's
//     batch_size_cap).  Without that evidence the batch runs whole.
struct LittleSizer {
    struct Rec {
        double a, u, l;
    };
    std::vector<Rec> h;
    u64 resident = 0;
    void reset() { h.clear(); }
    void record(u64 attempted, u64 useful, double latency) {
        if (attempted && latency > 0) h.push_back({(double)attempted, (double)useful, latency});
    }
    // the cap level A* (0: no measured evidence for a cap)
    u64 level() const {
        if (h.empty()) return 0;
        size_t b = 0;
        for (size_t i = 1; i < h.size(); ++i)
            if (h[i].u / h[i].l > h[b].u / h[b].l) b = i;
        const double tb = h[b].u / h[b].l;
        for (const Rec& r : h)
            if (r.a > 1.05 * h[b].a && r.u / r.l < tb)
                return std::max<u64>(resident, (u64)h[b].a);
        return 0;
    }
    u64 cap(u64 C) const {
        if (C <= resident) return 0;
        const u64 lv = level();
        return lv && C > lv ? lv : 0;
    }
};

constexpr u32 kTailMax = 256;   // batches per tail-loop launch

struct gdp2d_ctx {
    int device = 0;
    Tracer tr;
    cudaStream_t st = nullptr;
    MeshStore work, pristine;
    u32 epoch = 0, pristine_epoch = 0;
    ull alive_v = 0, alive_t = 0, alive_s = 0;            // working-mesh alive counts
    ull p_alive_v = 0, p_alive_t = 0, p_alive_s = 0;
    // per-triangle scratch
    TriAux aux;
    u32 aux_cap = 0;
    uint8_t* flags = nullptr;
    size_t flags_cap = 0;
    // candidates
    DevCands c{};
    u32 ccap = 0;
    u32* regions = nullptr;
    u32* region_len = nullptr;
    u32* bfs_len = nullptr;
    size_t reg_cap = 0;   // entries in regions
    u32 rl_cap = 0;       // entries in region_len / bfs_len
    InsertBufs ib;
    FreshInfo fresh;
    WorkLists wl;
    ScanScratch scan;
    Counters* d_ctr = nullptr;
    Counters* h_ctr = nullptr;    // pinned
    RoundCtr* h_rc = nullptr;     // pinned
    u32* h_tot = nullptr;         // pinned [4]
    void* qscratch = nullptr;
    u32 round = 0;
    bool full_scan = true;        // next collect recomputes every triangle
    bool full_collect = false;    // GDP2D_COLLECT=full: never reuse cached flags
    int lawson_grid = 0;          // persistent Lawson kernel grid (co-resident blocks)
    int insert_grid = 0;          // persistent insertion kernel grid
    int rollback_grid = 0;        // persistent rollback kernel grid
    void* sel_state = nullptr;    // batch_size_cap radix-select state
    uint2* in_sv = nullptr;       // input segments by parent index (validators)
    u32 n_in = 0;
    bool in_valid = false;        // in_sv derived from the current pristine mesh
    void* vscratch = nullptr;     // validator scratch
    size_t vscratch_bytes = 0;
    LittleSizer little;           // Little's-law batch sizing (measured C / L per batch)
    RoundCtr* ring = nullptr;     // [4] step counters of the persistent insertion kernel
    u32* ins_state = nullptr;     // [16] status words (see k_insert.cu; [8] = unsafe flag)
    u32* h_state = nullptr;       // pinned copy
    cudaEvent_t ev_k[3] = {};     // around the split and rollback kernels
    double k_split_s = 0, k_rb_s = 0;   // per refine call: roofline accumulators
    u64 k_split_b = 0, k_rb_b = 0, k_launches = 0, k_rb_launches = 0;
    u32* d_C = nullptr;           // candidate count written by collect (device)
    // One device block holds everything the host reads after a batch, so the
    // end-of-batch readback is a single copy: ins_state [0,16), insertion
    // totals [16,19), the candidate count [19], the Counters from word 20.
    // h_status is its pinned mirror; the pointers above alias into both.
    u32* status = nullptr;
    u32* h_status = nullptr;
    u32 c_prev = 0;               // previous batch's candidate count (host, after its sync)
    bool have_c_prev = false;
    bool sync_collect = false;    // GDP2D_SYNC_COLLECT=1: host round trip after every collect
    u32 half_grid_c = 100000;     // GDP2D_HALF_GRID_C: batches below this many candidates run the
                                  // persistent kernels on one CTA per SM (cheaper grid barriers)
    u32 quarter_grid_c = 10000;   // GDP2D_QUARTER_GRID_C: ... below this on half the SMs
    u32 eighth_grid_c = 0;        // GDP2D_EIGHTH_GRID_C: ... below this on a quarter of the SMs
    u32 cluster_c = 4096;         // GDP2D_CLUSTER_C: ... below this as ONE thread-block cluster
                                  // (barrier.cluster instead of grid barriers)
    int cluster_size = 0;         // GDP2D_CLUSTER (default 16): CTAs of that cluster (0 = off)
    bool regions_tight = false;   // GDP2D_REGIONS_TIGHT=1 (tests): advertise half the region
                                  // capacity to no-round-trip batches, forcing the redo path
    u32 small_nv = 256;           // GDP2D_SMALL_NV: block-mode insertion at or below
    u32 small_wl = 256;           // GDP2D_SMALL_WL: block-mode Lawson below this list size
    u32 rm_warp = 4;              // GDP2D_RM_WARP: warp-per-removal rounds up to this many per warp
    u32 small_c = 256;            // GDP2D_SMALL_C: whole batch in one CTA at or below
    u32 standalone_c = 30000;     // GDP2D_STANDALONE_C: Lines 5-7 as standalone kernels only above this
                                  // (smaller batches filter inside the grid-mode batch kernel)
    bool dep_mis = false;         // GDP2D_DEP=mis: dependent pairs by the priority-MIS rule
    bool check = false;           // GDP2D_CHECK=1: validate after each insertion kernel
    u32* scan_part = nullptr;     // [3 * insert_grid] plan chunk sums
    u32* small_list = nullptr;    // [SMALL_LIST_WORDS]: the small-list collect (+ klist)
    u32* dlist = nullptr;         // [DLIST_CAP] + count: the tail loop's dirty elements
    bool dlist_on = false;        // this batch records its dirty elements
    bool klist_ok = false;        // klist = the last collect's list (the tail loop may start)
    bool tail_on = true;          // GDP2D_TAIL_LOOP=0: no device-resident tail loop
    TailRec* tail_rec = nullptr;  // [kTailMax] device records + pinned mirror
    TailRec* h_tail_rec = nullptr;
    u32* tail_out = nullptr;      // [8] + pinned mirror
    u32* h_tail_out = nullptr;
    u32 small_collect_c = 2048;   // GDP2D_SMALL_COLLECT: previous batch at or below -> small-list collect
    RoundCtr* rcs = nullptr;      // per-round counters of the persistent kernel
    u32* d_res = nullptr;
    u32* d_val = nullptr;
    const char* phase = "";
    cudaEvent_t ev[GDP2D_NPHASES + 4];   // phases, loop start/end, scan start/end
    // device CDT builder (k_cdt.cu) scratch
    struct {
        u32* ptri = nullptr; int8_t* pedge = nullptr; u32* pother = nullptr; u64* pkey = nullptr;
        uint8_t* pwin = nullptr; u32 ncap = 0;
        u64* tkey = nullptr; u32* newid = nullptr; u32 tcap = 0;
        uint2* pc = nullptr; u32* ppar = nullptr; u32* plist[2] = {nullptr, nullptr};
        u32* poff = nullptr; u32* plen = nullptr; u32* plive = nullptr; u32* pmap = nullptr;
        u32 pcap = 0;
        u32* claims = nullptr; u32 claim_cap = 0;
        u32* seeds = nullptr; u32 seed_cap = 0;
        CdtLocal* pool = nullptr; uint2* queue = nullptr; u32 pool_cap = 0;
        u32* part = nullptr; u32 part_cap = 0;
        RoundCtr* ring = nullptr; u32* state = nullptr; ull* bbox = nullptr;
    } cdt;
    // pageable host <-> device copies go through two pinned chunks (see xfer)
    void* pin_chunk[2] = {nullptr, nullptr};
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    // upload / download staging
    u32* stage_u32[3] = {nullptr, nullptr, nullptr};
    uint8_t* stage_u8 = nullptr;
    size_t stage_cap = 0;
    // AoS records of gdp2d_refine_aos (bytes)
    uint8_t* aos_stage = nullptr;
    size_t aos_cap = 0;
};

namespace {

void cands_free(DevCands& c) {
    dfree(c.pt); dfree(c.key); dfree(c.id); dfree(c.tie); dfree(c.loc);
    dfree(c.kind); dfree(c.alive); dfree(c.lkind); dfree(c.ledge); dfree(c.fb);
    dfree(c.red); dfree(c.unsafe); dfree(c.far);
}

void ensure_cands(gdp2d_ctx* x, u32 n) {
    if (n <= x->ccap) return;
    cands_free(x->c);
    const u32 cap = std::max<u32>(n + n / 2, 1024);
    dalloc(x->c.pt, cap); dalloc(x->c.key, cap); dalloc(x->c.id, cap); dalloc(x->c.tie, cap);
    dalloc(x->c.loc, cap); dalloc(x->c.kind, cap); dalloc(x->c.alive, cap);
    dalloc(x->c.lkind, cap); dalloc(x->c.ledge, cap); dalloc(x->c.fb, cap);
    dalloc(x->c.red, cap); dalloc(x->c.unsafe, cap); dalloc(x->c.far, cap);
    x->ccap = cap;
    // per-candidate insertion buffers
    dfree(x->ib.nv); dfree(x->ib.nt); dfree(x->ib.ns); dfree(x->ib.ov); dfree(x->ib.ot);
    dfree(x->ib.os);
    dalloc(x->ib.nv, cap); dalloc(x->ib.nt, cap); dalloc(x->ib.ns, cap);
    dalloc(x->ib.ov, cap); dalloc(x->ib.ot, cap); dalloc(x->ib.os, cap);
    x->ib.cap = cap;
}

void ensure_regions(gdp2d_ctx* x, u32 n, u32 ncav, u32 stride = 0) {
    const size_t rs = stride ? stride : ncav + 1 + MAX_CLAIM_EXTRA;
    if ((size_t)n * rs > x->reg_cap) {
        dfree(x->regions);
        x->reg_cap = std::max<size_t>((size_t)n * rs * 3 / 2, 4096);
        dalloc(x->regions, x->reg_cap);
    }
    if (n > x->rl_cap) {
        dfree(x->region_len);
        dfree(x->bfs_len);
        x->rl_cap = std::max<u32>(n + n / 2, 1024);
        dalloc(x->region_len, x->rl_cap);
        dalloc(x->bfs_len, x->rl_cap);
    }
}

void ensure_aux(gdp2d_ctx* x) {
    const u32 T = x->work.tcap;
    if (T > x->aux_cap) {
        dfree(x->aux.ckey); x->aux.ctie = nullptr; dfree(x->aux.owner); dfree(x->aux.se);
        dfree(x->aux.fkey); x->aux.ftie = nullptr; dfree(x->aux.fown);
        dalloc(x->aux.fown, T);
        dalloc(x->aux.ckey, 2ull * T); x->aux.ctie = x->aux.ckey + 1; dalloc(x->aux.owner, T);
        dalloc(x->aux.se, 4ull * T);
        dalloc(x->aux.fkey, 2ull * T); x->aux.ftie = x->aux.fkey + 1;
        // interleaved records: keys 0, ties ~0
        CK(cudaMemset2DAsync(x->aux.ckey, 2 * sizeof(u64), 0, sizeof(u64), T, x->st));
        CK(cudaMemset2DAsync(x->aux.ctie, 2 * sizeof(u64), 0xFF, sizeof(u64), T, x->st));
        CK(cudaMemset2DAsync(x->aux.fkey, 2 * sizeof(u64), 0, sizeof(u64), T, x->st));
        CK(cudaMemset2DAsync(x->aux.ftie, 2 * sizeof(u64), 0xFF, sizeof(u64), T, x->st));
        CK(cudaMemsetAsync(x->aux.owner, 0xFF, sizeof(u32) * T, x->st));
        CK(cudaMemsetAsync(x->aux.se, 0, sizeof(u32) * 4ull * T, x->st));
        // flip claims are tagged with the round, which restarts here
        CK(cudaMemsetAsync(x->aux.fown, 0, sizeof(u64) * T, x->st));
        x->aux_cap = T;
        x->round = 0;
    }
    const size_t fl = ((size_t)(x->work.scap + SCAN_TILE - 1) / SCAN_TILE +
                       (size_t)(x->work.tcap + SCAN_TILE - 1) / SCAN_TILE + 2) *
                      SCAN_TILE;
    if (fl > x->flags_cap) {
        dfree(x->flags);
        dalloc(x->flags, fl);
        x->flags_cap = fl;
    }
    // work lists: sized by triangle capacity
    const u32 wcap = 2 * T + (1u << 20);
    if (wcap > x->wl.cap) {
        dfree(x->wl.w[0]); dfree(x->wl.w[1]); dfree(x->wl.fc); dfree(x->wl.fu);
        dfree(x->wl.touched); dfree(x->wl.fwin);
        dalloc(x->wl.w[0], wcap); dalloc(x->wl.w[1], wcap); dalloc(x->wl.fc, wcap);
        dalloc(x->wl.fu, wcap); dalloc(x->wl.touched, wcap); dalloc(x->wl.fwin, wcap);
        x->wl.cap = wcap;
    }
}

// Lawson / touched work lists of at least n entries (contents are transient).
void ensure_worklists(gdp2d_ctx* x, u64 n) {
    if (n <= x->wl.cap) return;
    const u32 wcap = (u32)std::min<u64>(0xFFFFFFF0ull, n + n / 2);
    dfree(x->wl.w[0]); dfree(x->wl.w[1]); dfree(x->wl.fc); dfree(x->wl.fu);
    dfree(x->wl.touched); dfree(x->wl.fwin);
    dalloc(x->wl.w[0], wcap); dalloc(x->wl.w[1], wcap); dalloc(x->wl.fc, wcap);
    dalloc(x->wl.fu, wcap); dalloc(x->wl.touched, wcap); dalloc(x->wl.fwin, wcap);
    x->wl.cap = wcap;
}

void ensure_fresh(gdp2d_ctx* x, u32 n) {
    if (n <= x->fresh.cap) return;
    FreshInfo& f = x->fresh;
    dfree(f.key); dfree(f.tie); dfree(f.cc); dfree(f.removed); dfree(f.mark); dfree(f.dirty);
    dfree(f.dstat); dfree(f.hcnt); dfree(f.hlist);
    const u32 cap = std::max<u32>(n + n / 2, 1024);
    dalloc(f.key, cap); dalloc(f.tie, cap); dalloc(f.cc, cap); dalloc(f.removed, cap);
    dalloc(f.mark, cap); dalloc(f.dirty, cap);
    dalloc(f.dstat, cap); dalloc(f.hcnt, cap); dalloc(f.hlist, (size_t)cap * DEP_HMAX);
    f.cap = cap;
    dfree(x->wl.rm[0]); dfree(x->wl.rm[1]); dfree(x->wl.star); dfree(x->wl.star_len);
    dalloc(x->wl.rm[0], cap); dalloc(x->wl.rm[1], cap);
    dalloc(x->wl.star, (size_t)cap * MAX_STAR);
    dalloc(x->wl.star_len, cap);
    x->wl.rm_cap = cap;
}

// Working-mesh capacity for the next insertion (amortised growth).
void ensure_mesh(gdp2d_ctx* x, u32 V, u32 T, u32 S) {
    MeshStore& w = x->work;
    if (V <= w.vcap && T <= w.tcap && S <= w.scap) return;
    const auto grow = [](u32 need, u32 cap) {
        return need <= cap ? cap : (u32)std::min<u64>(0xFFFFFFF0ull, (u64)need * 3 / 2 + 1024);
    };
    mesh_reserve(w, grow(V, w.vcap), grow(T, w.tcap), grow(S, w.scap), x->st);
    ensure_aux(x);
}

void zero_rc(gdp2d_ctx* x) { CK(cudaMemsetAsync(x->wl.rc, 0, sizeof(RoundCtr), x->st)); }

RoundCtr read_rc(gdp2d_ctx* x) {
    CK(cudaMemcpyAsync(x->h_rc, x->wl.rc, sizeof(RoundCtr), cudaMemcpyDeviceToHost, x->st));
    CK(cudaStreamSynchronize(x->st));
    return *x->h_rc;
}

void raise_dev_err(gdp2d_ctx* x);

void check_dev_err(gdp2d_ctx* x) {
    CK(cudaMemcpyAsync(x->h_ctr, x->d_ctr, sizeof(Counters), cudaMemcpyDeviceToHost, x->st));
    CK(cudaStreamSynchronize(x->st));
    raise_dev_err(x);
}

// Throw if the (already downloaded) device counters carry an error.
void raise_dev_err(gdp2d_ctx* x) {
    if (x->h_ctr->err_code) {
        char buf[512];
        const double* d = x->h_ctr->dbg;
        snprintf(buf, sizeof buf,
                 "device error %u (%s), info %u, dbg [%.17g %.17g %.17g %.17g %.17g %.17g %.17g %.17g]",
                 x->h_ctr->err_code, dev_err_name(x->h_ctr->err_code), x->h_ctr->err_info, d[0],
                 d[1], d[2], d[3], d[4], d[5], d[6], d[7]);
        const u32 ec = x->h_ctr->err_code;
        throw Fail{ec == DERR_WORKLIST_OVERFLOW ? GDP2D_ECAPACITY
                   : ec >= DERR_DUPLICATE       ? GDP2D_ECDT
                                                : GDP2D_EMESH,
                   buf};
    }
}

}  // namespace

// Lawson driver (cdt.hpp:111-123): the persistent cooperative kernel runs
// every round of the fixpoint in one launch; the host continues only when a
// launch used up its round budget.
static void lawson_from(gdp2d_ctx* x, u32 start_buf, u32 n, u32* rounds) {
    u32 cur = start_buf;
    u32 guard = 0;
    constexpr u32 kMax = 1024;
    while (n > 0) {
        if (n > x->wl.cap) throw Fail{GDP2D_ECAPACITY, "Lawson work list overflow"};
        if (++guard > 1000) throw Fail{GDP2D_EMESH, "Lawson flip rounds did not converge"};
        CK(cudaMemsetAsync(x->rcs, 0, sizeof(RoundCtr) * kMax, x->st));
        launch_lawson_persistent(x->work.m, x->round + 1, cur, n, kMax, x->aux, x->wl, x->rcs,
                                 x->d_res, x->d_ctr, x->lawson_grid, x->st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(x->h_tot, x->d_res, 3 * sizeof(u32), cudaMemcpyDeviceToHost, x->st));
        CK(cudaStreamSynchronize(x->st));
        x->round += x->h_tot[0];
        if (rounds) *rounds += x->h_tot[0];
        cur = x->h_tot[1];
        n = x->h_tot[2];
    }
}

namespace {

void ctx_init(gdp2d_ctx* x, int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw Fail{GDP2D_ENODEVICE, "no CUDA device visible"};
    if (device < 0 || device >= n) throw Fail{GDP2D_ENODEVICE, "device index out of range"};
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        throw Fail{GDP2D_ENODEVICE, std::string("sm_100a required, found ") + prop.name};
    x->device = device;
    CK(cudaStreamCreateWithFlags(&x->st, cudaStreamNonBlocking));
    dalloc(x->status, kStatusWords);
    CK(cudaMallocHost(&x->h_status, kStatusWords * sizeof(u32)));
    x->ins_state = x->status;
    x->ib.totals = x->status + 16;
    x->d_C = x->status + 19;
    x->d_ctr = reinterpret_cast<Counters*>(x->status + 20);
    x->h_state = x->h_status;
    x->h_tot = x->h_status + 16;
    x->h_ctr = reinterpret_cast<Counters*>(x->h_status + 20);
    dalloc(x->wl.rc, 1);
    CK(cudaMallocHost(&x->h_rc, sizeof(RoundCtr)));
    CK(cudaMalloc(&x->qscratch, 256));
    dalloc(x->d_val, 4);
    dalloc(x->wl.dbg, 4 + 2 * MAX_STAR);
    CK(cudaMemsetAsync(x->wl.dbg, 0, sizeof(double) * (4 + 2 * MAX_STAR), x->st));
    if (const char* e = std::getenv("GDP2D_SYNC_COLLECT")) x->sync_collect = e[0] == '1';
    if (const char* e = std::getenv("GDP2D_STANDALONE_C")) x->standalone_c = (u32)std::atoll(e);
    if (const char* e = std::getenv("GDP2D_REGIONS_TIGHT")) x->regions_tight = e[0] == '1';
    if (const char* e = std::getenv("GDP2D_HALF_GRID_C")) x->half_grid_c = (u32)std::atoll(e);
    if (const char* e = std::getenv("GDP2D_QUARTER_GRID_C")) x->quarter_grid_c = (u32)std::atoll(e);
    if (const char* e = std::getenv("GDP2D_EIGHTH_GRID_C")) x->eighth_grid_c = (u32)std::atoll(e);
    if (const char* e = std::getenv("GDP2D_CLUSTER_C")) x->cluster_c = (u32)std::atoll(e);
    {
        const char* e = std::getenv("GDP2D_CLUSTER");
        x->cluster_size = insert_cluster_size(device, e ? std::atoi(e) : 16);
    }
    x->lawson_grid = lawson_persistent_grid(device);
    x->insert_grid = insert_persistent_grid(device);
    x->rollback_grid = rollback_persistent_grid(device);
    if (const char* e = std::getenv("GDP2D_GRID")) {   // experiments: fewer co-resident CTAs
        const int g = std::atoi(e);
        if (g > 0) {
            x->insert_grid = std::min(x->insert_grid, g);
            x->rollback_grid = std::min(x->rollback_grid, g);
        }
    }
    CK(cudaMalloc(&x->sel_state, select_state_bytes()));
    x->little.resident = cavity_resident_candidates(device);
    dalloc(x->ring, 5);   // 4-slot step ring + the removal-seed accumulator
    if (const char* e = std::getenv("GDP2D_TRACE"); e && (e[0] == '1' || e[0] == '2')) {
        x->tr.on = true;
        x->tr.rounds = e[0] == '2';
        x->tr.init();
    }
    if (const char* e = std::getenv("GDP2D_SMALL_NV")) x->small_nv = (u32)std::strtoul(e, nullptr, 10);
    if (const char* e = std::getenv("GDP2D_SMALL_WL")) x->small_wl = (u32)std::strtoul(e, nullptr, 10);
    if (const char* e = std::getenv("GDP2D_RM_WARP")) x->rm_warp = (u32)std::strtoul(e, nullptr, 10);
    if (const char* e = std::getenv("GDP2D_SMALL_C")) x->small_c = (u32)std::strtoul(e, nullptr, 10);
    if (const char* e = std::getenv("GDP2D_DEP")) x->dep_mis = std::string(e) == "mis";
    if (const char* e = std::getenv("GDP2D_CHECK")) x->check = e[0] == '1';
    dalloc(x->scan_part, 3ull * x->insert_grid + 3);
    dalloc(x->small_list, SMALL_LIST_WORDS);
    CK(cudaMemsetAsync(x->small_list, 0, sizeof(u32) * SMALL_LIST_WORDS, x->st));
    dalloc(x->dlist, DLIST_CAP + 1);
    CK(cudaMemsetAsync(x->dlist + DLIST_CAP, 0, sizeof(u32), x->st));
    dalloc(x->tail_rec, kTailMax);
    CK(cudaMallocHost(&x->h_tail_rec, sizeof(TailRec) * kTailMax));
    dalloc(x->tail_out, 8);
    CK(cudaMallocHost(&x->h_tail_out, sizeof(u32) * 8));
    if (const char* e = std::getenv("GDP2D_TAIL_LOOP")) x->tail_on = e[0] != '0';
    if (const char* e = std::getenv("GDP2D_SMALL_COLLECT")) x->small_collect_c = (u32)std::atoll(e);
    const char* fc = std::getenv("GDP2D_COLLECT");
    x->full_collect = fc && std::string(fc) == "full";
    dalloc(x->rcs, 1024);
    dalloc(x->d_res, 4);
    for (auto& e : x->ev) CK(cudaEventCreate(&e));
    for (auto& e : x->ev_k) CK(cudaEventCreate(&e));
}

void ctx_release(gdp2d_ctx* x) {
    cudaSetDevice(x->device);
    mesh_free(x->work);
    mesh_free(x->pristine);
    dfree(x->aux.ckey); x->aux.ctie = nullptr; dfree(x->aux.owner); dfree(x->aux.se);
    dfree(x->aux.fkey); x->aux.ftie = nullptr; dfree(x->aux.fown);
    dfree(x->flags);
    cands_free(x->c);
    dfree(x->regions); dfree(x->region_len); dfree(x->bfs_len);
    dfree(x->ib.nv); dfree(x->ib.nt); dfree(x->ib.ns); dfree(x->ib.ov); dfree(x->ib.ot);
    dfree(x->ib.os);
    dfree(x->fresh.key); dfree(x->fresh.tie); dfree(x->fresh.cc); dfree(x->fresh.removed);
    dfree(x->fresh.mark); dfree(x->fresh.dirty);
    dfree(x->fresh.dstat); dfree(x->fresh.hcnt); dfree(x->fresh.hlist);
    dfree(x->wl.w[0]); dfree(x->wl.w[1]); dfree(x->wl.fc); dfree(x->wl.fu);
    dfree(x->wl.touched); dfree(x->wl.fwin); dfree(x->wl.rm[0]); dfree(x->wl.rm[1]);
    dfree(x->wl.star); dfree(x->wl.star_len); dfree(x->wl.rc);
    dfree(x->scan.partial);
    x->ins_state = x->ib.totals = x->d_C = nullptr;
    x->d_ctr = nullptr;
    dfree(x->status);
    if (x->h_status) cudaFreeHost(x->h_status);
    x->h_status = x->h_state = x->h_tot = nullptr;
    x->h_ctr = nullptr;
    for (auto& s : x->stage_u32) dfree(s);
    dfree(x->stage_u8);
    dfree(x->aos_stage);
    if (x->h_rc) cudaFreeHost(x->h_rc);
    if (x->qscratch) cudaFree(x->qscratch);
    dfree(x->d_val);
    dfree(x->wl.dbg);
    dfree(x->rcs);
    dfree(x->d_res);
    dfree(x->ring);
    dfree(x->scan_part);
    dfree(x->small_list);
    dfree(x->dlist);
    dfree(x->tail_rec);
    dfree(x->tail_out);
    if (x->h_tail_rec) cudaFreeHost(x->h_tail_rec);
    if (x->h_tail_out) cudaFreeHost(x->h_tail_out);
    {
        auto& c = x->cdt;
        dfree(c.ptri); dfree(c.pedge); dfree(c.pother); dfree(c.pkey); dfree(c.pwin);
        dfree(c.tkey); dfree(c.newid); dfree(c.pc); dfree(c.ppar); dfree(c.plist[0]);
        dfree(c.plist[1]); dfree(c.poff); dfree(c.plen); dfree(c.plive); dfree(c.pmap);
        dfree(c.claims); dfree(c.seeds); dfree(c.pool); dfree(c.queue); dfree(c.part);
        dfree(c.ring); dfree(c.state); dfree(c.bbox);
    }
    if (x->sel_state) cudaFree(x->sel_state);
    dfree(x->in_sv);
    if (x->vscratch) cudaFree(x->vscratch);
    x->tr.release();
    for (auto& e : x->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : x->ev_k)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
        if (x->pin_chunk[i]) cudaFreeHost(x->pin_chunk[i]);
        if (x->pin_ev[i]) cudaEventDestroy(x->pin_ev[i]);
    }
    if (x->st) cudaStreamDestroy(x->st);
}

void ensure_stage(gdp2d_ctx* x, size_t n) {
    if (n <= x->stage_cap) return;
    for (auto& s : x->stage_u32) {
        dfree(s);
        dalloc(s, n);
    }
    dfree(x->stage_u8);
    dalloc(x->stage_u8, n);
    x->stage_cap = n;
}

void validate_view(const gdp2d_mesh_view* v) {
    if (!v) throw Fail{GDP2D_EINVAL, "null mesh view"};
    if (v->n_triangles && (!v->tri_v || !v->tri_n || !v->tri_seg || !v->tri_alive))
        throw Fail{GDP2D_EINVAL, "missing triangle arrays"};
    if (v->n_vertices && (!v->xy || !v->vert_kind || !v->vert_birth || !v->vert_alive ||
                          !v->vert_tri))
        throw Fail{GDP2D_EINVAL, "missing vertex arrays"};
    if (v->n_subsegments && (!v->seg_v || !v->seg_parent || !v->seg_encroached ||
                             !v->seg_alive || !v->seg_tri))
        throw Fail{GDP2D_EINVAL, "missing subsegment arrays"};
    if (v->n_triangles >= (1u << 30)) throw Fail{GDP2D_EINVAL, "too many triangles"};
}

// ---- host <-> device copies -----------------------------------------------------
// Pinned caller memory is copied directly.  Pageable memory (malloc'ed output
// of gdp2d_refine, the C++ shim's vectors) goes through two 32 MB pinned
// chunks: the DMA of one chunk overlaps the multi-threaded host copy of the
// other, instead of the driver's single-threaded pageable path.
constexpr size_t kPinChunk = 32u << 20;

bool host_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void ensure_pin_chunks(gdp2d_ctx* x) {
    for (int i = 0; i < 2; ++i) {
        if (!x->pin_chunk[i]) CK(cudaMallocHost(&x->pin_chunk[i], kPinChunk));
        if (!x->pin_ev[i]) CK(cudaEventCreateWithFlags(&x->pin_ev[i], cudaEventDisableTiming));
    }
}

void par_memcpy(void* dst, const void* src, size_t n) {
    const unsigned hw = std::thread::hardware_concurrency();
    const size_t parts = std::min<size_t>(std::min(8u, hw ? hw : 1u), std::max<size_t>(1, n >> 22));
    if (parts <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    for (size_t p = 0; p < parts; ++p)
        th.emplace_back([=] {
            const size_t lo = n * p / parts, hi = n * (p + 1) / parts;
            std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
        });
    for (auto& t : th) t.join();
}

void d2h(gdp2d_ctx* x, void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    cudaStream_t st = x->st;
    if (bytes < (4u << 20) || host_pinned(dst)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        return;
    }
    ensure_pin_chunks(x);
    size_t prev_off = 0, prev_n = 0;
    int k = 0;
    for (size_t off = 0; off < bytes; off += kPinChunk, ++k) {
        const size_t n = std::min(kPinChunk, bytes - off);
        CK(cudaMemcpyAsync(x->pin_chunk[k & 1], static_cast<const char*>(src) + off, n,
                           cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(x->pin_ev[k & 1], st));
        if (k > 0) {
            CK(cudaEventSynchronize(x->pin_ev[(k - 1) & 1]));
            par_memcpy(static_cast<char*>(dst) + prev_off, x->pin_chunk[(k - 1) & 1], prev_n);
        }
        prev_off = off;
        prev_n = n;
    }
    CK(cudaEventSynchronize(x->pin_ev[(k - 1) & 1]));
    par_memcpy(static_cast<char*>(dst) + prev_off, x->pin_chunk[(k - 1) & 1], prev_n);
}

void h2d(gdp2d_ctx* x, void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    cudaStream_t st = x->st;
    if (bytes < (4u << 20) || host_pinned(src)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    ensure_pin_chunks(x);
    int k = 0;
    for (size_t off = 0; off < bytes; off += kPinChunk, ++k) {
        const size_t n = std::min(kPinChunk, bytes - off);
        CK(cudaEventSynchronize(x->pin_ev[k & 1]));   // the chunk's previous DMA is done
        par_memcpy(x->pin_chunk[k & 1], static_cast<const char*>(src) + off, n);
        CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, x->pin_chunk[k & 1], n,
                           cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(x->pin_ev[k & 1], st));
    }
    // the last chunks stay in flight; any later reuse of a chunk waits on its
    // event (or follows it in stream order)
}

void upload_finish(gdp2d_ctx* x, u32 batch_epoch);

void upload(gdp2d_ctx* x, const gdp2d_mesh_view* v) {
    validate_view(v);
    const u32 V = v->n_vertices, T = v->n_triangles, S = v->n_subsegments;
    MeshStore& p = x->pristine;
    p.m.nV = p.m.nT = p.m.nS = 0;
    mesh_reserve(p, V, T, S, x->st);
    DevMesh& m = p.m;
    m.nV = V;
    m.nT = T;
    m.nS = S;
    cudaStream_t st = x->st;
    h2d(x, m.xy, v->xy, 16ull * V);
    h2d(x, m.vkind, v->vert_kind, V);
    h2d(x, m.vbirth, v->vert_birth, 4ull * V);
    h2d(x, m.valive, v->vert_alive, V);
    h2d(x, m.vtri, v->vert_tri, 4ull * V);
    ensure_stage(x, std::max<size_t>(3ull * T, 2ull * S) + T + S + 16);
    if (T) {
        h2d(x, x->stage_u32[0], v->tri_v, 12ull * T);
        h2d(x, x->stage_u32[1], v->tri_seg, 12ull * T);
        h2d(x, x->stage_u32[2], v->tri_n, 12ull * T);
        h2d(x, x->stage_u8, v->tri_alive, T);
        note_launch(), k_pack_tris<<<grid(T), 256, 0, st>>>(m, x->stage_u32[0], x->stage_u32[1], x->stage_u8);
        launch_encode_neighbors(m, x->stage_u32[2], st);
    }
    if (S) {
        h2d(x, m.sv, v->seg_v, 8ull * S);
        h2d(x, m.sparent, v->seg_parent, 4ull * S);
        h2d(x, m.salive, v->seg_alive, S);
        h2d(x, m.stri, v->seg_tri, 4ull * S);
        CK(cudaMemcpyAsync(x->stage_u8 + T + 8, v->seg_encroached, S, cudaMemcpyHostToDevice,
                           st));
        note_launch(), k_u8_to_u32<<<grid(S), 256, 0, st>>>(x->stage_u8 + T + 8, m.senc, S);
        CK(cudaMemsetAsync(m.sdepth, 0, 4ull * S, st));
    }
    CK(cudaGetLastError());
    upload_finish(x, v->batch_epoch);
}

// The tail of every upload: epoch, lazily derived input segments, alive counts.
void upload_finish(gdp2d_ctx* x, u32 batch_epoch) {
    const DevMesh& m = x->pristine.m;
    const u32 V = m.nV, T = m.nT, S = m.nS;
    cudaStream_t st = x->st;
    x->pristine_epoch = batch_epoch;
    x->n_in = 0;   // input segments are derived lazily by gdp2d_ctx_validate
    x->in_valid = false;
    // alive counts (batch metrics) on the device, read back with the upload
    ull* cnt = reinterpret_cast<ull*>(x->qscratch);
    CK(cudaMemsetAsync(cnt, 0, 3 * sizeof(ull), st));
    note_launch(), k_count_alive<<<grid(std::max(V, std::max(T, S))), 256, 0, st>>>(m, cnt);
    ull h[3];
    CK(cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    x->p_alive_v = h[0];
    x->p_alive_t = h[1];
    x->p_alive_s = h[2];
}

// theta_hint (degrees, 0 = unknown): the one-shot gdp2d_refine sizes the
// working mesh for the growth the quality bound implies (the mesh grows about
// 2.1x at B = sqrt(2) and 5.4x at 30 degrees on the BASELINE PSLGs), so a single
// call does not pay reallocations mid-refinement.
void reset_work(gdp2d_ctx* x, double theta_hint = 0.0) {
    const DevMesh& p = x->pristine.m;
    // headroom: 2.5x the input (amortised growth handles the rest);
    // GDP2D_HEADROOM overrides the factor (tests use 1.0 to force growth)
    double hr = theta_hint >= 28.0 ? 6.0 : theta_hint >= 24.0 ? 4.0 : 2.5;
    if (const char* e = std::getenv("GDP2D_HEADROOM")) hr = std::max(1.0, std::atof(e));
    x->work.m.nV = x->work.m.nT = x->work.m.nS = 0;
    mesh_reserve(x->work, std::max<u32>((u32)(p.nV * hr), 64), std::max<u32>((u32)(p.nT * hr), 128),
                 std::max<u32>((u32)(p.nS * hr), 64), x->st);
    mesh_copy(x->work, x->pristine, x->st);
    // subsegment depth restarts at 0 for every refine call (refine.hpp:655)
    if (x->work.m.nS) CK(cudaMemsetAsync(x->work.m.sdepth, 0, 4ull * x->work.m.nS, x->st));
    x->epoch = x->pristine_epoch;
    x->alive_v = x->p_alive_v;
    x->alive_t = x->p_alive_t;
    x->alive_s = x->p_alive_s;
    ensure_aux(x);
    x->full_scan = true;
}

// Copy the working mesh into host arrays already present in *b.
void download_into(gdp2d_ctx* x, gdp2d_mesh_buf* b) {
    const DevMesh& m = x->work.m;
    const u32 V = m.nV, T = m.nT, S = m.nS;
    cudaStream_t st = x->st;
    b->n_vertices = V;
    b->n_triangles = T;
    b->n_subsegments = S;
    b->batch_epoch = x->epoch;
    ensure_stage(x, std::max<size_t>(3ull * T, 2ull * S) + T + S + 16);
    if (V) {
        d2h(x, b->xy, m.xy, 16ull * V);
        d2h(x, b->vert_kind, m.vkind, V);
        d2h(x, b->vert_birth, m.vbirth, 4ull * V);
        d2h(x, b->vert_alive, m.valive, V);
        d2h(x, b->vert_tri, m.vtri, 4ull * V);
    }
    if (T) {
        note_launch(), k_unpack_tris<<<grid(T), 256, 0, st>>>(m, x->stage_u32[0], x->stage_u32[1], x->stage_u8);
        launch_decode_neighbors(m, x->stage_u32[2], st);
        d2h(x, b->tri_v, x->stage_u32[0], 12ull * T);
        d2h(x, b->tri_seg, x->stage_u32[1], 12ull * T);
        d2h(x, b->tri_n, x->stage_u32[2], 12ull * T);
        d2h(x, b->tri_alive, x->stage_u8, T);
    }
    if (S) {
        d2h(x, b->seg_v, m.sv, 8ull * S);
        d2h(x, b->seg_parent, m.sparent, 4ull * S);
        d2h(x, b->seg_alive, m.salive, S);
        d2h(x, b->seg_tri, m.stri, 4ull * S);
        note_launch(), k_u32_to_u8<<<grid(S), 256, 0, st>>>(m.senc, x->stage_u8 + T + 8, S);
        d2h(x, b->seg_encroached, x->stage_u8 + T + 8, S);
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
}

// Library-owned output arrays (freed by gdp2d_free): 2 MB aligned, with a
// transparent-huge-page hint for the big ones, so the first touch by the
// staged D2H copy faults 2 MB pages, not 4 KB ones.
void* host_out_alloc(size_t bytes) {
    constexpr size_t kHuge = 2u << 20;
    if (bytes < kHuge) return std::malloc(bytes ? bytes : 1);
    const size_t n = (bytes + kHuge - 1) / kHuge * kHuge;
    void* p = std::aligned_alloc(kHuge, n);
#ifdef MADV_HUGEPAGE
    if (p) madvise(p, n, MADV_HUGEPAGE);
#endif
    return p;
}

void download(gdp2d_ctx* x, gdp2d_mesh_buf* b) {
    const DevMesh& m = x->work.m;
    const u32 V = m.nV, T = m.nT, S = m.nS;
    std::memset(b, 0, sizeof *b);
    auto hm = [](size_t bytes) { return host_out_alloc(bytes); };
    b->xy = (double*)hm(16ull * V);
    b->vert_kind = (uint8_t*)hm(V);
    b->vert_birth = (u32*)hm(4ull * V);
    b->vert_alive = (uint8_t*)hm(V);
    b->vert_tri = (u32*)hm(4ull * V);
    b->tri_v = (u32*)hm(12ull * T);
    b->tri_n = (u32*)hm(12ull * T);
    b->tri_seg = (u32*)hm(12ull * T);
    b->tri_alive = (uint8_t*)hm(T);
    b->seg_v = (u32*)hm(8ull * S);
    b->seg_parent = (u32*)hm(4ull * S);
    b->seg_encroached = (uint8_t*)hm(S);
    b->seg_alive = (uint8_t*)hm(S);
    b->seg_tri = (u32*)hm(4ull * S);
    download_into(x, b);
}

// ---- AoS records (gdp2d_refine_aos) ----

void check_aos_layout(const gdp2d_aos_layout* L) {
    auto in = [](u32 off, u32 bytes, u32 size, u32 align) {
        return off % align == 0 && (u64)off + bytes <= size;
    };
    const bool ok = L && L->vert_size % 8 == 0 && L->tri_size % 4 == 0 && L->seg_size % 4 == 0 &&
                    in(L->vert_pos, 16, L->vert_size, 8) && in(L->vert_kind, 1, L->vert_size, 1) &&
                    in(L->vert_birth, 4, L->vert_size, 4) && in(L->vert_alive, 1, L->vert_size, 1) &&
                    in(L->tri_v, 12, L->tri_size, 4) && in(L->tri_nbr, 12, L->tri_size, 4) &&
                    in(L->tri_seg, 12, L->tri_size, 4) && in(L->tri_alive, 1, L->tri_size, 1) &&
                    in(L->seg_v, 8, L->seg_size, 4) && in(L->seg_parent, 4, L->seg_size, 4) &&
                    in(L->seg_encroached, 1, L->seg_size, 1) && in(L->seg_alive, 1, L->seg_size, 1);
    if (!ok) throw Fail{GDP2D_EINVAL, "AoS layout: field outside its record or misaligned"};
}

void ensure_aos(gdp2d_ctx* x, size_t bytes) {
    if (bytes <= x->aos_cap) return;
    dfree(x->aos_stage);
    dalloc(x->aos_stage, bytes);
    x->aos_cap = bytes;
}

void upload_aos(gdp2d_ctx* x, const gdp2d_aos_layout* L, const gdp2d_aos_mesh* a) {
    check_aos_layout(L);
    const u32 V = a->n_vertices, T = a->n_triangles, S = a->n_subsegments;
    if ((V && (!a->verts || !a->vert_tri)) || (T && !a->tris) || (S && (!a->segs || !a->seg_tri)))
        throw Fail{GDP2D_EINVAL, "missing AoS arrays"};
    MeshStore& p = x->pristine;
    p.m.nV = p.m.nT = p.m.nS = 0;
    mesh_reserve(p, V, T, S, x->st);
    DevMesh& m = p.m;
    m.nV = V;
    m.nT = T;
    m.nS = S;
    cudaStream_t st = x->st;
    ensure_aos(x, std::max({(size_t)V * L->vert_size, (size_t)T * L->tri_size,
                            (size_t)S * L->seg_size, (size_t)16}));
    ensure_stage(x, std::max<size_t>(3ull * T, 2ull * S) + T + S + 16);
    if (V) {
        h2d(x, x->aos_stage, a->verts, (size_t)V * L->vert_size);
        note_launch(), k_aos_verts_in<<<grid(V), 256, 0, st>>>(x->aos_stage, *L, m, V);
        h2d(x, m.vtri, a->vert_tri, 4ull * V);
    }
    if (T) {   // the records' bytes reuse the staging once the vertex kernel ran (stream order)
        h2d(x, x->aos_stage, a->tris, (size_t)T * L->tri_size);
        note_launch(), k_aos_tris_in<<<grid(T), 256, 0, st>>>(x->aos_stage, *L, x->stage_u32[0],
                                                            x->stage_u32[1], x->stage_u32[2],
                                                            x->stage_u8, T);
        note_launch(), k_pack_tris<<<grid(T), 256, 0, st>>>(m, x->stage_u32[0], x->stage_u32[1], x->stage_u8);
        launch_encode_neighbors(m, x->stage_u32[2], st);
    }
    if (S) {
        h2d(x, x->aos_stage, a->segs, (size_t)S * L->seg_size);
        note_launch(), k_aos_segs_in<<<grid(S), 256, 0, st>>>(x->aos_stage, *L, m, S);
        h2d(x, m.stri, a->seg_tri, 4ull * S);
    }
    CK(cudaGetLastError());
    upload_finish(x, a->batch_epoch);
}

// The working mesh into the caller's AoS arrays, sized by its resize callback.
void download_aos(gdp2d_ctx* x, const gdp2d_aos_layout* L, gdp2d_aos_mesh* a) {
    const DevMesh& m = x->work.m;
    const u32 V = m.nV, T = m.nT, S = m.nS;
    cudaStream_t st = x->st;
    ensure_aos(x, std::max({(size_t)V * L->vert_size, (size_t)T * L->tri_size,
                            (size_t)S * L->seg_size, (size_t)16}));
    ensure_stage(x, std::max<size_t>(3ull * T, 2ull * S) + T + S + 16);
    auto dst = [&](int what, u64 n) {
        void* d = a->resize(a->user, what, n);
        if (!d && n) throw Fail{GDP2D_EINVAL, "AoS resize callback returned null"};
        return d;
    };
    // the record padding goes out as zeros
    if (V) {
        CK(cudaMemsetAsync(x->aos_stage, 0, (size_t)V * L->vert_size, st));
        note_launch(), k_aos_verts_out<<<grid(V), 256, 0, st>>>(m, *L, x->aos_stage, V);
        d2h(x, dst(GDP2D_AOS_VERTS, V), x->aos_stage, (size_t)V * L->vert_size);
        d2h(x, dst(GDP2D_AOS_VERT_TRI, V), m.vtri, 4ull * V);
    } else {
        dst(GDP2D_AOS_VERTS, 0);
        dst(GDP2D_AOS_VERT_TRI, 0);
    }
    if (T) {
        CK(cudaMemsetAsync(x->aos_stage, 0, (size_t)T * L->tri_size, st));
        note_launch(), k_unpack_tris<<<grid(T), 256, 0, st>>>(m, x->stage_u32[0], x->stage_u32[1], x->stage_u8);
        launch_decode_neighbors(m, x->stage_u32[2], st);
        note_launch(), k_aos_tris_out<<<grid(T), 256, 0, st>>>(x->stage_u32[0], x->stage_u32[1],
                                                             x->stage_u32[2], x->stage_u8, *L,
                                                             x->aos_stage, T);
        d2h(x, dst(GDP2D_AOS_TRIS, T), x->aos_stage, (size_t)T * L->tri_size);
    } else {
        dst(GDP2D_AOS_TRIS, 0);
    }
    if (S) {
        CK(cudaMemsetAsync(x->aos_stage, 0, (size_t)S * L->seg_size, st));
        note_launch(), k_aos_segs_out<<<grid(S), 256, 0, st>>>(m, *L, x->aos_stage, S);
        d2h(x, dst(GDP2D_AOS_SEGS, S), x->aos_stage, (size_t)S * L->seg_size);
        d2h(x, dst(GDP2D_AOS_SEG_TRI, S), m.stri, 4ull * S);
    } else {
        dst(GDP2D_AOS_SEGS, 0);
        dst(GDP2D_AOS_SEG_TRI, 0);
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    a->n_vertices = V;
    a->n_triangles = T;
    a->n_subsegments = S;
    a->batch_epoch = x->epoch;
}

double ev_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return (double)ms;
}

// GDP2D_CHECK=1: device structural validation of the working mesh grown by
// this batch's reserved ids (totals read back first).
void check_structure_now(gdp2d_ctx* x, u32 nV, u32 nT, u32 nS, const char* where) {
    CK(cudaMemcpyAsync(x->h_tot, x->ib.totals, 3 * sizeof(u32), cudaMemcpyDeviceToHost, x->st));
    CK(cudaMemcpyAsync(x->h_state, x->ins_state, 16 * sizeof(u32), cudaMemcpyDeviceToHost, x->st));
    CK(cudaStreamSynchronize(x->st));
    if (x->h_state[0] != 0u) return;   // growth request: nothing was written
    DevMesh m = x->work.m;
    m.nV = nV + x->h_tot[0];
    m.nT = nT + x->h_tot[1];
    m.nS = nS + x->h_tot[2];
    launch_vtri_rebuild(m, x->st);   // batches keep vert_tri for fresh vertices only
    launch_validate(m, x->d_val, x->st);
    u32 h[4];
    CK(cudaMemcpyAsync(h, x->d_val, sizeof h, cudaMemcpyDeviceToHost, x->st));
    CK(cudaStreamSynchronize(x->st));
    check_dev_err(x);
    if (h[0]) {
        char buf[200];
        snprintf(buf, sizeof buf, "check after %s (batch %u): failure %u at triangle %u edge %d",
                 where, x->epoch, h[0], h[1], (int)h[2]);
        throw Fail{GDP2D_EMESH, buf};
    }
}

// The launch record every batch kernel shares (insert_persistent, tail_loop).
InsertLaunch base_launch(gdp2d_ctx* x, const gdp2d_params* p, u32 batch, u32 ncav, u32 rs,
                         int isolate) {
    InsertLaunch L;
    L.m = x->work.m;
    L.c = x->c;
    L.b = x->ib;
    L.x = x->aux;
    L.f = x->fresh;
    L.w = x->wl;
    L.w.vdirty = x->fresh.dirty;          // fixup flags detection suspects
    L.w.fresh_cc = x->fresh.cc;
    L.w.fresh_v0 = x->work.m.nV;          // fresh ids start here ...
    L.w.fresh_n = x->fresh.cap;           // ... and never exceed the buffer
    L.w.vtri_from = x->work.m.nV;         // vert_tri kept for the fresh ids only
    if (x->dlist_on) {                    // the next batch may run in the tail loop
        L.w.dlist = x->dlist;
        L.w.dlist_n = x->dlist + DLIST_CAP;
        L.w.dlist_cap = DLIST_CAP;
    }
    L.ring = x->ring;
    L.state = x->ins_state;
    L.ctr = x->d_ctr;
    L.d_C = x->d_C;
    L.depth_cap = p->split_depth_cap;
    L.batch = batch;
    L.round0 = x->round + 1;
    L.vcap = x->work.vcap;
    L.tcap = x->work.tcap;
    L.scap = x->work.scap;
    L.small_nv = x->small_nv;
    L.small_wl = x->small_wl;
    L.rm_warp = x->rm_warp;
    L.max_steps = 1u << 20;
    L.ncav = ncav;
    L.rs = rs;
    L.isolate = isolate;
    L.dep_mis = x->dep_mis ? 1 : 0;
    L.extras = 2;   // refinement claims: the rewrite table (launch_cavity)
    L.regions = x->regions;
    L.region_len = x->region_len;
    L.scan_part = x->scan_part;
    L.small_c = x->small_c;
    return L;
}

// Insertion phase as one persistent cooperative launch (k_insert.cu): no host
// round trip inside; the capacity check runs on the device and a batch that
// does not fit is re-launched after growing the buffers (the mesh is not
// touched by a launch that reports INS_GROW).
// Returns false when the candidate list outgrew the region buffers (the batch
// did nothing; the caller grows them and redoes it).  x->h_tot[3] = C.
bool insert_persistent(gdp2d_ctx* x, const gdp2d_params* p, int prefiltered, u32 reg_cap,
                       u32 c_est, u32 ncav, u32 rs, int isolate, u32 batch, u32& nv, u32& nt,
                       u32& ns, u32& flip_rounds, u32& rm_rounds, cudaEvent_t start_ev) {
    cudaStream_t st = x->st;
    // Smaller batches run the persistent kernels on fewer co-resident CTAs:
    // their phases have little parallel work and a grid barrier's cost grows
    // with the CTA count (measured: cfg 2 42.6 -> 40.5 ms with the half grid
    // below 100K candidates; identical output for any grid size).
    const int div = c_est < x->eighth_grid_c     ? 8
                    : c_est < x->quarter_grid_c ? 4
                    : c_est < x->half_grid_c    ? 2
                                                : 1;
    // Mid-size batches: both kernels as ONE thread-block cluster, whose
    // barriers are hardware cluster barriers (~0.2 us) instead of grid
    // barriers (~1.2 us); same output for any grid size or launch shape.
    const bool as_cluster = x->cluster_size > 0 && c_est < x->cluster_c;
    const int g_ins =
        as_cluster ? x->cluster_size : std::max(1, x->insert_grid / div);
    static const int rb_div = [] {
        const char* e = std::getenv("GDP2D_RB_DIV");   // experiments: extra divisor, rollback kernel
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    const int g_rb =
        as_cluster ? x->cluster_size : std::max(1, x->rollback_grid / (div * rb_div));
    bool started = false;   // an earlier attempt got past the filter and plan
    int grow = 0;
    for (int attempt = 0;; ++attempt) {
        if (attempt > 0) CK(cudaMemsetAsync(x->ring, 0, 5 * sizeof(RoundCtr), st));
        InsertLaunch L = base_launch(x, p, batch, ncav, rs, isolate);
        L.resume = started ? 1 : 0;
        L.prefiltered = prefiltered;
        L.planned = prefiltered && !isolate;
        L.reg_cap = reg_cap;
        L.cluster = as_cluster ? 1 : 0;
        if (x->tr.on) {
            L.trace = x->tr.d_trace;
            L.trace_val = x->tr.d_trace_val;
            L.trace_n = x->tr.d_trace_n;
            L.trace_cap = Tracer::kCap;
            CK(cudaMemsetAsync(x->tr.d_trace_n, 0, sizeof(u32), st));
        }
        x->tr.mark("pre_ins", st);
        // word 8 = unsafe flag stays; attempt 0's words were zeroed by the scan
        if (attempt > 0) CK(cudaMemsetAsync(x->ins_state, 0, 8 * sizeof(u32), st));
        // the caller's last phase event marks the kernel start when nothing
        // was queued since (each event record costs ~3 us of stream time)
        cudaEvent_t k_start = start_ev;
        if (attempt > 0 || x->tr.on || !start_ev) {
            CK(cudaEventRecord(x->ev_k[0], st));
            k_start = x->ev_k[0];
        }
        const int mode = p->mode == GDP2D_CHEW ? 1 : 0;
        if (!x->check) {
            // (the split/rollback boundary comes from the kernels' start stamps)
            launch_insert_persistent(L, mode, g_ins, g_rb, st, nullptr, 1 | 2);
        } else {
            // GDP2D_CHECK=1: structural validation after each kernel
            launch_insert_persistent(L, mode, g_ins, g_rb, st, x->ev_k[1], 1);
            check_structure_now(x, x->work.m.nV, x->work.m.nT, x->work.m.nS, "split kernel");
            launch_insert_persistent(L, mode, g_ins, g_rb, st, nullptr, 2);
            check_structure_now(x, x->work.m.nV, x->work.m.nT, x->work.m.nS, "rollback kernel");
        }
        CK(cudaEventRecord(x->ev_k[2], st));
        x->tr.mark("insert_kernel", st);
        CK(cudaGetLastError());
        // status words, totals, C and the counters in one copy
        CK(cudaMemcpyAsync(x->h_status, x->status, kStatusWords * sizeof(u32),
                           cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const u32 C = x->h_tot[3];
        if (x->h_state[0] == 3u) return false;   // INS_REGIONS
        nv = x->h_tot[0];
        nt = x->h_tot[1];
        ns = x->h_tot[2];
        if (x->h_state[0] == 1u) {   // INS_GROW
            if (++grow > 2) throw Fail{GDP2D_ECAPACITY, "insertion does not fit after growth"};
            started = true;
            ensure_mesh(x, x->work.m.nV + nv, x->work.m.nT + nt, x->work.m.nS + ns);
            ensure_fresh(x, nv);
            ensure_worklists(x, 12ull * nv);
            continue;
        }
        if (x->h_state[0] == 2u) throw Fail{GDP2D_EMESH, "insertion exceeded its step bound"};
        {
            // roofline instrumentation of the two persistent kernels
            const Counters& h = *x->h_ctr;
            const u64 ins = h.ins_mid + h.ins_cc;
            const u64 f_split = x->h_state[7];
            const u64 f_rb = h.flips >= f_split ? h.flips - f_split : 0;
            const u64 b_split = 32ull * C + 128ull * ins + 128ull * f_split;
            const u64 b_rb = 64ull * nv + 128ull * f_rb + 128ull * h.rm_done;
            x->k_launches += 1;
            // the pair's span by events, split at the rollback kernel's
            // start (globaltimer stamps in state words 10-13; GDP2D_CHECK
            // records an event between the launches instead)
            const double pair = ev_ms(k_start, x->ev_k[2]) * 1e-3;
            double s_split;
            if (x->check) {
                s_split = ev_ms(k_start, x->ev_k[1]) * 1e-3;
            } else {
                u64 t0, t1;
                std::memcpy(&t0, x->h_state + 10, sizeof t0);
                std::memcpy(&t1, x->h_state + 12, sizeof t1);
                s_split = t1 > t0 ? std::min(pair, double(t1 - t0) * 1e-9) : 0.0;
            }
            x->k_split_s += s_split;
            x->k_split_b += b_split;
            x->k_rb_s += pair - s_split;
            x->k_rb_b += b_rb;
            x->k_rb_launches += 1;
        }
        x->round += x->h_state[1] + 1;
        flip_rounds = x->h_state[2];
        rm_rounds = x->h_state[3];
        x->work.m.nV += nv;
        x->work.m.nT += nt;
        x->work.m.nS += ns;
        return true;
    }
}

// Algorithmic bytes of one Line-3 scan: every element reads its 1 B cached
// verdict, every subsegment reads alive + the sticky encroached flag (5 B); a
// re-evaluated (dirty) element moves its 16 B record + three 16 B corner
// gathers (64 B, SURVEY 8(d)'s per-triangle figure; the subsegment record +
// apex gathers are taken as the same 64 B) and every element writes its 1 B
// flag (k_collect_flags).  When the timed region includes the scatter (the
// no-round-trip path), each candidate adds its element's record + corners
// (64 B) and its 41 B candidate record.
u64 scan_alg_bytes(u64 nT, u64 nS, u64 dirty, u64 cands, bool scatter) {
    return 2 * (nT + nS) + 5 * nS + 64 * dirty + (scatter ? 105 * cands : 0);
}

// The bookkeeping of one finished batch (alive counts, record_batch metrics,
// ruleskit.hpp:128-142, the Little's-law measurement, the report totals);
// bm.phase_seconds is filled by the caller.  Returns the retained insertions.
u32 account_batch(gdp2d_ctx* x, gdp2d_report* r, gdp2d_batch_metrics& bm, u32 attempted,
                  const Counters& h, u32 nt, u32 flip_rounds, u32 rm_rounds) {
    const u32 inserted = h.ins_mid + h.ins_cc;
    const u32 retained = inserted - std::min(inserted, h.rm_done);
    x->alive_v += inserted;
    x->alive_v -= std::min<ull>(x->alive_v, h.rm_done);
    x->alive_t += nt;
    x->alive_t -= std::min<ull>(x->alive_t, 2ull * h.rm_done);
    x->alive_s += h.ins_mid;
    bm.attempted = attempted;
    bm.concurrency = retained;
    bm.latency = 0;
    for (double s : bm.phase_seconds) bm.latency += s;
    bm.throughput = bm.latency > 0 ? retained / bm.latency : 0.0;
    x->little.record(attempted, retained, bm.latency);
    bm.waste_fraction = attempted ? double(attempted - retained) / attempted : 0.0;
    bm.walk_steps = h.walk_steps;
    bm.cavity_visits = h.cavity_visits;
    bm.survivors_claim = h.surv_claim;
    bm.survivors_cavity = h.surv_cavity;
    bm.inserted_midpoints = h.ins_mid;
    bm.inserted_circumcenters = h.ins_cc;
    bm.removed_redundant = h.rm_red;
    bm.removed_dependent = h.rm_dep;
    bm.dropped = h.dropped;
    bm.marked_encroached = h.marked;
    bm.flips = h.flips;
    bm.flip_rounds = flip_rounds;
    bm.removal_rounds = rm_rounds;
    bm.removals_kept = h.rm_kept;
    if (r->batches && r->n_batches < r->batches_capacity) r->batches[r->n_batches] = bm;
    r->n_batches++;
    r->total_candidates += attempted;
    r->total_walk_steps += h.walk_steps;
    r->total_cavity_visits += h.cavity_visits;
    r->total_inserted += inserted;
    r->total_flips += h.flips;
    r->total_removed += h.rm_done;
    r->sum_tris_alive += bm.tris_alive;
    r->sum_verts_alive += bm.verts_alive;
    r->sum_subsegs_alive += bm.subsegs_alive;
    return retained;
}

// k_tail_loop on the working mesh (see its header in k_insert.cu): up to
// `budget` batches; `ran` = batches done.  Returns true when the refinement
// is finished.
bool tail_loop(gdp2d_ctx* x, const gdp2d_params* p, const Quality& q, gdp2d_report* r,
               u32 ncav, u64 budget, u64& ran) {
    cudaStream_t st = x->st;
    const int isolate = ncav == 0 ? 0
                        : p->insert_mode == GDP2D_INSERT_ISOLATED   ? 1
                        : p->insert_mode == GDP2D_INSERT_PRECEDENCE ? 2
                                                                    : 0;
    const u32 rs = isolate ? isolated_stride(ncav) : ncav + 1 + MAX_CLAIM_EXTRA;
    // every buffer a batch of <= small_c candidates needs (nothing grows inside)
    ensure_regions(x, x->small_c, ncav, rs);
    ensure_fresh(x, x->small_c);
    ensure_worklists(x, 12ull * x->small_c);
    const u32 reg_cap = (u32)std::min<size_t>(x->reg_cap / rs, x->rl_cap);
    const u32 nb_max = (u32)std::min<u64>(budget, kTailMax);
    InsertLaunch L = base_launch(x, p, x->epoch + 1, ncav, rs, isolate);
    L.w.dlist = x->dlist;
    L.w.dlist_n = x->dlist + DLIST_CAP;
    L.w.dlist_cap = DLIST_CAP;
    L.reg_cap = reg_cap;
    TailArgs t;
    t.rec = x->tail_rec;
    t.max_batches = nb_max;
    t.klist = x->small_list + SMALL_LIST_CAP + 1;
    t.klist_n = x->small_list + 2 * SMALL_LIST_CAP + 1;
    t.q = q;
    t.out = x->tail_out;
    CK(cudaMemsetAsync(x->d_ctr, 0, sizeof(Counters), st));
    CK(cudaEventRecord(x->ev[0], st));
    launch_tail_loop(L, t, p->mode == GDP2D_CHEW ? 1 : 0, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(x->h_tail_out, x->tail_out, 8 * sizeof(u32), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(x->h_tail_rec, x->tail_rec, sizeof(TailRec) * nb_max,
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const u32 exitr = x->h_tail_out[0], nb = x->h_tail_out[1];
    ran = nb;
    bool done = false;
    for (u32 k = 0; k < nb; ++k) {
        const TailRec& rec = x->h_tail_rec[k];
        if (rec.ctr.err_code) {
            *x->h_ctr = rec.ctr;
            raise_dev_err(x);
        }
        gdp2d_batch_metrics bm;
        std::memset(&bm, 0, sizeof bm);
        bm.batch_index = r->n_batches;
        bm.tris_alive = x->alive_t;
        bm.verts_alive = x->alive_v;
        bm.subsegs_alive = x->alive_s;
        bm.phase_seconds[GDP2D_PH_COLLECT] = double(rec.t1 - rec.t0) * 1e-9;
        bm.phase_seconds[GDP2D_PH_INSERT] = double(rec.t2 - rec.t1) * 1e-9;
        r->scan_seconds += double(rec.t1 - rec.t0) * 1e-9;
        r->scan_bytes += 64ull * rec.ctr.scan_dirty + 105ull * rec.attempted;
        r->scan_launches += 1;
        const u32 retained =
            account_batch(x, r, bm, rec.attempted, rec.ctr, rec.nt, rec.flip_rounds, rec.rm_rounds);
        if (retained == 0 && rec.ctr.marked == 0) done = true;
    }
    if (exitr == TAIL_ERR) throw Fail{GDP2D_EMESH, "tail loop: device error"};
    x->epoch += nb;
    x->round = x->h_tail_out[5] - 1;
    x->work.m.nV = x->h_tail_out[2];
    x->work.m.nT = x->h_tail_out[3];
    x->work.m.nS = x->h_tail_out[4];
    x->c_prev = x->h_tail_out[6];
    x->have_c_prev = true;
    // after BIG / GROW the klist is the list of the batch the host runs next;
    // NOKEYS: the dirty list overflowed, the host collects from scratch
    x->klist_ok = exitr != TAIL_NOKEYS;
    if (exitr == TAIL_NOKEYS || exitr == TAIL_GROW || exitr == TAIL_BIG) x->klist_ok = false;
    if (exitr == TAIL_DONE) done = true;
    return done;
}

// The refinement loop (refine.hpp:651-713) on the working mesh.
void refine_loop(gdp2d_ctx* x, const gdp2d_params* p, gdp2d_report* r) {
    const auto wall0 = std::chrono::steady_clock::now();
    cudaStream_t st = x->st;
    const Quality q = make_quality(p);
    const u32 ncav = p->rule2_filtering_enabled ? p->cavity_n : 0;
    if (ncav > (u32)MAX_CAVITY_N) throw Fail{GDP2D_EINVAL, "cavity_n exceeds 64"};
    const gdp2d_report keep = *r;
    const unsigned long long launches0 = gdp2d::launch_counter();
    std::memset(r, 0, sizeof *r);
    r->batches = keep.batches;
    r->batches_capacity = keep.batches_capacity;
    x->k_split_s = x->k_rb_s = 0;
    x->k_split_b = x->k_rb_b = x->k_launches = x->k_rb_launches = 0;
    x->have_c_prev = false;
    x->klist_ok = false;
    x->dlist_on = false;
    x->little.reset();
    CK(cudaEventRecord(x->ev[GDP2D_NPHASES + 1], st));  // loop start
    for (u64 iter = 0;; ++iter) {
        if (iter >= p->iteration_cap) {
            r->iteration_cap_hit = 1;
            break;
        }
        // The long tail of small batches: run them back to back on the device
        // (k_tail_loop) while the list stays small; the loop returns here when
        // it does not, or the refinement is done.
        if (x->tail_on && x->have_c_prev && x->klist_ok && x->c_prev <= x->small_c &&
            !x->tr.on && !x->check && p->rule4_unified_collection != 0 &&
            p->batch_size_cap == 0) {
            u64 ran = 0;
            const bool done = tail_loop(x, p, q, r, ncav, p->iteration_cap - iter, ran);
            iter += ran;
            if (done) break;
            --iter;   // the for loop's increment: the next batch is iteration iter + ran
            continue;
        }
        DevMesh& m = x->work.m;
        gdp2d_batch_metrics bm;
        std::memset(&bm, 0, sizeof bm);
        bm.batch_index = r->n_batches;
        bm.tris_alive = x->alive_t;
        bm.verts_alive = x->alive_v;
        bm.subsegs_alive = x->alive_s;
        CK(cudaMemsetAsync(x->d_ctr, 0, sizeof(Counters), st));
        ensure_cands(x, m.nS + m.nT);
        CK(cudaEventRecord(x->ev[0], st));
        x->tr.mark("start", st);
        CollectCache cache;
        cache.full = (x->full_scan || x->full_collect) ? 1 : 0;
        cache.zero[0] = reinterpret_cast<u32*>(x->ring);
        cache.zero_n[0] = (u32)(5 * sizeof(RoundCtr) / 4);
        cache.zero[1] = x->ins_state;
        cache.zero_n[1] = 9;   // status words + the unsafe flag
        bool tris_scanned = false;
        // No host round trip after collect (ncs): the count stays on the
        // device; the filter kernels read it, the loop learns it with the
        // batch's end-of-batch readback.  The first batch of a call, the
        // batch caps and rule 4 off take the synchronous path.
        // Little's-law sizing needs C on the host only where a cap can
        // apply: a measured cap level exists and the previous batch came
        // within half of it (batches shrink over a refinement)
        const u64 little_lv = p->little_batch_sizing ? x->little.level() : 0;
        const bool little_sync = little_lv && (u64)x->c_prev * 2 > little_lv;
        const bool ncs = !x->sync_collect && x->have_c_prev &&
                         p->rule4_unified_collection != 0 && p->batch_size_cap == 0 &&
                         !little_sync;
        const bool small = ncs && x->c_prev <= x->small_collect_c;
        x->dlist_on = small;   // its rewrites feed a tail loop's next collect
        u32 C = launch_collect(m, q, p->rule4_unified_collection != 0, x->flags, x->c, x->ccap,
                               x->scan, x->d_ctr, st, cache, &tris_scanned, x->d_C,
                               nullptr, ncs ? nullptr : x->ev[GDP2D_NPHASES + 3], !ncs,
                               small ? x->small_list : nullptr, x->dlist + DLIST_CAP);
        // the no-round-trip collect is timed to ev[1], scatter included (one
        // event record less per batch)
        const cudaEvent_t scan_end = ncs ? x->ev[1] : x->ev[GDP2D_NPHASES + 3];
        // a full scan has refreshed every cached verdict it covered; with
        // rule 4 off and subsegment candidates, triangles were not scanned
        if (tris_scanned) x->full_scan = false;
        CK(cudaGetLastError());
        // scan bytes (scan_alg_bytes); the dirty count arrives with the
        // end-of-batch counters
        const u64 scan_nT = m.nT, scan_nS = m.nS;
        r->scan_launches += 1;
        x->tr.mark("collect", st);
        if (!ncs && C == 0) {
            check_dev_err(x);
            r->scan_seconds += ev_ms(x->ev[0], x->ev[GDP2D_NPHASES + 3]) * 1e-3;
            r->scan_bytes += scan_alg_bytes(scan_nT, scan_nS, x->h_ctr->scan_dirty, 0, false);
            break;
        }
        // Batch sizing (refine.hpp:252-261 + the Little's-law cap): keep the
        // highest priorities; the list keeps its order, the rest is dead
        u64 cap = p->batch_size_cap;
        if (p->little_batch_sizing && !ncs) {
            const u64 lc = x->little.cap(C);
            if (lc && (cap == 0 || lc < cap)) cap = lc;
        }
        u32 attempted = (!ncs && cap > 0 && C > cap) ? (u32)cap : C;
        if (!ncs && attempted < C) launch_select_topk(x->c, C, attempted, x->sel_state, st);
        // split points are fused into collect: one event ends both phases
        CK(cudaEventRecord(x->ev[1], st));
        bool filtered_events = false;   // ev[3..5] recorded (standalone filters)
        // isolated insertion needs the cavity filter (rule 2)
        const int isolate = ncav == 0 ? 0
                            : p->insert_mode == GDP2D_INSERT_ISOLATED   ? 1
                            : p->insert_mode == GDP2D_INSERT_PRECEDENCE ? 2
                                                                        : 0;
        const u32 rs = isolate ? isolated_stride(ncav) : ncav + 1 + MAX_CLAIM_EXTRA;
        if (!ncs) ensure_regions(x, C, ncav, rs);
        u32 reg_cap = (u32)std::min<size_t>(x->reg_cap / rs, x->rl_cap);
        if (ncs && x->regions_tight) reg_cap = std::min(reg_cap, x->c_prev / 2);
        // (the scan zeroed the step ring, the status words and the unsafe flag)
        const u32 batch = ++x->epoch;
        u32 flip_rounds = 0, rm_rounds = 0;
        u32 nv = 0, nt = 0, ns = 0;
        {
            // Lines 5-7 as high-occupancy standalone kernels for big batches
            // (they skip C <= small_c: the batch kernel filters in one CTA)
            NArg na = NArg::host(C);
            bool standalone = C > std::max(x->small_c, x->standalone_c);
            if (ncs) {
                standalone = x->c_prev > std::max(x->small_c, x->standalone_c);   // predicted
                na.d_n = x->d_C;
                na.skip_le = x->small_c;
                na.cap = reg_cap;
                na.grid_n = (u32)std::min<u64>((u64)m.nS + m.nT,
                                               std::max<u64>(x->c_prev + x->c_prev / 2, 4096));
            }
            if (standalone) {
                launch_locate(m, x->c, na, x->d_ctr, st);
                CK(cudaEventRecord(x->ev[3], st));
                launch_claim(m, x->c, na, x->aux, x->d_ctr, st);
                CK(cudaEventRecord(x->ev[4], st));
                if (isolate)
                    launch_cavity_isolated(m, x->c, na, ncav, rs, p->mode == GDP2D_CHEW ? 1 : 0,
                                           p->split_depth_cap, isolate == 1, x->aux, x->regions,
                                           x->region_len, x->ins_state + 8, x->d_ctr, st);
                else
                    launch_cavity(m, x->c, na, ncav, 2, x->aux, x->regions,
                                  x->region_len, nullptr, x->d_ctr, st, &x->ib,
                                  p->split_depth_cap);
                CK(cudaEventRecord(x->ev[5], st));
                filtered_events = true;
            }
            // (tail batch: everything runs inside the block-mode kernels; the
            // filter phases get no events of their own)
            if (!insert_persistent(x, p, standalone ? 1 : 0, reg_cap, ncs ? x->c_prev : C, ncav,
                                   rs, isolate, batch, nv, nt, ns, flip_rounds, rm_rounds,
                                   standalone ? x->ev[5] : x->ev[1])) {
                // the list outgrew the region buffers: grow them, redo the batch
                // (collect recomputes the same list from its cached verdicts)
                // (the redo takes the synchronous path: it knows C exactly);
                // C = NONE: the small-list collect overflowed, nothing to grow
                if (x->h_tot[3] != NONE) ensure_regions(x, x->h_tot[3], ncav, rs);
                --x->epoch;
                x->c_prev = x->h_tot[3] != NONE ? x->h_tot[3] : x->c_prev;
                x->have_c_prev = false;
                --iter;
                continue;
            }
            if (ncs) {
                C = x->h_tot[3];
                attempted = C;
            }
        }
        r->scan_seconds += ev_ms(x->ev[0], scan_end) * 1e-3;
        x->c_prev = C;
        x->have_c_prev = true;
        if (C == 0) {   // ncs: the batch found no candidates (its kernels did nothing)
            raise_dev_err(x);
            r->scan_bytes += scan_alg_bytes(scan_nT, scan_nS, x->h_ctr->scan_dirty, 0, true);
            --x->epoch;
            break;
        }
        // end of the insertion phase: the rollback kernel's end event
        const cudaEvent_t ins_end = x->ev_k[2];
        x->tr.mark("sync", st);
        x->tr.flush(bm.batch_index, st);
        if (x->tr.on)
            fprintf(stderr, "[trace] batch %u counters: C=%u surv=%u/%u mid=%u cc=%u red=%u dep=%u "
                            "marked=%u flips=%llu rm=%u\n",
                    bm.batch_index, C, x->h_ctr->surv_claim, x->h_ctr->surv_cavity,
                    x->h_ctr->ins_mid, x->h_ctr->ins_cc, x->h_ctr->rm_red, x->h_ctr->rm_dep,
                    x->h_ctr->marked, (unsigned long long)x->h_ctr->flips, x->h_ctr->rm_done);
        CK(cudaGetLastError());
        raise_dev_err(x);   // counters came back with the insertion's status
        const Counters& h = *x->h_ctr;
        r->scan_bytes += scan_alg_bytes(scan_nT, scan_nS, h.scan_dirty, C, ncs);
        // metrics (record_batch, ruleskit.hpp:128-142)
        bm.phase_seconds[GDP2D_PH_COLLECT] = ev_ms(x->ev[0], x->ev[1]) * 1e-3;
        bm.phase_seconds[GDP2D_PH_SPLIT_POINTS] = 0.0;   // fused into collect
        if (filtered_events) {
            bm.phase_seconds[GDP2D_PH_LOCATE] = ev_ms(x->ev[1], x->ev[3]) * 1e-3;
            bm.phase_seconds[GDP2D_PH_CLAIM] = ev_ms(x->ev[3], x->ev[4]) * 1e-3;
            bm.phase_seconds[GDP2D_PH_CAVITY] = ev_ms(x->ev[4], x->ev[5]) * 1e-3;
            bm.phase_seconds[GDP2D_PH_INSERT] = ev_ms(x->ev[5], ins_end) * 1e-3;
        } else {   // filtered inside the batch kernel
            bm.phase_seconds[GDP2D_PH_INSERT] = ev_ms(x->ev[1], ins_end) * 1e-3;
        }
        x->klist_ok = small && C != NONE;   // the next batch may take the tail loop
        const u32 retained = account_batch(x, r, bm, attempted, h, nt, flip_rounds, rm_rounds);
        if (retained == 0 && h.marked == 0) break;
    }
    // the batches kept vert_tri for their own fresh vertices only
    launch_vtri_rebuild(x->work.m, st);
    CK(cudaEventRecord(x->ev[GDP2D_NPHASES], st));
    CK(cudaEventSynchronize(x->ev[GDP2D_NPHASES]));
    if (const char* dbg = std::getenv("GDP2D_DEBUG"); dbg && dbg[0] == '1') {
        double h[4 + 2 * MAX_STAR];
        CK(cudaMemcpy(h, x->wl.dbg, sizeof h, cudaMemcpyDeviceToHost));
        if (h[0] != 0.0) {
            fprintf(stderr, "gdp2d debug: kept removal k=%d v=(%.17g, %.17g) link:", (int)h[1], h[2], h[3]);
            for (int q = 0; q < (int)h[1] && q < MAX_STAR; ++q)
                fprintf(stderr, " (%.17g, %.17g)", h[4 + 2 * q], h[5 + 2 * q]);
            fprintf(stderr, "\n");
        }
    }
    r->device_seconds = ev_ms(x->ev[GDP2D_NPHASES + 1], x->ev[GDP2D_NPHASES]) * 1e-3;
    r->kernel_launches = gdp2d::launch_counter() - launches0;
    r->split_seconds = x->k_split_s;
    r->split_bytes = x->k_split_b;
    r->split_launches = x->k_launches;
    r->rollback_seconds = x->k_rb_s;
    r->rollback_bytes = x->k_rb_b;
    r->rollback_launches = x->k_rb_launches;
    r->wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
}

void fill_summary(gdp2d_ctx* x, const gdp2d_params* p, gdp2d_report* r) {
    const QualitySummary s = launch_quality(x->work.m, make_quality(p), x->qscratch, x->st);
    r->output_points = s.alive_v;
    r->steiner_points = s.steiner;
    r->bad_triangles = s.bad;
    r->bad_area_percent = s.total_area > 0 ? s.bad_area / s.total_area * 100.0 : 0.0;
    r->min_angle_deg = s.min_angle;
    r->max_edge = s.max_edge;
}

}  // namespace


// ---- Line 1 on the device (k_cdt.cu) ------------------------------------------------

namespace {

template <class T>
void cdt_grow(T*& p, u32& cap, size_t n) {
    (void)cap;
    dfree(p);
    dalloc(p, n);
}

void build_cdt(gdp2d_ctx* x, const double* xy, u32 N, const u32* seg, u32 M,
               gdp2d_cdt_report* rep) {
    if (N < 3) throw Fail{GDP2D_ECDT, "need at least 3 points"};
    if (!xy || (M && !seg)) throw Fail{GDP2D_EINVAL, "missing point / segment arrays"};
    if (N >= (1u << 29) - 8) throw Fail{GDP2D_EINVAL, "too many points"};
    for (u32 i = 0; i < M; ++i) {
        const u32 a = seg[2 * i], b = seg[2 * i + 1];
        if (a >= N || b >= N) throw Fail{GDP2D_EINVAL, "segment endpoint out of range"};
        if (a == b) throw Fail{GDP2D_ECDT, "degenerate segment"};
    }
    cudaStream_t st = x->st;
    auto& c = x->cdt;
    const u32 T = 2 * N + 1;          // triangles of the DT of N points inside the super triangle
    const u32 pcap = 2 * M + 1024;    // pieces (segments + collinear splits)
    cudaEvent_t e0, e1, e2, e3;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&e2));
    CK(cudaEventCreate(&e3));
    struct EvFree {
        cudaEvent_t* e;
        ~EvFree() { for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]); }
    };
    cudaEvent_t evs[4] = {e0, e1, e2, e3};
    EvFree evfree{evs};
    CK(cudaEventRecord(e0, st));

    // working mesh: the DT of the points + super triangle
    MeshStore& w = x->work;
    w.m.nV = w.m.nT = w.m.nS = 0;
    mesh_reserve(w, N + 3, T, pcap, st);
    ensure_aux(x);
    ensure_worklists(x, 3ull * T + (1u << 20));
    DevMesh& m = w.m;
    CK(cudaMemcpyAsync(m.xy, xy, 16ull * N, cudaMemcpyHostToDevice, st));
    if (c.bbox == nullptr) {
        dalloc(c.bbox, 4);
        dalloc(c.ring, 4);
        dalloc(c.state, 16);
    }
    CK(cudaMemsetAsync(x->d_ctr, 0, sizeof(Counters), st));
    launch_cdt_bbox(m.xy, N, c.bbox, x->d_ctr, st);
    ull hb[4];
    CK(cudaMemcpyAsync(hb, c.bbox, sizeof hb, cudaMemcpyDeviceToHost, st));
    check_dev_err(x);   // synchronises
    const auto unkey = [](ull k) {
        const ull b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
        double d;
        std::memcpy(&d, &b, 8);
        return d;
    };
    const double x0 = unkey(hb[0]), y0 = unkey(hb[1]), x1 = unkey(hb[2]), y1 = unkey(hb[3]);
    const double R = std::max(x1 - x0, y1 - y0);
    if (!(R > 0)) throw Fail{GDP2D_ECDT, "duplicate point"};
    const double cx = 0.5 * (x0 + x1), cy = 0.5 * (y0 + y1), K = 32.0 * R;
    const double2 sup[3] = {make_double2(cx - K, cy - K), make_double2(cx + K, cy - K),
                            make_double2(cx, cy + K)};
    CK(cudaMemcpyAsync(m.xy + N, sup, sizeof sup, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(m.vkind, 0, N + 3, st));
    CK(cudaMemsetAsync(m.vbirth, 0, 4ull * (N + 3), st));
    CK(cudaMemsetAsync(m.valive, 1, N + 3, st));
    CK(cudaMemsetAsync(m.vtri, 0xFF, 4ull * (N + 3), st));
    const uint4 t0v[3] = {make_uint4(N, N + 1, N + 2, 1u), make_uint4(NONE, NONE, NONE, 0u),
                          make_uint4(NONE, NONE, NONE, 0u)};
    const TriRec t0r = {t0v[0], t0v[1]};
    CK(cudaMemcpyAsync(m.tr, &t0r, sizeof t0r, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(m.ts, &t0v[2], 16, cudaMemcpyHostToDevice, st));
    m.nV = N + 3;
    m.nT = T;
    m.nS = 0;

    // builder scratch
    if (N > c.ncap) {
        const u32 n2 = N + N / 4 + 1024;
        cdt_grow(c.ptri, c.ncap, n2);
        cdt_grow(c.pedge, c.ncap, n2);
        cdt_grow(c.pother, c.ncap, n2);
        cdt_grow(c.pkey, c.ncap, n2);
        cdt_grow(c.pwin, c.ncap, n2);
        c.ncap = n2;
    }
    if (T > c.tcap) {
        const u32 t2 = T + T / 4 + 1024;
        cdt_grow(c.tkey, c.tcap, t2);
        cdt_grow(c.newid, c.tcap, t2);
        cdt_grow(c.pool, c.tcap, t2);
        cdt_grow(c.queue, c.tcap, t2);
        c.pool_cap = t2;
        const u32 cc2 = 2 * t2 + (1u << 20);
        cdt_grow(c.claims, c.claim_cap, cc2);
        c.claim_cap = cc2;
        const u32 sc2 = 3 * t2 + (1u << 20);
        cdt_grow(c.seeds, c.seed_cap, sc2);
        c.seed_cap = sc2;
        c.tcap = t2;
    }
    if (pcap > c.pcap) {
        cdt_grow(c.pc, c.pcap, pcap);
        cdt_grow(c.ppar, c.pcap, pcap);
        cdt_grow(c.plist[0], c.pcap, pcap);
        cdt_grow(c.plist[1], c.pcap, pcap);
        cdt_grow(c.poff, c.pcap, pcap);
        cdt_grow(c.plen, c.pcap, pcap);
        cdt_grow(c.plive, c.pcap, pcap);
        cdt_grow(c.pmap, c.pcap, pcap);
        c.pcap = pcap;
    }
    int g1 = cdt_grid(x->device, 0), g2 = cdt_grid(x->device, 1);
    // segment recovery is latency-bound with few rounds: below 300K pieces one
    // CTA per SM (measured 1.7 -> 1.1 ms at 100K segments)
    if (M < 300000) g2 = std::max(1, g2 / 2);
    if (const char* e = std::getenv("GDP2D_CDT_GRID")) {   // experiments
        const int g = std::atoi(e);
        if (g > 0) {
            g1 = std::min(g1, g);
            g2 = std::min(g2, g);
        }
    }
    if ((u32)std::max(g1, g2) > c.part_cap) {
        c.part_cap = (u32)std::max(g1, g2);
        dfree(c.part);
        dalloc(c.part, c.part_cap);
    }
    CK(cudaMemsetAsync(c.tkey, 0xFF, 8ull * T, st));
    CK(cudaMemsetAsync(c.ring, 0, 4 * sizeof(RoundCtr), st));
    CK(cudaMemsetAsync(c.state, 0, 16 * sizeof(u32), st));

    CdtArgs a{};
    a.m = m;
    a.N = N;
    a.stride0 = 1;
    {
        // GDP2D_CDT_LEVELS=1: insertion levels of 32x (the first keeps >= 256
        // points).  Measured slower at 1M (9.3 vs 7.7 ms: 24 vs 20 rounds, 154
        // vs 94 Lawson rounds) -- the rounds are flip-bound, not scan-bound.
        const char* e = std::getenv("GDP2D_CDT_LEVELS");
        const bool levels = e && e[0] == '1';
        while (levels && (u64)N / ((u64)a.stride0 * 32) >= 256) a.stride0 *= 32;
    }
    a.x = x->aux;
    a.w = x->wl;
    a.w.vdirty = nullptr;
    a.w.fresh_n = 0;
    a.ring = c.ring;
    a.state = c.state;
    a.ctr = x->d_ctr;
    a.round0 = x->round + 1;
    a.ptri = c.ptri;
    a.pedge = c.pedge;
    a.pother = c.pother;
    a.pkey = c.pkey;
    a.pwin = c.pwin;
    a.tkey = c.tkey;
    a.part = c.part;
    a.pc = c.pc;
    a.ppar = c.ppar;
    a.plist[0] = c.plist[0];
    a.plist[1] = c.plist[1];
    a.poff = c.poff;
    a.plen = c.plen;
    a.claims = c.claims;
    a.seeds = c.seeds;
    a.pool = c.pool;
    a.queue = c.queue;
    a.pcap = c.pcap;
    a.claim_cap = c.claim_cap;
    a.seed_cap = c.seed_cap;
    a.pool_cap = c.pool_cap;

    // 1. Delaunay triangulation (one persistent launch)
    launch_cdt_delaunay(a, g1, st);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, st));
    u32 hs[16];
    CK(cudaMemcpyAsync(hs, c.state, sizeof hs, cudaMemcpyDeviceToHost, st));
    check_dev_err(x);
    if (hs[0] != T) throw Fail{GDP2D_ECDT, "CDT insertion rounds stopped early"};
    const u32 ins_rounds = hs[CDT_ST_ROUNDS], ins_flip_rounds = hs[CDT_ST_FLIP_ROUNDS];
    x->round += hs[CDT_ST_STEPS] + 8;

    // 2. segment recovery
    u32 np = M, found = 0, pipes = 0, splits = 0, rec_rounds = 0, pmax = 0, nseeds = 0;
    if (M) {
        std::vector<u32> iota(M);
        for (u32 i = 0; i < M; ++i) iota[i] = i;
        CK(cudaMemcpyAsync(c.pc, seg, 8ull * M, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(c.ppar, iota.data(), 4ull * M, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(c.plist[0], iota.data(), 4ull * M, cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(c.ring, 0, 4 * sizeof(RoundCtr), st));
        CK(cudaMemsetAsync(c.state, 0, 16 * sizeof(u32), st));
        CK(cudaMemcpyAsync(c.state + CDT_ST_NPIECES, &M, 4, cudaMemcpyHostToDevice, st));
        a.round0 = x->round + 1;
        launch_cdt_recover(a, M, g2, st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(hs, c.state, sizeof hs, cudaMemcpyDeviceToHost, st));
        check_dev_err(x);   // synchronises (iota stays alive until here)
        np = hs[CDT_ST_NPIECES];
        found = hs[CDT_ST_FOUND];
        pipes = hs[CDT_ST_PIPES];
        splits = hs[CDT_ST_SPLITS];
        rec_rounds = hs[CDT_ST_RECOVER_ROUNDS];
        pmax = hs[CDT_ST_PIPE_MAX];
        nseeds = std::min(hs[CDT_ST_SEEDS], c.seed_cap);
        x->round += hs[12] + 8;
    }
    CK(cudaEventRecord(e2, st));

    // 3. cut away the super triangle's fan; constrained Lawson from the pipes
    launch_cdt_strip(m, N, st);
    u32 fin_rounds = 0;
    if (nseeds) {
        CK(cudaMemcpyAsync(x->wl.w[0], c.seeds, 4ull * nseeds, cudaMemcpyDeviceToDevice, st));
        lawson_from(x, 0, nseeds, &fin_rounds);
        check_dev_err(x);
    }
    // subsegment ids: live pieces in (segment, position along it) order
    u32 nS = 0;
    CK(cudaMemsetAsync(c.plive, 0, 4ull * np, st));
    launch_cdt_piece_live(m, c.plive, st);
    if (splits == 0) {
        u32* d_tot = x->d_res;
        scan_exclusive(c.plive, c.newid, np, d_tot, x->scan, st);
        launch_cdt_pmap(c.plive, c.newid, c.pmap, np, st);
        CK(cudaMemcpyAsync(&nS, d_tot, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    } else {
        std::vector<uint2> hpc(np);
        std::vector<u32> hpar(np), hlive(np), hmap(np, NONE);
        CK(cudaMemcpyAsync(hpc.data(), c.pc, 8ull * np, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hpar.data(), c.ppar, 4ull * np, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hlive.data(), c.plive, 4ull * np, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::vector<std::pair<std::pair<u32, double>, u32>> order;
        for (u32 p = 0; p < np; ++p) {
            if (!hlive[p]) continue;
            const u32 par = hpar[p];
            const u32 sa = seg[2 * par], sb = seg[2 * par + 1], u = hpc[p].x;
            const double dx = xy[2 * sb] - xy[2 * sa], dy = xy[2 * sb + 1] - xy[2 * sa + 1];
            const double t = (xy[2 * u] - xy[2 * sa]) * dx + (xy[2 * u + 1] - xy[2 * sa + 1]) * dy;
            order.push_back({{par, t}, p});
        }
        std::sort(order.begin(), order.end());
        for (const auto& o : order) hmap[o.second] = nS++;
        CK(cudaMemcpyAsync(c.pmap, hmap.data(), 4ull * np, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
    // compaction into the context's input mesh
    launch_alive_flags(m, c.newid, st);
    // newid doubles as the flag array: scan in place is not supported, use the pool
    u32* flags = reinterpret_cast<u32*>(c.pool);
    CK(cudaMemcpyAsync(flags, c.newid, 4ull * T, cudaMemcpyDeviceToDevice, st));
    scan_exclusive(flags, c.newid, T, x->d_res, x->scan, st);
    u32 nTf = 0;
    CK(cudaMemcpyAsync(&nTf, x->d_res, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (nTf == 0) throw Fail{GDP2D_ECDT, "all points collinear"};
    MeshStore& pr = x->pristine;
    pr.m.nV = pr.m.nT = pr.m.nS = 0;
    mesh_reserve(pr, N, nTf, std::max<u32>(nS, 1), st);
    pr.m.nV = N;
    pr.m.nT = nTf;
    pr.m.nS = nS;
    launch_cdt_compact(m, pr.m, N, c.newid, c.pc, c.ppar, c.pmap, np, st);
    CK(cudaGetLastError());
    x->pristine_epoch = 0;
    x->p_alive_v = N;
    x->p_alive_t = nTf;
    x->p_alive_s = nS;
    x->n_in = 0;
    x->in_valid = false;
    reset_work(x);
    CK(cudaEventRecord(e3, st));
    CK(cudaStreamSynchronize(st));
    float ms01 = 0, ms12 = 0, ms23 = 0;
    cudaEventElapsedTime(&ms01, e0, e1);
    cudaEventElapsedTime(&ms12, e1, e2);
    cudaEventElapsedTime(&ms23, e2, e3);
    if (rep) {
        rep->struct_size = sizeof(gdp2d_cdt_report);
        rep->n_triangles = nTf;
        rep->n_subsegments = nS;
        rep->insert_rounds = ins_rounds;
        rep->flip_rounds = ins_flip_rounds;
        rep->recover_rounds = rec_rounds;
        rep->segments_present = found;
        rep->pipes_recovered = pipes;
        rep->collinear_splits = splits;
        rep->max_pipe = pmax;
        rep->final_flip_rounds = fin_rounds;
        rep->reserved = 0;
        rep->flips = x->h_ctr->flips;
        rep->delaunay_seconds = ms01 * 1e-3;
        rep->recover_seconds = ms12 * 1e-3;
        rep->finish_seconds = ms23 * 1e-3;
        rep->seconds = (ms01 + ms12 + ms23) * 1e-3;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

namespace {
int run_guarded(const std::function<void()>& fn) {
    try {
        fn();
        return GDP2D_OK;
    } catch (const Fail& f) {
        g_err = f.what;
        return f.code;
    } catch (const CudaError& e) {
        g_err = e.what;
        return GDP2D_ECUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return GDP2D_EINTERNAL;
    }
}

void upload_cands(gdp2d_ctx* x, const gdp2d_candidate* c, u32 n) {
    ensure_cands(x, n);
    std::vector<double2> pt(n);
    std::vector<u64> key(n);
    std::vector<u32> id(n), tie(n), loc(n);
    std::vector<uint8_t> kind(n), alive(n), lk(n, 0), fb(n);
    std::vector<int8_t> le(n, -1);
    for (u32 i = 0; i < n; ++i) {
        pt[i] = make_double2(c[i].x, c[i].y);
        double meas = c[i].measure;
        u64 bits;
        std::memcpy(&bits, &meas, 8);
        key[i] = ((u64)(c[i].band ? 1 : 0) << 63) | (bits & 0x7FFFFFFFFFFFFFFFull);
        id[i] = c[i].id;
        tie[i] = c[i].tiebreak;
        loc[i] = c[i].located;
        kind[i] = c[i].kind == GDP2D_CAND_SUBSEG ? 0 : 1;
        alive[i] = c[i].alive ? 1 : 0;
        fb[i] = c[i].fallback;
    }
    cudaStream_t st = x->st;
    CK(cudaMemcpyAsync(x->c.pt, pt.data(), 16ull * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(x->c.key, key.data(), 8ull * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(x->c.id, id.data(), 4ull * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(x->c.tie, tie.data(), 4ull * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(x->c.loc, loc.data(), 4ull * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(x->c.kind, kind.data(), n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(x->c.alive, alive.data(), n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(x->c.lkind, lk.data(), n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(x->c.ledge, le.data(), n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(x->c.fb, fb.data(), n, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
}

void download_cands(gdp2d_ctx* x, gdp2d_candidate* c, u32 n) {
    std::vector<double2> pt(n);
    std::vector<u64> key(n);
    std::vector<u32> id(n), tie(n), loc(n);
    std::vector<uint8_t> kind(n), alive(n), fb(n);
    cudaStream_t st = x->st;
    CK(cudaMemcpyAsync(pt.data(), x->c.pt, 16ull * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(key.data(), x->c.key, 8ull * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(id.data(), x->c.id, 4ull * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(tie.data(), x->c.tie, 4ull * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(loc.data(), x->c.loc, 4ull * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(kind.data(), x->c.kind, n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(alive.data(), x->c.alive, n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(fb.data(), x->c.fb, n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (u32 i = 0; i < n; ++i) {
        c[i].x = pt[i].x;
        c[i].y = pt[i].y;
        const u64 bits = key[i] & 0x7FFFFFFFFFFFFFFFull;
        std::memcpy(&c[i].measure, &bits, 8);
        c[i].band = (uint8_t)(key[i] >> 63);
        c[i].id = id[i];
        c[i].tiebreak = tie[i];
        c[i].located = loc[i];
        c[i].kind = kind[i] == 0 ? GDP2D_CAND_SUBSEG : GDP2D_CAND_TRI;
        c[i].alive = alive[i];
        c[i].fallback = fb[i];
    }
}

constexpr int kMaxDevices = 64;
std::mutex g_cache_mu[kMaxDevices];
gdp2d_ctx* g_cache[kMaxDevices] = {};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        cudaSetDevice(d);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

extern "C" {

const char* gdp2d_last_error(void) { return g_err.c_str(); }
const char* gdp2d_version(void) { return "gdp2d-b200 0.1 (sm_100a)"; }

uint64_t gdp2d_kernel_launches(void) { return __atomic_load_n(&launch_counter(), __ATOMIC_RELAXED); }

size_t gdp2d_struct_size(int which) {
    switch (which) {
        case 0: return sizeof(gdp2d_mesh_view);
        case 1: return sizeof(gdp2d_mesh_buf);
        case 2: return sizeof(gdp2d_params);
        case 3: return sizeof(gdp2d_batch_metrics);
        case 4: return sizeof(gdp2d_report);
        case 5: return sizeof(gdp2d_candidate);
        case 6: return sizeof(gdp2d_validation);
        case 7: return sizeof(gdp2d_node_ele);
        case 8: return sizeof(gdp2d_cdt_report);
        case 9: return sizeof(gdp2d_aos_layout);
        case 10: return sizeof(gdp2d_aos_mesh);
        default: return 0;
    }
}

void gdp2d_params_init(gdp2d_params* p, double theta_deg, double ell, uint32_t mode) {
    std::memset(p, 0, sizeof *p);
    p->theta_deg = theta_deg;
    // refine.hpp:195-196, evaluated on the host exactly as the reference does
    const double c = std::cos(theta_deg * 3.14159265358979323846 / 180.0);
    p->cos2_theta = c * c;
    p->ell = ell;
    p->mode = mode;
    p->cavity_n = 32;
    p->rule1_compaction_threshold = 1024;
    p->rule2_filtering_enabled = 1;
    p->rule4_unified_collection = 1;
    p->little_batch_sizing = 1;   // measured-C/L sizing (LittleSizer), on by default
    p->insert_mode = GDP2D_INSERT_ROLLBACK;
    p->reserved0 = 0;
    p->iteration_cap = 10000;
    p->split_depth_cap = 64;
    p->batch_size_cap = 0;
}

int gdp2d_ctx_create(gdp2d_ctx** out, int device) {
    if (!out) return GDP2D_EINVAL;
    *out = nullptr;
    gdp2d_ctx* x = new gdp2d_ctx();
    const int rc = run_guarded([&] { ctx_init(x, device); });
    if (rc != GDP2D_OK) {
        ctx_release(x);
        delete x;
        return rc;
    }
    *out = x;
    return GDP2D_OK;
}

void gdp2d_ctx_destroy(gdp2d_ctx* x) {
    if (!x) return;
    ctx_release(x);
    delete x;
}

int gdp2d_ctx_upload(gdp2d_ctx* x, const gdp2d_mesh_view* in) {
    if (!x) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] {
        upload(x, in);
        reset_work(x);
        CK(cudaStreamSynchronize(x->st));
    });
}

int gdp2d_ctx_reset(gdp2d_ctx* x) {
    if (!x) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] { reset_work(x); });
}

int gdp2d_ctx_refine(gdp2d_ctx* x, const gdp2d_params* p, gdp2d_report* r) {
    if (!x || !p || !r) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] {
        refine_loop(x, p, r);
        fill_summary(x, p, r);
    });
}

int gdp2d_ctx_download(gdp2d_ctx* x, gdp2d_mesh_buf* out) {
    if (!x || !out) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] { download(x, out); });
}

uint64_t gdp2d_ctx_device_bytes(gdp2d_ctx* x) {
    if (!x) return 0;
    const MeshStore& w = x->work;
    const MeshStore& p = x->pristine;
    auto mesh_bytes = [](const MeshStore& s) {
        return (u64)s.vcap * (16 + 1 + 4 + 1 + 4) + (u64)s.tcap * 48 + (u64)s.scap * (8 + 4 + 4 + 1 + 4 + 4);
    };
    return mesh_bytes(w) + mesh_bytes(p) + (u64)x->aux_cap * (8 + 8 + 4 + 4 + 12) + x->flags_cap +
           (u64)x->ccap * 41 + x->reg_cap * 4 + (u64)x->wl.cap * 21 +
           (u64)x->wl.rm_cap * (4 * MAX_STAR + 30);
}

int gdp2d_refine(const gdp2d_mesh_view* in, gdp2d_mesh_buf* out, const gdp2d_params* p,
                 gdp2d_report* r, int device) {
    if (!in || !out || !p || !r) return GDP2D_EINVAL;
    if (device < 0 || device >= kMaxDevices) return GDP2D_ENODEVICE;
    std::lock_guard<std::mutex> lock(g_cache_mu[device]);
    if (!g_cache[device]) {
        const int rc = gdp2d_ctx_create(&g_cache[device], device);
        if (rc) return rc;
    }
    gdp2d_ctx* x = g_cache[device];
    return run_guarded([&] {
        DeviceGuard g(x->device);
        // e2e clock: from the held lock and a live context to the refined
        // mesh in host memory; refine_loop sets wall_seconds (loop only)
        const auto t0 = std::chrono::steady_clock::now();
        upload(x, in);
        reset_work(x, p->theta_deg);
        refine_loop(x, p, r);
        download(x, out);
        r->e2e_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        fill_summary(x, p, r);
    });
}

int gdp2d_refine_aos(const gdp2d_aos_layout* layout, gdp2d_aos_mesh* mesh,
                     const gdp2d_params* p, gdp2d_report* r, int device) {
    if (!layout || !mesh || !mesh->resize || !p || !r) return GDP2D_EINVAL;
    if (device < 0 || device >= kMaxDevices) return GDP2D_ENODEVICE;
    std::lock_guard<std::mutex> lock(g_cache_mu[device]);
    if (!g_cache[device]) {
        const int rc = gdp2d_ctx_create(&g_cache[device], device);
        if (rc) return rc;
    }
    gdp2d_ctx* x = g_cache[device];
    return run_guarded([&] {
        DeviceGuard g(x->device);
        const auto t0 = std::chrono::steady_clock::now();
        upload_aos(x, layout, mesh);
        reset_work(x, p->theta_deg);
        refine_loop(x, p, r);
        download_aos(x, layout, mesh);
        r->e2e_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        fill_summary(x, p, r);
    });
}

int gdp2d_warmup(int device) {
    if (device < 0 || device >= kMaxDevices) return GDP2D_ENODEVICE;
    std::lock_guard<std::mutex> lock(g_cache_mu[device]);
    if (!g_cache[device]) {
        const int rc = gdp2d_ctx_create(&g_cache[device], device);
        if (rc) return rc;
    }
    gdp2d_ctx* x = g_cache[device];
    return run_guarded([&] {
        DeviceGuard g(x->device);
        // unit square + five interior points: every Line-1 and refinement
        // kernel launches at least once
        static const double xy[] = {0.0,  0.0,  1.0,  0.0,  1.0,  1.0,  0.0,  1.0,  0.31,
                                    0.27, 0.72, 0.33, 0.45, 0.71, 0.18, 0.62, 0.83, 0.79};
        static const uint32_t seg[] = {0, 1, 1, 2, 2, 3, 3, 0};
        build_cdt(x, xy, 9, seg, 4, nullptr);
        gdp2d_params p;
        gdp2d_params_init(&p, 30.0, std::numeric_limits<double>::infinity(), GDP2D_RUPPERT);
        gdp2d_report r;
        std::memset(&r, 0, sizeof r);
        refine_loop(x, &p, &r);
    });
}

void* gdp2d_pinned_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
        g_err = "cudaHostAlloc failed";
        return nullptr;
    }
    return p;
}

void gdp2d_pinned_free(void* p) {
    if (p) cudaFreeHost(p);
}

void gdp2d_release_cached(void) {
    for (int d = 0; d < kMaxDevices; ++d) {
        std::lock_guard<std::mutex> lock(g_cache_mu[d]);
        if (g_cache[d]) gdp2d_ctx_destroy(g_cache[d]);
        g_cache[d] = nullptr;
    }
}

int gdp2d_ctx_sizes(gdp2d_ctx* x, uint32_t* v, uint32_t* t, uint32_t* s) {
    if (!x || !v || !t || !s) return GDP2D_EINVAL;
    *v = x->work.m.nV;
    *t = x->work.m.nT;
    *s = x->work.m.nS;
    return GDP2D_OK;
}

int gdp2d_ctx_download_to(gdp2d_ctx* x, gdp2d_mesh_buf* dst) {
    if (!x || !dst) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] { download_into(x, dst); });
}

void gdp2d_free(gdp2d_mesh_buf* b) {
    if (!b) return;
    void* ptrs[] = {b->xy,      b->vert_kind, b->vert_birth, b->vert_alive, b->vert_tri,
                    b->tri_v,   b->tri_n,     b->tri_seg,    b->tri_alive,  b->seg_v,
                    b->seg_parent, b->seg_encroached, b->seg_alive, b->seg_tri};
    for (void* q : ptrs) std::free(q);
    std::memset(b, 0, sizeof *b);
}

int gdp2d_collect(gdp2d_ctx* x, const gdp2d_params* p, gdp2d_candidate* out, uint32_t cap,
                  uint32_t* n) {
    if (!x || !p || !n) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    int status = GDP2D_OK;
    const int rc = run_guarded([&] {
        DevMesh& m = x->work.m;
        ensure_cands(x, m.nS + m.nT);
        CK(cudaMemsetAsync(x->d_ctr, 0, sizeof(Counters), x->st));
        CollectCache cache;
        cache.full = 1;
        bool tris_scanned = false;
        u32 C = launch_collect(m, make_quality(p), p->rule4_unified_collection != 0,
                               x->flags, x->c, x->ccap, x->scan, x->d_ctr, x->st, cache,
                               &tris_scanned, x->d_C);
        std::vector<gdp2d_candidate> tmp(C);
        if (C) {
            // batch_size_cap (refine.hpp:252-261): the kept candidates in list
            // order, with their original tiebreaks
            const bool capped = p->batch_size_cap > 0 && C > p->batch_size_cap;
            if (capped) launch_select_topk(x->c, C, (u32)p->batch_size_cap, x->sel_state, x->st);
            download_cands(x, tmp.data(), C);
            if (capped) {
                u32 k = 0;
                for (u32 i = 0; i < C; ++i)
                    if (tmp[i].alive) tmp[k++] = tmp[i];
                tmp.resize(k);
                C = k;
            }
        }
        *n = C;
        if (C > cap) {
            status = GDP2D_ECAPACITY;
            g_err = "candidate buffer too small";
        }
        if (out && C) std::memcpy(out, tmp.data(), sizeof(gdp2d_candidate) * std::min(C, cap));
    });
    return rc ? rc : status;
}

namespace {
// Input segments by parent index from the pristine mesh: the chain endpoints
// of each parent's subsegments (vertices of odd degree within the parent).
void derive_input_segments(gdp2d_ctx* x) {
    const DevMesh& pm = x->pristine.m;
    const u32 S = pm.nS;
    std::vector<uint2> sv(S);
    std::vector<u32> par(S);
    std::vector<uint8_t> al(S);
    if (S) {
        CK(cudaMemcpyAsync(sv.data(), pm.sv, sizeof(uint2) * S, cudaMemcpyDeviceToHost, x->st));
        CK(cudaMemcpyAsync(par.data(), pm.sparent, 4ull * S, cudaMemcpyDeviceToHost, x->st));
        CK(cudaMemcpyAsync(al.data(), pm.salive, S, cudaMemcpyDeviceToHost, x->st));
        CK(cudaStreamSynchronize(x->st));
    }
    u32 np = 0;
    for (u32 i = 0; i < S; ++i)
        if (al[i] && par[i] != GDP2D_NONE) np = std::max(np, par[i] + 1);
    std::vector<std::vector<u32>> ends(np);
    for (u32 i = 0; i < S; ++i) {
        if (!al[i] || par[i] == GDP2D_NONE) continue;
        auto& e = ends[par[i]];
        for (const u32 w : {sv[i].x, sv[i].y}) {
            auto it = std::find(e.begin(), e.end(), w);
            if (it == e.end()) e.push_back(w);
            else e.erase(it);
        }
    }
    std::vector<uint2> in(np, make_uint2(0, 0));
    for (u32 q = 0; q < np; ++q)
        if (ends[q].size() == 2) in[q] = make_uint2(ends[q][0], ends[q][1]);
    dfree(x->in_sv);
    dalloc(x->in_sv, std::max<u32>(np, 1));
    if (np) CK(cudaMemcpyAsync(x->in_sv, in.data(), sizeof(uint2) * np, cudaMemcpyHostToDevice, x->st));
    CK(cudaStreamSynchronize(x->st));
    x->n_in = np;
    x->in_valid = true;
}
}  // namespace

int gdp2d_ctx_validate(gdp2d_ctx* x, const gdp2d_params* p, gdp2d_validation* out) {
    if (!x || !p || !out) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] {
        if (!x->in_valid) derive_input_segments(x);
        VerifySummary v = launch_verify(x->work.m, make_quality(p), x->in_sv, x->n_in,
                                        x->vscratch, x->vscratch_bytes, x->d_val, x->st);
        if (v.scratch_needed) {
            if (x->vscratch) cudaFree(x->vscratch);
            x->vscratch_bytes = v.scratch_needed;
            CK(cudaMalloc(&x->vscratch, x->vscratch_bytes));
            v = launch_verify(x->work.m, make_quality(p), x->in_sv, x->n_in, x->vscratch,
                              x->vscratch_bytes, x->d_val, x->st);
        }
        CK(cudaGetLastError());
        out->structure_failure = v.structure_failure;
        out->structure_tri = v.structure_tri;
        out->cdt_violations = v.cdt_violations;
        out->bad_triangles = v.bad_triangles;
        out->conformity_failures = v.conformity_failures;
        out->min_angle_deg = v.min_angle_deg;
        out->mean_min_angle_deg = v.mean_min_angle_deg;
        for (int i = 0; i < GDP2D_HIST_BINS; ++i) out->min_angle_hist[i] = v.min_angle_hist[i];
    });
}

int gdp2d_ctx_build_cdt(gdp2d_ctx* x, const double* xy, uint32_t n_points, const uint32_t* seg,
                        uint32_t n_segments, gdp2d_cdt_report* rep) {
    if (!x) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] { build_cdt(x, xy, n_points, seg, n_segments, rep); });
}

int gdp2d_build_cdt(const double* xy, uint32_t n_points, const uint32_t* seg,
                    uint32_t n_segments, gdp2d_mesh_buf* out, gdp2d_cdt_report* rep,
                    int device) {
    if (!out) return GDP2D_EINVAL;
    if (device < 0 || device >= kMaxDevices) return GDP2D_ENODEVICE;
    std::lock_guard<std::mutex> lock(g_cache_mu[device]);
    if (!g_cache[device]) {
        const int rc = gdp2d_ctx_create(&g_cache[device], device);
        if (rc) return rc;
    }
    gdp2d_ctx* x = g_cache[device];
    return run_guarded([&] {
        DeviceGuard g(x->device);
        build_cdt(x, xy, n_points, seg, n_segments, rep);
        download(x, out);
    });
}

int gdp2d_ctx_export(gdp2d_ctx* x, gdp2d_node_ele* out) {
    if (!x || !out || !out->xy || !out->marker || !out->tri) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] {
        const DevMesh& m = x->work.m;
        const u32 V = m.nV, T = m.nT;
        cudaStream_t st = x->st;
        // device scratch: flags + offsets + compacted outputs
        const size_t need = 8ull * V + 8ull * T + 16ull * V + V + 12ull * T + 64;
        if (need > x->vscratch_bytes) {
            if (x->vscratch) cudaFree(x->vscratch);
            x->vscratch_bytes = need;
            CK(cudaMalloc(&x->vscratch, need));
        }
        char* b = static_cast<char*>(x->vscratch);
        double2* xy = reinterpret_cast<double2*>(b);
        b += 16ull * V;
        u32* fv = reinterpret_cast<u32*>(b);
        u32* ov = fv + V;
        u32* ft = ov + V;
        u32* ot = ft + T;
        u32* tri = ot + T;
        u32* totals = tri + 3ull * T;
        uint8_t* marker = reinterpret_cast<uint8_t*>(totals + 4);
        launch_export(m, fv, ov, ft, ot, xy, marker, tri, totals, x->scan, st);
        CK(cudaGetLastError());
        u32 h[2];
        CK(cudaMemcpyAsync(h, totals, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        out->n_nodes = h[0];
        out->n_tris = h[1];
        if (h[0]) {
            CK(cudaMemcpyAsync(out->xy, xy, 16ull * h[0], cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(out->marker, marker, h[0], cudaMemcpyDeviceToHost, st));
        }
        if (h[1]) CK(cudaMemcpyAsync(out->tri, tri, 12ull * h[1], cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

int gdp2d_split_points(gdp2d_ctx* x, gdp2d_candidate* c, uint32_t n) {
    if (!x || (!c && n)) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] {
        if (!n) return;
        upload_cands(x, c, n);
        CK(cudaMemsetAsync(x->d_ctr, 0, sizeof(Counters), x->st));
        launch_split_points(x->work.m, x->c, n, x->d_ctr, x->st);
        CK(cudaGetLastError());
        download_cands(x, c, n);
    });
}

int gdp2d_locate(gdp2d_ctx* x, gdp2d_candidate* c, uint32_t n) {
    if (!x || (!c && n)) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] {
        if (!n) return;
        upload_cands(x, c, n);
        CK(cudaMemsetAsync(x->d_ctr, 0, sizeof(Counters), x->st));
        launch_locate(x->work.m, x->c, n, x->d_ctr, x->st);
        CK(cudaGetLastError());
        download_cands(x, c, n);
    });
}

int gdp2d_claim(gdp2d_ctx* x, gdp2d_candidate* c, uint32_t n) {
    if (!x || (!c && n)) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] {
        if (!n) return;
        upload_cands(x, c, n);
        CK(cudaMemsetAsync(x->d_ctr, 0, sizeof(Counters), x->st));
        launch_claim(x->work.m, x->c, n, x->aux, x->d_ctr, x->st);
        CK(cudaGetLastError());
        download_cands(x, c, n);
    });
}

int gdp2d_cavity(gdp2d_ctx* x, gdp2d_candidate* c, uint32_t n, uint32_t n_cav,
                 uint32_t* regions, uint32_t* region_len) {
    if (!x || (!c && n)) return GDP2D_EINVAL;
    if (n_cav > (u32)MAX_CAVITY_N) {
        g_err = "cavity_n exceeds 64";
        return GDP2D_EINVAL;
    }
    DeviceGuard g(x->device);
    return run_guarded([&] {
        if (!n) return;
        upload_cands(x, c, n);
        ensure_regions(x, n, n_cav);
        CK(cudaMemsetAsync(x->d_ctr, 0, sizeof(Counters), x->st));
        launch_cavity(x->work.m, x->c, n, n_cav, 0, x->aux, x->regions, x->region_len,
                      x->bfs_len, x->d_ctr, x->st);
        CK(cudaGetLastError());
        download_cands(x, c, n);
        if (regions && region_len) {
            const u32 rs = n_cav + 1 + MAX_CLAIM_EXTRA;
            std::vector<u32> reg((size_t)n * rs), len(n);
            CK(cudaMemcpyAsync(reg.data(), x->regions, 4ull * n * rs, cudaMemcpyDeviceToHost,
                               x->st));
            CK(cudaMemcpyAsync(len.data(), x->bfs_len, 4ull * n, cudaMemcpyDeviceToHost, x->st));
            CK(cudaStreamSynchronize(x->st));
            for (u32 i = 0; i < n; ++i) {
                region_len[i] = len[i];
                for (u32 k = 0; k < len[i]; ++k)
                    regions[(size_t)i * (n_cav + 1) + k] = reg[(size_t)i * rs + k];
            }
        }
    });
}

int gdp2d_flip_fixpoint(gdp2d_ctx* x, const uint32_t* seed_tri, const uint8_t* seed_edge,
                        uint32_t n, uint64_t* flips) {
    if (!x || (n && (!seed_tri || !seed_edge))) return GDP2D_EINVAL;
    DeviceGuard g(x->device);
    return run_guarded([&] {
        ensure_aux(x);
        if (n > x->wl.cap) throw Fail{GDP2D_ECAPACITY, "too many seeds"};
        std::vector<u32> codes(n);
        for (u32 i = 0; i < n; ++i) codes[i] = enc(seed_tri[i], seed_edge[i]);
        CK(cudaMemsetAsync(x->d_ctr, 0, sizeof(Counters), x->st));
        if (n)
            CK(cudaMemcpyAsync(x->wl.w[0], codes.data(), 4ull * n, cudaMemcpyHostToDevice,
                               x->st));
        u32 rounds = 0;
        lawson_from(x, 0, n, &rounds);
        check_dev_err(x);
        if (flips) *flips = x->h_ctr->flips;
    });
}

int gdp2d_predicates_batch(int device, int kind, const double* pts, uint32_t n,
                           const gdp2d_params* p, int8_t* out) {
    if ((n && (!pts || !out)) || kind < 0 || kind > 4) return GDP2D_EINVAL;
    return run_guarded([&] {
        int cnt = 0;
        if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt == 0)
            throw Fail{GDP2D_ENODEVICE, "no CUDA device visible"};
        DeviceGuard g(device);
        if (!n) return;
        const int arity = kind == GDP2D_PRED_INCIRCLE ? 4 : 3;
        double* dp = nullptr;
        int8_t* dout = nullptr;
        dalloc(dp, (size_t)n * arity * 2);
        dalloc(dout, n);
        CK(cudaMemcpy(dp, pts, 16ull * n * arity, cudaMemcpyHostToDevice));
        gdp2d_params def;
        if (!p) {
            gdp2d_params_init(&def, 20.0, INFINITY, 0);
            p = &def;
        }
        launch_predicates(kind, dp, n, make_quality(p), dout, 0);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, dout, n, cudaMemcpyDeviceToHost));
        dfree(dp);
        dfree(dout);
    });
}

int gdp2d_circumcenter_batch(int device, const double* pts, uint32_t n, double* out,
                             uint8_t* ok) {
    if (n && (!pts || !out || !ok)) return GDP2D_EINVAL;
    return run_guarded([&] {
        int cnt = 0;
        if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt == 0)
            throw Fail{GDP2D_ENODEVICE, "no CUDA device visible"};
        DeviceGuard g(device);
        if (!n) return;
        double *dp = nullptr, *dout = nullptr;
        uint8_t* dok = nullptr;
        dalloc(dp, 6ull * n);
        dalloc(dout, 2ull * n);
        dalloc(dok, n);
        CK(cudaMemcpy(dp, pts, 48ull * n, cudaMemcpyHostToDevice));
        launch_circumcenters(dp, n, dout, dok, 0);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, dout, 16ull * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(ok, dok, n, cudaMemcpyDeviceToHost));
        dfree(dp);
        dfree(dout);
        dfree(dok);
    });
}

}  // extern "C"
