// k_filter.cu -- Lines 6-7 of Algorithm 1 as standalone kernels for the
// gdp2d_claim / gdp2d_cavity parity entry points: the per-triangle claim
// (claim_filter, refine.hpp:367-376) and the cavity-approximation filter
// (cavity_filter, refine.hpp:382-429 -> expand, expandlist.hpp:93-157).  The
// per-candidate bodies live in gdp2d_phases.cuh and are the ones the
// persistent batch kernel runs.
#include <algorithm>

#include "gdp2d_phases.cuh"
#include "scan.cuh"

namespace gdp2d {

__global__ void k_claim_max(DevCands c, NArg na, u64* __restrict__ ckey) {
    const u32 n = narg(na);
    GRID_STRIDE(i, n) claim_max_one(c, i, ckey);
}

__global__ void k_claim_tie(DevCands c, NArg na, const u64* __restrict__ ckey,
                            u64* __restrict__ ctie) {
    const u32 n = narg(na);
    GRID_STRIDE(i, n) claim_tie_one(c, i, ckey, ctie);
}

__global__ void k_claim_check(DevCands c, NArg na, const u64* __restrict__ ckey,
                              const u64* __restrict__ ctie, Counters* ctr) {
    const u32 n = narg(na);
    u32 surv = 0;
    GRID_STRIDE(i, n) surv += claim_check_one(c, i, ckey, ctie);
    block_add<u32>(&ctr->surv_claim, surv);
}

__global__ void k_claim_reset(DevCands c, NArg na, u32 nT, u64* __restrict__ ckey,
                              u64* __restrict__ ctie) {
    const u32 n = narg(na);
    GRID_STRIDE(i, n) claim_reset_one(c, i, nT, ckey, ctie);
}

void launch_claim(const DevMesh& m, DevCands c, NArg n, TriAux a, Counters* d_ctr,
                  cudaStream_t st) {
    if (!n.grid_n) return;
    const u32 g = (n.grid_n + 255) / 256;
    note_launch(), k_claim_max<<<g, 256, 0, st>>>(c, n, a.ckey);
    note_launch(), k_claim_tie<<<g, 256, 0, st>>>(c, n, a.ckey, a.ctie);
    note_launch(), k_claim_check<<<g, 256, 0, st>>>(c, n, a.ckey, a.ctie, d_ctr);
    note_launch(), k_claim_reset<<<g, 256, 0, st>>>(c, n, m.nT, a.ckey, a.ctie);
}

#ifndef GDP2D_CAVITY_MINB
#define GDP2D_CAVITY_MINB 1
#endif
__global__ void __launch_bounds__(128, GDP2D_CAVITY_MINB) k_cavity_bfs(const __grid_constant__ DevMesh m, const __grid_constant__ DevCands c, NArg na, u32 ncav,
                                                    int extras, u32 rs,
                                                    u32* __restrict__ regions,
                                                    u32* __restrict__ region_len,
                                                    u32* __restrict__ bfs_len,
                                                    u64* __restrict__ ckey, Counters* ctr) {
    const u32 n = narg(na);
    ull visits = 0;
    GRID_STRIDE(i, n) visits += cavity_bfs_one(m, c, i, ncav, extras, rs, regions, region_len, bfs_len, ckey);
    block_add<ull>(&ctr->cavity_visits, visits);
}

// rewrite table (gdp2d_phases.cuh)
__global__ void k_rw_claim(DevMesh m, DevCands c, NArg na, u64* __restrict__ fkey) {
    const u32 n = narg(na);
    GRID_STRIDE(i, n) rw_claim_one(m, c, i, fkey);
}
__global__ void k_rw_tie(DevCands c, NArg na, const u64* __restrict__ fkey, u64* __restrict__ ftie) {
    const u32 n = narg(na);
    GRID_STRIDE(i, n) rw_tie_one(c, i, fkey, ftie);
}

__global__ void k_cavity_tie(DevCands c, NArg na, u32 rs, const u32* __restrict__ regions,
                             const u32* __restrict__ region_len, const u64* __restrict__ ckey,
                             u64* __restrict__ ctie) {
    const u32 n = narg(na);
    GRID_STRIDE(i, n) cavity_tie_one(c, i, rs, regions, region_len, ckey, ctie);
}

// fkey != null: a survivor must also own its rewritten triangles
__global__ void k_cavity_check(DevCands c, NArg na, u32 rs, const u32* __restrict__ regions,
                               const u32* __restrict__ region_len, const u64* __restrict__ ckey,
                               const u64* __restrict__ ctie, const u64* __restrict__ fkey,
                               const u64* __restrict__ ftie, Counters* ctr) {
    const u32 n = narg(na);
    u32 surv = 0;
    GRID_STRIDE(i, n) {
        const bool rw_ok = !fkey || !c.alive[i] || rw_owns(c, i, fkey, ftie);
        u32 sv = cavity_check_one(c, i, rs, regions, region_len, ckey, ctie);
        if (sv && !rw_ok) {
            c.alive[i] = 0;
            sv = 0;
        }
        surv += sv;
    }
    block_add<u32>(&ctr->surv_cavity, surv);
}

// plan.nv != null: the phase-1 plan of each survivor (plan_one) is made here,
// by every candidate's thread at full occupancy, instead of inside the
// persistent insertion kernel (InsertLaunch::planned).
__global__ void k_cavity_reset(const __grid_constant__ DevMesh m, DevCands c, NArg na, u32 rs,
                               const u32* __restrict__ regions,
                               const u32* __restrict__ region_len, u64* __restrict__ ckey,
                               u64* __restrict__ ctie, u64* __restrict__ fkey,
                               u64* __restrict__ ftie, InsertBufs plan, u64 depth_cap,
                               Counters* ctr) {
    const u32 n = narg(na);
    u32 dropped = 0;
    GRID_STRIDE(i, n) {
        cavity_reset_one(i, rs, regions, region_len, ckey, ctie);
        if (fkey) rw_reset_one(c, i, m.nT, fkey, ftie);
        if (plan.nv) {
            u32 nv, nt, ns;
            dropped += plan_one(m, c, i, depth_cap, nv, nt, ns);
            plan.nv[i] = nv;
            plan.nt[i] = nt;
            plan.ns[i] = ns;
        }
    }
    if (plan.nv) warp_add_u32(&ctr->dropped, dropped);
}

// ---- isolated claims (GDP2D_INSERT_ISOLATED, gdp2d_phases.cuh) ----

template <int MODE>
__global__ void __launch_bounds__(128) k_cavity_claims(const __grid_constant__ DevMesh m, const __grid_constant__ DevCands c, NArg na, u32 ncav,
                                                       u32 rs, u32* __restrict__ regions,
                                                       u32* __restrict__ region_len,
                                                       u64* __restrict__ ckey, u64 depth_cap,
                                                       int ring, Counters* ctr) {
    const u32 n = narg(na);
    ull visits = 0;
    GRID_STRIDE(i, n)
        visits += cavity_claims_one<MODE>(m, c, i, ncav, rs, regions, region_len, ckey, depth_cap,
                                          ring != 0);
    block_add<ull>(&ctr->cavity_visits, visits);
}

__global__ void k_isolated_check(DevMesh m, DevCands c, NArg na, u32 rs,
                                 const u32* __restrict__ regions,
                                 const u32* __restrict__ region_len, const u64* __restrict__ ckey,
                                 const u64* __restrict__ ctie, const u64* __restrict__ fkey,
                                 const u64* __restrict__ ftie, u32* unsafe_flag, Counters* ctr) {
    const u32 n = narg(na);
    u32 surv = 0, marked = 0, unsafe = 0;
    GRID_STRIDE(i, n) {
        if (c.alive[i] && !rw_owns(c, i, fkey, ftie)) {
            c.alive[i] = 0;
        } else {
            u32 mk = 0, us = 0;
            surv += isolated_check_one(m, c, i, rs, regions, region_len, ckey, ctie, mk, us);
            marked += mk;
            unsafe |= us;
        }
    }
    if (unsafe) atomicOr(unsafe_flag, 1u);
    block_add<u32>(&ctr->surv_cavity, surv);
    block_add<u32>(&ctr->marked, marked);
}

void launch_cavity_isolated(const DevMesh& m, DevCands c, NArg n, u32 ncav, u32 rs, int mode,
                            u64 depth_cap, bool ring, TriAux a, u32* regions, u32* region_len,
                            u32* unsafe_flag, Counters* d_ctr, cudaStream_t st) {
    if (!n.grid_n) return;
    if (mode == 0)
        note_launch(), k_cavity_claims<0><<<(n.grid_n + 127) / 128, 128, 0, st>>>(m, c, n, ncav, rs, regions, region_len, a.ckey, depth_cap, ring ? 1 : 0, d_ctr);
    else
        note_launch(), k_cavity_claims<1><<<(n.grid_n + 127) / 128, 128, 0, st>>>(m, c, n, ncav, rs, regions, region_len, a.ckey, depth_cap, ring ? 1 : 0, d_ctr);
    const u32 g = (n.grid_n + 255) / 256;
    note_launch(), k_rw_claim<<<g, 256, 0, st>>>(m, c, n, a.fkey);
    note_launch(), k_cavity_tie<<<g, 256, 0, st>>>(c, n, rs, regions, region_len, a.ckey, a.ctie);
    note_launch(), k_rw_tie<<<g, 256, 0, st>>>(c, n, a.fkey, a.ftie);
    note_launch(), k_isolated_check<<<g, 256, 0, st>>>(m, c, n, rs, regions, region_len, a.ckey, a.ctie, a.fkey, a.ftie, unsafe_flag, d_ctr);
    note_launch(), k_cavity_reset<<<g, 256, 0, st>>>(m, c, n, rs, regions, region_len, a.ckey, a.ctie, a.fkey, a.ftie, InsertBufs{}, 0, d_ctr);
}

void launch_cavity(const DevMesh& m, DevCands c, NArg n, u32 ncav, int extras, TriAux a,
                   u32* regions, u32* region_len, u32* bfs_len, Counters* d_ctr,
                   cudaStream_t st, const InsertBufs* plan, u64 depth_cap) {
    if (!n.grid_n) return;
    const u32 rs = ncav + 1 + MAX_CLAIM_EXTRA;
    const bool rw = extras >= 2;   // refinement: the rewrite table
    note_launch(), k_cavity_bfs<<<(n.grid_n + 127) / 128, 128, 0, st>>>(m, c, n, ncav, extras, rs, regions,
                                                   region_len, bfs_len, a.ckey, d_ctr);
    const u32 g = (n.grid_n + 255) / 256;
    if (rw) note_launch(), k_rw_claim<<<g, 256, 0, st>>>(m, c, n, a.fkey);
    note_launch(), k_cavity_tie<<<g, 256, 0, st>>>(c, n, rs, regions, region_len, a.ckey, a.ctie);
    if (rw) note_launch(), k_rw_tie<<<g, 256, 0, st>>>(c, n, a.fkey, a.ftie);
    note_launch(), k_cavity_check<<<g, 256, 0, st>>>(c, n, rs, regions, region_len, a.ckey, a.ctie,
                                                     rw ? a.fkey : nullptr, rw ? a.ftie : nullptr,
                                                     d_ctr);
    note_launch(), k_cavity_reset<<<g, 256, 0, st>>>(m, c, n, rs, regions, region_len, a.ckey,
                                                     a.ctie, rw ? a.fkey : nullptr,
                                                     rw ? a.ftie : nullptr,
                                                     plan ? *plan : InsertBufs{}, depth_cap,
                                                     d_ctr);
}

// Little's law against measured occupancy: the number of candidates the
// cavity filter (the heaviest per-candidate kernel) keeps in flight at once
// on this device -- SMs x resident CTAs x threads.  A batch larger than this
// only queues (latency grows linearly) while its waste (conflicts) grows.
u32 cavity_resident_candidates(int device) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cavity_bfs, 128, 0);
    return (u32)std::max(1, sms * std::max(1, per_sm) * 128);
}

}  // namespace gdp2d
