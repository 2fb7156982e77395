// k_locate.cu -- Line 6 of Algorithm 1, point location (locate,
// refine.hpp:301-335 -> locate_point cdt.hpp:68-105 with subsegment
// interception), as a standalone kernel for the gdp2d_locate parity entry
// point.  One thread per candidate: walks average < 1 step,
// so a lane-per-walk keeps every lane busy; the warp's walks are independent
// gathers that overlap in the memory system.  The refinement itself runs the
// same body (locate_one, gdp2d_phases.cuh) inside the persistent batch kernel.
#include "gdp2d_phases.cuh"
#include "scan.cuh"

namespace gdp2d {

__global__ void __launch_bounds__(256) k_locate(const __grid_constant__ DevMesh m,
                                                const __grid_constant__ DevCands c, NArg na,
                                                Counters* ctr) {
    const u32 n = narg(na);
    ull steps = 0;
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        steps += locate_one(m, c, i);
    block_add<ull>(&ctr->walk_steps, steps);
}

void launch_locate(const DevMesh& m, DevCands c, NArg n, Counters* d_ctr, cudaStream_t st) {
    if (!n.grid_n) return;
    note_launch(), k_locate<<<(n.grid_n + 255) / 256, 256, 0, st>>>(m, c, n, d_ctr);
}

}  // namespace gdp2d
