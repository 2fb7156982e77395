// k_locate.cu -- Line 6 of Algorithm 1, point location (locate,
// refine.hpp:301-335 -> locate_point cdt.hpp:68-105 with subsegment
// interception).  One thread per candidate: walks average < 1 step (SURVEY
// §8a a13), so a lane-per-walk keeps every lane busy; the warp's walks are
// independent gathers that overlap in the memory system.
#include "engine.h"

namespace gdp2d {

__global__ void __launch_bounds__(256) k_locate(DevMesh m, DevCands c, u32 n, Counters* ctr) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    ull steps = 0;
    if (i < n && c.alive[i]) {
        if (c.kind[i] == 0) {
            c.loc[i] = m.stri[c.id[i]];
            c.lkind[i] = 4;   // subsegment midpoint: split along the subsegment
            c.ledge[i] = -1;
        } else {
            const double2 p = c.pt[i];
            const Loc loc = locate_point(m, c.id[i], p, true);
            steps = loc.steps;
            u32 hit = NONE;
            bool done = false;
            switch (loc.kind) {
                case 0:  // Inside
                    c.loc[i] = loc.tri;
                    c.lkind[i] = 0;
                    c.ledge[i] = -1;
                    done = true;
                    break;
                case 1: {  // OnEdge
                    const u32 s = comp(m.ts[loc.tri], loc.edge);
                    if (s == NONE) {
                        c.loc[i] = loc.tri;
                        c.lkind[i] = 1;
                        c.ledge[i] = (int8_t)loc.edge;
                        done = true;
                    } else {
                        hit = s;
                    }
                    break;
                }
                case 4:
                    hit = loc.seg;
                    break;
                default:  // OnVertex, OutsideHull
                    c.alive[i] = 0;
                    done = true;
                    break;
            }
            if (!done) {
                // Interception: split the blocking subsegment (refine.hpp:329-334).
                c.kind[i] = 0;
                c.id[i] = hit;
                c.pt[i] = subseg_mid(m, hit);
                c.key[i] = make_key(1, subseg_len(m, hit));
                c.loc[i] = m.stri[hit];
                c.lkind[i] = 4;
                c.ledge[i] = -1;
            }
        }
    }
    warp_add_ull(&ctr->walk_steps, steps);
}

void launch_locate(const DevMesh& m, DevCands c, u32 n, Counters* d_ctr, cudaStream_t st) {
    if (!n) return;
    note_launch(), k_locate<<<(n + 255) / 256, 256, 0, st>>>(m, c, n, d_ctr);
}

}  // namespace gdp2d
