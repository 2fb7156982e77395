/* oracle/cdt_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's hot-path primitives (predicates,
 * quality test, collect + splitting points, locate, claim, cavity), written
 * from /root/reference/proj/include/cdtref/*.hpp and pinned against the
 * compiled reference itself (oracle/_ref/libcdtref_ref.so, see
 * tests/test_oracle.py).  It is the checker for the GPU path, never the
 * product: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.
 */
#ifndef CDT_ORACLE_H
#define CDT_ORACLE_H

#include <stdint.h>

#include "gdp2d.h"

#ifdef __cplusplus
extern "C" {
#endif

int orc_orient2d(const double* a, const double* b, const double* c);
int orc_incircle(const double* a, const double* b, const double* c, const double* d);
int orc_in_diametric(const double* sa, const double* sb, const double* p);
int orc_in_lens(const double* sa, const double* sb, const double* p);
int orc_circumcenter(const double* a, const double* b, const double* c, double* out);
int orc_is_bad(const double* a, const double* b, const double* c, double cos2, double ell);

/* batch form matching gdp2d_predicates_batch */
void orc_predicates_batch(int kind, const double* pts, uint32_t n, const gdp2d_params* p,
                          int8_t* out);

/* collect + compute_splitting_points; returns the candidate count. */
uint32_t orc_collect(const gdp2d_mesh_view* m, const gdp2d_params* p, gdp2d_candidate* out,
                     uint32_t cap);
void orc_locate(const gdp2d_mesh_view* m, gdp2d_candidate* c, uint32_t n);
void orc_claim(const gdp2d_mesh_view* m, gdp2d_candidate* c, uint32_t n);
/* regions: n*(n_cav+1) entries (may be NULL) */
void orc_cavity(const gdp2d_mesh_view* m, gdp2d_candidate* c, uint32_t n, uint32_t n_cav,
                uint32_t* regions, uint32_t* region_len);

#ifdef __cplusplus
}
#endif

#endif
