/* oracle/cdt_oracle.c -- TEST INFRASTRUCTURE ONLY (see cdt_oracle.h).
 *
 * Plain-C restatement of the reference hot-path primitives; every function
 * cites the reference file:line it restates.  Compiled with -ffp-contract=off
 * so the floating-point formulas evaluate exactly as the reference's.
 */
#include "cdt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define NONE 0xFFFFFFFFu
static const double kEps = 1.1102230246251565e-16; /* predicates.hpp:21 */

static int sgn(double d) { return (d > 0.0) - (d < 0.0); }
static int nx(int i) { return (i + 1) % 3; } /* mesh.hpp:97 */
static int pv(int i) { return (i + 2) % 3; } /* mesh.hpp:98 */

/* ---- expansion arithmetic (detail/expansion.hpp:21-94) ---------------------- */

static void two_sum(double a, double b, double* x, double* y) {
    const double s = a + b, bv = s - a, av = s - bv, br = b - bv, ar = a - av;
    *x = s;
    *y = ar + br;
}

static void two_prod(double a, double b, double* x, double* y) {
    *x = a * b;
    *y = fma(a, b, -*x);
}

static int exp_sum(const double* e, int el, const double* f, int fl, double* h) {
    int ei = 0, fi = 0, hi = 0;
    double q;
    if (fabs(f[0]) < fabs(e[0])) {
        q = f[0];
        fi = 1;
    } else {
        q = e[0];
        ei = 1;
    }
    while (ei < el || fi < fl) {
        double n, s, lo;
        if (ei >= el || (fi < fl && fabs(f[fi]) < fabs(e[ei])))
            n = f[fi++];
        else
            n = e[ei++];
        two_sum(q, n, &s, &lo);
        if (lo != 0.0) h[hi++] = lo;
        q = s;
    }
    if (q != 0.0 || hi == 0) h[hi++] = q;
    return hi;
}

static int exp_scale(const double* e, int el, double b, double* h) {
    int hi = 0;
    double px, py, q;
    two_prod(e[0], b, &px, &py);
    if (py != 0.0) h[hi++] = py;
    q = px;
    for (int i = 1; i < el; ++i) {
        double tx, ty, s1, l1, s2, l2;
        two_prod(e[i], b, &tx, &ty);
        two_sum(q, ty, &s1, &l1);
        if (l1 != 0.0) h[hi++] = l1;
        two_sum(tx, s1, &s2, &l2);
        if (l2 != 0.0) h[hi++] = l2;
        q = s2;
    }
    if (q != 0.0 || hi == 0) h[hi++] = q;
    return hi;
}

static int prod2(double a, double b, double* h) {
    double x, y;
    int n = 0;
    two_prod(a, b, &x, &y);
    if (y != 0.0) h[n++] = y;
    if (x != 0.0 || n == 0) h[n++] = x;
    return n;
}

static void acc_add(double* acc, int* n, double* t, int tl, int sign, double* tmp) {
    if (sign < 0)
        for (int i = 0; i < tl; ++i) t[i] = -t[i];
    const int m = exp_sum(acc, *n, t, tl, tmp);
    memcpy(acc, tmp, sizeof(double) * (size_t)m);
    *n = m;
}

/* exact orient2d determinant in raw coordinates (predicates.hpp:30-46) */
static int orient_exp(const double* a, const double* b, const double* c, double* out) {
    double p[2], tmp[16];
    int n = prod2(a[0], b[1], out), k;
    k = prod2(a[0], c[1], p); acc_add(out, &n, p, k, -1, tmp);
    k = prod2(b[0], c[1], p); acc_add(out, &n, p, k, +1, tmp);
    k = prod2(b[0], a[1], p); acc_add(out, &n, p, k, -1, tmp);
    k = prod2(c[0], a[1], p); acc_add(out, &n, p, k, +1, tmp);
    k = prod2(c[0], b[1], p); acc_add(out, &n, p, k, -1, tmp);
    return n;
}

/* ---- predicates ------------------------------------------------------------- */

/* orient2d (predicates.hpp:63-79) */
int orc_orient2d(const double* a, const double* b, const double* c) {
    const double dl = (a[0] - c[0]) * (b[1] - c[1]);
    const double dr = (a[1] - c[1]) * (b[0] - c[0]);
    const double det = dl - dr;
    if (dl > 0.0) {
        if (dr <= 0.0) return sgn(det);
    } else if (dl < 0.0) {
        if (dr >= 0.0) return sgn(det);
    } else {
        return (dr < 0.0) - (dr > 0.0);
    }
    const double ds = fabs(dl) + fabs(dr);
    if (fabs(det) > (3.0 + 16.0 * kEps) * kEps * ds) return sgn(det);
    double e[16];
    const int n = orient_exp(a, b, c, e);
    return sgn(e[n - 1]);
}

/* incircle (predicates.hpp:82-103, exact :50-59) */
int orc_incircle(const double* a, const double* b, const double* c, const double* d) {
    const double adx = a[0] - d[0], ady = a[1] - d[1];
    const double bdx = b[0] - d[0], bdy = b[1] - d[1];
    const double cdx = c[0] - d[0], cdy = c[1] - d[1];
    const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
    const double alift = adx * adx + ady * ady;
    const double cdxady = cdx * ady, adxcdy = adx * cdy;
    const double blift = bdx * bdx + bdy * bdy;
    const double adxbdy = adx * bdy, bdxady = bdx * ady;
    const double clift = cdx * cdx + cdy * cdy;
    const double det =
        alift * (bdxcdy - cdxbdy) + blift * (cdxady - adxcdy) + clift * (adxbdy - bdxady);
    const double perm = (fabs(bdxcdy) + fabs(cdxbdy)) * alift +
                        (fabs(cdxady) + fabs(adxcdy)) * blift +
                        (fabs(adxbdy) + fabs(bdxady)) * clift;
    if (fabs(det) > (10.0 + 96.0 * kEps) * kEps * perm) return sgn(det);
    const double* pts[4] = {a, b, c, d};
    double acc[400], tmp[400], term[100], orient[16], lift[4], part[32], p2[2], q2[2];
    int n = 1;
    acc[0] = 0.0;
    for (int k = 0; k < 4; ++k) {
        const double* p = pts[k];
        const int lp = prod2(p[0], p[0], p2), lq = prod2(p[1], p[1], q2);
        const int ll = exp_sum(p2, lp, q2, lq, lift);
        int on;
        if (k == 0) on = orient_exp(b, c, d, orient);
        else if (k == 1) on = orient_exp(a, c, d, orient);
        else if (k == 2) on = orient_exp(a, b, d, orient);
        else on = orient_exp(a, b, c, orient);
        int tn = 1;
        term[0] = 0.0;
        for (int i = 0; i < ll; ++i) {
            const int pn = exp_scale(orient, on, lift[i], part);
            const int m = exp_sum(term, tn, part, pn, tmp);
            memcpy(term, tmp, sizeof(double) * (size_t)m);
            tn = m;
        }
        acc_add(acc, &n, term, tn, (k & 1) ? -1 : +1, tmp);
    }
    return sgn(acc[n - 1]);
}

/* in_diametric_circle (predicates.hpp:107-119) */
int orc_in_diametric(const double* sa, const double* sb, const double* p) {
    const double ux = sa[0] - p[0], uy = sa[1] - p[1], vx = sb[0] - p[0], vy = sb[1] - p[1];
    const double d = ux * vx + uy * vy;
    const double mag = fabs(ux * vx) + fabs(uy * vy);
    if (fabs(d) > 8.0 * kEps * mag) return d < 0.0;
    double acc[20], tmp[20], t[2];
    int n = prod2(sa[0], sb[0], acc), k;
    k = prod2(sa[0], p[0], t); acc_add(acc, &n, t, k, -1, tmp);
    k = prod2(p[0], sb[0], t); acc_add(acc, &n, t, k, -1, tmp);
    k = prod2(p[0], p[0], t); acc_add(acc, &n, t, k, +1, tmp);
    k = prod2(sa[1], sb[1], t); acc_add(acc, &n, t, k, +1, tmp);
    k = prod2(sa[1], p[1], t); acc_add(acc, &n, t, k, -1, tmp);
    k = prod2(p[1], sb[1], t); acc_add(acc, &n, t, k, -1, tmp);
    k = prod2(p[1], p[1], t); acc_add(acc, &n, t, k, +1, tmp);
    return sgn(acc[n - 1]) < 0;
}

static int mul_exp(const double* a, int na, const double* b, int nb, double* out) {
    double part[64], tmp[2048];
    int n = 1;
    out[0] = 0.0;
    for (int i = 0; i < na; ++i) {
        const int pn = exp_scale(b, nb, a[i], part);
        const int m = exp_sum(out, n, part, pn, tmp);
        memcpy(out, tmp, sizeof(double) * (size_t)m);
        n = m;
    }
    return n;
}

/* in_diametral_lens (predicates.hpp:126-162) */
int orc_in_lens(const double* sa, const double* sb, const double* p) {
    if ((p[0] == sa[0] && p[1] == sa[1]) || (p[0] == sb[0] && p[1] == sb[1])) return 0;
    const double ux = sa[0] - p[0], uy = sa[1] - p[1], vx = sb[0] - p[0], vy = sb[1] - p[1];
    const double d = ux * vx + uy * vy;
    if (d >= 0.0) return 0;
    const double uu = ux * ux + uy * uy, vv = vx * vx + vy * vy;
    const double lhs = 4.0 * d * d, rhs = uu * vv;
    if (fabs(lhs - rhs) > 64.0 * kEps * (lhs + rhs)) return lhs >= rhs;
    double e[4][2];
    int ne[4];
    const double hi_in[4][2] = {{sa[0], p[0]}, {sa[1], p[1]}, {sb[0], p[0]}, {sb[1], p[1]}};
    for (int k = 0; k < 4; ++k) {
        double h, l;
        two_sum(hi_in[k][0], -hi_in[k][1], &h, &l);
        ne[k] = 0;
        if (l != 0.0) e[k][ne[k]++] = l;
        e[k][ne[k]++] = h;
    }
    double t1[16], t2[16], dote[32], ulen[32], vlen[32];
    int n1 = mul_exp(e[0], ne[0], e[2], ne[2], t1), n2 = mul_exp(e[1], ne[1], e[3], ne[3], t2);
    const int nd = exp_sum(t1, n1, t2, n2, dote);
    n1 = mul_exp(e[0], ne[0], e[0], ne[0], t1);
    n2 = mul_exp(e[1], ne[1], e[1], ne[1], t2);
    const int nu = exp_sum(t1, n1, t2, n2, ulen);
    n1 = mul_exp(e[2], ne[2], e[2], ne[2], t1);
    n2 = mul_exp(e[3], ne[3], e[3], ne[3], t2);
    const int nv = exp_sum(t1, n1, t2, n2, vlen);
    double sq[1100], uv[1100], res[2200];
    double four_d[32];
    for (int i = 0; i < nd; ++i) four_d[i] = 4.0 * dote[i];
    const int ns = mul_exp(four_d, nd, dote, nd, sq);
    const int nuv = mul_exp(ulen, nu, vlen, nv, uv);
    for (int i = 0; i < nuv; ++i) uv[i] = -uv[i];
    const int nr = exp_sum(sq, ns, uv, nuv, res);
    return sgn(dote[nd - 1]) < 0 && sgn(res[nr - 1]) >= 0;
}

/* circumcenter (predicates.hpp:172-185); returns well_conditioned */
int orc_circumcenter(const double* a, const double* b, const double* c, double* out) {
    const double abx = b[0] - a[0], aby = b[1] - a[1], acx = c[0] - a[0], acy = c[1] - a[1];
    const double d = 2.0 * (abx * acy - aby * acx);
    const double ab2 = abx * abx + aby * aby, ac2 = acx * acx + acy * acy;
    const double ux = (acy * ab2 - aby * ac2) / d;
    const double uy = (abx * ac2 - acx * ab2) / d;
    out[0] = a[0] + ux;
    out[1] = a[1] + uy;
    const double scale = ab2 < ac2 ? ac2 : ab2;
    return isfinite(out[0]) && isfinite(out[1]) && fabs(d) > 1e-12 * scale;
}

/* is_bad_triangle (refine.hpp:192-206) with the host cos^2(theta) */
int orc_is_bad(const double* a, const double* b, const double* c, double c2, double ell) {
    const double* p3[3] = {a, b, c};
    const double ell2 = ell * ell;
    for (int i = 0; i < 3; ++i) {
        const double* p = p3[i];
        const double ux = p3[nx(i)][0] - p[0], uy = p3[nx(i)][1] - p[1];
        const double vx = p3[pv(i)][0] - p[0], vy = p3[pv(i)][1] - p[1];
        if (isfinite(ell) && ux * ux + uy * uy > ell2) return 1;
        const double d = ux * vx + uy * vy;
        if (d > 0.0 && d * d > c2 * (ux * ux + uy * uy) * (vx * vx + vy * vy)) return 1;
    }
    return 0;
}

void orc_predicates_batch(int kind, const double* pts, uint32_t n, const gdp2d_params* p,
                          int8_t* out) {
    for (uint32_t i = 0; i < n; ++i) {
        const double* r = pts + (size_t)i * (kind == GDP2D_PRED_INCIRCLE ? 8 : 6);
        switch (kind) {
            case GDP2D_PRED_ORIENT2D: out[i] = (int8_t)orc_orient2d(r, r + 2, r + 4); break;
            case GDP2D_PRED_INCIRCLE: out[i] = (int8_t)orc_incircle(r, r + 2, r + 4, r + 6); break;
            case GDP2D_PRED_DIAMETRIC: out[i] = (int8_t)orc_in_diametric(r, r + 2, r + 4); break;
            case GDP2D_PRED_LENS: out[i] = (int8_t)orc_in_lens(r, r + 2, r + 4); break;
            default: out[i] = (int8_t)orc_is_bad(r, r + 2, r + 4, p->cos2_theta, p->ell);
        }
    }
}

/* ---- mesh-level primitives on the reference SoA layout ------------------------ */

#define XY(m, v) ((m)->xy + 2 * (size_t)(v))
#define TV(m, t, i) ((m)->tri_v[3 * (size_t)(t) + (i)])
#define TN(m, t, i) ((m)->tri_n[3 * (size_t)(t) + (i)])
#define TS(m, t, i) ((m)->tri_seg[3 * (size_t)(t) + (i)])

static int index_of_neighbor(const gdp2d_mesh_view* m, uint32_t t, uint32_t u) { /* mesh.hpp:107 */
    for (int i = 0; i < 3; ++i)
        if (TN(m, t, i) == u) return i;
    return -1;
}

static int pe(const gdp2d_mesh_view* m, uint32_t s, const double* p, int mode) { /* refine.hpp:180 */
    const double* a = XY(m, m->seg_v[2 * s]);
    const double* b = XY(m, m->seg_v[2 * s + 1]);
    return mode == GDP2D_CHEW ? orc_in_lens(a, b, p) : orc_in_diametric(a, b, p);
}

static int is_encroached(const gdp2d_mesh_view* m, uint32_t s, int mode) { /* refine.hpp:126,210 */
    const uint32_t t = m->seg_tri[s];
    for (int e = 0; e < 3; ++e) {
        if (TS(m, t, e) != s) continue;
        if (pe(m, s, XY(m, TV(m, t, e)), mode)) return 1;
        const uint32_t u = TN(m, t, e);
        if (u != NONE) {
            const int f = index_of_neighbor(m, u, t);
            if (f >= 0 && pe(m, s, XY(m, TV(m, u, f)), mode)) return 1;
        }
        break;
    }
    return 0;
}

static double sqd(const double* a, const double* b) {
    const double dx = a[0] - b[0], dy = a[1] - b[1];
    return dx * dx + dy * dy;
}

static int resolvable(const gdp2d_mesh_view* m, uint32_t t) { /* refine.hpp:169-178 */
    double mag = 0.0, len2 = 0.0;
    for (int i = 0; i < 3; ++i) {
        const double* p = XY(m, TV(m, t, i));
        mag = fmax(mag, fmax(fabs(p[0]), fabs(p[1])));
        len2 = fmax(len2, sqd(p, XY(m, TV(m, t, nx(i)))));
    }
    const double fl = mag * 1e-12;
    return len2 > fl * fl;
}

static void mid(const double* a, const double* b, double* o) { /* geometry.hpp:31 */
    o[0] = 0.5 * (a[0] + b[0]);
    o[1] = 0.5 * (a[1] + b[1]);
}

static void split_point(const gdp2d_mesh_view* m, gdp2d_candidate* c) { /* refine.hpp:267-296 */
    double o[2];
    c->fallback = 0;
    if (c->kind == GDP2D_CAND_SUBSEG) {
        mid(XY(m, m->seg_v[2 * c->id]), XY(m, m->seg_v[2 * c->id + 1]), o);
    } else {
        const uint32_t t = c->id;
        if (!orc_circumcenter(XY(m, TV(m, t, 0)), XY(m, TV(m, t, 1)), XY(m, TV(m, t, 2)), o) ||
            !isfinite(o[0]) || !isfinite(o[1])) {
            int best = 0;
            double bl = -1.0;
            for (int e = 0; e < 3; ++e) {
                const double l = sqd(XY(m, TV(m, t, nx(e))), XY(m, TV(m, t, pv(e))));
                if (l > bl) {
                    bl = l;
                    best = e;
                }
            }
            mid(XY(m, TV(m, t, nx(best))), XY(m, TV(m, t, pv(best))), o);
            c->fallback = 1;
        }
    }
    c->x = o[0];
    c->y = o[1];
}

/* collect (refine.hpp:226-263) + compute_splitting_points (:267) */
uint32_t orc_collect(const gdp2d_mesh_view* m, const gdp2d_params* p, gdp2d_candidate* out,
                     uint32_t cap) {
    uint32_t n = 0;
    for (uint32_t s = 0; s < m->n_subsegments; ++s) {
        if (!m->seg_alive[s]) continue;
        if (!m->seg_encroached[s] && !is_encroached(m, s, (int)p->mode)) continue;
        if (n < cap) {
            gdp2d_candidate* c = &out[n];
            memset(c, 0, sizeof *c);
            c->kind = GDP2D_CAND_SUBSEG;
            c->id = s;
            c->band = GDP2D_BAND_MIDPOINT;
            c->measure = sqrt(sqd(XY(m, m->seg_v[2 * s]), XY(m, m->seg_v[2 * s + 1])));
            c->tiebreak = n;
            c->located = GDP2D_PENDING;
            c->alive = 1;
            split_point(m, c);
        }
        ++n;
    }
    if (!p->rule4_unified_collection && n > 0) return n;
    for (uint32_t t = 0; t < m->n_triangles; ++t) {
        if (!m->tri_alive[t]) continue;
        const double *a = XY(m, TV(m, t, 0)), *b = XY(m, TV(m, t, 1)), *c3 = XY(m, TV(m, t, 2));
        if (!orc_is_bad(a, b, c3, p->cos2_theta, p->ell) || !resolvable(m, t)) continue;
        if (n < cap) {
            gdp2d_candidate* c = &out[n];
            memset(c, 0, sizeof *c);
            c->kind = GDP2D_CAND_TRI;
            c->id = t;
            c->band = GDP2D_BAND_CIRCUMCENTER;
            c->measure =
                0.5 * fabs((b[0] - a[0]) * (c3[1] - a[1]) - (b[1] - a[1]) * (c3[0] - a[0]));
            c->tiebreak = n;
            c->located = GDP2D_PENDING;
            c->alive = 1;
            split_point(m, c);
        }
        ++n;
    }
    return n;
}

/* classify_in_triangle (cdt.hpp:41-60) -> kind, edge */
static int classify(const gdp2d_mesh_view* m, uint32_t t, const double* p, int* edge) {
    int ze = -1, zc = 0;
    for (int e = 0; e < 3; ++e) {
        const int o = orc_orient2d(XY(m, TV(m, t, nx(e))), XY(m, TV(m, t, pv(e))), p);
        if (o < 0) {
            *edge = e;
            return GDP2D_LOC_OUTSIDE;
        }
        if (o == 0) {
            ze = e;
            ++zc;
        }
    }
    *edge = ze;
    if (zc == 0) return GDP2D_LOC_INSIDE;
    if (zc == 1) return GDP2D_LOC_ONEDGE;
    return GDP2D_LOC_ONVERTEX;
}

/* locate_point (cdt.hpp:68-105) with interception; returns kind */
static int locate_point(const gdp2d_mesh_view* m, uint32_t start, const double* p, uint32_t* tri,
                        int* edge, uint32_t* seg) {
    uint32_t cur = start, prev = NONE;
    const uint64_t cap = 8 + 2 * (uint64_t)m->n_triangles;
    for (uint64_t step = 0; step < cap; ++step) {
        int ex = -1;
        for (int e = 0; e < 3; ++e) {
            if (TN(m, cur, e) == prev && prev != NONE) continue;
            if (orc_orient2d(XY(m, TV(m, cur, nx(e))), XY(m, TV(m, cur, pv(e))), p) < 0) {
                ex = e;
                break;
            }
        }
        if (ex < 0) {
            int e2;
            const int k = classify(m, cur, p, &e2);
            if (k != GDP2D_LOC_OUTSIDE) {
                *tri = cur;
                *edge = e2;
                return k;
            }
            ex = e2;
        }
        if (TS(m, cur, ex) != NONE) {
            *tri = cur;
            *edge = ex;
            *seg = TS(m, cur, ex);
            return GDP2D_LOC_INTERCEPTED;
        }
        const uint32_t nxt = TN(m, cur, ex);
        if (nxt == NONE) {
            *tri = cur;
            *edge = ex;
            return GDP2D_LOC_OUTSIDE;
        }
        prev = cur;
        cur = nxt;
    }
    for (uint32_t t = 0; t < m->n_triangles; ++t) {
        if (!m->tri_alive[t]) continue;
        int e2;
        const int k = classify(m, t, p, &e2);
        if (k != GDP2D_LOC_OUTSIDE) {
            *tri = t;
            *edge = e2;
            return k;
        }
    }
    return GDP2D_LOC_OUTSIDE;
}

/* locate (refine.hpp:301-335) */
void orc_locate(const gdp2d_mesh_view* m, gdp2d_candidate* cs, uint32_t n) {
    for (uint32_t i = 0; i < n; ++i) {
        gdp2d_candidate* c = &cs[i];
        if (!c->alive) continue;
        if (c->kind == GDP2D_CAND_SUBSEG) {
            c->located = m->seg_tri[c->id];
            continue;
        }
        const double p[2] = {c->x, c->y};
        uint32_t tri = NONE, seg = NONE, hit = NONE;
        int edge = -1;
        const int k = locate_point(m, c->id, p, &tri, &edge, &seg);
        if (k == GDP2D_LOC_INSIDE) {
            c->located = tri;
            continue;
        }
        if (k == GDP2D_LOC_ONEDGE) {
            if (TS(m, tri, edge) == NONE) {
                c->located = tri;
                continue;
            }
            hit = TS(m, tri, edge);
        } else if (k == GDP2D_LOC_INTERCEPTED) {
            hit = seg;
        } else {
            c->alive = 0;
            continue;
        }
        double o[2];
        const double *a = XY(m, m->seg_v[2 * hit]), *b = XY(m, m->seg_v[2 * hit + 1]);
        mid(a, b, o);
        c->kind = GDP2D_CAND_SUBSEG;
        c->id = hit;
        c->x = o[0];
        c->y = o[1];
        c->band = GDP2D_BAND_MIDPOINT;
        c->measure = sqrt(sqd(a, b));
        c->located = m->seg_tri[hit];
    }
}

/* priority_less (refine.hpp:65-69) */
static int prio_less(const gdp2d_candidate* a, const gdp2d_candidate* b) {
    if (a->band != b->band) return a->band < b->band;
    if (a->measure != b->measure) return a->measure < b->measure;
    return a->tiebreak > b->tiebreak;
}

/* ClaimTable::claim_max (refine.hpp:349-354), sequential */
static void claim_max(uint32_t* slots, uint32_t t, uint32_t cand, const gdp2d_candidate* l) {
    const uint32_t cur = slots[t];
    if (cur == NONE || prio_less(&l[cur], &l[cand])) slots[t] = cand;
}

/* claim_filter (refine.hpp:367-376) */
void orc_claim(const gdp2d_mesh_view* m, gdp2d_candidate* c, uint32_t n) {
    uint32_t* slots = (uint32_t*)malloc(sizeof(uint32_t) * (m->n_triangles + 1));
    for (uint32_t t = 0; t < m->n_triangles; ++t) slots[t] = NONE;
    for (uint32_t i = 0; i < n; ++i)
        if (c[i].alive) claim_max(slots, c[i].located, i, c);
    for (uint32_t i = 0; i < n; ++i)
        if (c[i].alive && slots[c[i].located] != i) c[i].alive = 0;
    free(slots);
}

/* cavity_filter (refine.hpp:382-429) with expand()'s window order */
void orc_cavity(const gdp2d_mesh_view* m, gdp2d_candidate* c, uint32_t n, uint32_t n_cav,
                uint32_t* regions, uint32_t* region_len) {
    uint32_t* slots = (uint32_t*)malloc(sizeof(uint32_t) * (m->n_triangles + 1));
    for (uint32_t t = 0; t < m->n_triangles; ++t) slots[t] = NONE;
    const uint32_t rs = n_cav + 1;
    uint32_t* reg = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n * rs + 1));
    uint32_t* rl = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
    uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * (4 + 3 * (size_t)rs) * 4);
    for (uint32_t i = 0; i < n; ++i) {
        if (!c[i].alive) continue;
        uint32_t* r = reg + (size_t)i * rs;
        uint32_t len = 0, head = 0, tail = 0;
        const double p[2] = {c[i].x, c[i].y};
        q[tail++] = c[i].located;
        while (head < tail) {
            const uint32_t t = q[head++];
            int pred = t == c[i].located;
            if (!pred && m->tri_alive[t])
                pred = orc_incircle(XY(m, TV(m, t, 0)), XY(m, TV(m, t, 1)), XY(m, TV(m, t, 2)),
                                    p) > 0;
            if (!pred) continue;
            int in = 0;
            for (uint32_t k = 0; k < len; ++k) in |= r[k] == t;
            if (in || len > n_cav) continue;
            r[len++] = t;
            claim_max(slots, t, i, c);
            for (int e = 0; e < 3; ++e) {
                if (TS(m, t, e) != NONE) continue;
                const uint32_t nb = TN(m, t, e);
                if (nb == NONE) continue;
                int seen = 0;
                for (uint32_t k = 0; k < len; ++k) seen |= r[k] == nb;
                if (!seen) q[tail++] = nb;
            }
        }
        rl[i] = len;
    }
    for (uint32_t i = 0; i < n; ++i) {
        if (!c[i].alive) continue;
        for (uint32_t k = 0; k < rl[i]; ++k)
            if (slots[reg[(size_t)i * rs + k]] != i) {
                c[i].alive = 0;
                break;
            }
    }
    if (regions && region_len) {
        for (uint32_t i = 0; i < n; ++i) {
            region_len[i] = rl[i];
            for (uint32_t k = 0; k < rl[i]; ++k) regions[(size_t)i * rs + k] = reg[(size_t)i * rs + k];
        }
    }
    free(q);
    free(rl);
    free(reg);
    free(slots);
}
