// gdp2d_predicates.cuh -- device geometric predicates with exact fallbacks.
//
// Sign decisions are exact (Shewchuk-style non-overlapping expansions), so
// they equal the reference's decisions bit for bit on identical inputs:
//   orient2d            predicates.hpp:63-79   (filter + exact :30-35)
//   incircle            predicates.hpp:82-103  (permanent filter + exact :50-59)
//   in_diametric_circle predicates.hpp:107-119
//   in_diametral_lens   predicates.hpp:126-162
//   circumcenter        predicates.hpp:172-185 (FP formula, bit-exact: the
//                       translation unit is compiled with -fmad=false so no
//                       a*b+c is contracted into an FMA)
// Expansion primitives restate detail/expansion.hpp:21-94 (two_sum, two_prod
// with an explicit fma error term, zero-eliminating sum and scale).  The exact
// paths are __noinline__ so their local-memory stacks stay off the fast path.
#pragma once

#include "gdp2d_common.cuh"

namespace gdp2d {

static constexpr double kEps = 1.1102230246251565e-16;  // DBL_EPSILON / 2
static constexpr double kOrientErrBound = (3.0 + 16.0 * kEps) * kEps;
static constexpr double kIncircleErrBound = (10.0 + 96.0 * kEps) * kEps;

__device__ __forceinline__ int sgn(double d) { return (d > 0.0) - (d < 0.0); }

// ---- expansion arithmetic ---------------------------------------------------

__device__ __forceinline__ void two_sum(double a, double b, double& x, double& y) {
    x = __dadd_rn(a, b);
    const double bv = __dsub_rn(x, a);
    const double av = __dsub_rn(x, bv);
    const double br = __dsub_rn(b, bv);
    const double ar = __dsub_rn(a, av);
    y = __dadd_rn(ar, br);
}

__device__ __forceinline__ void two_prod(double a, double b, double& x, double& y) {
    x = __dmul_rn(a, b);
    y = fma(a, b, -x);
}

// h = e + f (zero-eliminated); e, f non-empty; returns >= 1 component.
static __device__ __noinline__ int exp_sum(const double* e, int elen, const double* f, int flen,
                                    double* h) {
    int ei = 0, fi = 0, hi = 0;
    double q;
    if (fabs(f[0]) < fabs(e[0])) {
        q = f[0];
        fi = 1;
    } else {
        q = e[0];
        ei = 1;
    }
    while (ei < elen || fi < flen) {
        double nx;
        if (ei >= elen || (fi < flen && fabs(f[fi]) < fabs(e[ei]))) {
            nx = f[fi++];
        } else {
            nx = e[ei++];
        }
        double s, lo;
        two_sum(q, nx, s, lo);
        if (lo != 0.0) h[hi++] = lo;
        q = s;
    }
    if (q != 0.0 || hi == 0) h[hi++] = q;
    return hi;
}

// h = e * b (zero-eliminated); returns >= 1 component.
static __device__ __noinline__ int exp_scale(const double* e, int elen, double b, double* h) {
    int hi = 0;
    double px, py;
    two_prod(e[0], b, px, py);
    if (py != 0.0) h[hi++] = py;
    double q = px;
    for (int i = 1; i < elen; ++i) {
        double tx, ty, s1, l1, s2, l2;
        two_prod(e[i], b, tx, ty);
        two_sum(q, ty, s1, l1);
        if (l1 != 0.0) h[hi++] = l1;
        two_sum(tx, s1, s2, l2);
        if (l2 != 0.0) h[hi++] = l2;
        q = s2;
    }
    if (q != 0.0 || hi == 0) h[hi++] = q;
    return hi;
}

__device__ __forceinline__ int exp_product2(double a, double b, double* h) {
    double x, y;
    two_prod(a, b, x, y);
    int n = 0;
    if (y != 0.0) h[n++] = y;
    if (x != 0.0 || n == 0) h[n++] = x;
    return n;
}

__device__ __forceinline__ int exp_sign(const double* e, int n) { return sgn(e[n - 1]); }

__device__ __forceinline__ void exp_negate(double* e, int n) {
    for (int i = 0; i < n; ++i) e[i] = -e[i];
}

// acc (len *n) += sign * term; uses tmp as scratch (capacity >= *n + tlen).
__device__ __forceinline__ void exp_accumulate(double* acc, int* n, double* term, int tlen,
                                               int sign, double* tmp) {
    if (sign < 0) exp_negate(term, tlen);
    const int m = exp_sum(acc, *n, term, tlen, tmp);
    for (int i = 0; i < m; ++i) acc[i] = tmp[i];
    *n = m;
}

// Exact orient2d determinant in raw coordinates (predicates.hpp:30-46).
static __device__ __noinline__ int orient2d_expansion(double2 a, double2 b, double2 c, double* out) {
    double p[2], acc[12], tmp[12];
    int n = exp_product2(a.x, b.y, acc);
    int k;
    k = exp_product2(a.x, c.y, p); exp_accumulate(acc, &n, p, k, -1, tmp);
    k = exp_product2(b.x, c.y, p); exp_accumulate(acc, &n, p, k, +1, tmp);
    k = exp_product2(b.x, a.y, p); exp_accumulate(acc, &n, p, k, -1, tmp);
    k = exp_product2(c.x, a.y, p); exp_accumulate(acc, &n, p, k, +1, tmp);
    k = exp_product2(c.x, b.y, p); exp_accumulate(acc, &n, p, k, -1, tmp);
    for (int i = 0; i < n; ++i) out[i] = acc[i];
    return n;
}

static __device__ __noinline__ int orient2d_exact(double2 a, double2 b, double2 c) {
    double e[12];
    const int n = orient2d_expansion(a, b, c, e);
    return exp_sign(e, n);
}

// Exact incircle sign: sum over the lifted column (predicates.hpp:50-59).
static __device__ __noinline__ int incircle_exact(double2 a, double2 b, double2 c, double2 d) {
    double acc[384], tmp[384], term[96], orient[12], lift[4], part[24], p2[2], q2[2];
    int n = 1;
    acc[0] = 0.0;
    const double2 pts[4] = {a, b, c, d};
    for (int k = 0; k < 4; ++k) {
        // lift(p_k) * orient(other three, in cyclic-preserving order)
        const double2 p = pts[k];
        int lp = exp_product2(p.x, p.x, p2);
        int lq = exp_product2(p.y, p.y, q2);
        const int ll = exp_sum(p2, lp, q2, lq, lift);
        int on;
        if (k == 0) on = orient2d_expansion(b, c, d, orient);
        else if (k == 1) on = orient2d_expansion(a, c, d, orient);
        else if (k == 2) on = orient2d_expansion(a, b, d, orient);
        else on = orient2d_expansion(a, b, c, orient);
        // term = lift * orient
        int tn = 1;
        term[0] = 0.0;
        for (int i = 0; i < ll; ++i) {
            const int pn = exp_scale(orient, on, lift[i], part);
            const int m = exp_sum(term, tn, part, pn, tmp);
            for (int j = 0; j < m; ++j) term[j] = tmp[j];
            tn = m;
        }
        // det = (ta - tb) + (tc - td)
        exp_accumulate(acc, &n, term, tn, (k & 1) ? -1 : +1, tmp);
    }
    return exp_sign(acc, n);
}

// ---- filtered predicates -----------------------------------------------------

// predicates.hpp:63-79
__device__ __forceinline__ int orient2d(double2 a, double2 b, double2 c) {
    const double detleft = (a.x - c.x) * (b.y - c.y);
    const double detright = (a.y - c.y) * (b.x - c.x);
    const double det = detleft - detright;
    if (detleft > 0.0) {
        if (detright <= 0.0) return sgn(det);
    } else if (detleft < 0.0) {
        if (detright >= 0.0) return sgn(det);
    } else {
        return (detright < 0.0) - (detright > 0.0);
    }
    const double detsum = fabs(detleft) + fabs(detright);
    if (fabs(det) > kOrientErrBound * detsum) return sgn(det);
    return orient2d_exact(a, b, c);
}

// predicates.hpp:82-103
__device__ __forceinline__ int incircle(double2 a, double2 b, double2 c, double2 d) {
    const double adx = a.x - d.x, ady = a.y - d.y;
    const double bdx = b.x - d.x, bdy = b.y - d.y;
    const double cdx = c.x - d.x, cdy = c.y - d.y;
    const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
    const double alift = adx * adx + ady * ady;
    const double cdxady = cdx * ady, adxcdy = adx * cdy;
    const double blift = bdx * bdx + bdy * bdy;
    const double adxbdy = adx * bdy, bdxady = bdx * ady;
    const double clift = cdx * cdx + cdy * cdy;
    const double det =
        alift * (bdxcdy - cdxbdy) + blift * (cdxady - adxcdy) + clift * (adxbdy - bdxady);
    const double permanent = (fabs(bdxcdy) + fabs(cdxbdy)) * alift +
                             (fabs(cdxady) + fabs(adxcdy)) * blift +
                             (fabs(adxbdy) + fabs(bdxady)) * clift;
    if (fabs(det) > kIncircleErrBound * permanent) return sgn(det);
    return incircle_exact(a, b, c, d);
}

__device__ __forceinline__ double dot2(double2 a, double2 b) { return a.x * b.x + a.y * b.y; }
__device__ __forceinline__ double cross2(double2 a, double2 b) { return a.x * b.y - a.y * b.x; }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) {
    return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double sqdist(double2 a, double2 b) {
    const double dx = a.x - b.x, dy = a.y - b.y;
    return dx * dx + dy * dy;
}
__device__ __forceinline__ double2 midpoint2(double2 a, double2 b) {
    return make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
}
__device__ __forceinline__ bool peq(double2 a, double2 b) { return a.x == b.x && a.y == b.y; }

static __device__ __noinline__ bool in_diametric_exact(double2 sa, double2 sb, double2 p) {
    double acc[16], tmp[16], t[2];
    int n = exp_product2(sa.x, sb.x, acc);
    int k;
    k = exp_product2(sa.x, p.x, t); exp_accumulate(acc, &n, t, k, -1, tmp);
    k = exp_product2(p.x, sb.x, t); exp_accumulate(acc, &n, t, k, -1, tmp);
    k = exp_product2(p.x, p.x, t);  exp_accumulate(acc, &n, t, k, +1, tmp);
    k = exp_product2(sa.y, sb.y, t); exp_accumulate(acc, &n, t, k, +1, tmp);
    k = exp_product2(sa.y, p.y, t); exp_accumulate(acc, &n, t, k, -1, tmp);
    k = exp_product2(p.y, sb.y, t); exp_accumulate(acc, &n, t, k, -1, tmp);
    k = exp_product2(p.y, p.y, t);  exp_accumulate(acc, &n, t, k, +1, tmp);
    return exp_sign(acc, n) < 0;
}

// predicates.hpp:107-119
__device__ __forceinline__ bool in_diametric_circle(double2 sa, double2 sb, double2 p) {
    const double2 u = sub2(sa, p);
    const double2 v = sub2(sb, p);
    const double d = dot2(u, v);
    const double mag = fabs(u.x * v.x) + fabs(u.y * v.y);
    if (fabs(d) > 8.0 * kEps * mag) return d < 0.0;
    return in_diametric_exact(sa, sb, p);
}

// Exact 4*dot^2 - |u|^2 |v|^2 over two-component differences (predicates.hpp:141-161).
static __device__ __noinline__ bool in_lens_exact(double2 sa, double2 sb, double2 p) {
    double ex[2], ey[2], fx[2], fy[2];
    int nex, ney, nfx, nfy;
    auto comp2 = [](double a, double b, double* o) {
        double hi, lo;
        two_sum(a, -b, hi, lo);
        int n = 0;
        if (lo != 0.0) o[n++] = lo;
        o[n++] = hi;
        return n;
    };
    nex = comp2(sa.x, p.x, ex);
    ney = comp2(sa.y, p.y, ey);
    nfx = comp2(sb.x, p.x, fx);
    nfy = comp2(sb.y, p.y, fy);
    double dote[16], ulen[16], vlen[16], t4[8], t4b[8];
    auto mul22 = [&](const double* a, int na, const double* b, int nb, double* out, double* s1) {
        int n = 1;
        out[0] = 0.0;
        double part[4], tmp2[8];
        for (int i = 0; i < na; ++i) {
            const int pn = exp_scale(b, nb, a[i], part);
            const int m = exp_sum(out, n, part, pn, tmp2);
            for (int j = 0; j < m; ++j) out[j] = tmp2[j];
            n = m;
        }
        (void)s1;
        return n;
    };
    int n1 = mul22(ex, nex, fx, nfx, t4, nullptr);
    int n2 = mul22(ey, ney, fy, nfy, t4b, nullptr);
    const int nd = exp_sum(t4, n1, t4b, n2, dote);
    n1 = mul22(ex, nex, ex, nex, t4, nullptr);
    n2 = mul22(ey, ney, ey, ney, t4b, nullptr);
    const int nu = exp_sum(t4, n1, t4b, n2, ulen);
    n1 = mul22(fx, nfx, fx, nfx, t4, nullptr);
    n2 = mul22(fy, nfy, fy, nfy, t4b, nullptr);
    const int nv = exp_sum(t4, n1, t4b, n2, vlen);
    // result = 4 * dote^2 - ulen * vlen, accumulated component-wise.
    double acc[1024], tmp[1024], part[32];
    int n = 1;
    acc[0] = 0.0;
    for (int i = 0; i < nd; ++i) {
        const int pn = exp_scale(dote, nd, 4.0 * dote[i], part);
        exp_accumulate(acc, &n, part, pn, +1, tmp);
    }
    for (int i = 0; i < nu; ++i) {
        const int pn = exp_scale(vlen, nv, ulen[i], part);
        exp_accumulate(acc, &n, part, pn, -1, tmp);
    }
    return exp_sign(dote, nd) < 0 && exp_sign(acc, n) >= 0;
}

// predicates.hpp:126-162
__device__ __forceinline__ bool in_diametral_lens(double2 sa, double2 sb, double2 p) {
    if (peq(p, sa) || peq(p, sb)) return false;
    const double2 u = sub2(sa, p);
    const double2 v = sub2(sb, p);
    const double d = dot2(u, v);
    if (d >= 0.0) return false;
    const double uu = dot2(u, u);
    const double vv = dot2(v, v);
    const double lhs = 4.0 * d * d;
    const double rhs = uu * vv;
    if (fabs(lhs - rhs) > 64.0 * kEps * (lhs + rhs)) return lhs >= rhs;
    return in_lens_exact(sa, sb, p);
}

// predicates.hpp:172-185
__device__ __forceinline__ double2 circumcenter(double2 a, double2 b, double2 c, bool& ok) {
    const double2 ab = sub2(b, a);
    const double2 ac = sub2(c, a);
    const double d = 2.0 * cross2(ab, ac);
    const double ab2 = dot2(ab, ab);
    const double ac2 = dot2(ac, ac);
    const double ux = (ac.y * ab2 - ab.y * ac2) / d;
    const double uy = (ab.x * ac2 - ac.x * ab2) / d;
    const double2 center = make_double2(a.x + ux, a.y + uy);
    const double scale = fmax(ab2, ac2);
    ok = isfinite(center.x) && isfinite(center.y) && fabs(d) > 1e-12 * scale;
    return center;
}

}  // namespace gdp2d
