/*
 * XRL ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU FP64 implementation of what the hot path
 * of XRL (arXiv 2409.12375) computes.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares
 * no code with the CUDA path (paper_2409_12375_b200/csrc) and includes none of
 * its headers.  Compiled with -O2 -ffp-contract=off (no FMA contraction) so
 * the near-pair decisions are correctly-rounded FP64, operation by operation.
 *
 * What it computes:
 *   P_kk = I(c_k; T_k) / A_k                                       (self)
 *   P_kl = 1/2 [ I(c_k; T_l)/A_l + I(c_l; T_k)/A_k ]   if (k,l) near   (near)
 *   P_kl = 1 / |c_k - c_l|                             otherwise       (far)
 *   y_t[k] = sum_l P_kl x_t[l],   t = 1..3, re and im separately.
 * Panels are triangles or rectangles (a rectangle's I is the sum
 * over its two diagonal triangles).  Galerkin option (NEXT f4):
 * self and vertex-adjacent pairs average I over an outer quadrature of the
 * observation panel instead of taking it at the centroid.
 * with I(r;T) = \int_T dS'/|r - r'| (Eq. 1 kernel, PAPER.md:88
 * Eq. 6 second term with j*omega*mu0/4pi pulled out as PAPER.md:144 says;
 * PAPER.md:116 "P directly computed on centroids" = particle format).
 *
 * Pins: tests/test_oracle_pins.py (closed forms, scipy quadrature brute force,
 * additivity, isometry, far-field limit, symmetry).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- geometry */

/* Panels: pv[stride*k + 0..2] triangle vertex indices; with stride 4 and
 * pv[4k+3] >= 0 the panel is a rectangle (a planar parallelogram a, b, c, d in
 * cyclic order; "hybrid of triangles and
 * rectangles"). */
static int orc_is_quad(const int32_t *pv, int32_t stride, int64_t k)
{
    return stride == 4 && pv[4 * k + 3] >= 0;
}

static double orc_len(const double *e)
{
    return sqrt((e[0] * e[0] + e[1] * e[1]) + e[2] * e[2]);
}

/* Panel geometry, PAPER.md:56 (centroid = PEEC circuit node).
 * Triangle: centroid = ((v0 + v1) + v2) / 3 in this order; area =
 * |(v1-v0)x(v2-v0)|/2; D = longest edge length.
 * Rectangle (parallelogram a b c d): centroid = intersection of the diagonals
 * = (a + c) * 0.5; area = |(b-a)x(d-a)|; D = the longer diagonal
 * (the panel's diameter; reading R16). */
void orc_geometry(int64_t nt, const double *vert, const int32_t *pv, int32_t stride,
                  double *cent, double *area, double *dmax)
{
    for (int64_t k = 0; k < nt; ++k) {
        const double *a = vert + 3 * (int64_t)pv[stride * k + 0];
        const double *b = vert + 3 * (int64_t)pv[stride * k + 1];
        const double *c = vert + 3 * (int64_t)pv[stride * k + 2];
        if (orc_is_quad(pv, stride, k)) {
            const double *q = vert + 3 * (int64_t)pv[4 * k + 3];
            double e1[3], e2[3], d1[3], d2[3];
            for (int d = 0; d < 3; ++d) {
                cent[3 * k + d] = (a[d] + c[d]) * 0.5;
                e1[d] = b[d] - a[d];
                e2[d] = q[d] - a[d];
                d1[d] = c[d] - a[d];
                d2[d] = q[d] - b[d];
            }
            double cx = e1[1] * e2[2] - e1[2] * e2[1];
            double cy = e1[2] * e2[0] - e1[0] * e2[2];
            double cz = e1[0] * e2[1] - e1[1] * e2[0];
            area[k] = sqrt(cx * cx + cy * cy + cz * cz);
            double l1 = orc_len(d1), l2 = orc_len(d2);
            dmax[k] = l1 > l2 ? l1 : l2;
            continue;
        }
        for (int d = 0; d < 3; ++d) cent[3 * k + d] = ((a[d] + b[d]) + c[d]) / 3.0;
        double e1[3], e2[3], e3[3];
        for (int d = 0; d < 3; ++d) { e1[d] = b[d] - a[d]; e2[d] = c[d] - a[d]; e3[d] = c[d] - b[d]; }
        double cx = e1[1] * e2[2] - e1[2] * e2[1];
        double cy = e1[2] * e2[0] - e1[0] * e2[2];
        double cz = e1[0] * e2[1] - e1[1] * e2[0];
        area[k] = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
        double l1 = orc_len(e1), l2 = orc_len(e2), l3 = orc_len(e3);
        double m = l1 > l2 ? l1 : l2;
        dmax[k] = m > l3 ? m : l3;
    }
}

/* ------------------------------------------------ single-triangle integral */

/* I(r; T) = \int_T dS' / |r - r'| for a flat triangle with uniform density.
 * Closed form (edge decomposition of the potential of a uniform polygon
 * source, e.g. Wilton et al. 1984):
 *   I = sum_i P0_i ln[(R+_i + l+_i)/(R-_i + l-_i)]
 *       - |h| sum_i [ atan(P0_i l+_i/(R0_i^2 + |h| R+_i))
 *                   - atan(P0_i l-_i/(R0_i^2 + |h| R-_i)) ]
 * h: signed height of r over the plane, rho: projection of r on the plane;
 * for edge i from vertex a to b (counter-clockwise about the winding normal)
 * with unit tangent t and outward in-plane normal u = t x n:
 *   P0 = (a - rho).u, l- = (a - rho).t, l+ = (b - rho).t,
 *   R0^2 = P0^2 + h^2, R- = |r - a|, R+ = |r - b|.
 * The log ratio is evaluated in whichever of the equivalent forms
 * (R+ + l+)/(R- + l-) = (R- - l-)/(R+ - l+) has no cancellation.  An edge
 * with P0 == 0 contributes nothing. */
double orc_tri_potential(const double *r, const double *v0, const double *v1, const double *v2)
{
    const double *V[3] = {v0, v1, v2};
    double e1[3], e2[3], n[3];
    for (int d = 0; d < 3; ++d) { e1[d] = v1[d] - v0[d]; e2[d] = v2[d] - v0[d]; }
    n[0] = e1[1] * e2[2] - e1[2] * e2[1];
    n[1] = e1[2] * e2[0] - e1[0] * e2[2];
    n[2] = e1[0] * e2[1] - e1[1] * e2[0];
    double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    for (int d = 0; d < 3; ++d) n[d] /= nn;
    double h = (r[0] - v0[0]) * n[0] + (r[1] - v0[1]) * n[1] + (r[2] - v0[2]) * n[2];
    double ah = fabs(h);
    double rho[3];
    for (int d = 0; d < 3; ++d) rho[d] = r[d] - h * n[d];
    double sum_log = 0.0, sum_atan = 0.0;
    for (int i = 0; i < 3; ++i) {
        const double *a = V[i], *b = V[(i + 1) % 3];
        double t[3], u[3];
        for (int d = 0; d < 3; ++d) t[d] = b[d] - a[d];
        double lt = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
        for (int d = 0; d < 3; ++d) t[d] /= lt;
        u[0] = t[1] * n[2] - t[2] * n[1];
        u[1] = t[2] * n[0] - t[0] * n[2];
        u[2] = t[0] * n[1] - t[1] * n[0];
        double am[3], bm[3];
        for (int d = 0; d < 3; ++d) { am[d] = a[d] - rho[d]; bm[d] = b[d] - rho[d]; }
        double P0 = am[0] * u[0] + am[1] * u[1] + am[2] * u[2];
        if (P0 == 0.0) continue;
        double lm = am[0] * t[0] + am[1] * t[1] + am[2] * t[2];
        double lp = bm[0] * t[0] + bm[1] * t[1] + bm[2] * t[2];
        double R02 = P0 * P0 + h * h;
        double ra[3], rb[3];
        for (int d = 0; d < 3; ++d) { ra[d] = r[d] - a[d]; rb[d] = r[d] - b[d]; }
        double Rm = sqrt(ra[0] * ra[0] + ra[1] * ra[1] + ra[2] * ra[2]);
        double Rp = sqrt(rb[0] * rb[0] + rb[1] * rb[1] + rb[2] * rb[2]);
        double lg;
        if (lm >= 0.0)          lg = log((Rp + lp) / (Rm + lm));
        else if (lp <= 0.0)     lg = log((Rm - lm) / (Rp - lp));
        else                    lg = log(Rp + lp) + log(Rm - lm) - log(R02);
        sum_log += P0 * lg;
        if (ah > 0.0)
            sum_atan += atan(P0 * lp / (R02 + ah * Rp)) - atan(P0 * lm / (R02 + ah * Rm));
    }
    return sum_log - ah * sum_atan;
}

/* I(r; S_k) for panel k: a triangle, or a rectangle as its two triangles
 * (a, b, c) + (a, c, d) split on the diagonal ac (additivity of the integral). */
static double orc_panel_potential(const double *r, const double *vert, const int32_t *pv, int32_t stride, int64_t k)
{
    const double *a = vert + 3 * (int64_t)pv[stride * k + 0];
    const double *b = vert + 3 * (int64_t)pv[stride * k + 1];
    const double *c = vert + 3 * (int64_t)pv[stride * k + 2];
    double I = orc_tri_potential(r, a, b, c);
    if (orc_is_quad(pv, stride, k)) I += orc_tri_potential(r, a, c, vert + 3 * (int64_t)pv[4 * k + 3]);
    return I;
}

/* Outer quadrature over panel k for the Galerkin near rule:
 * triangles: Radon's 7-point degree-5 rule (centroid weight 9/40; points
 * (a, a, 1-2a) with a = (6 -+ sqrt 15)/21, weights (155 -+ sqrt 15)/1200);
 * rectangles: the 2 x 2 Gauss product rule (points a + s (b-a) + t (d-a), s, t
 * = (1 -+ 1/sqrt 3)/2, weights 1/4).  Weights sum to 1 (the mean over the
 * panel).  Returns the number of points. */
static int orc_outer_rule(const double *vert, const int32_t *pv, int32_t stride, int64_t k, double *x, double *w)
{
    const double *a = vert + 3 * (int64_t)pv[stride * k + 0];
    const double *b = vert + 3 * (int64_t)pv[stride * k + 1];
    const double *c = vert + 3 * (int64_t)pv[stride * k + 2];
    if (orc_is_quad(pv, stride, k)) {
        const double *q = vert + 3 * (int64_t)pv[4 * k + 3];
        const double g[2] = {(1.0 - 1.0 / sqrt(3.0)) / 2.0, (1.0 + 1.0 / sqrt(3.0)) / 2.0};
        int m = 0;
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j, ++m) {
                for (int d = 0; d < 3; ++d) x[3 * m + d] = a[d] + g[i] * (b[d] - a[d]) + g[j] * (q[d] - a[d]);
                w[m] = 0.25;
            }
        return 4;
    }
    const double s15 = sqrt(15.0);
    const double al[2] = {(6.0 - s15) / 21.0, (6.0 + s15) / 21.0};
    const double wt[2] = {(155.0 - s15) / 1200.0, (155.0 + s15) / 1200.0};
    for (int d = 0; d < 3; ++d) x[d] = (a[d] + b[d] + c[d]) / 3.0;
    w[0] = 9.0 / 40.0;
    int m = 1;
    for (int s = 0; s < 2; ++s)
        for (int v = 0; v < 3; ++v, ++m) {
            /* barycentric (1-2a) on vertex v, a on the other two */
            const double *P[3] = {a, b, c};
            for (int d = 0; d < 3; ++d)
                x[3 * m + d] = (1.0 - 2.0 * al[s]) * P[v][d] + al[s] * P[(v + 1) % 3][d] + al[s] * P[(v + 2) % 3][d];
            w[m] = wt[s];
        }
    return 7;
}

/* Panels k and l share a vertex index (edge- or vertex-adjacent). */
static int orc_adjacent(const int32_t *pv, int32_t stride, int64_t k, int64_t l)
{
    int nk = orc_is_quad(pv, stride, k) ? 4 : 3, nl = orc_is_quad(pv, stride, l) ? 4 : 3;
    for (int i = 0; i < nk; ++i)
        for (int j = 0; j < nl; ++j)
            if (pv[stride * k + i] == pv[stride * l + j]) return 1;
    return 0;
}

/* (1/A_k) int_{S_k} I(r; S_l) dS / A_l by the outer rule of panel k. */
static double orc_galerkin_term(const double *vert, const int32_t *pv, int32_t stride, const double *area,
                                int64_t k, int64_t l)
{
    double x[3 * 7], w[7];
    int m = orc_outer_rule(vert, pv, stride, k, x, w);
    double s = 0.0;
    for (int q = 0; q < m; ++q) s += w[q] * orc_panel_potential(x + 3 * q, vert, pv, stride, l);
    return s / area[l];
}

/* Test access to the panel integral and the outer rule (pins). */
double orc_panel_potential_ext(const double *r, const double *vert, const int32_t *pv, int32_t stride, int64_t k)
{
    return orc_panel_potential(r, vert, pv, stride, k);
}
int orc_outer_rule_ext(const double *vert, const int32_t *pv, int32_t stride, int64_t k, double *x, double *w)
{
    return orc_outer_rule(vert, pv, stride, k, x, w);
}

/* ------------------------------------------------------- near criterion */

/* (k,l), k != l, is near iff d^2 < (eta * max(D_k, D_l))^2 with
 * d^2 = ((dx*dx + dy*dy) + dz*dz) over FP64 centroid differences, every
 * operation correctly rounded, no contraction (reading R3). */
static int orc_is_near(const double *ck, const double *cl, double Dk, double Dl, double eta)
{
    double dx = ck[0] - cl[0], dy = ck[1] - cl[1], dz = ck[2] - cl[2];
    double d2 = (dx * dx + dy * dy) + dz * dz;
    double t = eta * (Dk > Dl ? Dk : Dl);
    return d2 < t * t;
}

/* Entry P_kl of the discrete operator (definition C1 above).  galerkin != 0:
 * self and vertex-adjacent pairs use the outer quadrature of SPEC.md:345
 * instead of the centroid (symmetrised the same way); other near pairs stay
 * centroid-collocated (reading R17). */
static double orc_pkl(int64_t k, int64_t l, const double *vert, const int32_t *pv, int32_t stride,
                      const double *cent, const double *area, const double *dmax, double eta, int galerkin)
{
    const double *ck = cent + 3 * k, *cl = cent + 3 * l;
    if (k == l) {
        if (galerkin) return orc_galerkin_term(vert, pv, stride, area, k, k);
        return orc_panel_potential(ck, vert, pv, stride, k) / area[k];
    }
    if (orc_is_near(ck, cl, dmax[k], dmax[l], eta)) {
        if (galerkin && orc_adjacent(pv, stride, k, l))
            return 0.5 * (orc_galerkin_term(vert, pv, stride, area, k, l) +
                          orc_galerkin_term(vert, pv, stride, area, l, k));
        double Ikl = orc_panel_potential(ck, vert, pv, stride, l) / area[l];
        double Ilk = orc_panel_potential(cl, vert, pv, stride, k) / area[k];
        return 0.5 * (Ikl + Ilk);
    }
    double dx = ck[0] - cl[0], dy = ck[1] - cl[1], dz = ck[2] - cl[2];
    return 1.0 / sqrt((dx * dx + dy * dy) + dz * dz);
}

/* Dense entries P[rows[i], cols[j]] (small cases / symmetry checks). */
void orc_p_entries(int64_t nt, const double *vert, const int32_t *pv, int32_t stride, const double *cent,
                   const double *area, const double *dmax, double eta, int32_t galerkin,
                   int64_t nr, const int64_t *rows, int64_t nc, const int64_t *cols, double *out)
{
    (void)nt;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nr; ++i)
        for (int64_t j = 0; j < nc; ++j)
            out[i * nc + j] = orc_pkl(rows[i], cols[j], vert, pv, stride, cent, area, dmax, eta, galerkin);
}

/* Direct O(N^2) sum on selected target rows.
 * x: [nvec][nt] complex as interleaved (re,im) doubles; y: [nvec][nr] same.
 * y[v][i] = sum_l P_{rows[i], l} x[v][l]   (C4; P real -> re, im separately) */
void orc_mvm_rows(int64_t nt, const double *vert, const int32_t *pv, int32_t stride, const double *cent,
                  const double *area, const double *dmax, double eta, int32_t galerkin,
                  int32_t nvec, const double *x, int64_t nr, const int64_t *rows, double *y,
                  int32_t nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * 2 * (size_t)nvec);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < nr; ++i) {
            int64_t k = rows[i];
            for (int v = 0; v < 2 * nvec; ++v) acc[v] = 0.0;
            for (int64_t l = 0; l < nt; ++l) {
                double p = orc_pkl(k, l, vert, pv, stride, cent, area, dmax, eta, galerkin);
                for (int v = 0; v < nvec; ++v) {
                    acc[2 * v + 0] += p * x[2 * ((int64_t)v * nt + l) + 0];
                    acc[2 * v + 1] += p * x[2 * ((int64_t)v * nt + l) + 1];
                }
            }
            for (int v = 0; v < nvec; ++v) {
                y[2 * ((int64_t)v * nr + i) + 0] = acc[2 * v + 0];
                y[2 * ((int64_t)v * nr + i) + 1] = acc[2 * v + 1];
            }
        }
        free(acc);
    }
}

/* Near-field rows: for each selected row k, the sorted set of l (including l=k)
 * with (k,l) near or l == k, and the near entry value P_kl (symmetrised
 * integral, self term on the diagonal).  Pass cols/vals = NULL to get the
 * per-row counts only (cnt[i]); otherwise row i is written at offset off[i]. */
void orc_near_rows(int64_t nt, const double *vert, const int32_t *pv, int32_t stride, const double *cent,
                   const double *area, const double *dmax, double eta, int32_t galerkin,
                   int64_t nr, const int64_t *rows, int64_t *cnt, const int64_t *off,
                   int64_t *cols, double *vals, double *inv_r)
{
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < nr; ++i) {
        int64_t k = rows[i];
        int64_t c = 0;
        for (int64_t l = 0; l < nt; ++l) {
            int near = (l == k) || orc_is_near(cent + 3 * k, cent + 3 * l, dmax[k], dmax[l], eta);
            if (!near) continue;
            if (cols) {
                cols[off[i] + c] = l;
                vals[off[i] + c] = orc_pkl(k, l, vert, pv, stride, cent, area, dmax, eta, galerkin);
                if (inv_r) {
                    if (l == k) inv_r[off[i] + c] = 0.0;
                    else {
                        const double *ck = cent + 3 * k, *cl = cent + 3 * l;
                        double dx = ck[0] - cl[0], dy = ck[1] - cl[1], dz = ck[2] - cl[2];
                        inv_r[off[i] + c] = 1.0 / sqrt((dx * dx + dy * dy) + dz * dz);
                    }
                }
            }
            ++c;
        }
        cnt[i] = c;
    }
}

/* Count pairs within a relative distance `rel` of the near threshold
 * (|d - eta*D| / (eta*D) < rel), k < l  -- the tie audit. */
int64_t orc_tie_audit(int64_t nt, const double *cent, const double *dmax, double eta, double rel)
{
    int64_t ties = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : ties)
    for (int64_t k = 0; k < nt; ++k)
        for (int64_t l = k + 1; l < nt; ++l) {
            const double *ck = cent + 3 * k, *cl = cent + 3 * l;
            double dx = ck[0] - cl[0], dy = ck[1] - cl[1], dz = ck[2] - cl[2];
            double d = sqrt((dx * dx + dy * dy) + dz * dz);
            double t = eta * (dmax[k] > dmax[l] ? dmax[k] : dmax[l]);
            if (fabs(d - t) < rel * t) ++ties;
        }
    return ties;
}

/* The tie audit restricted to target rows: pairs (rows[i], l), l != rows[i],
 * all l, within `rel` of the threshold (full-size configs, sampled rows). */
int64_t orc_tie_audit_rows(int64_t nt, const double *cent, const double *dmax, double eta, double rel,
                           int64_t nr, const int64_t *rows)
{
    int64_t ties = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : ties)
    for (int64_t i = 0; i < nr; ++i) {
        const int64_t k = rows[i];
        for (int64_t l = 0; l < nt; ++l) {
            if (l == k) continue;
            const double *ck = cent + 3 * k, *cl = cent + 3 * l;
            double dx = ck[0] - cl[0], dy = ck[1] - cl[1], dz = ck[2] - cl[2];
            double d = sqrt((dx * dx + dy * dy) + dz * dz);
            double t = eta * (dmax[k] > dmax[l] ? dmax[k] : dmax[l]);
            if (fabs(d - t) < rel * t) ++ties;
        }
    }
    return ties;
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
