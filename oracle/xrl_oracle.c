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

/* Panel geometry, PAPER.md:56 (centroid = PEEC circuit node).
 * centroid = ((v0 + v1) + v2) / 3 in this order; area = |(v1-v0)x(v2-v0)|/2;
 * D = longest edge length. */
void orc_geometry(int64_t nt, const double *vert, const int32_t *tri,
                  double *cent, double *area, double *dmax)
{
    for (int64_t k = 0; k < nt; ++k) {
        const double *a = vert + 3 * (int64_t)tri[3 * k + 0];
        const double *b = vert + 3 * (int64_t)tri[3 * k + 1];
        const double *c = vert + 3 * (int64_t)tri[3 * k + 2];
        for (int d = 0; d < 3; ++d) cent[3 * k + d] = ((a[d] + b[d]) + c[d]) / 3.0;
        double e1[3], e2[3], e3[3];
        for (int d = 0; d < 3; ++d) { e1[d] = b[d] - a[d]; e2[d] = c[d] - a[d]; e3[d] = c[d] - b[d]; }
        double cx = e1[1] * e2[2] - e1[2] * e2[1];
        double cy = e1[2] * e2[0] - e1[0] * e2[2];
        double cz = e1[0] * e2[1] - e1[1] * e2[0];
        area[k] = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
        double l1 = sqrt((e1[0] * e1[0] + e1[1] * e1[1]) + e1[2] * e1[2]);
        double l2 = sqrt((e2[0] * e2[0] + e2[1] * e2[1]) + e2[2] * e2[2]);
        double l3 = sqrt((e3[0] * e3[0] + e3[1] * e3[1]) + e3[2] * e3[2]);
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

/* Entry P_kl of the discrete operator (definition C1 above). */
static double orc_pkl(int64_t k, int64_t l, const double *vert, const int32_t *tri,
                      const double *cent, const double *area, const double *dmax, double eta)
{
    const double *ck = cent + 3 * k, *cl = cent + 3 * l;
    if (k == l) {
        return orc_tri_potential(ck, vert + 3 * (int64_t)tri[3 * k], vert + 3 * (int64_t)tri[3 * k + 1],
                                 vert + 3 * (int64_t)tri[3 * k + 2]) / area[k];
    }
    if (orc_is_near(ck, cl, dmax[k], dmax[l], eta)) {
        double Ikl = orc_tri_potential(ck, vert + 3 * (int64_t)tri[3 * l], vert + 3 * (int64_t)tri[3 * l + 1],
                                       vert + 3 * (int64_t)tri[3 * l + 2]) / area[l];
        double Ilk = orc_tri_potential(cl, vert + 3 * (int64_t)tri[3 * k], vert + 3 * (int64_t)tri[3 * k + 1],
                                       vert + 3 * (int64_t)tri[3 * k + 2]) / area[k];
        return 0.5 * (Ikl + Ilk);
    }
    double dx = ck[0] - cl[0], dy = ck[1] - cl[1], dz = ck[2] - cl[2];
    return 1.0 / sqrt((dx * dx + dy * dy) + dz * dz);
}

/* Dense entries P[rows[i], cols[j]] (small cases / symmetry checks). */
void orc_p_entries(int64_t nt, const double *vert, const int32_t *tri, const double *cent,
                   const double *area, const double *dmax, double eta,
                   int64_t nr, const int64_t *rows, int64_t nc, const int64_t *cols, double *out)
{
    (void)nt;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nr; ++i)
        for (int64_t j = 0; j < nc; ++j)
            out[i * nc + j] = orc_pkl(rows[i], cols[j], vert, tri, cent, area, dmax, eta);
}

/* Direct O(N^2) sum on selected target rows.
 * x: [nvec][nt] complex as interleaved (re,im) doubles; y: [nvec][nr] same.
 * y[v][i] = sum_l P_{rows[i], l} x[v][l]   (C4; P real -> re, im separately) */
void orc_mvm_rows(int64_t nt, const double *vert, const int32_t *tri, const double *cent,
                  const double *area, const double *dmax, double eta,
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
                double p = orc_pkl(k, l, vert, tri, cent, area, dmax, eta);
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
void orc_near_rows(int64_t nt, const double *vert, const int32_t *tri, const double *cent,
                   const double *area, const double *dmax, double eta,
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
                vals[off[i] + c] = orc_pkl(k, l, vert, tri, cent, area, dmax, eta);
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

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
