// Host FP64 check of the FMM conventions in csrc/harmonics.h + operators.cpp:
// P2M, M2M, M2L, L2L, L2P, P2L, M2P against direct 1/r sums.  Development tool
// and CPU test (tests/test_host_math.py); not part of the product path.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2409_12375_b200/csrc/harmonics.h"
#include "../paper_2409_12375_b200/csrc/operators.h"

using namespace xrl;

static RecTables<double> tab;

struct Pt { double x, y, z, q; };

static std::vector<Pt> box_points(std::mt19937_64& g, const double c[3], double s, int n)
{
    std::uniform_real_distribution<double> u(-0.5, 0.5), uq(-1, 1);
    std::vector<Pt> p(n);
    for (auto& a : p) { a.x = c[0] + s * u(g); a.y = c[1] + s * u(g); a.z = c[2] + s * u(g); a.q = uq(g); }
    return p;
}

static void p2m(const std::vector<Pt>& src, const double c[3], double s, double* mu)
{
    double h[kNC];
    for (int i = 0; i < kNC; ++i) mu[i] = 0;
    for (auto& p : src) {
        regular_harmonics<kP>((p.x - c[0]) / s, (p.y - c[1]) / s, (p.z - c[2]) / s, tab, h);
        for (int i = 0; i < kNC; ++i) mu[i] += p.q * h[i];
    }
}

static double l2p(const double* ell, const double c[3], double s, const Pt& t)
{
    double h[kNC];
    regular_harmonics<kP>((t.x - c[0]) / s, (t.y - c[1]) / s, (t.z - c[2]) / s, tab, h);
    double phi = 0;
    for (int i = 0; i < kNC; ++i) phi += ell[i] * h[i];
    return phi / s;
}

static double m2p(const double* mu, const double c[3], double s, const Pt& t)
{
    double h[kNC];
    irregular_harmonics<kP>((t.x - c[0]) / s, (t.y - c[1]) / s, (t.z - c[2]) / s, tab, h);
    double phi = 0;
    for (int i = 0; i < kNC; ++i) phi += cweight(i) * mu[i] * h[i];
    return phi / s;
}

static void p2l(const std::vector<Pt>& src, const double c[3], double s, double* ell)
{
    double h[kNC];
    for (int i = 0; i < kNC; ++i) ell[i] = 0;
    for (auto& p : src) {
        irregular_harmonics<kP>((p.x - c[0]) / s, (p.y - c[1]) / s, (p.z - c[2]) / s, tab, h);
        for (int i = 0; i < kNC; ++i) ell[i] += p.q * cweight(i) * h[i];
    }
}

static double direct(const std::vector<Pt>& src, const Pt& t)
{
    double s = 0;
    for (auto& p : src) s += p.q / std::sqrt((t.x - p.x) * (t.x - p.x) + (t.y - p.y) * (t.y - p.y) + (t.z - p.z) * (t.z - p.z));
    return s;
}

static void matvec(const double* T, const double* x, double* y)
{
    for (int i = 0; i < kNC; ++i) {
        double s = 0;
        for (int j = 0; j < kNC; ++j) s += T[i * kNC + j] * x[j];
        y[i] = s;
    }
}

int main()
{
    fill_recurrence_tables(tab);
    HostOperators ops;
    build_operators(ops);
    std::mt19937_64 g(7);
    int fails = 0;
    auto report = [&](const char* name, double err, double tol) {
        std::printf("%-28s rel err %.3e  (tol %.1e) %s\n", name, err, tol, err < tol ? "ok" : "FAIL");
        if (!(err < tol)) ++fails;
    };
    const double s = 0.25;
    const double cs[3] = {0.125, 0.375, 0.625};

    // P2M -> M2P, source box, targets 2 boxes away
    {
        auto src = box_points(g, cs, s, 60);
        double mu[kNC];
        p2m(src, cs, s, mu);
        double e2 = 0, n2 = 0;
        for (int it = 0; it < 50; ++it) {
            double ct[3] = {cs[0] + 2 * s, cs[1] + (it % 3 - 1) * s, cs[2] + 2 * s};
            auto t = box_points(g, ct, s, 1)[0];
            double a = m2p(mu, cs, s, t), b = direct(src, t);
            e2 += (a - b) * (a - b); n2 += b * b;
        }
        report("P2M->M2P", std::sqrt(e2 / n2), 1e-4);
    }
    // P2L -> L2P
    {
        auto src = box_points(g, cs, s, 60);
        double ct[3] = {cs[0] - 2 * s, cs[1] + 2 * s, cs[2]};
        double ell[kNC];
        p2l(src, ct, s, ell);
        double e2 = 0, n2 = 0;
        for (int it = 0; it < 50; ++it) {
            auto t = box_points(g, ct, s, 1)[0];
            double a = l2p(ell, ct, s, t), b = direct(src, t);
            e2 += (a - b) * (a - b); n2 += b * b;
        }
        report("P2L->L2P", std::sqrt(e2 / n2), 1e-4);
    }
    // M2L over all 316 offsets: P2M -> M2L -> L2P vs direct
    {
        double worst = 0, sum_e = 0, sum_n = 0;
        for (int o = 0; o < kNM2L; ++o) {
            auto src = box_points(g, cs, s, 40);
            double mu[kNC], ell[kNC];
            p2m(src, cs, s, mu);
            double ct[3] = {cs[0] + ops.m2l_off[o][0] * s, cs[1] + ops.m2l_off[o][1] * s, cs[2] + ops.m2l_off[o][2] * s};
            matvec(&ops.m2l[size_t(o) * kNC * kNC], mu, ell);
            double e2 = 0, n2 = 0;
            for (int it = 0; it < 20; ++it) {
                auto t = box_points(g, ct, s, 1)[0];
                double a = l2p(ell, ct, s, t), b = direct(src, t);
                e2 += (a - b) * (a - b); n2 += b * b;
            }
            worst = std::max(worst, std::sqrt(e2 / n2));
            sum_e += e2; sum_n += n2;
        }
        report("M2L all offsets (joint)", std::sqrt(sum_e / sum_n), 2e-5);
        report("M2L worst offset", worst, 2e-3);
    }
    // M2M: 8 children -> parent -> M2P far away
    {
        const double cp[3] = {0.5, 0.5, 0.5};
        const double sp = 0.5;
        std::vector<Pt> all;
        double mup[kNC] = {0};
        for (int oc = 0; oc < 8; ++oc) {
            double cc[3] = {cp[0] + ((oc & 1) ? 0.25 : -0.25) * sp, cp[1] + ((oc & 2) ? 0.25 : -0.25) * sp,
                            cp[2] + ((oc & 4) ? 0.25 : -0.25) * sp};
            auto src = box_points(g, cc, sp / 2, 10);
            all.insert(all.end(), src.begin(), src.end());
            double muc[kNC], tmp[kNC];
            p2m(src, cc, sp / 2, muc);
            matvec(&ops.m2m[size_t(oc) * kNC * kNC], muc, tmp);
            for (int i = 0; i < kNC; ++i) mup[i] += tmp[i];
        }
        double mud[kNC];
        p2m(all, cp, sp, mud);
        double e = 0, n = 0;
        for (int i = 0; i < kNC; ++i) { e += (mup[i] - mud[i]) * (mup[i] - mud[i]); n += mud[i] * mud[i]; }
        report("M2M == direct P2M (exact)", std::sqrt(e / n), 1e-13);
    }
    // L2L: P2L into parent, L2L to children == P2L into children (exact)
    {
        const double cp[3] = {0.5, 0.5, 0.5};
        const double sp = 0.5;
        double cf[3] = {cp[0] + 3 * sp, cp[1] - 2 * sp, cp[2] + 2.5 * sp};
        auto src = box_points(g, cf, sp, 30);
        double ellp[kNC];
        p2l(src, cp, sp, ellp);
        double e = 0, n = 0, e_eval = 0, n_eval = 0;
        for (int oc = 0; oc < 8; ++oc) {
            double cc[3] = {cp[0] + ((oc & 1) ? 0.25 : -0.25) * sp, cp[1] + ((oc & 2) ? 0.25 : -0.25) * sp,
                            cp[2] + ((oc & 4) ? 0.25 : -0.25) * sp};
            double ellc[kNC];
            matvec(&ops.l2l[size_t(oc) * kNC * kNC], ellp, ellc);
            // evaluating the shifted local must equal evaluating the parent local (exact)
            for (int it = 0; it < 5; ++it) {
                auto t = box_points(g, cc, sp / 2, 1)[0];
                double a = l2p(ellc, cc, sp / 2, t), b = l2p(ellp, cp, sp, t);
                e += (a - b) * (a - b); n += b * b;
                double d = direct(src, t);
                e_eval += (a - d) * (a - d); n_eval += d * d;
            }
        }
        report("L2L == parent local (exact)", std::sqrt(e / n), 1e-12);
        report("L2L local vs direct", std::sqrt(e_eval / n_eval), 1e-5);
    }
    std::printf("%s\n", fails ? "FAILED" : "ALL OK");
    return fails ? 1 : 0;
}
