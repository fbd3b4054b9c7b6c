// Host FP64 emulation of the M2L operand splits (development tool): 3xTF32 (the round-2 kernel) against
// 3xFP16 with power-of-2 scaling (one scale for all operators, one for all multipoles of an MVM), measured as the potential error of
// P2M -> M2L -> L2P against the FP64 chain.  Prints the operator magnitude ranges per degree as well.
// Build: g++ -O2 -fopenmp -I paper_2409_12375_b200/csrc tools/m2l_prec_check.cpp paper_2409_12375_b200/csrc/operators.cpp
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "harmonics.h"
#include "operators.h"

using namespace xrl;

static RecTables<double> tab;

static int deg(int i) { int n = 0; while ((n + 1) * (n + 1) <= i) ++n; return n; }

static float tf32_rna(float x)
{
    uint32_t u; std::memcpy(&u, &x, 4);
    u = (u + 0x1000u) & ~0x1fffu;
    float r; std::memcpy(&r, &u, 4); return r;
}
// round to fp16 (RN even), subnormals down to 2^-24, overflow -> inf
static double fp16(double x)
{
    if (x == 0) return 0;
    int e; std::frexp(x, &e);             // x = f 2^e, 0.5 <= |f| < 1
    int ee = std::max(e, -13);            // normal: 11 significant bits; exponent floor 2^-14 (e - 1 >= -14)
    const double q = std::ldexp(1.0, ee - 11);
    double r = std::nearbyint(x / q) * q;
    if (std::fabs(r) > 65504.0) return INFINITY;
    return r;
}

int main(int argc, char** argv)
{
    const int mode_pts = argc > 1 ? atoi(argv[1]) : 0;  // 0: volume, 1: plane, 2: few points
    fill_recurrence_tables(tab);
    HostOperators ops;
    build_operators(ops);
    // magnitude table of the operators: max |T| per (n_i, n_k) over all offsets, and per offset range
    double lo_all = 1e300, hi_all = 0;
    for (int o = 0; o < kNM2L; ++o) {
        const double* T = &ops.m2l[size_t(o) * kNC * kNC];
        double mx = 0, mn = 1e300;
        for (int i = 0; i < kNC * kNC; ++i) if (T[i] != 0) { mx = std::max(mx, std::fabs(T[i])); mn = std::min(mn, std::fabs(T[i])); }
        lo_all = std::min(lo_all, mn); hi_all = std::max(hi_all, mx);
        if (o == 0 || o == 100 || o == 315) std::printf("offset %d (%d,%d,%d): |T| in [%.3e, %.3e]\n", o, ops.m2l_off[o][0], ops.m2l_off[o][1], ops.m2l_off[o][2], mn, mx);
    }
    std::printf("all offsets: |T| in [%.3e, %.3e]\n", lo_all, hi_all);
    std::printf("max |T| by (n_i rows, n_k cols), offset (2,0,0):\n");
    {
        const int o = ops.m2l_index[(2 + 3) * 49 + 3 * 7 + 3];
        const double* T = &ops.m2l[size_t(o) * kNC * kNC];
        for (int ni = 0; ni <= kP; ++ni) {
            for (int nk = 0; nk <= kP; ++nk) {
                double mx = 0;
                for (int i = ni * ni; i < (ni + 1) * (ni + 1); ++i)
                    for (int k = nk * nk; k < (nk + 1) * (nk + 1); ++k) mx = std::max(mx, std::fabs(T[i * kNC + k]));
                std::printf(" %8.1e", mx);
            }
            std::printf("\n");
        }
    }
    std::mt19937_64 g(11);
    std::uniform_real_distribution<double> u(-0.5, 0.5), uq(-1, 1), ud(0, 1);
    double e_tf[3] = {0, 0, 0}, e_h[3] = {0, 0, 0}, nn[3] = {0, 0, 0};
    double mudeg[kP + 1] = {0};
    // the shipped scheme: ONE power-of-2 scale for all operators (largest |T| in [2^14, 2^15)) and one for all
    // multipoles of the MVM (largest |mu| in [2^14, 2^15)); boxes carry charges of magnitude 10^-(0..4)
    double tmax = 0;
    for (size_t i = 0; i < ops.m2l.size(); ++i) tmax = std::max(tmax, std::fabs(ops.m2l[i]));
    int eb; std::frexp(tmax, &eb); const double sb = std::ldexp(1.0, 15 - eb);
    for (int trial = 0; trial < 3; ++trial) {
        std::vector<std::vector<float>> mus(kNM2L, std::vector<float>(kNC));
        std::vector<std::vector<double>> mud(kNM2L, std::vector<double>(kNC));
        float amax = 0;
        for (int o = 0; o < kNM2L; ++o) {
            const int np = mode_pts == 2 ? 3 : 200;
            const double mag = std::pow(10.0, -4.0 * ud(g));
            std::vector<double> px(np), py(np), pz(np), pq(np);
            const double nz = u(g), ax = uq(g), ay = uq(g);
            for (int l = 0; l < np; ++l) {
                px[l] = u(g); py[l] = u(g);
                pz[l] = mode_pts == 1 ? std::max(-0.5, std::min(0.5, nz + 0.3 * ax * px[l] + 0.3 * ay * py[l])) : u(g);
                pq[l] = mag * (trial == 2 ? 1.0 + 0.01 * uq(g) : uq(g));  // trial 2: nearly uniform charges
            }
            double h[kNC];
            for (int i = 0; i < kNC; ++i) mud[o][i] = 0;
            for (int l = 0; l < np; ++l) {
                regular_harmonics<kP>(px[l], py[l], pz[l], tab, h);
                for (int i = 0; i < kNC; ++i) mud[o][i] += pq[l] * h[i];
            }
            for (int i = 0; i < kNC; ++i) {
                mus[o][i] = (float)mud[o][i];
                amax = std::max(amax, std::fabs(mus[o][i]));
                mudeg[deg(i)] = std::max(mudeg[deg(i)], std::fabs(mud[o][i]) / std::fabs(mud[o][0] != 0 ? mud[o][0] : 1));
            }
        }
        int ea; std::frexp((double)amax, &ea); const double sa = std::ldexp(1.0, 15 - ea);
        for (int o = 0; o < kNM2L; ++o) {
            const double* T = &ops.m2l[size_t(o) * kNC * kNC];
            const double* mu = mud[o].data();
            const float* muf = mus[o].data();
            double ell[kNC], ell_tf[kNC], ell_h[kNC], h[kNC];
            for (int i = 0; i < kNC; ++i) {
                double s = 0, stf = 0, sh = 0;
                for (int k = 0; k < kNC; ++k) {
                    s += T[i * kNC + k] * mu[k];
                    const float bf = (float)T[i * kNC + k];
                    const float ah = tf32_rna(muf[k]), al = muf[k] - ah, bh = tf32_rna(bf), bl = bf - bh;
                    stf += (double)al * bh + (double)ah * bl + (double)ah * bh;
                    const double xa = muf[k] * sa, xb = T[i * kNC + k] * sb;
                    const double hah = fp16(xa), hal = fp16(xa - hah), hbh = fp16(xb), hbl = fp16(xb - hbh);
                    sh += hal * hbh + hah * hbl + hah * hbh;
                }
                ell[i] = s; ell_tf[i] = (float)stf; ell_h[i] = (float)(sh / (sa * sb));
            }
            // potential at 20 targets in the target box (unit box coordinates), each box's error relative to its
            // own potential (the magnitudes differ by up to 10^4 between boxes)
            double eb2 = 0, eh2 = 0, n2 = 0;
            for (int it = 0; it < 20; ++it) {
                regular_harmonics<kP>(u(g), u(g), u(g), tab, h);
                double a = 0, b = 0, c = 0;
                for (int i = 0; i < kNC; ++i) { a += ell[i] * h[i]; b += ell_tf[i] * h[i]; c += ell_h[i] * h[i]; }
                eb2 += (b - a) * (b - a); eh2 += (c - a) * (c - a); n2 += a * a;
            }
            e_tf[trial] += eb2 / n2; e_h[trial] += eh2 / n2; nn[trial] += 1;
        }
        std::printf("trial %d (%s charges, box magnitudes 1..1e-4): per-box potential rel err (rms) 3xTF32 %.3e, "
                    "3xFP16 (global scales) %.3e\n", trial, trial == 2 ? "uniform" : "random",
                    std::sqrt(e_tf[trial] / nn[trial]), std::sqrt(e_h[trial] / nn[trial]));
    }
    std::printf("max |mu_n| / |mu_0| by degree:");
    for (int n = 0; n <= kP; ++n) std::printf(" %.1e", mudeg[n]);
    std::printf("\n");
    return 0;
}
