// Host FP64 construction of the FMM translation operators (see operators.h).
//
// The complex translation theorems used (factorial normalisation of
// harmonics.h, unit box width):
//   M2M  M_p{n,m} = sum_{j,k} (M_c{j,k} / 2^j) conj(R_{n-j}^{m-k}(t)),  t = (c_c - c_p)/s_p
//   L2L  L_c{j,k} = 2^{-(j+1)} sum_{n,m} L_p{n,m} R_{n-j}^{m-k}(t)
//   M2L  L{n,m}   = (-1)^{n+m} sum_{j,k} M{j,k} I_{j+n}^{k-m}(d),        d = (c_L - c_M)/s
// (from R(a+b) = sum R_j^k(a) R_{n-j}^{m-k}(b) and
//  I_n^m(a - b) = sum conj(R_j^k(b)) I_{n+j}^{m+k}(a), |b| < |a|).
// Each complex operator is turned into a real (p+1)^2 x (p+1)^2 matrix acting on
// the real storage by applying it to every real basis vector.
#include "operators.h"

#include <cmath>
#include <complex>
#include <cstring>

namespace xrl {

using cd = std::complex<double>;

namespace {

double fact(int n)
{
    double f = 1;
    for (int i = 2; i <= n; ++i) f *= i;
    return f;
}

// full-range index for complex arrays: n*n + n + m
inline int fidx(int n, int m) { return n * n + n + m; }

// Factorial-normalised complex harmonics for n <= L, all m.
void cplx_harmonics(double x, double y, double z, int L, std::vector<cd>& R, std::vector<cd>& I)
{
    const int N = (L + 1) * (L + 1);
    R.assign(N, cd(0));
    I.assign(N, cd(0));
    const double r2 = x * x + y * y + z * z;
    const cd w(x, y);
    cd rm(1.0, 0.0);                     // R_m^m
    cd im = (r2 > 0) ? cd(1.0 / std::sqrt(r2), 0.0) : cd(0);  // I_m^m
    for (int m = 0; m <= L; ++m) {
        if (m > 0) {
            rm = -w / double(2 * m) * rm;
            im = -double(2 * m - 1) * w / r2 * im;
        }
        cd rp = rm, rq = 0, ip = im, iq = 0;
        R[fidx(m, m)] = rm;
        I[fidx(m, m)] = im;
        for (int n = m + 1; n <= L; ++n) {
            cd rn = (double(2 * n - 1) * z * rp - r2 * rq) / double((n + m) * (n - m));
            cd in = (double(2 * n - 1) * z * ip - double((n + m - 1) * (n - m - 1)) * iq) / r2;
            rq = rp; rp = rn; iq = ip; ip = in;
            R[fidx(n, m)] = rn;
            I[fidx(n, m)] = in;
        }
    }
    for (int n = 1; n <= L; ++n)
        for (int m = 1; m <= n; ++m) {
            const double sg = (m & 1) ? -1.0 : 1.0;
            R[fidx(n, -m)] = sg * std::conj(R[fidx(n, m)]);
            I[fidx(n, -m)] = sg * std::conj(I[fidx(n, m)]);
        }
}

inline double Nnm(int n, int m) { return std::sqrt(fact(n + m) * fact(n - m)); }

// real mu (tilde) -> complex factorial M, all m
void mu_to_M(const double* mu, std::vector<cd>& M)
{
    M.assign(kNC, cd(0));
    for (int n = 0; n <= kP; ++n) {
        M[fidx(n, 0)] = cd(mu[hidx(n, 0)], 0) / Nnm(n, 0);
        for (int m = 1; m <= n; ++m) {
            cd t = cd(mu[hidx(n, m)], -mu[hidx(n, m) + 1]) / Nnm(n, m);
            M[fidx(n, m)] = t;
            M[fidx(n, -m)] = ((m & 1) ? -1.0 : 1.0) * std::conj(t);
        }
    }
}

void M_to_mu(const std::vector<cd>& M, double* mu)
{
    for (int n = 0; n <= kP; ++n) {
        mu[hidx(n, 0)] = (M[fidx(n, 0)] * Nnm(n, 0)).real();
        for (int m = 1; m <= n; ++m) {
            cd t = M[fidx(n, m)] * Nnm(n, m);
            mu[hidx(n, m)] = t.real();
            mu[hidx(n, m) + 1] = -t.imag();
        }
    }
}

void ell_to_L(const double* ell, std::vector<cd>& L)
{
    L.assign(kNC, cd(0));
    for (int n = 0; n <= kP; ++n) {
        L[fidx(n, 0)] = cd(ell[hidx(n, 0)], 0) * Nnm(n, 0);
        for (int m = 1; m <= n; ++m) {
            cd t = cd(ell[hidx(n, m)], -ell[hidx(n, m) + 1]) * 0.5 * Nnm(n, m);
            L[fidx(n, m)] = t;
            L[fidx(n, -m)] = ((m & 1) ? -1.0 : 1.0) * std::conj(t);
        }
    }
}

void L_to_ell(const std::vector<cd>& L, double* ell)
{
    for (int n = 0; n <= kP; ++n) {
        ell[hidx(n, 0)] = (L[fidx(n, 0)] / Nnm(n, 0)).real();
        for (int m = 1; m <= n; ++m) {
            cd t = L[fidx(n, m)] / Nnm(n, m);
            ell[hidx(n, m)] = 2.0 * t.real();
            ell[hidx(n, m) + 1] = -2.0 * t.imag();
        }
    }
}

template <typename F>
void realify(F&& apply, double* out /* [kNC][kNC] row = output */)
{
    std::vector<double> e(kNC), col(kNC);
    for (int j = 0; j < kNC; ++j) {
        std::fill(e.begin(), e.end(), 0.0);
        e[j] = 1.0;
        apply(e.data(), col.data());
        for (int i = 0; i < kNC; ++i) out[i * kNC + j] = col[i];
    }
}

}  // namespace

void build_operators(HostOperators& ops)
{
    ops.m2m.assign(8 * kNC * kNC, 0.0);
    ops.l2l.assign(8 * kNC * kNC, 0.0);
    ops.m2l.assign(size_t(kNM2L) * kNC * kNC, 0.0);

    std::vector<cd> Rt, It, A, B;
    for (int oc = 0; oc < 8; ++oc) {
        const double t[3] = {((oc & 1) ? 0.25 : -0.25), ((oc & 2) ? 0.25 : -0.25), ((oc & 4) ? 0.25 : -0.25)};
        cplx_harmonics(t[0], t[1], t[2], kP, Rt, It);
        // M2M: child -> parent
        realify([&](const double* mu_c, double* mu_p) {
            mu_to_M(mu_c, A);
            B.assign(kNC, cd(0));
            for (int n = 0; n <= kP; ++n)
                for (int m = -n; m <= n; ++m) {
                    cd s = 0;
                    for (int j = 0; j <= n; ++j)
                        for (int k = -j; k <= j; ++k) {
                            const int nn = n - j, mm = m - k;
                            if (mm < -nn || mm > nn) continue;
                            s += A[fidx(j, k)] * std::ldexp(1.0, -j) * std::conj(Rt[fidx(nn, mm)]);
                        }
                    B[fidx(n, m)] = s;
                }
            M_to_mu(B, mu_p);
        }, &ops.m2m[size_t(oc) * kNC * kNC]);
        // L2L: parent -> child
        realify([&](const double* ell_p, double* ell_c) {
            ell_to_L(ell_p, A);
            B.assign(kNC, cd(0));
            for (int j = 0; j <= kP; ++j)
                for (int k = -j; k <= j; ++k) {
                    cd s = 0;
                    for (int n = j; n <= kP; ++n)
                        for (int m = -n; m <= n; ++m) {
                            const int nn = n - j, mm = m - k;
                            if (mm < -nn || mm > nn) continue;
                            s += A[fidx(n, m)] * Rt[fidx(nn, mm)];
                        }
                    B[fidx(j, k)] = s * std::ldexp(1.0, -(j + 1));
                }
            L_to_ell(B, ell_c);
        }, &ops.l2l[size_t(oc) * kNC * kNC]);
    }

    int idx = 0;
    for (int i = 0; i < 343; ++i) ops.m2l_index[i] = -1;
    for (int dx = -3; dx <= 3; ++dx)
        for (int dy = -3; dy <= 3; ++dy)
            for (int dz = -3; dz <= 3; ++dz) {
                if (std::abs(dx) <= 1 && std::abs(dy) <= 1 && std::abs(dz) <= 1) continue;
                ops.m2l_off[idx][0] = dx;
                ops.m2l_off[idx][1] = dy;
                ops.m2l_off[idx][2] = dz;
                ops.m2l_index[(dx + 3) * 49 + (dy + 3) * 7 + (dz + 3)] = idx;
                ++idx;
            }
    // the 316 offsets are independent: one per OpenMP thread (context creation; ~1 s single-threaded)
#pragma omp parallel for schedule(dynamic) firstprivate(Rt, It, A, B)
    for (int o = 0; o < kNM2L; ++o) {
        const int* d = ops.m2l_off[o];
        cplx_harmonics(double(d[0]), double(d[1]), double(d[2]), 2 * kP, Rt, It);
        realify([&](const double* mu, double* ell) {
            mu_to_M(mu, A);
            B.assign(kNC, cd(0));
            for (int n = 0; n <= kP; ++n)
                for (int m = -n; m <= n; ++m) {
                    cd s = 0;
                    for (int j = 0; j <= kP; ++j)
                        for (int k = -j; k <= j; ++k) {
                            const int nn = j + n, mm = k - m;
                            if (mm < -nn || mm > nn) continue;
                            s += A[fidx(j, k)] * It[fidx(nn, mm)];
                        }
                    B[fidx(n, m)] = (((n + m) & 1) ? -1.0 : 1.0) * s;
                }
            L_to_ell(B, ell);
        }, &ops.m2l[size_t(o) * kNC * kNC]);
    }
}

}  // namespace xrl
