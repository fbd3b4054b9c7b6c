// Real storage of the semi-normalised solid harmonics used by the FMM passes.
//
// Laplace kernel 1/|r - r'| (Eq. 1; FMM over centroids PAPER.md:116,
// refs [22],[23]).  Complex factorial-normalised harmonics (Condon-Shortley
// phase):
//   R_n^m(r) = r^n P_n^m(cos t) e^{i m phi} / (n+m)!
//   I_n^m(r) = (n-m)! P_n^m(cos t) e^{i m phi} / r^{n+1}
// with 1/|a - b| = sum_{n,m} conj(R_n^m(b)) I_n^m(a) for |b| < |a|.
// Stored semi-normalised:  Rt = R * N,  It = I / N,  N_n^m = sqrt((n+m)!(n-m)!)
// so that |Rt| <= r^n and |It| <= r^{-n-1} (O(1) numbers in box units).
//
// Real vector of (p+1)^2 entries for m >= 0 (negative m follow from
// X_n^{-m} = (-1)^m conj(X_n^m)):
//   h[n*n]          = Re X_n^0
//   h[n*n + 2m - 1] = Re X_n^m     (m = 1..n)
//   h[n*n + 2m]     = Im X_n^m
//
// Recurrences (both families share the constants A, B, D):
//   Rt_m^m = -D_m (x + i y) Rt_{m-1}^{m-1},          Rt_0^0 = 1
//   Rt_n^m = A_nm z Rt_{n-1}^m - B_nm r^2 Rt_{n-2}^m
//   It_m^m = -D_m (x + i y)/r^2 It_{m-1}^{m-1},      It_0^0 = 1/r
//   It_n^m = (A_nm z It_{n-1}^m - B_nm It_{n-2}^m) / r^2
//   D_m = sqrt((2m-1)/(2m)),  A_nm = (2n-1)/sqrt((n+m)(n-m)),
//   B_nm = sqrt((n+m-1)(n-m-1)/((n+m)(n-m))).
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define XRL_HD __host__ __device__ __forceinline__
#else
#define XRL_HD inline
#endif

namespace xrl {

constexpr int kP = 10;                       // expansion order p (north star: p = 10)
constexpr int kNC = (kP + 1) * (kP + 1);     // 121 real coefficients
constexpr int kNRHS = 6;                     // 3 complex components = 6 real RHS

XRL_HD int hidx(int n, int m) { return n * n + (m == 0 ? 0 : 2 * m - 1); }

// Constant tables indexed by (n, m) -> n*(P+1)+m.  Filled by fill_recurrence_tables.
template <typename T>
struct RecTables {
    T A[(kP + 1) * (kP + 1)];
    T B[(kP + 1) * (kP + 1)];
    T D[kP + 1];
};

template <typename T>
inline void fill_recurrence_tables(RecTables<T>& t)
{
    for (int n = 0; n <= kP; ++n)
        for (int m = 0; m <= kP; ++m) {
            double a = 0, b = 0;
            if (m < n) {
                a = (2.0 * n - 1) / std::sqrt(double(n + m) * double(n - m));
                b = (n - m - 1 > 0) ? std::sqrt(double(n + m - 1) * double(n - m - 1) / (double(n + m) * double(n - m))) : 0.0;
            }
            t.A[n * (kP + 1) + m] = T(a);
            t.B[n * (kP + 1) + m] = T(b);
        }
    t.D[0] = T(0);
    for (int m = 1; m <= kP; ++m) t.D[m] = T(std::sqrt((2.0 * m - 1) / (2.0 * m)));
}

// Regular semi-normalised harmonics Rt_n^m(x,y,z), n <= P, real storage into h.
template <int P, typename T, typename Tab>
XRL_HD void regular_harmonics(T x, T y, T z, const Tab& tab, T* h)
{
    const T r2 = x * x + y * y + z * z;
    T cr = T(1), ci = T(0);  // Rt_m^m
#pragma unroll
    for (int m = 0; m <= P; ++m) {
        if (m > 0) {
            const T d = -tab.D[m];
            const T nr = d * (x * cr - y * ci);
            const T ni = d * (x * ci + y * cr);
            cr = nr; ci = ni;
        }
        T pr = cr, pi = ci;       // n = m
        T qr = T(0), qi = T(0);   // n = m - 1
        if (m == 0) h[0] = cr;
        else { h[hidx(m, m)] = cr; h[hidx(m, m) + 1] = ci; }
#pragma unroll
        for (int n = 1; n <= P; ++n) {
            if (n <= m) continue;
            const T a = tab.A[n * (P + 1) + m] * z;
            const T b = tab.B[n * (P + 1) + m] * r2;
            const T nr = a * pr - b * qr;
            const T ni = a * pi - b * qi;
            qr = pr; qi = pi; pr = nr; pi = ni;
            if (m == 0) h[n * n] = nr;
            else { h[hidx(n, m)] = nr; h[hidx(n, m) + 1] = ni; }
        }
    }
}

// Irregular semi-normalised harmonics It_n^m(x,y,z), n <= P, real storage into h.
template <int P, typename T, typename Tab>
XRL_HD void irregular_harmonics(T x, T y, T z, const Tab& tab, T* h)
{
    const T r2 = x * x + y * y + z * z;
    const T ir2 = T(1) / r2;
    T cr = T(1) / std::sqrt(r2), ci = T(0);
#pragma unroll
    for (int m = 0; m <= P; ++m) {
        if (m > 0) {
            const T d = -tab.D[m] * ir2;
            const T nr = d * (x * cr - y * ci);
            const T ni = d * (x * ci + y * cr);
            cr = nr; ci = ni;
        }
        T pr = cr, pi = ci;
        T qr = T(0), qi = T(0);
        if (m == 0) h[0] = cr;
        else { h[hidx(m, m)] = cr; h[hidx(m, m) + 1] = ci; }
#pragma unroll
        for (int n = 1; n <= P; ++n) {
            if (n <= m) continue;
            const T a = tab.A[n * (P + 1) + m] * z;
            const T b = tab.B[n * (P + 1) + m];
            const T nr = (a * pr - b * qr) * ir2;
            const T ni = (a * pi - b * qi) * ir2;
            qr = pr; qi = pi; pr = nr; pi = ni;
            if (m == 0) h[n * n] = nr;
            else { h[hidx(n, m)] = nr; h[hidx(n, m) + 1] = ni; }
        }
    }
}

// Streaming variants: f(i, value) for every real coefficient i (same order of
// evaluation, no (p+1)^2 array: L2P/M2P contract on the fly).
template <int P, bool kUnrollM = true, typename T, typename Tab, typename F>
XRL_HD void regular_harmonics_visit(T x, T y, T z, const Tab& tab, F&& f)
{
    const T r2 = x * x + y * y + z * z;
    T cr = T(1), ci = T(0);
#pragma unroll (kUnrollM ? P + 1 : 1)
    for (int m = 0; m <= P; ++m) {
        if (m > 0) {
            const T d = -tab.D[m];
            const T nr = d * (x * cr - y * ci);
            const T ni = d * (x * ci + y * cr);
            cr = nr; ci = ni;
        }
        T pr = cr, pi = ci;
        T qr = T(0), qi = T(0);
        if (m == 0) f(0, cr);
        else { f(hidx(m, m), cr); f(hidx(m, m) + 1, ci); }
#pragma unroll
        for (int n = 1; n <= P; ++n) {
            if (n <= m) continue;
            const T a = tab.A[n * (P + 1) + m] * z;
            const T b = tab.B[n * (P + 1) + m] * r2;
            const T nr = a * pr - b * qr;
            const T ni = a * pi - b * qi;
            qr = pr; qi = pi; pr = nr; pi = ni;
            if (m == 0) f(n * n, nr);
            else { f(hidx(n, m), nr); f(hidx(n, m) + 1, ni); }
        }
    }
}

template <int P, bool kUnrollM = true, typename T, typename Tab, typename F>
XRL_HD void irregular_harmonics_visit(T x, T y, T z, const Tab& tab, F&& f)
{
    const T r2 = x * x + y * y + z * z;
    const T ir2 = T(1) / r2;
    T cr = T(1) / std::sqrt(r2), ci = T(0);
#pragma unroll (kUnrollM ? P + 1 : 1)
    for (int m = 0; m <= P; ++m) {
        if (m > 0) {
            const T d = -tab.D[m] * ir2;
            const T nr = d * (x * cr - y * ci);
            const T ni = d * (x * ci + y * cr);
            cr = nr; ci = ni;
        }
        T pr = cr, pi = ci;
        T qr = T(0), qi = T(0);
        if (m == 0) f(0, cr);
        else { f(hidx(m, m), cr); f(hidx(m, m) + 1, ci); }
#pragma unroll
        for (int n = 1; n <= P; ++n) {
            if (n <= m) continue;
            const T a = tab.A[n * (P + 1) + m] * z;
            const T b = tab.B[n * (P + 1) + m];
            const T nr = (a * pr - b * qr) * ir2;
            const T ni = (a * pi - b * qi) * ir2;
            qr = pr; qi = pi; pr = nr; pi = ni;
            if (m == 0) f(n * n, nr);
            else { f(hidx(n, m), nr); f(hidx(n, m) + 1, ni); }
        }
    }
}

// Weight c of the real contraction phi*s = sum c_i mu_i It_i (M2P) and of
// ell = sum q c_i It_i (P2L): 1 for m = 0, 2 for the (re, im) pair of m > 0.
XRL_HD float cweight(int i)
{
    // i = n*n + j with j = 0..2n; m = (j+1)/2
    int n = 0;
    while ((n + 1) * (n + 1) <= i) ++n;
    return (i == n * n) ? 1.f : 2.f;
}

}  // namespace xrl
