// xrl_extract: the R/L extraction sweep, host orchestration over the C-ABI.
//
// For each frequency f ("solve ... at each frequency point"): the loop-space operator
// (Eq. 8-9, xrl_operator_create), the diagonal-of-P preconditioner (Eq. 10: xrl_precond_build, or the
// exact Q^-1 of xrl_precond_build_exact when block_size < 0),
// one preconditioned GMRES with the n_ports port excitations batched as right-hand sides
// (xrl_port_rhs, xrl_gmres), the port currents (xrl_port_currents) give the admittance
// Y[:, q] = I(unit volts on port q); Z = Y^-1 (FP64 Gauss-Jordan, partial pivoting),
// R = Re Z, L = Im Z / (2 pi f) (R and L per frequency).
#include <cmath>
#include <complex>
#include <vector>

#include <cuda_runtime.h>

#include "xrl_internal.h"

using cplx = std::complex<double>;

namespace {

bool invert(std::vector<cplx>& a, int n)  // in place, row-major
{
    std::vector<cplx> inv(n * n, 0.0);
    for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
    for (int c = 0; c < n; ++c) {
        int p = c;
        for (int r = c + 1; r < n; ++r)
            if (std::abs(a[r * n + c]) > std::abs(a[p * n + c])) p = r;
        if (std::abs(a[p * n + c]) == 0.0) return false;
        if (p != c)
            for (int k = 0; k < n; ++k) { std::swap(a[p * n + k], a[c * n + k]); std::swap(inv[p * n + k], inv[c * n + k]); }
        const cplx d = 1.0 / a[c * n + c];
        for (int k = 0; k < n; ++k) { a[c * n + k] *= d; inv[c * n + k] *= d; }
        for (int r = 0; r < n; ++r) {
            if (r == c) continue;
            const cplx f = a[r * n + c];
            if (f == 0.0) continue;
            for (int k = 0; k < n; ++k) { a[r * n + k] -= f * a[c * n + k]; inv[r * n + k] -= f * inv[c * n + k]; }
        }
    }
    a = inv;
    return true;
}

}  // namespace

extern "C" xrl_status xrl_extract(xrl_tree tree, xrl_near near, xrl_topo topo, const double* zs, double sigma,
                                  double zeta, int32_t n_freq, const double* freqs, int32_t block_size,
                                  const xrl_gmres_opts* opts, double* z, double* r, double* l, int32_t* iters,
                                  double* true_rre)
{
    if (!tree || !near || !topo || !freqs || n_freq < 1) {
        xrl::set_error("xrl_extract: null argument or n_freq < 1");
        return XRL_EINVAL;
    }
    if (tree->part_world > 1) {
        xrl::set_error("xrl_extract: the extraction sweep runs on single-rank trees only (part_world = %d)",
                       tree->part_world);
        return XRL_EUNSUPPORTED;
    }
    const int np = topo->n_ports;
    if (np < 1) { xrl::set_error("xrl_extract: the topology has no ports"); return XRL_EINVAL; }
    for (int j = 0; j < n_freq; ++j)
        if (!(freqs[j] > 0)) { xrl::set_error("xrl_extract: frequencies must be > 0"); return XRL_EINVAL; }
    const int64_t nl = topo->n_loops;
    void *b = nullptr, *x = nullptr;
    if (cudaSetDevice(tree->ctx->device) != cudaSuccess || cudaMalloc(&b, (size_t)np * nl * 8) != cudaSuccess ||
        cudaMalloc(&x, (size_t)np * nl * 8) != cudaSuccess) {
        cudaFree(b);
        xrl::set_error("xrl_extract: device allocation failed");
        return XRL_ENOMEM;
    }
    xrl_status result = XRL_OK;
    std::vector<int32_t> it(np), conv(np);
    std::vector<double> rre(np), trre(np), ip((size_t)np * np * 2);
    for (int j = 0; j < n_freq && result >= 0; ++j) {
        xrl_op op = nullptr;
        xrl_precond pc = nullptr;
        xrl_status s = xrl_operator_create(tree, near, topo, zs, sigma, zeta, freqs[j], &op);
        if (s == XRL_OK) s = block_size < 0 ? xrl_precond_build_exact(op, &pc) : xrl_precond_build(op, block_size > 0 ? block_size : 64, &pc);
        for (int q = 0; q < np && s == XRL_OK; ++q) s = xrl_port_rhs(topo, q, 1.0, (char*)b + (size_t)q * nl * 8);
        if (s == XRL_OK && cudaMemset(x, 0, (size_t)np * nl * 8) != cudaSuccess) s = XRL_ECUDA;
        if (s == XRL_OK || s == XRL_ENOCONV) {
            s = xrl_gmres(op, pc, b, x, np, opts, it.data(), rre.data(), trre.data(), conv.data());
            if (s == XRL_ENOCONV) result = XRL_ENOCONV;
        }
        if (s == XRL_OK || s == XRL_ENOCONV) s = xrl_port_currents(topo, x, np, ip.data());
        if (s < 0) result = s;
        xrl_precond_destroy(pc);
        xrl_operator_destroy(op);
        if (s < 0) break;
        // Y[p][q] = current on port p for unit volts on port q (ip is [rhs q][port p][re, im])
        std::vector<cplx> Y((size_t)np * np);
        for (int q = 0; q < np; ++q)
            for (int p = 0; p < np; ++p) Y[p * np + q] = cplx(ip[((size_t)q * np + p) * 2], ip[((size_t)q * np + p) * 2 + 1]);
        if (!invert(Y, np)) { xrl::set_error("xrl_extract: singular port admittance at f = %g Hz", freqs[j]); result = XRL_ESINGULAR; break; }
        const double w = 2.0 * M_PI * freqs[j];
        for (int e = 0; e < np * np; ++e) {
            const size_t o = (size_t)j * np * np + e;
            if (z) { z[2 * o] = Y[e].real(); z[2 * o + 1] = Y[e].imag(); }
            if (r) r[o] = Y[e].real();
            if (l) l[o] = Y[e].imag() / w;
        }
        for (int q = 0; q < np; ++q) {
            if (iters) iters[(size_t)j * np + q] = it[q];
            if (true_rre) true_rre[(size_t)j * np + q] = trre[q];
        }
    }
    cudaFree(b);
    cudaFree(x);
    return result;
}
