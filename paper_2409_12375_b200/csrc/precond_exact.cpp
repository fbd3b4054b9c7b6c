// Exact diagonal-of-P preconditioner: Q^-1 of Eq. 10,
//     Q = sum_t C_t diag(d) C_t^T,  d_k = Z_s,k / A_k + j alpha P_kk,  C_t = M A_t,
// applied exactly as Eq. 11 prescribes (the paper factorises Q once per frequency with
// Pardiso and solves per GMRES iteration).  Here: Q assembled on the host in FP64 complex
// (sparse, pattern = loops sharing a panel), nested-dissection (METIS) ordering, else approximate minimum
// degree, then a host sparse LU with partial pivoting (cuSOLVER's low-level csrlu, the library analogue of
// Pardiso), factorised once per operator; every apply copies v to the host, runs the two triangular solves
// per right-hand side and copies z back (synchronous on the context stream).
//
// cuSOLVER/cuSPARSE are opened at run time (dlopen) on the first exact build, so the rest of libxrl never
// depends on them; a missing library makes xrl_precond_build_exact fail with a message (no fallback).
#include <dlfcn.h>

#include <algorithm>
#include <complex>
#include <cstdlib>
#include <numeric>
#include <vector>

#include <cuComplex.h>
#include <cuda_runtime.h>

#include "xrl_internal.h"

using namespace xrl;

namespace {

// ---- the few cuSOLVER / cuSPARSE entry points used (C ABI, opaque handles)
typedef void* SpHandle;
typedef void* MatDescr;
typedef void* LuInfo;
struct Api {
    bool ok = false;
    int (*spCreate)(SpHandle*);
    int (*spDestroy)(SpHandle);
    int (*createLuInfo)(LuInfo*);
    int (*destroyLuInfo)(LuInfo);
    int (*luAnalysis)(SpHandle, int, int, const MatDescr, const int*, const int*, LuInfo);
    int (*luBufferInfo)(SpHandle, int, int, const MatDescr, const cuDoubleComplex*, const int*, const int*, LuInfo,
                        size_t*, size_t*);
    int (*luFactor)(SpHandle, int, int, const MatDescr, const cuDoubleComplex*, const int*, const int*, LuInfo, double,
                    void*);
    int (*luZeroPivot)(SpHandle, LuInfo, double, int*);
    int (*luSolve)(SpHandle, int, const cuDoubleComplex*, cuDoubleComplex*, LuInfo, void*);
    int (*metisnd)(SpHandle, int, int, const MatDescr, const int*, const int*, const int64_t*, int*);
    int (*symamd)(SpHandle, int, int, const MatDescr, const int*, const int*, int*);
    int (*createDescr)(MatDescr*);
    int (*destroyDescr)(MatDescr);
    int (*setType)(MatDescr, int);
    int (*setBase)(MatDescr, int);
    std::string err;
};

Api& api()
{
    static Api a;
    static bool tried = false;
    if (tried) return a;
    tried = true;
    void* hs = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
    void* hp = dlopen("libcusparse.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!hs || !hp) {
        a.err = std::string("cannot load cuSOLVER/cuSPARSE: ") + dlerror();
        return a;
    }
    bool ok = true;
    auto sym = [&](void* h, const char* name) {
        void* f = dlsym(h, name);
        if (!f) { ok = false; a.err += std::string(" missing ") + name; }
        return f;
    };
    a.spCreate = (decltype(a.spCreate))sym(hs, "cusolverSpCreate");
    a.spDestroy = (decltype(a.spDestroy))sym(hs, "cusolverSpDestroy");
    a.createLuInfo = (decltype(a.createLuInfo))sym(hs, "cusolverSpCreateCsrluInfoHost");
    a.destroyLuInfo = (decltype(a.destroyLuInfo))sym(hs, "cusolverSpDestroyCsrluInfoHost");
    a.luAnalysis = (decltype(a.luAnalysis))sym(hs, "cusolverSpXcsrluAnalysisHost");
    a.luBufferInfo = (decltype(a.luBufferInfo))sym(hs, "cusolverSpZcsrluBufferInfoHost");
    a.luFactor = (decltype(a.luFactor))sym(hs, "cusolverSpZcsrluFactorHost");
    a.luZeroPivot = (decltype(a.luZeroPivot))sym(hs, "cusolverSpZcsrluZeroPivotHost");
    a.luSolve = (decltype(a.luSolve))sym(hs, "cusolverSpZcsrluSolveHost");
    a.symamd = (decltype(a.symamd))sym(hs, "cusolverSpXcsrsymamdHost");
    a.createDescr = (decltype(a.createDescr))sym(hp, "cusparseCreateMatDescr");
    a.destroyDescr = (decltype(a.destroyDescr))sym(hp, "cusparseDestroyMatDescr");
    a.setType = (decltype(a.setType))sym(hp, "cusparseSetMatType");
    a.setBase = (decltype(a.setBase))sym(hp, "cusparseSetMatIndexBase");
    a.metisnd = (decltype(a.metisnd))dlsym(hs, "cusolverSpXcsrmetisndHost");  // optional
    a.ok = ok;
    return a;
}

struct Exact {
    int n = 0;
    std::vector<int> perm;  // row i of the factored matrix = loop perm[i]
    SpHandle h = nullptr;
    MatDescr descr = nullptr;
    LuInfo info = nullptr;
    std::vector<char> work;
    std::vector<cuDoubleComplex> b, x;
    std::vector<float2> hv;
    int64_t nnz_q = 0;
    ~Exact()
    {
        Api& A = api();
        if (info) A.destroyLuInfo(info);
        if (descr) A.destroyDescr(descr);
        if (h) A.spDestroy(h);
    }
};

}  // namespace

namespace xrl {

xrl_status exact_build(xrl_precond pc)
{
    Api& A = api();
    if (!A.ok) { set_error("xrl_precond_build_exact: %s", A.err.c_str()); return XRL_EINVAL; }
    xrl_op op = pc->op;
    xrl_topo T = op->topo;
    const int64_t n = op->tree->n, nl = T->n_loops;
    if (nl >= ((int64_t)1 << 31)) { set_error("xrl_precond_build_exact: too many loops for 32-bit LU"); return XRL_EINVAL; }
    std::vector<double2> d;
    precond_diag(op, d);
    // ---- assemble Q (CSR, FP64 complex): Q_ab = sum_k d_k (c_a(k) . c_b(k)) over panels k shared by a, b
    const std::vector<int64_t>& cp = T->c_ptr_h;
    const std::vector<int32_t>& cc = T->c_col_h;
    const std::vector<double>& cv = T->c_val_h;
    std::vector<int64_t> kp(n + 1, 0);  // panel -> entries of C (transpose)
    for (int64_t q = 0; q < cp[nl]; ++q) ++kp[cc[q] + 1];
    for (int64_t k = 0; k < n; ++k) kp[k + 1] += kp[k];
    std::vector<int32_t> kl(cp[nl]);
    std::vector<int64_t> kq(cp[nl]);
    {
        std::vector<int64_t> fill(kp.begin(), kp.end() - 1);
        for (int64_t a = 0; a < nl; ++a)
            for (int64_t q = cp[a]; q < cp[a + 1]; ++q) {
                const int64_t f = fill[cc[q]]++;
                kl[f] = (int32_t)a;
                kq[f] = q;
            }
    }
    std::vector<std::vector<int32_t>> rc(nl);
    std::vector<std::vector<std::complex<double>>> rv(nl);
#pragma omp parallel
    {
        std::vector<std::complex<double>> acc(nl, 0.0);
        std::vector<char> mark(nl, 0);
        std::vector<int32_t> touched;
#pragma omp for schedule(dynamic, 256)
        for (int64_t a = 0; a < nl; ++a) {
            touched.clear();
            for (int64_t q = cp[a]; q < cp[a + 1]; ++q) {
                const int32_t k = cc[q];
                const double* ca = &cv[3 * q];
                const std::complex<double> dk(d[k].x, d[k].y);
                for (int64_t f = kp[k]; f < kp[k + 1]; ++f) {
                    const int32_t b = kl[f];
                    const double* cb = &cv[3 * kq[f]];
                    const double s = ca[0] * cb[0] + ca[1] * cb[1] + ca[2] * cb[2];
                    if (!mark[b]) { mark[b] = 1; touched.push_back(b); acc[b] = 0.0; }
                    acc[b] += dk * s;
                }
            }
            std::sort(touched.begin(), touched.end());
            rc[a] = touched;
            rv[a].resize(touched.size());
            for (size_t i = 0; i < touched.size(); ++i) {
                rv[a][i] = acc[touched[i]];
                mark[touched[i]] = 0;
            }
        }
    }
    const int N = (int)nl;
    std::vector<int> qp(N + 1, 0);
    for (int a = 0; a < N; ++a) qp[a + 1] = qp[a] + (int)rc[a].size();
    const int nnz = qp[N];
    std::vector<int> qc(nnz);
    for (int a = 0; a < N; ++a) std::copy(rc[a].begin(), rc[a].end(), qc.begin() + qp[a]);
    auto E = std::make_unique<Exact>();
    E->n = N;
    E->nnz_q = nnz;
    if (A.spCreate(&E->h) || A.createDescr(&E->descr) || A.setType(E->descr, 0 /* general */) ||
        A.setBase(E->descr, 0 /* zero */)) {
        set_error("xrl_precond_build_exact: cuSOLVER/cuSPARSE handle creation failed");
        return XRL_ECUDA;
    }
    // ---- fill-reducing ordering (Q's pattern is symmetric)
    E->perm.resize(N);
    int st = A.metisnd ? A.metisnd(E->h, N, nnz, E->descr, qp.data(), qc.data(), nullptr, E->perm.data()) : 1;
    if (st) st = A.symamd(E->h, N, nnz, E->descr, qp.data(), qc.data(), E->perm.data());
    if (st) std::iota(E->perm.begin(), E->perm.end(), 0);
    std::vector<int> inv(N);
    for (int i = 0; i < N; ++i) inv[E->perm[i]] = i;
    // B = Q(perm, perm)
    std::vector<int> bp(N + 1, 0), bc(nnz);
    std::vector<cuDoubleComplex> bv(nnz);
    for (int i = 0; i < N; ++i) bp[i + 1] = bp[i] + (int)rc[E->perm[i]].size();
    {
        std::vector<std::pair<int, std::complex<double>>> row;
        for (int i = 0; i < N; ++i) {
            const int a = E->perm[i];
            row.clear();
            for (size_t q = 0; q < rc[a].size(); ++q) row.emplace_back(inv[rc[a][q]], rv[a][q]);
            std::sort(row.begin(), row.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
            for (size_t q = 0; q < row.size(); ++q) {
                bc[bp[i] + q] = row[q].first;
                bv[bp[i] + q] = make_cuDoubleComplex(row[q].second.real(), row[q].second.imag());
            }
        }
    }
    // ---- LU with partial pivoting (threshold 1), factorised once
    size_t internal = 0, wbytes = 0;
    if (A.createLuInfo(&E->info) || A.luAnalysis(E->h, N, nnz, E->descr, bp.data(), bc.data(), E->info) ||
        A.luBufferInfo(E->h, N, nnz, E->descr, bv.data(), bp.data(), bc.data(), E->info, &internal, &wbytes)) {
        set_error("xrl_precond_build_exact: LU analysis failed");
        return XRL_ECUDA;
    }
    E->work.resize(std::max<size_t>(wbytes, 16));
    if (A.luFactor(E->h, N, nnz, E->descr, bv.data(), bp.data(), bc.data(), E->info, 1.0, E->work.data())) {
        set_error("xrl_precond_build_exact: LU factorisation failed");
        return XRL_ECUDA;
    }
    int zp = -1;
    A.luZeroPivot(E->h, E->info, 1e-14, &zp);
    if (zp >= 0) { set_error("xrl_precond_build_exact: singular Q (zero pivot at row %d)", zp); return XRL_ESINGULAR; }
    E->b.resize(N);
    E->x.resize(N);
    pc->exact = E.release();
    return XRL_OK;
}

void exact_apply(xrl_precond pc, const float2* v, float2* z, int nrhs)
{
    Exact* E = static_cast<Exact*>(pc->exact);
    Api& A = api();
    cudaStream_t st = pc->op->tree->ctx->stream;
    const int N = E->n;
    E->hv.resize((size_t)nrhs * N);
    XRL_CUDA(cudaMemcpyAsync(E->hv.data(), v, 8 * E->hv.size(), cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    for (int c = 0; c < nrhs; ++c) {
        float2* col = E->hv.data() + (size_t)c * N;
        for (int i = 0; i < N; ++i) {
            const float2 w = col[E->perm[i]];
            E->b[i] = make_cuDoubleComplex(w.x, w.y);
        }
        if (A.luSolve(E->h, N, E->b.data(), E->x.data(), E->info, E->work.data())) {
            set_error("xrl_precond_apply: LU solve failed");
            throw CudaError{XRL_ECUDA};
        }
        for (int i = 0; i < N; ++i) col[E->perm[i]] = make_float2((float)E->x[i].x, (float)E->x[i].y);
    }
    XRL_CUDA(cudaMemcpyAsync(z, E->hv.data(), 8 * E->hv.size(), cudaMemcpyHostToDevice, st));
    XRL_CUDA(cudaStreamSynchronize(st));
}

void exact_free(xrl_precond pc)
{
    delete static_cast<Exact*>(pc->exact);
    pc->exact = nullptr;
}

}  // namespace xrl
