// Exact diagonal-of-P preconditioner: Q^-1 of Eq. 10,
//     Q = sum_t C_t diag(d) C_t^T,  d_k = Z_s,k / A_k + j alpha P_kk,  C_t = M A_t,
// applied exactly as Eq. 11 prescribes (the paper factorises Q once per frequency with
// Pardiso and solves per GMRES iteration).  Here: Q assembled on the host in FP64 complex
// (sparse, pattern = loops sharing a panel), nested-dissection (METIS) ordering, else approximate minimum
// degree, then a host sparse LU with partial pivoting (cuSOLVER's low-level csrlu, the library analogue of
// Pardiso), factorised once per operator.  The factors P B Q^T = L U are moved to the GPU (FP64 complex
// CSR) and every apply runs on the context stream: gather-permute v, cuSPARSE triangular solves with L
// (unit diagonal) and U, scatter-permute into z (XRL_EXACT_HOST=1: the host solve instead, for checks).
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
#include <cusparse.h>

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
    int (*luNnz)(SpHandle, int*, int*, LuInfo);
    int (*luExtract)(SpHandle, int*, int*, const MatDescr, cuDoubleComplex*, int*, int*, const MatDescr,
                     cuDoubleComplex*, int*, int*, LuInfo, void*);
    // cuSPARSE generic triangular solve
    decltype(&cusparseCreate) spCreateH;
    decltype(&cusparseDestroy) spDestroyH;
    decltype(&cusparseSetStream) spSetStream;
    decltype(&cusparseCreateCsr) createCsr;
    decltype(&cusparseDestroySpMat) destroySpMat;
    decltype(&cusparseSpMatSetAttribute) setAttr;
    decltype(&cusparseCreateDnVec) createDnVec;
    decltype(&cusparseDestroyDnVec) destroyDnVec;
    decltype(&cusparseSpSV_createDescr) svCreate;
    decltype(&cusparseSpSV_destroyDescr) svDestroy;
    decltype(&cusparseSpSV_bufferSize) svBuffer;
    decltype(&cusparseSpSV_analysis) svAnalysis;
    decltype(&cusparseSpSV_solve) svSolve;
    // incomplete LU(0) on the GPU (legacy csrilu02, complex FP64)
    int (*iluCreate)(void**);
    int (*iluDestroy)(void*);
    int (*iluBuffer)(cusparseHandle_t, int, int, const MatDescr, cuDoubleComplex*, const int*, const int*, void*, int*);
    int (*iluAnalysis)(cusparseHandle_t, int, int, const MatDescr, const cuDoubleComplex*, const int*, const int*,
                       void*, int, void*);
    int (*iluFactor)(cusparseHandle_t, int, int, const MatDescr, cuDoubleComplex*, const int*, const int*, void*, int,
                     void*);
    int (*iluZeroPivot)(cusparseHandle_t, void*, int*);
    int (*rcm)(SpHandle, int, int, const MatDescr, const int*, const int*, int*);
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
    a.luNnz = (decltype(a.luNnz))sym(hs, "cusolverSpXcsrluNnzHost");
    a.luExtract = (decltype(a.luExtract))sym(hs, "cusolverSpZcsrluExtractHost");
    a.spCreateH = (decltype(a.spCreateH))sym(hp, "cusparseCreate");
    a.spDestroyH = (decltype(a.spDestroyH))sym(hp, "cusparseDestroy");
    a.spSetStream = (decltype(a.spSetStream))sym(hp, "cusparseSetStream");
    a.createCsr = (decltype(a.createCsr))sym(hp, "cusparseCreateCsr");
    a.destroySpMat = (decltype(a.destroySpMat))sym(hp, "cusparseDestroySpMat");
    a.setAttr = (decltype(a.setAttr))sym(hp, "cusparseSpMatSetAttribute");
    a.createDnVec = (decltype(a.createDnVec))sym(hp, "cusparseCreateDnVec");
    a.destroyDnVec = (decltype(a.destroyDnVec))sym(hp, "cusparseDestroyDnVec");
    a.svCreate = (decltype(a.svCreate))sym(hp, "cusparseSpSV_createDescr");
    a.svDestroy = (decltype(a.svDestroy))sym(hp, "cusparseSpSV_destroyDescr");
    a.svBuffer = (decltype(a.svBuffer))sym(hp, "cusparseSpSV_bufferSize");
    a.svAnalysis = (decltype(a.svAnalysis))sym(hp, "cusparseSpSV_analysis");
    a.svSolve = (decltype(a.svSolve))sym(hp, "cusparseSpSV_solve");
    a.metisnd = (decltype(a.metisnd))dlsym(hs, "cusolverSpXcsrmetisndHost");  // optional
    a.iluCreate = (decltype(a.iluCreate))sym(hp, "cusparseCreateCsrilu02Info");
    a.iluDestroy = (decltype(a.iluDestroy))sym(hp, "cusparseDestroyCsrilu02Info");
    a.iluBuffer = (decltype(a.iluBuffer))sym(hp, "cusparseZcsrilu02_bufferSize");
    a.iluAnalysis = (decltype(a.iluAnalysis))sym(hp, "cusparseZcsrilu02_analysis");
    a.iluFactor = (decltype(a.iluFactor))sym(hp, "cusparseZcsrilu02");
    a.iluZeroPivot = (decltype(a.iluZeroPivot))sym(hp, "cusparseXcsrilu02_zeroPivot");
    a.rcm = (decltype(a.rcm))sym(hs, "cusolverSpXcsrsymrcmHost");
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
    int64_t nnz_q = 0, nnz_l = 0, nnz_u = 0;
    // device factors and triangular-solve state (P B Q^T = L U)
    bool dev = false;
    DBuf<int> gin, gout;                      // z-permutations: b[i] = v[gin[i]], z[gout[i]] = w[i]
    DBuf<int> lp, lc, up, uc;
    DBuf<cuDoubleComplex> lv, uv, db, dy;
    DBuf<char> bufL, bufU;
    cusparseHandle_t sh = nullptr;
    cusparseSpMatDescr_t mL = nullptr, mU = nullptr;
    cusparseDnVecDescr_t vB = nullptr, vY = nullptr;
    cusparseSpSVDescr_t sL = nullptr, sU = nullptr;
    void* ilu_info = nullptr;
    ~Exact()
    {
        Api& A = api();
        if (ilu_info) A.iluDestroy(ilu_info);
        if (sL) A.svDestroy(sL);
        if (sU) A.svDestroy(sU);
        if (vB) A.destroyDnVec(vB);
        if (vY) A.destroyDnVec(vY);
        if (mL) A.destroySpMat(mL);
        if (mU) A.destroySpMat(mU);
        if (sh) A.spDestroyH(sh);
        if (info) A.destroyLuInfo(info);
        if (descr) A.destroyDescr(descr);
        if (h) A.spDestroy(h);
    }
};

__global__ void k_exact_gather(int n, const float2* __restrict__ v, const int* __restrict__ gin, cuDoubleComplex* b)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const float2 w = v[gin[i]];
        b[i] = make_cuDoubleComplex(w.x, w.y);
    }
}

__global__ void k_exact_scatter(int n, const cuDoubleComplex* __restrict__ w, const int* __restrict__ gout, float2* z)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) z[gout[i]] = make_float2((float)w[i].x, (float)w[i].y);
}

}  // namespace

namespace xrl {

void assemble_q(xrl_op op, int qkind, std::vector<std::vector<int32_t>>& rc,
                std::vector<std::vector<std::complex<double>>>& rv)
{
    xrl_topo T = op->topo;
    const int64_t n = op->tree->n, nl = T->n_loops;
    // panel part: Q_ab = sum_k d_k (c_a(k) . c_b(k)) over panels k shared by loops a, b, with
    //   diag-of-P (Eq. 10): d_k = Z_s,k / A_k + j alpha P_kk;  diag-of-L: d_k = Z_s,k / A_k (the ESI part only)
    std::vector<double2> d;
    precond_diag(op, d);
    if (qkind == 1)
        for (int64_t k = 0; k < n; ++k) d[k] = make_double2(op->zsa_h[2 * k], op->zsa_h[2 * k + 1]);
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
    // branch part of diag-of-L: alpha L_ee M_ae M_be over the physical edges (branch e < n_edges is edge e)
    std::vector<double> lee;
    std::vector<int64_t> bp;   // edge -> loops (transpose of M restricted to edges)
    std::vector<int32_t> bl;
    std::vector<int8_t> bs;
    if (qkind == 1) {
        precond_ldiag(op, lee);
        const int64_t ne = T->n_edges;
        bp.assign(ne + 1, 0);
        for (int64_t a = 0; a < nl; ++a)
            for (int64_t q = T->m_ptr[a]; q < T->m_ptr[a + 1]; ++q)
                if (T->m_idx[q] < ne) ++bp[T->m_idx[q] + 1];
        for (int64_t e = 0; e < ne; ++e) bp[e + 1] += bp[e];
        bl.resize(bp[ne]);
        bs.resize(bp[ne]);
        std::vector<int64_t> fill(bp.begin(), bp.end() - 1);
        for (int64_t a = 0; a < nl; ++a)
            for (int64_t q = T->m_ptr[a]; q < T->m_ptr[a + 1]; ++q)
                if (T->m_idx[q] < ne) {
                    const int64_t f = fill[T->m_idx[q]]++;
                    bl[f] = (int32_t)a;
                    bs[f] = T->m_val[q];
                }
    }
    const double alpha = op->alpha_im;
    rc.assign(nl, {});
    rv.assign(nl, {});
#pragma omp parallel
    {
        std::vector<std::complex<double>> acc(nl, 0.0);
        std::vector<char> mark(nl, 0);
        std::vector<int32_t> touched;
        auto add = [&](int32_t b, std::complex<double> v) {
            if (!mark[b]) { mark[b] = 1; touched.push_back(b); acc[b] = 0.0; }
            acc[b] += v;
        };
#pragma omp for schedule(dynamic, 256)
        for (int64_t a = 0; a < nl; ++a) {
            touched.clear();
            for (int64_t q = cp[a]; q < cp[a + 1]; ++q) {
                const int32_t k = cc[q];
                const double* ca = &cv[3 * q];
                const std::complex<double> dk(d[k].x, d[k].y);
                for (int64_t f = kp[k]; f < kp[k + 1]; ++f) {
                    const double* cb = &cv[3 * kq[f]];
                    add(kl[f], dk * (ca[0] * cb[0] + ca[1] * cb[1] + ca[2] * cb[2]));
                }
            }
            if (qkind == 1)
                for (int64_t q = T->m_ptr[a]; q < T->m_ptr[a + 1]; ++q) {
                    const int32_t e = T->m_idx[q];
                    if (e >= T->n_edges) continue;
                    const std::complex<double> le(0.0, alpha * lee[e] * T->m_val[q]);
                    for (int64_t f = bp[e]; f < bp[e + 1]; ++f) add(bl[f], le * (double)bs[f]);
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
}

// ILU(0) of B = Q(perm, perm) on the GPU (cuSPARSE csrilu02, FP64 complex, in place on B's pattern): the
// incomplete factors L (unit lower) and U share B's arrays; the apply is the exact path's two triangular
// solves with gin = gout = perm.
static xrl_status ilu_build(xrl_precond pc, std::unique_ptr<Exact>& E, const std::vector<int>& bp,
                            const std::vector<int>& bc, const std::vector<cuDoubleComplex>& bv)
{
    Api& A = api();
    const int N = E->n, nnz = (int)bc.size();
    cudaStream_t st = pc->op->tree->ctx->stream;
    E->gin.alloc(N);
    E->gout.alloc(N);
    XRL_CUDA(cudaMemcpyAsync(E->gin.p, E->perm.data(), 4 * (size_t)N, cudaMemcpyHostToDevice, st));
    XRL_CUDA(cudaMemcpyAsync(E->gout.p, E->perm.data(), 4 * (size_t)N, cudaMemcpyHostToDevice, st));
    E->lp.alloc(N + 1);
    E->lc.alloc(std::max(1, nnz));
    E->lv.alloc(std::max(1, nnz));
    XRL_CUDA(cudaMemcpyAsync(E->lp.p, bp.data(), 4 * (size_t)(N + 1), cudaMemcpyHostToDevice, st));
    XRL_CUDA(cudaMemcpyAsync(E->lc.p, bc.data(), 4 * (size_t)nnz, cudaMemcpyHostToDevice, st));
    XRL_CUDA(cudaMemcpyAsync(E->lv.p, bv.data(), 16 * (size_t)nnz, cudaMemcpyHostToDevice, st));
    E->db.alloc(N);
    E->dy.alloc(N);
    if (A.spCreateH(&E->sh) || A.spSetStream(E->sh, st) || A.iluCreate(&E->ilu_info)) {
        set_error("xrl_precond_build_kind: cuSPARSE ILU(0) setup failed");
        return XRL_ECUDA;
    }
    int bytes = 0;
    if (A.iluBuffer(E->sh, N, nnz, E->descr, E->lv.p, E->lp.p, E->lc.p, E->ilu_info, &bytes)) {
        set_error("xrl_precond_build_kind: ILU(0) buffer size failed");
        return XRL_ECUDA;
    }
    DBuf<char> buf(std::max(bytes, 16));
    const int policy = CUSPARSE_SOLVE_POLICY_USE_LEVEL;
    if (A.iluAnalysis(E->sh, N, nnz, E->descr, E->lv.p, E->lp.p, E->lc.p, E->ilu_info, policy, buf.p) ||
        A.iluFactor(E->sh, N, nnz, E->descr, E->lv.p, E->lp.p, E->lc.p, E->ilu_info, policy, buf.p)) {
        set_error("xrl_precond_build_kind: ILU(0) factorisation failed");
        return XRL_ECUDA;
    }
    int zp = -1;
    const int zs = A.iluZeroPivot(E->sh, E->ilu_info, &zp);  // synchronises
    if (zs == CUSPARSE_STATUS_ZERO_PIVOT || zp >= 0) {
        set_error("xrl_precond_build_kind: ILU(0) zero pivot at row %d", zp);
        return XRL_ESINGULAR;
    }
    E->nnz_l = E->nnz_u = nnz;
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
    cusparseFillMode_t lo = CUSPARSE_FILL_MODE_LOWER, upm = CUSPARSE_FILL_MODE_UPPER;
    cusparseDiagType_t unit = CUSPARSE_DIAG_TYPE_UNIT, nonunit = CUSPARSE_DIAG_TYPE_NON_UNIT;
    bool bad = A.createCsr(&E->mL, N, N, nnz, E->lp.p, E->lc.p, E->lv.p, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                           CUSPARSE_INDEX_BASE_ZERO, CUDA_C_64F) ||
               A.createCsr(&E->mU, N, N, nnz, E->lp.p, E->lc.p, E->lv.p, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                           CUSPARSE_INDEX_BASE_ZERO, CUDA_C_64F) ||
               A.setAttr(E->mL, CUSPARSE_SPMAT_FILL_MODE, &lo, sizeof(lo)) ||
               A.setAttr(E->mL, CUSPARSE_SPMAT_DIAG_TYPE, &unit, sizeof(unit)) ||
               A.setAttr(E->mU, CUSPARSE_SPMAT_FILL_MODE, &upm, sizeof(upm)) ||
               A.setAttr(E->mU, CUSPARSE_SPMAT_DIAG_TYPE, &nonunit, sizeof(nonunit)) ||
               A.createDnVec(&E->vB, N, E->db.p, CUDA_C_64F) || A.createDnVec(&E->vY, N, E->dy.p, CUDA_C_64F) ||
               A.svCreate(&E->sL) || A.svCreate(&E->sU);
    size_t szL = 0, szU = 0;
    bad = bad || A.svBuffer(E->sh, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, E->mL, E->vB, E->vY, CUDA_C_64F,
                            CUSPARSE_SPSV_ALG_DEFAULT, E->sL, &szL) ||
          A.svBuffer(E->sh, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, E->mU, E->vY, E->vB, CUDA_C_64F,
                     CUSPARSE_SPSV_ALG_DEFAULT, E->sU, &szU);
    if (!bad) {
        E->bufL.alloc(std::max<size_t>(szL, 16));
        E->bufU.alloc(std::max<size_t>(szU, 16));
        bad = A.svAnalysis(E->sh, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, E->mL, E->vB, E->vY, CUDA_C_64F,
                           CUSPARSE_SPSV_ALG_DEFAULT, E->sL, E->bufL.p) ||
              A.svAnalysis(E->sh, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, E->mU, E->vY, E->vB, CUDA_C_64F,
                           CUSPARSE_SPSV_ALG_DEFAULT, E->sU, E->bufU.p);
    }
    if (bad) { set_error("xrl_precond_build_kind: cuSPARSE triangular-solve setup failed"); return XRL_ECUDA; }
    XRL_CUDA(cudaStreamSynchronize(st));
    E->dev = true;
    pc->exact = E.release();
    return XRL_OK;
}

xrl_status exact_build(xrl_precond pc)
{
    Api& A = api();
    if (!A.ok) { set_error("xrl_precond_build_exact: %s", A.err.c_str()); return XRL_EINVAL; }
    xrl_op op = pc->op;
    xrl_topo T = op->topo;
    const int64_t nl = T->n_loops;
    if (nl >= ((int64_t)1 << 31)) { set_error("xrl_precond_build_exact: too many loops for 32-bit LU"); return XRL_EINVAL; }
    std::vector<std::vector<int32_t>> rc;
    std::vector<std::vector<std::complex<double>>> rv;
    assemble_q(op, pc->qkind, rc, rv);
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
    // (ILU(0): reverse Cuthill-McKee, a bandwidth ordering -- nested dissection orders the separators last,
    // which suits a complete factorisation but leaves an incomplete one with the weakest couplings)
    int st = 1;
    if (pc->ilu) {
        static const bool natural = getenv("XRL_ILU_NATURAL") != nullptr;
        st = natural ? 1 : A.rcm(E->h, N, nnz, E->descr, qp.data(), qc.data(), E->perm.data());
        if (st) std::iota(E->perm.begin(), E->perm.end(), 0);
        st = 0;
    }
    if (st) st = A.metisnd ? A.metisnd(E->h, N, nnz, E->descr, qp.data(), qc.data(), nullptr, E->perm.data()) : 1;
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
    if (pc->ilu) return ilu_build(pc, E, bp, bc, bv);
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
    static const bool host_only = getenv("XRL_EXACT_HOST") != nullptr;
    if (!host_only) {
        // ---- factors to the GPU: P B Q^T = L U (L unit lower, U upper); B = Q(perm, perm)
        int nl_ = 0, nu_ = 0;
        if (A.luNnz(E->h, &nl_, &nu_, E->info)) { set_error("xrl_precond_build_exact: LU nnz failed"); return XRL_ECUDA; }
        std::vector<int> P(N), Qp(N), hlp(N + 1), hlc(nl_), hup(N + 1), huc(nu_);
        std::vector<cuDoubleComplex> hlv(nl_), huv(nu_);
        if (A.luExtract(E->h, P.data(), Qp.data(), E->descr, hlv.data(), hlp.data(), hlc.data(), E->descr, huv.data(),
                        hup.data(), huc.data(), E->info, E->work.data())) {
            set_error("xrl_precond_build_exact: LU extract failed");
            return XRL_ECUDA;
        }
        E->nnz_l = nl_;
        E->nnz_u = nu_;
        // z = Qmat^-1 v:  b[i] = v[perm[P[i]]], L y = b, U w = y, z[perm[Q[i]]] = w[i]
        std::vector<int> gi(N), go(N);
        for (int i = 0; i < N; ++i) { gi[i] = E->perm[P[i]]; go[i] = E->perm[Qp[i]]; }
        cudaStream_t st = op->tree->ctx->stream;
        auto up_i = [&](DBuf<int>& d, const std::vector<int>& h) {
            d.alloc(std::max<size_t>(1, h.size()));
            XRL_CUDA(cudaMemcpyAsync(d.p, h.data(), 4 * h.size(), cudaMemcpyHostToDevice, st));
        };
        auto up_z = [&](DBuf<cuDoubleComplex>& d, const std::vector<cuDoubleComplex>& h) {
            d.alloc(std::max<size_t>(1, h.size()));
            XRL_CUDA(cudaMemcpyAsync(d.p, h.data(), 16 * h.size(), cudaMemcpyHostToDevice, st));
        };
        up_i(E->gin, gi); up_i(E->gout, go);
        up_i(E->lp, hlp); up_i(E->lc, hlc); up_z(E->lv, hlv);
        up_i(E->up, hup); up_i(E->uc, huc); up_z(E->uv, huv);
        E->db.alloc(N);
        E->dy.alloc(N);
        XRL_CUDA(cudaStreamSynchronize(st));
        const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
        cusparseFillMode_t lo = CUSPARSE_FILL_MODE_LOWER, upm = CUSPARSE_FILL_MODE_UPPER;
        cusparseDiagType_t unit = CUSPARSE_DIAG_TYPE_UNIT, nonunit = CUSPARSE_DIAG_TYPE_NON_UNIT;
        bool bad = A.spCreateH(&E->sh) || A.spSetStream(E->sh, st) ||
                   A.createCsr(&E->mL, N, N, nl_, E->lp.p, E->lc.p, E->lv.p, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                               CUSPARSE_INDEX_BASE_ZERO, CUDA_C_64F) ||
                   A.createCsr(&E->mU, N, N, nu_, E->up.p, E->uc.p, E->uv.p, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                               CUSPARSE_INDEX_BASE_ZERO, CUDA_C_64F) ||
                   A.setAttr(E->mL, CUSPARSE_SPMAT_FILL_MODE, &lo, sizeof(lo)) ||
                   A.setAttr(E->mL, CUSPARSE_SPMAT_DIAG_TYPE, &unit, sizeof(unit)) ||
                   A.setAttr(E->mU, CUSPARSE_SPMAT_FILL_MODE, &upm, sizeof(upm)) ||
                   A.setAttr(E->mU, CUSPARSE_SPMAT_DIAG_TYPE, &nonunit, sizeof(nonunit)) ||
                   A.createDnVec(&E->vB, N, E->db.p, CUDA_C_64F) || A.createDnVec(&E->vY, N, E->dy.p, CUDA_C_64F) ||
                   A.svCreate(&E->sL) || A.svCreate(&E->sU);
        size_t szL = 0, szU = 0;
        bad = bad || A.svBuffer(E->sh, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, E->mL, E->vB, E->vY, CUDA_C_64F,
                                CUSPARSE_SPSV_ALG_DEFAULT, E->sL, &szL) ||
              A.svBuffer(E->sh, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, E->mU, E->vY, E->vB, CUDA_C_64F,
                         CUSPARSE_SPSV_ALG_DEFAULT, E->sU, &szU);
        if (!bad) {
            E->bufL.alloc(std::max<size_t>(szL, 16));
            E->bufU.alloc(std::max<size_t>(szU, 16));
            bad = A.svAnalysis(E->sh, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, E->mL, E->vB, E->vY, CUDA_C_64F,
                               CUSPARSE_SPSV_ALG_DEFAULT, E->sL, E->bufL.p) ||
                  A.svAnalysis(E->sh, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, E->mU, E->vY, E->vB, CUDA_C_64F,
                               CUSPARSE_SPSV_ALG_DEFAULT, E->sU, E->bufU.p);
        }
        if (bad) { set_error("xrl_precond_build_exact: cuSPARSE triangular-solve setup failed"); return XRL_ECUDA; }
        XRL_CUDA(cudaStreamSynchronize(st));
        E->dev = true;
    }
    pc->exact = E.release();
    return XRL_OK;
}

void exact_apply(xrl_precond pc, const float2* v, float2* z, int nrhs)
{
    Exact* E = static_cast<Exact*>(pc->exact);
    Api& A = api();
    cudaStream_t st = pc->op->tree->ctx->stream;
    const int N = E->n;
    if (E->dev) {
        const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
        for (int c = 0; c < nrhs; ++c) {
            k_exact_gather<<<(N + 255) / 256, 256, 0, st>>>(N, v + (size_t)c * N, E->gin.p, E->db.p);
            XRL_LAUNCH_CHECK();
            if (A.svSolve(E->sh, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, E->mL, E->vB, E->vY, CUDA_C_64F,
                          CUSPARSE_SPSV_ALG_DEFAULT, E->sL) ||
                A.svSolve(E->sh, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, E->mU, E->vY, E->vB, CUDA_C_64F,
                          CUSPARSE_SPSV_ALG_DEFAULT, E->sU)) {
                set_error("xrl_precond_apply: cuSPARSE triangular solve failed");
                throw CudaError{XRL_ECUDA};
            }
            k_exact_scatter<<<(N + 255) / 256, 256, 0, st>>>(N, E->db.p, E->gout.p, z + (size_t)c * N);
            XRL_LAUNCH_CHECK();
        }
        return;
    }
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
