// Tensor-core dot products for the u8 scan filter: one int8 IMMA GEMM per
// query chunk, D = Qop . Xs^T (s32), through cuBLASLt (a plain library GEMM;
// everything around it -- quantisation, offset correction, bounds, top-k and
// the exact re-rank -- is in scan.cu).
//
// Row-major D (m queries x ldD) is column-major D^T (n x m, ld = ldD):
// D^T = op(A) . op(B) with A = Xs (column-major k x n, lda = k, op = T) and
// B = Qop (column-major k x m, ldb = k, op = N): the "TN" int8 layout.
#include <cublasLt.h>

#include <mutex>
#include <vector>

#include "common.cuh"

namespace mrpt {

namespace {

struct Plan {
  int dev;
  int64_t n, m, k, ldD;
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulAlgo_t algo;
};

struct DevState {
  cublasLtHandle_t h = nullptr;
  void *ws = nullptr;
  size_t ws_bytes = 0;
};

std::mutex g_mu;
std::vector<DevState> g_dev;
std::vector<Plan> g_plans;

constexpr size_t kLtWorkspace = 32u << 20;

const char *lt_status(cublasStatus_t st) {
  switch (st) {
    case CUBLAS_STATUS_NOT_INITIALIZED: return "not initialized";
    case CUBLAS_STATUS_ALLOC_FAILED: return "allocation failed";
    case CUBLAS_STATUS_INVALID_VALUE: return "invalid value";
    case CUBLAS_STATUS_ARCH_MISMATCH: return "arch mismatch";
    case CUBLAS_STATUS_EXECUTION_FAILED: return "execution failed";
    case CUBLAS_STATUS_NOT_SUPPORTED: return "not supported";
    case CUBLAS_STATUS_INTERNAL_ERROR: return "internal error";
    default: return "error";
  }
}

}  // namespace

// D (m x ldD, row-major s32) = Qop (m x k s8) . Xs (n x k s8)^T.
int32_t igemm_rows_tn(const int8_t *Xs, int64_t n, const int8_t *Qop, int64_t m, int64_t k, int32_t *D,
                      int64_t ldD, cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(MRPT_ECUDA, "igemm: no device");
  std::lock_guard<std::mutex> lock(g_mu);
  if ((int)g_dev.size() <= dev) g_dev.resize(dev + 1);
  DevState &ds = g_dev[dev];
  cublasStatus_t st;
  if (!ds.h) {
    if ((st = cublasLtCreate(&ds.h)) != CUBLAS_STATUS_SUCCESS) {
      set_error("igemm: cublasLtCreate: %s", lt_status(st));
      return MRPT_ECUDA;
    }
    if (cudaMalloc(&ds.ws, kLtWorkspace) != cudaSuccess) {
      ds.ws = nullptr;
      return fail(MRPT_ECUDA, "igemm: workspace allocation failed");
    }
    ds.ws_bytes = kLtWorkspace;
  }
  Plan *pl = nullptr;
  for (Plan &p : g_plans)
    if (p.dev == dev && p.n == n && p.m == m && p.k == k && p.ldD == ldD) pl = &p;
  if (!pl) {
    Plan p;
    p.dev = dev;
    p.n = n;
    p.m = m;
    p.k = k;
    p.ldD = ldD;
    cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    bool ok = cublasLtMatmulDescCreate(&p.op, CUBLAS_COMPUTE_32I, CUDA_R_32I) == CUBLAS_STATUS_SUCCESS &&
              cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)) ==
                  CUBLAS_STATUS_SUCCESS &&
              cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)) ==
                  CUBLAS_STATUS_SUCCESS &&
              cublasLtMatrixLayoutCreate(&p.la, CUDA_R_8I, k, n, k) == CUBLAS_STATUS_SUCCESS &&
              cublasLtMatrixLayoutCreate(&p.lb, CUDA_R_8I, k, m, k) == CUBLAS_STATUS_SUCCESS &&
              cublasLtMatrixLayoutCreate(&p.lc, CUDA_R_32I, n, m, ldD) == CUBLAS_STATUS_SUCCESS;
    cublasLtMatmulPreference_t pref = nullptr;
    cublasLtMatmulHeuristicResult_t res;
    int nres = 0;
    if (ok) {
      ok = cublasLtMatmulPreferenceCreate(&pref) == CUBLAS_STATUS_SUCCESS &&
           cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES,
                                                &ds.ws_bytes, sizeof(ds.ws_bytes)) == CUBLAS_STATUS_SUCCESS;
      if (ok)
        ok = cublasLtMatmulAlgoGetHeuristic(ds.h, p.op, p.la, p.lb, p.lc, p.lc, pref, 1, &res, &nres) ==
                 CUBLAS_STATUS_SUCCESS &&
             nres > 0;
      if (pref) cublasLtMatmulPreferenceDestroy(pref);
    }
    if (!ok) {
      if (p.la) cublasLtMatrixLayoutDestroy(p.la);
      if (p.lb) cublasLtMatrixLayoutDestroy(p.lb);
      if (p.lc) cublasLtMatrixLayoutDestroy(p.lc);
      if (p.op) cublasLtMatmulDescDestroy(p.op);
      return fail(MRPT_ECUDA, "igemm: no cuBLASLt int8 algorithm for this shape");
    }
    p.algo = res.algo;
    g_plans.push_back(p);
    pl = &g_plans.back();
  }
  const int32_t alpha = 1, beta = 0;
  st = cublasLtMatmul(ds.h, pl->op, &alpha, Xs, pl->la, Qop, pl->lb, &beta, D, pl->lc, D, pl->lc, &pl->algo,
                      ds.ws, ds.ws_bytes, s);
  if (st != CUBLAS_STATUS_SUCCESS) {
    set_error("igemm: cublasLtMatmul: %s", lt_status(st));
    return MRPT_ECUDA;
  }
  return launch_status("igemm");
}

}  // namespace mrpt
