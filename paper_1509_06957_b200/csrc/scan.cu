// K4: exact squared-L2 scan of candidate rows and per-query top-k
// (replaces _cy.scan + np.unique/lexsort/sqrt of exact_knn_in_set,
// _kernels/_cy.pyx:81-97, pkg/src/mrpt/search.py:146-172).
//
// Parity: each d^2 is the reference's float64 sum taken sequentially over
// coordinates c = 0..d-1 of ((double)x_c - (double)q_c)^2 with a separate
// multiply and add (-ffp-contract=off in the reference build), so distances
// are bit-identical and the (d^2, id) order -- hence the returned ids -- is
// exactly the reference's.  The sequential chain is latency-bound per row,
// so each thread interleaves R candidate rows (R independent chains).
//
// Top-k: a shared-memory buffer collects (d^2, id) pairs that beat the
// running threshold; whenever it fills it is bitonic-sorted and truncated to
// the k best, which tightens the threshold.  Ties on d^2 order by id, as
// np.lexsort((S, d2)) does.
#include "common.cuh"

namespace mrpt {

constexpr int kScanNT = 256;
constexpr int kScanR = 4;

struct TopkArgs {
  const float *X;
  int64_t n;
  int d;
  int64_t ldx;
  const float *Q;
  int64_t nq;
  int64_t ldq;
  const int32_t *cand;
  int64_t cap;
  const int32_t *ncand;
  int k;        // entries written by this pass
  int kstride;  // row stride of ids/dists
  int64_t *ids;
  double *dists;
  unsigned long long *lb_key;  // optional lower bound per query (multi-pass)
  int32_t *lb_id;
  bool vec4;
};

__device__ __forceinline__ bool pair_less(unsigned long long ak, int ai, unsigned long long bk,
                                          int bi) {
  return ak < bk || (ak == bk && ai < bi);
}

template <int R>
__device__ __forceinline__ void dist_rows(const float *__restrict__ X, int64_t ldx, const int32_t *id,
                                          const double *qd, int d, bool vec4, double *acc) {
  const float *row[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    row[r] = X + (int64_t)id[r] * ldx;
    acc[r] = 0.0;
  }
  if (vec4) {
#pragma unroll 2
    for (int c = 0; c < d; c += 4) {
      const double q0 = qd[c], q1 = qd[c + 1], q2 = qd[c + 2], q3 = qd[c + 3];
      float4 x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = __ldg(reinterpret_cast<const float4 *>(row[r] + c));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double t;
        t = (double)x[r].x - q0;
        acc[r] = __dadd_rn(acc[r], __dmul_rn(t, t));
        t = (double)x[r].y - q1;
        acc[r] = __dadd_rn(acc[r], __dmul_rn(t, t));
        t = (double)x[r].z - q2;
        acc[r] = __dadd_rn(acc[r], __dmul_rn(t, t));
        t = (double)x[r].w - q3;
        acc[r] = __dadd_rn(acc[r], __dmul_rn(t, t));
      }
    }
  } else {
    for (int c = 0; c < d; ++c) {
      const double qc = qd[c];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double t = (double)__ldg(row[r] + c) - qc;
        acc[r] = __dadd_rn(acc[r], __dmul_rn(t, t));
      }
    }
  }
}

// Bitonic sort of BUF (key, id) pairs, ascending by (key, id).
template <int BUF>
__device__ void bitonic_sort(unsigned long long *bk, int32_t *bi) {
  for (int size = 2; size <= BUF; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < BUF / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const unsigned long long ka = bk[lo], kb = bk[hi];
        const int ia = bi[lo], ib = bi[hi];
        const bool gt = pair_less(kb, ib, ka, ia);
        if (gt == asc) {
          bk[lo] = kb;
          bk[hi] = ka;
          bi[lo] = ib;
          bi[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
}

template <int BUF>
__global__ void __launch_bounds__(kScanNT) k_scan_topk(TopkArgs a) {
  extern __shared__ unsigned long long topk_smem[];
  unsigned long long *bkey = topk_smem;                               // BUF
  int32_t *bid = reinterpret_cast<int32_t *>(bkey + BUF);            // BUF
  double *qd = reinterpret_cast<double *>(bid + BUF);                // d
  __shared__ int s_cnt;
  __shared__ unsigned long long s_tk;
  __shared__ int s_ti;
  const int tid = threadIdx.x;
  for (int64_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
    for (int c = tid; c < a.d; c += kScanNT) qd[c] = (double)a.Q[q * a.ldq + c];
    if (tid == 0) {
      s_cnt = 0;
      s_tk = ~0ull;
      s_ti = 0x7fffffff;
    }
    const unsigned long long lbk = a.lb_key ? a.lb_key[q] : 0ull;
    const int lbi = a.lb_key ? a.lb_id[q] : -1;
    const bool use_lb = a.lb_key != nullptr;
    __syncthreads();
    int64_t m;
    if (a.cand) {
      const int64_t nc = a.ncand[q];
      m = nc < a.cap ? nc : a.cap;
    } else {
      m = a.n;
    }
    const int32_t *qc = a.cand ? a.cand + q * a.cap : nullptr;
    for (int64_t base = 0; base < m; base += kScanNT * kScanR) {
      int32_t id[kScanR];
      bool valid[kScanR];
#pragma unroll
      for (int r = 0; r < kScanR; ++r) {
        const int64_t j = base + tid + r * kScanNT;
        valid[r] = j < m;
        id[r] = valid[r] ? (qc ? qc[j] : (int32_t)j) : 0;
      }
      double acc[kScanR];
      dist_rows<kScanR>(a.X, a.ldx, id, qd, a.d, a.vec4, acc);
      const unsigned long long tk = s_tk;
      const int ti = s_ti;
#pragma unroll
      for (int r = 0; r < kScanR; ++r) {
        const unsigned long long key = (unsigned long long)__double_as_longlong(acc[r]);
        if (valid[r] && pair_less(key, id[r], tk, ti) && (!use_lb || pair_less(lbk, lbi, key, id[r]))) {
          const int slot = atomicAdd(&s_cnt, 1);
          bkey[slot] = key;
          bid[slot] = id[r];
        }
      }
      __syncthreads();
      if (s_cnt > BUF - kScanNT * kScanR) {
        const int cnt = s_cnt;
        for (int i = cnt + tid; i < BUF; i += kScanNT) {
          bkey[i] = ~0ull;
          bid[i] = 0x7fffffff;
        }
        __syncthreads();
        bitonic_sort<BUF>(bkey, bid);
        if (tid == 0) {
          s_cnt = a.k;  // cnt > BUF - 1024 >= k
          s_tk = bkey[a.k - 1];
          s_ti = bid[a.k - 1];
        }
        __syncthreads();
      }
    }
    const int cnt = s_cnt;
    for (int i = cnt + tid; i < BUF; i += kScanNT) {
      bkey[i] = ~0ull;
      bid[i] = 0x7fffffff;
    }
    __syncthreads();
    bitonic_sort<BUF>(bkey, bid);
    const int kept = cnt < a.k ? cnt : a.k;
    for (int i = tid; i < a.k; i += kScanNT) {
      if (i < kept) {
        a.ids[q * a.kstride + i] = bid[i];
        a.dists[q * a.kstride + i] = sqrt(__longlong_as_double((long long)bkey[i]));
      } else {
        a.ids[q * a.kstride + i] = -1;
        a.dists[q * a.kstride + i] = __longlong_as_double(0x7ff0000000000000LL);
      }
    }
    if (use_lb && tid == 0 && kept > 0) {
      a.lb_key[q] = bkey[kept - 1];
      a.lb_id[q] = bid[kept - 1];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanNT)
k_scan(const float *__restrict__ X, int64_t ldx, int d, const int64_t *__restrict__ cand, int64_t m,
       const float *__restrict__ q, double *out, bool vec4) {
  extern __shared__ double qds[];
  for (int c = threadIdx.x; c < d; c += blockDim.x) qds[c] = (double)q[c];
  __syncthreads();
  for (int64_t base = (int64_t)blockIdx.x * kScanNT * kScanR; base < m;
       base += (int64_t)gridDim.x * kScanNT * kScanR) {
    int32_t id[kScanR];
    bool valid[kScanR];
#pragma unroll
    for (int r = 0; r < kScanR; ++r) {
      const int64_t j = base + threadIdx.x + r * kScanNT;
      valid[r] = j < m;
      id[r] = valid[r] ? (int32_t)cand[j] : 0;
    }
    double acc[kScanR];
    dist_rows<kScanR>(X, ldx, id, qds, d, vec4, acc);
#pragma unroll
    for (int r = 0; r < kScanR; ++r)
      if (valid[r]) out[base + threadIdx.x + r * kScanNT] = acc[r];
  }
}

}  // namespace mrpt

using namespace mrpt;

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

extern "C" int32_t mrpt_scan(const float *X, int64_t n, int32_t d, int64_t ldx, const int64_t *cand,
                             int64_t m, const float *q, double *out, void *stream) {
  clear_error();
  if (n < 1 || n >= (int64_t)1 << 31 || d < 1 || ldx < d || m < 0)
    return fail(MRPT_ESHAPE, "mrpt_scan: bad shape");
  if (m == 0) return MRPT_OK;
  cudaStream_t s = as_stream(stream);
  const bool vec4 = (d % 4 == 0) && (ldx % 4 == 0) && aligned16(X);
  const size_t smem = sizeof(double) * (size_t)d;
  if (smem > 200 * 1024) return fail(MRPT_EPARAM, "mrpt_scan: d too large");
  cudaFuncSetAttribute(k_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t blocks = ceil_div<int64_t>(m, kScanNT * kScanR);
  const int grid = (int)(blocks < (int64_t)num_sms() * 8 ? blocks : (int64_t)num_sms() * 8);
  k_scan<<<grid, kScanNT, smem, s>>>(X, ldx, d, cand, m, q, out, vec4);
  return launch_status("mrpt_scan");
}

typedef void (*topk_fn)(TopkArgs);

extern "C" int32_t mrpt_scan_topk(const float *X, int64_t n, int32_t d, int64_t ldx, const float *Q,
                                  int64_t nq, int64_t ldq, const int32_t *cand, int64_t cap,
                                  const int32_t *ncand, int32_t k, int64_t *ids, double *dists,
                                  void *stream) {
  clear_error();
  if (n < 1 || n >= (int64_t)1 << 31 || d < 1 || ldx < d || ldq < d || nq < 0)
    return fail(MRPT_ESHAPE, "mrpt_scan_topk: bad shape");
  if (k < 1) return fail(MRPT_EPARAM, "mrpt_scan_topk: k must be >= 1");
  if (cand && (cap < 1 || !ncand)) return fail(MRPT_EPARAM, "mrpt_scan_topk: bad candidate lists");
  if (nq == 0) return MRPT_OK;
  cudaStream_t s = as_stream(stream);
  TopkArgs a;
  a.X = X;
  a.n = n;
  a.d = d;
  a.ldx = ldx;
  a.Q = Q;
  a.nq = nq;
  a.ldq = ldq;
  a.cand = cand;
  a.cap = cap;
  a.ncand = ncand;
  a.kstride = k;
  a.lb_key = nullptr;
  a.lb_id = nullptr;
  a.vec4 = (d % 4 == 0) && (ldx % 4 == 0) && aligned16(X);
  const int chunk_max = 4096 - kScanNT * kScanR;  // 3072 entries per pass
  const int passes = (k + chunk_max - 1) / chunk_max;
  if (passes > 1) {
    if (cudaMallocAsync((void **)&a.lb_key, sizeof(unsigned long long) * nq, s) != cudaSuccess ||
        cudaMallocAsync((void **)&a.lb_id, sizeof(int32_t) * nq, s) != cudaSuccess)
      return fail(MRPT_ECUDA, "mrpt_scan_topk: scratch allocation failed");
    // lower bound below every key: (0, -1)
    cudaMemsetAsync(a.lb_key, 0, sizeof(unsigned long long) * nq, s);
    cudaMemsetAsync(a.lb_id, 0xff, sizeof(int32_t) * nq, s);
  }
  const int64_t grid = nq < (int64_t)num_sms() * 8 ? nq : (int64_t)num_sms() * 8;
  for (int p = 0; p < passes; ++p) {
    const int off = p * chunk_max;
    const int kk = (k - off) < chunk_max ? (k - off) : chunk_max;
    a.k = kk;
    a.ids = ids + off;
    a.dists = dists + off;
    topk_fn fn;
    int buf;
    if (kk + kScanNT * kScanR <= 2048) {
      fn = k_scan_topk<2048>;
      buf = 2048;
    } else {
      fn = k_scan_topk<4096>;
      buf = 4096;
    }
    const size_t smem = (size_t)buf * 12 + sizeof(double) * (size_t)d;
    if (smem > 220 * 1024) return fail(MRPT_EPARAM, "mrpt_scan_topk: d too large");
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fn<<<(unsigned)grid, kScanNT, smem, s>>>(a);
  }
  if (passes > 1) {
    cudaFreeAsync(a.lb_key, s);
    cudaFreeAsync(a.lb_id, s);
  }
  return launch_status("mrpt_scan_topk");
}
