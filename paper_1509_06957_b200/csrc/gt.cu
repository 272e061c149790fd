// f3: exact brute-force k-NN on the device -- the ground truth every recall
// number rests on (replaces evaluation.brute_force_knn / compute_ground_truth,
// pkg/src/mrpt/evaluation.py:28-81).
//
// Parity.  The reference computes, per query,
//     d2 = ((X.values.astype(f64) - q_f64) ** 2).sum(axis=1)
//     order = np.lexsort((ids, d2))[:k];  dist = sqrt(d2[order])
// (evaluation.py:40-44).  numpy reduces each contiguous row with its pairwise
// summation (loops_utils.h pairwise_sum): a run of n < 8 terms is summed in
// order from 0.0; a run of 8 <= n <= 128 terms goes into 8 interleaved
// accumulators r[j] (terms j, j+8, ...), combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n%8 tail is added in order;
// a longer run is split at n2 = n/2 - (n/2)%8 and the two halves' sums are
// added.  The host turns that recursion for the row length d into a postfix
// plan (leaf blocks of <= 128 terms, then ADDs); every (query, row) pair is
// summed by that plan with separate float64 subtract / multiply / add
// (__dsub_rn/__dmul_rn/__dadd_rn, never contracted), so d2 -- and the sqrt,
// correctly rounded on both sides -- are bit-identical to the reference's.
// tests/test_oracle_golden.py pins the plan against numpy on every width.
//
// Layout and selection.  A CTA owns QB queries (float64 in shared memory)
// and one chunk of rows; each thread sums one row for QG of them per round of
// 128 rows.  A pair enters its query's shared buffer if (d2, id) beats the
// query's running k-th (d2, id) -- np.lexsort order, ties by id; full
// buffers are bitonic-sorted and cut to the k best, which tightens the bound.
// Each chunk's sorted k best go to global memory; one CTA per query merges
// the chunks.  k above one pass's capacity runs several passes, each taking
// the next entries after the previous pass's last (d2, id).
// Bound: the float64 pipe (3 DP ops per term).
#include <stdlib.h>

#include "common.cuh"

namespace mrpt {

constexpr int kGtThreads = 256;
constexpr int kGtRound = 128;          // rows per round (threads per query group)
constexpr int kGtMaxLeaves = 80;
constexpr int kGtMaxOps = 2 * kGtMaxLeaves;
constexpr int kGtMaxD = 4096;
constexpr int kGtMergeMax = 8192;      // entries one merge CTA sorts
constexpr unsigned long long kGtInf = ~0ull;

struct GtPlan {
  int nops;
  int16_t op[kGtMaxOps];  // >= 0: leaf index; -1: add the two top sums
  int16_t lo[kGtMaxLeaves];
  int16_t len[kGtMaxLeaves];
};

struct GtArgs {
  const float *X;
  int64_t n;
  int d;
  int64_t ldx;
  const double *Q;
  int64_t nq;
  int64_t ldq;
  int kp;            // entries this pass keeps per query
  int kps;           // stride of a chunk's list (entries)
  int rch;           // row chunks
  int64_t rpc;       // rows per chunk (multiple of kGtRound)
  int B;             // buffer entries per query
  const unsigned long long *lb_key;  // previous pass's last entry, or null
  const int32_t *lb_id;
  unsigned long long *part_key;      // (nq, rch, kps)
  int32_t *part_id;
  bool vec4;
};

// numpy's pairwise recursion for n terms starting at lo, as a postfix plan.
static bool gt_plan_rec(GtPlan &p, int lo, int n, int &nleaf) {
  if (n <= 128) {
    if (nleaf >= kGtMaxLeaves || p.nops >= kGtMaxOps) return false;
    p.lo[nleaf] = (int16_t)lo;
    p.len[nleaf] = (int16_t)n;
    p.op[p.nops++] = (int16_t)nleaf++;
    return true;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  if (!gt_plan_rec(p, lo, n2, nleaf) || !gt_plan_rec(p, lo + n2, n - n2, nleaf)) return false;
  if (p.nops >= kGtMaxOps) return false;
  p.op[p.nops++] = -1;
  return true;
}

__device__ __forceinline__ double sq_diff(float x, double q) {
  const double t = __dsub_rn((double)x, q);
  return __dmul_rn(t, t);
}

// One leaf block of the plan for QG queries of one row.
template <int QG>
__device__ __forceinline__ void gt_leaf(const float *__restrict__ xr, const double *__restrict__ qs, int d,
                                        int lo, int len, bool vec4, double *res) {
  if (len < 8) {
#pragma unroll
    for (int j = 0; j < QG; ++j) res[j] = 0.0;
    for (int i = 0; i < len; ++i) {
      const float x = __ldg(xr + lo + i);
#pragma unroll
      for (int j = 0; j < QG; ++j) res[j] = __dadd_rn(res[j], sq_diff(x, qs[j * d + lo + i]));
    }
    return;
  }
  double acc[QG][8];
#pragma unroll
  for (int j = 0; j < QG; ++j)
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[j][u] = 0.0;  // 0.0 + a == a: same as numpy's r[j] = a[j]
  const int m = len - (len & 7);
  for (int i = 0; i < m; i += 8) {
    float x[8];
    if (vec4) {
      const float4 a = __ldg(reinterpret_cast<const float4 *>(xr + lo + i));
      const float4 b = __ldg(reinterpret_cast<const float4 *>(xr + lo + i) + 1);
      x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
      x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldg(xr + lo + i + u);
    }
#pragma unroll
    for (int j = 0; j < QG; ++j) {
      const double *q = qs + j * d + lo + i;
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[j][u] = __dadd_rn(acc[j][u], sq_diff(x[u], q[u]));
    }
  }
#pragma unroll
  for (int j = 0; j < QG; ++j)
    res[j] = __dadd_rn(__dadd_rn(__dadd_rn(acc[j][0], acc[j][1]), __dadd_rn(acc[j][2], acc[j][3])),
                       __dadd_rn(__dadd_rn(acc[j][4], acc[j][5]), __dadd_rn(acc[j][6], acc[j][7])));
  for (int i = m; i < len; ++i) {
    const float x = __ldg(xr + lo + i);
#pragma unroll
    for (int j = 0; j < QG; ++j) res[j] = __dadd_rn(res[j], sq_diff(x, qs[j * d + lo + i]));
  }
}

__device__ __forceinline__ bool gt_less(unsigned long long ak, int32_t ai, unsigned long long bk, int32_t bi) {
  return ak < bk || (ak == bk && ai < bi);
}

// Ascending bitonic sort of m (power of two) (key, id) pairs by the block.
__device__ void gt_bitonic(unsigned long long *k, int32_t *id, int m) {
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < m / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const unsigned long long ka = k[lo], kb = k[hi];
        const int32_t ia = id[lo], ib = id[hi];
        if (gt_less(kb, ib, ka, ia) == asc) {
          k[lo] = kb;
          k[hi] = ka;
          id[lo] = ib;
          id[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
}

template <int QG>
__global__ void __launch_bounds__(kGtThreads) k_gt_scan(GtArgs a, GtPlan plan) {
  constexpr int QB = QG * (kGtThreads / kGtRound);
  extern __shared__ unsigned long long gt_smem[];
  unsigned long long *bk = gt_smem;                                   // QB * B keys
  double *qs = reinterpret_cast<double *>(bk + (size_t)QB * a.B);    // QB * d queries
  int32_t *bi = reinterpret_cast<int32_t *>(qs + (size_t)QB * a.d);  // QB * B ids
  __shared__ int cnt[QB];
  __shared__ unsigned long long thk[QB];
  __shared__ int32_t thi[QB];
  const int tid = threadIdx.x;
  const int64_t q0 = (int64_t)blockIdx.x * QB;
  const int c = blockIdx.y;
  for (int i = tid; i < QB * a.d; i += kGtThreads) {
    const int j = i / a.d, col = i - j * a.d;
    qs[i] = q0 + j < a.nq ? a.Q[(q0 + j) * a.ldq + col] : 0.0;
  }
  if (tid < QB) {
    cnt[tid] = 0;
    thk[tid] = kGtInf;
    thi[tid] = 0x7fffffff;
  }
  __syncthreads();
  const int g = tid / kGtRound;  // query group of this thread
  const double *qg = qs + (size_t)g * QG * a.d;
  unsigned long long lbk[QG];
  int32_t lbi[QG];
#pragma unroll
  for (int j = 0; j < QG; ++j) {
    const int64_t q = q0 + g * QG + j;
    lbk[j] = (a.lb_key && q < a.nq) ? a.lb_key[q] : 0ull;
    lbi[j] = (a.lb_key && q < a.nq) ? a.lb_id[q] : -1;
  }
  const int64_t rbeg = (int64_t)c * a.rpc;
  const int64_t rend = rbeg + a.rpc < a.n ? rbeg + a.rpc : a.n;
  for (int64_t r0 = rbeg; r0 < rend; r0 += kGtRound) {
    const int64_t row = r0 + (tid % kGtRound);
    if (row < rend) {
      const float *xr = a.X + row * a.ldx;
      double st[QG][8];  // plan stack (depth <= 8 for d <= 4096)
      int sp = 0;
      for (int o = 0; o < plan.nops; ++o) {
        const int op = plan.op[o];
        if (op < 0) {
          --sp;
#pragma unroll
          for (int j = 0; j < QG; ++j) st[j][sp - 1] = __dadd_rn(st[j][sp - 1], st[j][sp]);
        } else {
          double res[QG];
          gt_leaf<QG>(xr, qg, a.d, plan.lo[op], plan.len[op], a.vec4, res);
#pragma unroll
          for (int j = 0; j < QG; ++j) st[j][sp] = res[j];
          ++sp;
        }
      }
#pragma unroll
      for (int j = 0; j < QG; ++j) {
        const int qj = g * QG + j;
        if (q0 + qj >= a.nq) continue;
        const unsigned long long key = (unsigned long long)__double_as_longlong(st[j][0]);
        const int32_t id = (int32_t)row;
        if (a.lb_key && !gt_less(lbk[j], lbi[j], key, id)) continue;  // taken by an earlier pass
        if (!gt_less(key, id, thk[qj], thi[qj])) continue;
        const int pos = atomicAdd(&cnt[qj], 1);
        bk[(size_t)qj * a.B + pos] = key;
        bi[(size_t)qj * a.B + pos] = id;
      }
    }
    __syncthreads();
    const bool last = r0 + kGtRound >= rend;
    for (int qj = 0; qj < QB; ++qj) {
      const int m = cnt[qj];
      if (!(m > a.B - kGtRound || (last && m > 0))) continue;  // block-uniform
      for (int i = m + tid; i < a.B; i += kGtThreads) {
        bk[(size_t)qj * a.B + i] = kGtInf;
        bi[(size_t)qj * a.B + i] = 0x7fffffff;
      }
      __syncthreads();
      gt_bitonic(bk + (size_t)qj * a.B, bi + (size_t)qj * a.B, a.B);
      if (tid == 0) {
        const int kept = m < a.kp ? m : a.kp;
        cnt[qj] = kept;
        if (kept == a.kp) {
          thk[qj] = bk[(size_t)qj * a.B + kept - 1];
          thi[qj] = bi[(size_t)qj * a.B + kept - 1];
        }
      }
      __syncthreads();
    }
  }
  // this chunk's sorted best (padded with +inf)
  for (int i = tid; i < QB * a.kp; i += kGtThreads) {
    const int qj = i / a.kp, e = i - qj * a.kp;
    if (q0 + qj >= a.nq) continue;
    const bool ok = e < cnt[qj];
    const size_t dst = ((size_t)(q0 + qj) * a.rch + c) * a.kps + e;
    a.part_key[dst] = ok ? bk[(size_t)qj * a.B + e] : kGtInf;
    a.part_id[dst] = ok ? bi[(size_t)qj * a.B + e] : 0x7fffffff;
  }
}

// One CTA per query: merge the chunks' lists, write this pass's entries and
// remember the last one as the next pass's lower bound.
__global__ void __launch_bounds__(kGtThreads) k_gt_merge(const unsigned long long *__restrict__ part_key,
                                                         const int32_t *__restrict__ part_id, int rch, int kps,
                                                         int kp, int m, int off, int kstride, int64_t *ids,
                                                         double *dists, unsigned long long *lb_key,
                                                         int32_t *lb_id) {
  extern __shared__ unsigned long long mg_smem[];
  unsigned long long *k = mg_smem;
  int32_t *id = reinterpret_cast<int32_t *>(k + m);
  const int64_t q = blockIdx.x;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const int c = i / kp, e = i - c * kp;
    const bool ok = c < rch;
    k[i] = ok ? part_key[((size_t)q * rch + c) * kps + e] : kGtInf;
    id[i] = ok ? part_id[((size_t)q * rch + c) * kps + e] : 0x7fffffff;
  }
  __syncthreads();
  gt_bitonic(k, id, m);
  for (int e = threadIdx.x; e < kp; e += blockDim.x) {
    ids[q * kstride + off + e] = k[e] == kGtInf ? -1 : (int64_t)id[e];
    dists[q * kstride + off + e] = k[e] == kGtInf ? __longlong_as_double(0x7ff0000000000000ll)
                                                  : sqrt(__longlong_as_double((long long)k[e]));
  }
  if (threadIdx.x == 0) {
    lb_key[q] = k[kp - 1];
    lb_id[q] = id[kp - 1];
  }
}

struct GtLayout {
  int qg, qb, B, kk, kp, passes, rch, m;
  int64_t rpc;
  size_t smem;
};

static int pow2_at_least(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

static bool gt_layout(int64_t n, int d, int64_t nq, int k, GtLayout &L) {
  if (n < 1 || d < 1 || d > kGtMaxD || k < 1 || nq < 0) return false;
  L.B = 1024;
  L.qg = 4;
  L.qb = L.qg * (kGtThreads / kGtRound);
  L.smem = (size_t)L.qb * L.B * 12 + (size_t)L.qb * d * 8;
  if (L.smem > 200 * 1024) {
    L.qg = 1;
    L.qb = L.qg * (kGtThreads / kGtRound);
    L.smem = (size_t)L.qb * L.B * 12 + (size_t)L.qb * d * 8;
  }
  L.kk = (int)((int64_t)k < n ? k : n);
  L.kp = L.kk < L.B / 2 ? L.kk : L.B / 2;
  L.passes = (L.kk + L.kp - 1) / L.kp;
  const int64_t nqb = nq > 0 ? (nq + L.qb - 1) / L.qb : 1;
  int64_t rch = (2 * num_sms() + nqb - 1) / nqb;
  const int64_t rmerge = kGtMergeMax / L.kp;
  const int64_t rrows = (n + kGtRound - 1) / kGtRound;
  if (rch > rmerge) rch = rmerge;
  if (rch > rrows) rch = rrows;
  if (rch < 1) rch = 1;
  L.rpc = ((n + rch - 1) / rch + kGtRound - 1) / kGtRound * kGtRound;
  L.rch = (int)((n + L.rpc - 1) / L.rpc);
  L.m = pow2_at_least(L.rch * L.kp);
  return true;
}

}  // namespace mrpt

using namespace mrpt;

extern "C" int32_t mrpt_brute_force_workspace_size(int64_t n, int32_t d, int64_t nq, int32_t k, int64_t *bytes) {
  clear_error();
  GtLayout L;
  if (!bytes || !gt_layout(n, d, nq, k, L)) return fail(MRPT_EPARAM, "mrpt_brute_force_workspace_size: bad shape");
  *bytes = (int64_t)(nq > 0 ? nq : 1) * (12 + (int64_t)L.rch * L.kp * 12) + 64;
  return MRPT_OK;
}

extern "C" int32_t mrpt_brute_force_knn(const float *X, int64_t n, int32_t d, int64_t ldx, const double *Q,
                                        int64_t nq, int64_t ldq, int32_t k, int64_t *ids, double *dists,
                                        void *ws, int64_t ws_bytes, void *stream) {
  clear_error();
  if (k < 1) return fail(MRPT_EPARAM, "mrpt_brute_force_knn: k must be >= 1");
  if (n < 1 || n >= ((int64_t)1 << 31) || d < 1 || ldx < d || ldq < d || nq < 0)
    return fail(MRPT_ESHAPE, "mrpt_brute_force_knn: bad shape");
  if (d > kGtMaxD) return fail(MRPT_EPARAM, "mrpt_brute_force_knn: d > 4096 is not supported");
  GtLayout L;
  gt_layout(n, d, nq, k, L);
  int64_t need = 0;
  mrpt_brute_force_workspace_size(n, d, nq, k, &need);
  if (ws_bytes < need || !ws) return fail(MRPT_EWORKSPACE, "mrpt_brute_force_knn: workspace too small");
  if (nq == 0) return MRPT_OK;
  GtPlan plan = {};
  int nleaf = 0;
  if (!gt_plan_rec(plan, 0, d, nleaf)) return fail(MRPT_EPARAM, "mrpt_brute_force_knn: summation plan too long");
  cudaStream_t s = as_stream(stream);
  char *w = reinterpret_cast<char *>(ws);
  unsigned long long *lb_key = reinterpret_cast<unsigned long long *>(w);
  int32_t *lb_id = reinterpret_cast<int32_t *>(lb_key + nq);
  size_t offp = ((size_t)nq * 12 + 15) & ~(size_t)15;
  unsigned long long *part_key = reinterpret_cast<unsigned long long *>(w + offp);
  int32_t *part_id = reinterpret_cast<int32_t *>(part_key + (size_t)nq * L.rch * L.kp);
  GtArgs a = {};
  a.X = X;
  a.n = n;
  a.d = d;
  a.ldx = ldx;
  a.Q = Q;
  a.nq = nq;
  a.ldq = ldq;
  a.kps = L.kp;
  a.rch = L.rch;
  a.rpc = L.rpc;
  a.B = L.B;
  a.part_key = part_key;
  a.part_id = part_id;
  a.vec4 = (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  auto fn = L.qg == 4 ? k_gt_scan<4> : k_gt_scan<1>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
  cudaFuncSetAttribute(k_gt_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, kGtMergeMax * 12);
  const dim3 grid((unsigned)((nq + L.qb - 1) / L.qb), (unsigned)L.rch);
  for (int p = 0; p < L.passes; ++p) {
    const int off = p * L.kp;
    const int kpt = L.kk - off < L.kp ? L.kk - off : L.kp;
    a.kp = kpt;
    a.lb_key = p ? lb_key : nullptr;
    a.lb_id = p ? lb_id : nullptr;
    (count_launch(), fn<<<grid, kGtThreads, L.smem, s>>>(a, plan));
    const int m = pow2_at_least(L.rch * kpt);
    (count_launch(), k_gt_merge<<<(unsigned)nq, kGtThreads, (size_t)m * 12, s>>>(
                         part_key, part_id, L.rch, L.kp, kpt, m, off, L.kk, ids, dists, lb_key, lb_id));
  }
  return launch_status("mrpt_brute_force_knn");
}
