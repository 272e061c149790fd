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
#include <cuda_fp16.h>
#include <stdlib.h>
#include <atomic>
#include <vector>

#include "common.cuh"
#include <cudaTypedefs.h>

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
  const int32_t *qlist;  // optional: process only these queries (count *qcount)
  const int32_t *qcount;
  const __half *Xh;      // optional fp16 shadow of X for the filter pass (row stride ldh)
  int64_t ldh;
  const float *radius;   // per row: upper bound of ||x - fp16(x)||_2
  int32_t *surv;         // optional (u8 filter): survivors per query, kSurvCap each, for k_rerank
  int32_t *nsurv;        // survivors per query, -1 when the query was finished in the filter kernel
  const uint32_t *cbits; // optional: candidate bitmaps (nq, bstride words) instead of cand lists
  int64_t bstride;
  int stat_slot;         // > 0: the exact fallback of route stat_slot (counts its queries)
};

// Queries that took the exact fallback, per route (1 fp32, 2 fp16, 3 u8,
// 4 tcgen05 filter), read by mrpt_fallback_stats; measurement only.
__device__ unsigned long long g_fallbacks[8];

constexpr int kSurvCap = 64;

__device__ __forceinline__ bool pair_less(unsigned long long ak, int ai, unsigned long long bk,
                                          int bi) {
  return ak < bk || (ak == bk && ai < bi);
}

// Exact squared distance of one row, summed in coordinate order exactly as
// the reference's float64 loop (_cy.pyx:81-97): one thread per row, but with
// 8 float4 loads (32 coordinates) in flight ahead of each run of dependent
// additions instead of one load round trip per coordinate.
__device__ __forceinline__ bool aligned16_dev(const void *p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

__device__ __forceinline__ double exact_dist2(const float *__restrict__ xr, const float *__restrict__ q, int d,
                                              bool vec4) {
  double e = 0.0;
  int c = 0;
  if (vec4) {
    for (; c + 32 <= d; c += 32) {
      float4 xv[8], qv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xv[u] = __ldg(reinterpret_cast<const float4 *>(xr + c) + u);
        qv[u] = __ldg(reinterpret_cast<const float4 *>(q + c) + u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        double t;
        t = (double)xv[u].x - (double)qv[u].x;
        e = __dadd_rn(e, __dmul_rn(t, t));
        t = (double)xv[u].y - (double)qv[u].y;
        e = __dadd_rn(e, __dmul_rn(t, t));
        t = (double)xv[u].z - (double)qv[u].z;
        e = __dadd_rn(e, __dmul_rn(t, t));
        t = (double)xv[u].w - (double)qv[u].w;
        e = __dadd_rn(e, __dmul_rn(t, t));
      }
    }
  }
  for (; c < d; ++c) {
    const double t = (double)__ldg(xr + c) - (double)__ldg(q + c);
    e = __dadd_rn(e, __dmul_rn(t, t));
  }
  return e;
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

// Coalesced variant (d % 4 == 0, 16-byte aligned rows).  Each warp scores 32
// candidates at a time: rows are read in 128-byte chunks by 8 lanes each
// (one LDG.128 instruction covers 4 rows), staged through a per-warp shared
// tile with a 36-word row stride (conflict-free STS.128 / LDS.128), and each
// lane then runs the reference's sequential float64 sum over its own row.
// The next chunk's loads are in flight while the current one is summed.
constexpr int kTileStride = 36;  // words per staged row (32 + 4 pad)

template <int BUF>
__global__ void __launch_bounds__(kScanNT, 3) k_scan_topk_tiled(TopkArgs a) {
  extern __shared__ unsigned long long topk_smem[];
  unsigned long long *bkey = topk_smem;                                   // BUF
  int32_t *bid = reinterpret_cast<int32_t *>(bkey + BUF);                 // BUF
  float *tiles = reinterpret_cast<float *>(bid + BUF);                    // 8 warps x 32 x 36
  double *qd = reinterpret_cast<double *>(tiles + (kScanNT / 32) * 32 * kTileStride);  // d
  __shared__ int s_cnt;
  __shared__ unsigned long long s_tk;
  __shared__ int s_ti;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.qcount && a.stat_slot > 0 && blockIdx.x == 0 && tid == 0)
    atomicAdd(&g_fallbacks[a.stat_slot], (unsigned long long)*a.qcount);
  float *tile = tiles + warp * 32 * kTileStride;
  const int d = a.d;
  const int nchunk = (d + 31) >> 5;
  const int sub = lane & 7;   // float4 slot within a 128-byte chunk
  const int rsub = lane >> 3; // row offset 0..3 within a load instruction
  const int64_t nwork = a.qlist ? (int64_t)*a.qcount : a.nq;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t q = a.qlist ? (int64_t)a.qlist[w] : w;
    for (int c = tid; c < d; c += kScanNT) qd[c] = (double)a.Q[q * a.ldq + c];
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
    const uint32_t *qbits = a.cbits ? a.cbits + q * a.bstride : nullptr;
    for (int64_t base = 0; base < m; base += kScanNT) {
      const int64_t j = base + warp * 32 + lane;
      const bool valid = j < m && (!qbits || ((__ldg(qbits + (j >> 5)) >> (j & 31)) & 1u));
      const int32_t myid = valid ? (qc ? qc[j] : (int32_t)j) : 0;
      // row ids of the 8 rows this lane loads (rows rsub + 4i of the group)
      int32_t rid[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rid[i] = __shfl_sync(0xffffffffu, myid, rsub + 4 * i);
      const float *xb = a.X + 4 * sub;
      const int64_t ldx = a.ldx;
      float4 buf[8];
      const bool full0 = 4 * sub < d;  // chunk 0 slot in range
#pragma unroll
      for (int i = 0; i < 8; ++i)
        buf[i] = full0 ? __ldg(reinterpret_cast<const float4 *>(xb + (int64_t)rid[i] * ldx))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      double acc = 0.0;
      for (int ch = 0; ch < nchunk; ++ch) {
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4 *>(tile + (rsub + 4 * i) * kTileStride + 4 * sub) = buf[i];
        __syncwarp();
        if (ch + 1 < nchunk) {
          const int off = (ch + 1) * 32;
          const bool in = off + 4 * sub < d;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            buf[i] = in ? __ldg(reinterpret_cast<const float4 *>(xb + (int64_t)rid[i] * ldx + off))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const int c0 = ch * 32;
        const int cn = (d - c0) < 32 ? (d - c0) : 32;
        const float *myrow = tile + lane * kTileStride;
        if (cn == 32) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const float4 x = *reinterpret_cast<const float4 *>(myrow + 4 * g);
            const double2 q01 = *reinterpret_cast<const double2 *>(qd + c0 + 4 * g);
            const double2 q23 = *reinterpret_cast<const double2 *>(qd + c0 + 4 * g + 2);
            double t;
            t = (double)x.x - q01.x;
            acc = __dadd_rn(acc, __dmul_rn(t, t));
            t = (double)x.y - q01.y;
            acc = __dadd_rn(acc, __dmul_rn(t, t));
            t = (double)x.z - q23.x;
            acc = __dadd_rn(acc, __dmul_rn(t, t));
            t = (double)x.w - q23.y;
            acc = __dadd_rn(acc, __dmul_rn(t, t));
          }
        } else {
          for (int c = 0; c < cn; ++c) {
            const double t = (double)myrow[c] - qd[c0 + c];
            acc = __dadd_rn(acc, __dmul_rn(t, t));
          }
        }
      }
      const unsigned long long tk = s_tk;
      const int ti = s_ti;
      const unsigned long long key = (unsigned long long)__double_as_longlong(acc);
      if (valid && pair_less(key, myid, tk, ti) && (!use_lb || pair_less(lbk, lbi, key, myid))) {
        const int slot = atomicAdd(&s_cnt, 1);
        bkey[slot] = key;
        bid[slot] = myid;
      }
      __syncthreads();
      if (s_cnt > BUF - kScanNT) {
        const int cnt = s_cnt;
        for (int i = cnt + tid; i < BUF; i += kScanNT) {
          bkey[i] = ~0ull;
          bid[i] = 0x7fffffff;
        }
        __syncthreads();
        bitonic_sort<BUF>(bkey, bid);
        if (tid == 0) {
          s_cnt = a.k;
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


// ---------------------------------------------------------------------------
// Filter-and-rerank top-k (d % 4 == 0, d <= 1024, k <= 120): bit-identical
// results at streaming cost.
//
// Pass 1 scores every candidate in float32: one warp per group of kFU
// candidates, lanes striding the coordinates with coalesced 16-byte loads,
// FFMA partial sums and a butterfly reduction.  Its value A obeys
// |A - E| <= eps*E + eta against the reference's float64 sum E (eps, eta
// from the float32 error analysis of a sum of non-negative terms, with a
// 2x safety factor).  Each warp keeps the candidates with
//     A <= ((T_a + eta) * (1 + eps) / (1 - eps)) + eta,
// T_a its k-th smallest A so far: if the k-th smallest E is E_k, the k
// smallest-A candidates all have E <= (T_a + eta)/(1 - eps), so every member
// of the exact top-k (ties included) satisfies the rule and survives.
// Pass 2 recomputes E for the few survivors with the reference's sequential
// float64 sum and orders them by (E, id).  A warp whose buffer cannot shrink
// (masses of exact ties) sends its query to the exact tiled kernel.
constexpr int kFMaxJ = 8;    // d <= 128 * kFMaxJ

__device__ __forceinline__ bool fpair_less(float ak, int ai, float bk, int bi) {
  return ak < bk || (ak == bk && ai < bi);
}

// warp-level bitonic sort of n (pow2) (float, id) pairs in shared memory
__device__ void warp_sort(float *k, int32_t *id, int n) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < n / 2; i += 32) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const float ka = k[lo], kb = k[hi];
        const int ia = id[lo], ib = id[hi];
        if (fpair_less(kb, ib, ka, ia) == asc) {
          k[lo] = kb;
          k[hi] = ka;
          id[lo] = ib;
          id[hi] = ia;
        }
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ double keep_bound(float ta, double eps, double eta) {
  return ((double)ta + eta) * (1.0 + eps) / (1.0 - eps) + eta;
}

// sort the first cnt entries (padding to n), return how many satisfy the
// keep rule for the current k-th value; *thr receives the bound.
__device__ int warp_shrink(float *k, int32_t *id, int cnt, int n, int kk, double eps, double eta,
                           double *thr) {
  const int lane = threadIdx.x & 31;
  for (int i = cnt + lane; i < n; i += 32) {
    k[i] = __int_as_float(0x7f800000);
    id[i] = 0x7fffffff;
  }
  __syncwarp();
  warp_sort(k, id, n);
  if (cnt < kk) {
    *thr = __longlong_as_double(0x7ff0000000000000LL);
    return cnt;
  }
  const double b = keep_bound(k[kk - 1], eps, eta);
  int keep = 0;
  for (int i0 = 0; i0 < cnt; i0 += 32) {
    const int i = i0 + lane;
    const bool in = i < cnt && (double)k[i] <= b;
    keep += __popc(__ballot_sync(0xffffffffu, in));
  }
  *thr = b;
  return keep;
}

template <int BUFW, int FU, int MINB>
__global__ void __launch_bounds__(kScanNT, MINB) k_scan_topk_filter(TopkArgs a, double eps, double eta,
                                                              int32_t *fb_list, int32_t *fb_count) {
  extern __shared__ unsigned long long topk_smem[];
  constexpr int NWARP = kScanNT / 32;
  constexpr int kFU = FU;
  float *qs = reinterpret_cast<float *>(topk_smem);                   // 128 * kFMaxJ
  float *wkey = qs + 128 * kFMaxJ;                                     // NWARP * BUFW
  int32_t *wid = reinterpret_cast<int32_t *>(wkey + NWARP * BUFW);    // NWARP * BUFW
  unsigned long long *ckey = reinterpret_cast<unsigned long long *>(wid + NWARP * BUFW);  // NWARP*BUFW
  int32_t *cid = reinterpret_cast<int32_t *>(ckey + NWARP * BUFW);    // NWARP * BUFW
  float *ck = reinterpret_cast<float *>(cid + NWARP * BUFW);          // NWARP * BUFW (merge keys)
  __shared__ int s_wcnt[NWARP];
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float *mk = wkey + warp * BUFW;
  int32_t *mi = wid + warp * BUFW;
  const int d = a.d;
  const int nj = (d + 127) >> 7;
  const int kk = a.k;
  for (int64_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
    const float *qrow = a.Q + q * a.ldq;
    for (int c = tid; c < 128 * kFMaxJ; c += kScanNT) qs[c] = c < d ? qrow[c] : 0.f;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    int64_t m;
    if (a.cand) {
      const int64_t nc = a.ncand[q];
      m = nc < a.cap ? nc : a.cap;
    } else {
      m = a.n;
    }
    const int32_t *qc = a.cand ? a.cand + q * a.cap : nullptr;
    int cnt = 0;
    double thr = __longlong_as_double(0x7ff0000000000000LL);
    bool bad = false;
    for (int64_t g = (int64_t)warp * kFU; g < m; g += (int64_t)NWARP * kFU) {
      int32_t cidv[kFU];
      const float *row[kFU];
#pragma unroll
      for (int u = 0; u < kFU; ++u) {
        const int64_t j = g + u;
        cidv[u] = j < m ? (qc ? __ldg(qc + j) : (int32_t)j) : -1;
        row[u] = a.X + (int64_t)(cidv[u] < 0 ? 0 : cidv[u]) * a.ldx;
      }
      float acc[kFU];
#pragma unroll
      for (int u = 0; u < kFU; ++u) acc[u] = 0.f;
#pragma unroll
      for (int j = 0; j < kFMaxJ; ++j) {
        const int c = j * 128 + 4 * lane;
        if (j < nj && c < d) {
          const float4 qj = *reinterpret_cast<const float4 *>(qs + c);
          float4 x[kFU];
#pragma unroll
          for (int u = 0; u < kFU; ++u) x[u] = __ldg(reinterpret_cast<const float4 *>(row[u] + c));
#pragma unroll
          for (int u = 0; u < kFU; ++u) {
            float t;
            t = x[u].x - qj.x;
            acc[u] = __fmaf_rn(t, t, acc[u]);
            t = x[u].y - qj.y;
            acc[u] = __fmaf_rn(t, t, acc[u]);
            t = x[u].z - qj.z;
            acc[u] = __fmaf_rn(t, t, acc[u]);
            t = x[u].w - qj.w;
            acc[u] = __fmaf_rn(t, t, acc[u]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kFU; ++u) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
      }
      // lane u decides for candidate u
      float mine = acc[0];
      int32_t myid = cidv[0];
#pragma unroll
      for (int u = 1; u < kFU; ++u)
        if (lane == u) {
          mine = acc[u];
          myid = cidv[u];
        }
      const bool take = lane < kFU && myid >= 0 && (double)mine <= thr;
      const unsigned tm = __ballot_sync(0xffffffffu, take);
      if (take) {
        const int slot = cnt + __popc(tm & lanemask_lt());
        mk[slot] = mine;
        mi[slot] = myid;
      }
      cnt += __popc(tm);
      if (cnt > BUFW - kFU) {
        __syncwarp();
        cnt = warp_shrink(mk, mi, cnt, BUFW, kk, eps, eta, &thr);
        if (cnt > BUFW - kFU) {  // cannot shrink: exact ties galore
          bad = true;
          cnt = 0;
          break;
        }
      }
    }
    __syncwarp();
    if (!bad) cnt = warp_shrink(mk, mi, cnt, BUFW, kk, eps, eta, &thr);
    if (lane == 0) {
      s_wcnt[warp] = cnt;
      if (bad) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) {
      if (tid == 0) fb_list[atomicAdd(fb_count, 1)] = (int32_t)q;
      __syncthreads();
      continue;
    }
    // merge the warp survivors (each a sorted prefix) into ck/cid
    int off = 0, total = 0;
    for (int w = 0; w < NWARP; ++w) {
      off += w < warp ? s_wcnt[w] : 0;
      total += s_wcnt[w];
    }
    for (int i = lane; i < cnt; i += 32) {
      ck[off + i] = mk[i];
      cid[off + i] = mi[i];
    }
    int np2 = 32;
    while (np2 < total) np2 <<= 1;
    for (int i = total + tid; i < np2; i += kScanNT) {
      ck[i] = __int_as_float(0x7f800000);
      cid[i] = 0x7fffffff;
    }
    __syncthreads();
    // CTA bitonic sort of np2 (approx, id)
    for (int size = 2; size <= np2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = tid; i < np2 / 2; i += kScanNT) {
          const int lo = 2 * i - (i & (stride - 1));
          const int hi = lo + stride;
          const bool asc = (lo & size) == 0;
          const float ka = ck[lo], kb = ck[hi];
          const int ia = cid[lo], ib = cid[hi];
          if (fpair_less(kb, ib, ka, ia) == asc) {
            ck[lo] = kb;
            ck[hi] = ka;
            cid[lo] = ib;
            cid[hi] = ia;
          }
        }
        __syncthreads();
      }
    }
    const double b = total >= kk ? keep_bound(ck[kk - 1], eps, eta)
                                 : __longlong_as_double(0x7ff0000000000000LL);
    // survivors: sorted prefix with approx <= b; exact float64 rerank
    int ns = 0;
    for (int i = 0; i < total; ++i) {
      if ((double)ck[i] <= b) ns = i + 1; else break;
    }
    int np3 = 1;
    while (np3 < ns) np3 <<= 1;
    for (int i = tid; i < np3; i += kScanNT) {
      if (i < ns) {
        const int32_t id = cid[i];
        const float *xr = a.X + (int64_t)id * a.ldx;
        const double e = exact_dist2(xr, qrow, d, a.vec4 && aligned16_dev(qrow));
        ckey[i] = (unsigned long long)__double_as_longlong(e);
        wid[i] = id;
      } else {
        ckey[i] = ~0ull;
        wid[i] = 0x7fffffff;
      }
    }
    __syncthreads();
    for (int size = 2; size <= np3; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = tid; i < np3 / 2; i += kScanNT) {
          const int lo = 2 * i - (i & (stride - 1));
          const int hi = lo + stride;
          const bool asc = (lo & size) == 0;
          const unsigned long long ka = ckey[lo], kb = ckey[hi];
          const int ia = wid[lo], ib = wid[hi];
          if (pair_less(kb, ib, ka, ia) == asc) {
            ckey[lo] = kb;
            ckey[hi] = ka;
            wid[lo] = ib;
            wid[hi] = ia;
          }
        }
        __syncthreads();
      }
    }
    const int kept = ns < kk ? ns : kk;
    for (int i = tid; i < kk; i += kScanNT) {
      if (i < kept) {
        a.ids[q * a.kstride + i] = wid[i];
        a.dists[q * a.kstride + i] = sqrt(__longlong_as_double((long long)ckey[i]));
      } else {
        a.ids[q * a.kstride + i] = -1;
        a.dists[q * a.kstride + i] = __longlong_as_double(0x7ff0000000000000LL);
      }
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// fp16 shadow rows for the filter pass.  x~ = fp16(x) (round to nearest),
// radius = ||x - x~||_2 rounded up.  For any query q the true distance then
// lies within radius of ||x~ - q|| (triangle inequality), so the filter can
// bound E from the fp16 row alone and the exact float64 rerank is unchanged.
// Rows are padded to 8 halves (16-byte loads) with zeros.
__global__ void k_quantize_fp16(const float *__restrict__ X, int64_t n, int d, int64_t ldx,
                                __half *Xh, int64_t ldh, float *radius, int32_t *bad) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += wstride) {
    const float *xr = X + i * ldx;
    __half *hr = Xh + i * ldh;
    double r2 = 0.0;
    for (int c = lane; c < ldh; c += 32) {
      float x = c < d ? xr[c] : 0.f;
      if (fabsf(x) > 65504.f) *bad = 1;
      const __half h = __float2half_rn(x);
      hr[c] = h;
      const double e = (double)x - (double)__half2float(h);
      r2 = fma(e, e, r2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    if (lane == 0) radius[i] = __double2float_ru(__dsqrt_ru(r2 * (1.0 + 1e-12)));
  }
}

// Packed float32 pairs in one 64-bit register (sm_100 FADD2 / FFMA2).
__device__ __forceinline__ unsigned long long f32x2_pack(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ unsigned long long f32x2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f32x2_fma(unsigned long long a, unsigned long long b,
                                                        unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float f32x2_sum(unsigned long long a) {
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a));
  return x + y;
}

// bounds of the reference distance E from the fp16-row filter value A and the
// row radius r:  sqrt(E) in [sqrt(D) - r, sqrt(D) + r],  D = ||x~ - q||^2 with
// |A - D| <= eps*D + eta (float32 arithmetic), E within 1e-12 relative of the
// real value (float64 reference sum).
__device__ __forceinline__ void dist_bounds(float A, float r, double eps, double eta, double &L,
                                            double &U) {
  const double a = (double)A;
  const double dlo = fmax(0.0, (a - eta) / (1.0 + eps));
  const double dhi = (a + eta) / (1.0 - eps);
  const double slo = fmax(0.0, sqrt(dlo) - (double)r);
  const double shi = sqrt(dhi) + (double)r;
  L = slo * slo * (1.0 - 1e-12);
  U = shi * shi * (1.0 + 1e-12);
}

// Filter on the fp16 shadow + exact rerank.  Per warp, a buffer of
// (A, r, id).  At every shrink the buffer's bounds L_i <= E_i <= U_i are
// evaluated in float64, U_k = k-th smallest U_i bounds the k-th smallest
// reference distance, and entries with L_i > U_k are dropped.  Between
// shrinks a candidate is admitted iff  A <= (1+eps)(sqrt(U_k) + r)^2 + eta,
// evaluated with upward rounding -- a superset of L <= U_k -- so every exact
// top-k member (ties included) survives to the float64 rerank.
__device__ __forceinline__ bool admit(float A, float r, float su, float onepe) {
  const float t = __fadd_ru(su, r);
  const float rhs = __fadd_ru(__fmul_ru(__fmul_ru(t, t), onepe), 1.1754944e-38f);
  return A <= rhs;
}

template <int BUFW>
__device__ int shrink_bounds(float *ma, float *mr, int32_t *mi, int cnt, int kk, double eps,
                             double eta, float *su_scr, int32_t *ix_scr, float *su_out) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < BUFW; i += 32) {
    if (i < cnt) {
      double L, U;
      dist_bounds(ma[i], mr[i], eps, eta, L, U);
      su_scr[i] = __double2float_ru(U);
    } else {
      su_scr[i] = __int_as_float(0x7f800000);
    }
    ix_scr[i] = i;
  }
  __syncwarp();
  warp_sort(su_scr, ix_scr, BUFW);
  const double uk = (double)su_scr[kk - 1];
  int keep = 0;
  for (int i0 = 0; i0 < cnt; i0 += 32) {
    const int i = i0 + lane;
    bool in = false;
    float av = 0.f, rv = 0.f;
    int32_t iv = 0;
    if (i < cnt) {
      av = ma[i];
      rv = mr[i];
      iv = mi[i];
      double L, U;
      dist_bounds(av, rv, eps, eta, L, U);
      in = L <= uk;
    }
    const unsigned bm = __ballot_sync(0xffffffffu, in);
    __syncwarp();
    if (in) {
      const int dst = keep + __popc(bm & lanemask_lt());
      ma[dst] = av;
      mr[dst] = rv;
      mi[dst] = iv;
    }
    __syncwarp();
    keep += __popc(bm);
  }
  *su_out = uk >= 3.0e38 ? __int_as_float(0x7f800000) : __double2float_ru(sqrt(uk));
  return keep;
}

template <int BUFW>
__global__ void __launch_bounds__(kScanNT, 4) k_scan_topk_filter_h(TopkArgs a, double eps, double eta,
                                                                  int32_t *fb_list, int32_t *fb_count) {
  extern __shared__ unsigned long long topk_smem[];
  constexpr int NWARP = kScanNT / 32;
  constexpr int kFU = 4;
  constexpr int kMaxJ = 4;  // ldh <= 256 * kMaxJ halves
  float *qs = reinterpret_cast<float *>(topk_smem);                   // 256 * kMaxJ
  float *wa = qs + 256 * kMaxJ;                                        // NWARP*BUFW filter values
  int32_t *wid = reinterpret_cast<int32_t *>(wa + NWARP * BUFW);      // NWARP*BUFW
  int32_t *cid = wid + NWARP * BUFW;                                   // NWARP*BUFW
  float *cl = reinterpret_cast<float *>(cid + NWARP * BUFW);          // NWARP*BUFW
  float *wr = cl + NWARP * BUFW;                                       // NWARP*BUFW radii
  float *cu = wr + NWARP * BUFW;                                       // NWARP*BUFW
  // the rerank keys (8 bytes each) overlay the radii and the upper bounds,
  // both dead by then: 52 KB per CTA at BUFW = 256, four CTAs per SM
  unsigned long long *ckey = reinterpret_cast<unsigned long long *>(wr);  // NWARP*BUFW
  __shared__ int s_wcnt[NWARP];
  __shared__ int s_bad, s_ns;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float *ma = wa + warp * BUFW;
  float *mr = wr + warp * BUFW;
  int32_t *mi = wid + warp * BUFW;
  const int d = a.d;
  const int dpad = (int)a.ldh;
  const int nj = (dpad + 255) >> 8;
  const int kk = a.k;
  const float onepe = __double2float_ru(1.0 + eps);
  for (int64_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
    const float *qrow = a.Q + q * a.ldq;
    for (int c = tid; c < 256 * kMaxJ; c += kScanNT) qs[c] = c < d ? qrow[c] : 0.f;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    int64_t m;
    if (a.cand) {
      const int64_t nc = a.ncand[q];
      m = nc < a.cap ? nc : a.cap;
    } else {
      m = a.n;
    }
    const int32_t *qc = a.cand ? a.cand + q * a.cap : nullptr;
    int cnt = 0;
    float su = __int_as_float(0x7f800000);  // sqrt(U_k), +inf until the first shrink
    bool bad = false;
    // A warp takes 32 * kFU consecutive candidates at a time: one coalesced
    // load puts lane l's kFU ids in registers, and each of the 32 iterations
    // broadcasts its kFU ids by shuffle -- the rows of an iteration wait for
    // one memory round trip instead of the id load and then the row load.
    for (int64_t c0 = (int64_t)warp * (32 * kFU); c0 < m && !bad; c0 += (int64_t)NWARP * 32 * kFU) {
      int32_t lane_ids[kFU];
#pragma unroll
      for (int u = 0; u < kFU; ++u) {
        const int64_t j = c0 + (int64_t)kFU * lane + u;
        lane_ids[u] = j < m ? (qc ? __ldg(qc + j) : (int32_t)j) : -1;
      }
      const int64_t left = m - c0;
      const int nit = left >= 32 * kFU ? 32 : (int)((left + kFU - 1) / kFU);
    for (int it = 0; it < nit; ++it) {
      int32_t cidv[kFU];
      const __half *row[kFU];
#pragma unroll
      for (int u = 0; u < kFU; ++u) {
        cidv[u] = __shfl_sync(0xffffffffu, lane_ids[u], it);
        row[u] = a.Xh + (int64_t)(cidv[u] < 0 ? 0 : cidv[u]) * a.ldh;
      }
      // after the transposed reduction below, lanes 8u .. 8u+7 hold candidate
      // u's value; lane 8u represents it
      static_assert(kFU == 4, "transposed reduction is written for 4 candidates");
      const int ci = (lane >> 3) & 3;
      int32_t myid = cidv[0];
#pragma unroll
      for (int u = 1; u < kFU; ++u) myid = ci == u ? cidv[u] : myid;
      const bool rep = (lane & 7) == 0;
      const float myr = (rep && myid >= 0) ? __ldg(a.radius + myid) : 0.f;
      // packed float32 pairs (FADD2 / FFMA2: two lanes of arithmetic per
      // instruction); even and odd coordinates accumulate separately
      unsigned long long acc2[kFU];
#pragma unroll
      for (int u = 0; u < kFU; ++u) acc2[u] = 0ull;
#pragma unroll
      for (int j = 0; j < kMaxJ; ++j) {
        const int c = j * 256 + 8 * lane;
        if (j < nj && c < dpad) {
          const float4 q0 = *reinterpret_cast<const float4 *>(qs + c);
          const float4 q1 = *reinterpret_cast<const float4 *>(qs + c + 4);
          const unsigned long long qp[4] = {f32x2_pack(q0.x, q0.y), f32x2_pack(q0.z, q0.w),
                                            f32x2_pack(q1.x, q1.y), f32x2_pack(q1.z, q1.w)};
          uint4 raw[kFU];
#pragma unroll
          for (int u = 0; u < kFU; ++u) raw[u] = __ldg(reinterpret_cast<const uint4 *>(row[u] + c));
#pragma unroll
          for (int u = 0; u < kFU; ++u) {
            const __half2 *h2 = reinterpret_cast<const __half2 *>(&raw[u]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __half22float2(h2[e]);
              const unsigned long long t = f32x2_sub(f32x2_pack(f.x, f.y), qp[e]);
              acc2[u] = f32x2_fma(t, t, acc2[u]);
            }
          }
        }
      }
      float acc[kFU];
#pragma unroll
      for (int u = 0; u < kFU; ++u) acc[u] = f32x2_sum(acc2[u]);
      // transposed warp reduction of the 4 sums (6 shuffles instead of 20):
      // exchange halves across lane bit 4, then bit 3, then sum the rest.
      // Any summation order is inside the eps bound (2 (ldh+16) u).
      const bool b16 = lane & 16, b8 = lane & 8;
      float k0 = b16 ? acc[2] : acc[0], k1 = b16 ? acc[3] : acc[1];
      const float s0 = b16 ? acc[0] : acc[2], s1 = b16 ? acc[1] : acc[3];
      k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
      k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
      float mine = (b8 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, b8 ? k0 : k1, 8);
      mine += __shfl_xor_sync(0xffffffffu, mine, 4);
      mine += __shfl_xor_sync(0xffffffffu, mine, 2);
      mine += __shfl_xor_sync(0xffffffffu, mine, 1);
      const bool take = rep && myid >= 0 && admit(mine, myr, su, onepe);
      const unsigned tm = __ballot_sync(0xffffffffu, take);
      if (take) {
        const int slot = cnt + __popc(tm & lanemask_lt());
        ma[slot] = mine;
        mr[slot] = myr;
        mi[slot] = myid;
      }
      cnt += __popc(tm);
      if (cnt > BUFW - kFU) {
        __syncwarp();
        cnt = shrink_bounds<BUFW>(ma, mr, mi, cnt, kk, eps, eta, cu + warp * BUFW,
                                  cid + warp * BUFW, &su);
        if (cnt > BUFW - kFU) {
          bad = true;
          cnt = 0;
          break;
        }
      }
    }
    }
    __syncwarp();
    if (lane == 0) {
      s_wcnt[warp] = cnt;
      if (bad) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) {
      if (tid == 0) fb_list[atomicAdd(fb_count, 1)] = (int32_t)q;
      __syncthreads();
      continue;
    }
    // merge every warp's buffer: bounds, global U_k, survivors L <= U_k
    int off = 0, total = 0;
    for (int w = 0; w < NWARP; ++w) {
      off += w < warp ? s_wcnt[w] : 0;
      total += s_wcnt[w];
    }
    for (int i = lane; i < cnt; i += 32) {
      double L, U;
      dist_bounds(ma[i], mr[i], eps, eta, L, U);
      cu[off + i] = __double2float_ru(U);
      cl[off + i] = __double2float_rd(L);
      cid[off + i] = mi[i];
    }
    __syncthreads();
    int np2 = 32;
    while (np2 < total) np2 <<= 1;
    float *su2 = wa;  // warp buffers are free now: sort scratch
    int32_t *sx = wid;
    for (int i = tid; i < np2; i += kScanNT) {
      su2[i] = i < total ? cu[i] : __int_as_float(0x7f800000);
      sx[i] = i;
    }
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = tid; i < np2 / 2; i += kScanNT) {
          const int lo = 2 * i - (i & (stride - 1));
          const int hi = lo + stride;
          const bool asc = (lo & size) == 0;
          const float ka = su2[lo], kb = su2[hi];
          const int ia = sx[lo], ib = sx[hi];
          if (fpair_less(kb, ib, ka, ia) == asc) {
            su2[lo] = kb;
            su2[hi] = ka;
            sx[lo] = ib;
            sx[hi] = ia;
          }
        }
        __syncthreads();
      }
    }
    const double uk = total >= kk ? (double)su2[kk - 1] : __longlong_as_double(0x7ff0000000000000LL);
    if (tid == 0) s_ns = 0;
    __syncthreads();
    for (int i = tid; i < total; i += kScanNT) {
      if ((double)cl[i] <= uk) sx[atomicAdd(&s_ns, 1)] = cid[i];
    }
    __syncthreads();
    const int ns = s_ns;
    int np3 = 1;
    while (np3 < ns) np3 <<= 1;
    for (int i = tid; i < np3; i += kScanNT) {
      if (i < ns) {
        const int32_t id = sx[i];
        const float *xr = a.X + (int64_t)id * a.ldx;
        const double e = exact_dist2(xr, qrow, d, a.vec4 && aligned16_dev(qrow));
        ckey[i] = (unsigned long long)__double_as_longlong(e);
        cid[i] = id;
      } else {
        ckey[i] = ~0ull;
        cid[i] = 0x7fffffff;
      }
    }
    __syncthreads();
    for (int size = 2; size <= np3; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = tid; i < np3 / 2; i += kScanNT) {
          const int lo = 2 * i - (i & (stride - 1));
          const int hi = lo + stride;
          const bool asc = (lo & size) == 0;
          const unsigned long long ka = ckey[lo], kb = ckey[hi];
          const int ia = cid[lo], ib = cid[hi];
          if (pair_less(kb, ib, ka, ia) == asc) {
            ckey[lo] = kb;
            ckey[hi] = ka;
            cid[lo] = ib;
            cid[hi] = ia;
          }
        }
        __syncthreads();
      }
    }
    const int kept = ns < kk ? ns : kk;
    for (int i = tid; i < kk; i += kScanNT) {
      if (i < kept) {
        a.ids[q * a.kstride + i] = cid[i];
        a.dists[q * a.kstride + i] = sqrt(__longlong_as_double((long long)ckey[i]));
      } else {
        a.ids[q * a.kstride + i] = -1;
        a.dists[q * a.kstride + i] = __longlong_as_double(0x7ff0000000000000LL);
      }
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// u8 shadow rows (non-negative data): X_i = rint(x_i / s) in [0, 255] with a
// per-row scale s (s = 1 when the whole dataset is integer-valued in
// [0, 255], which makes the shadow exact), radius r >= ||x - s X||_2 and
// N = sum X_i^2.  The filter then scores a candidate with exact integer dot
// products (dp4a, int32 accumulate -- no rounding at all):
//   D = s_x^2 N_x + s_q^2 N_q - 2 s_x s_q (X . Q)   (float64, |error| <= eta)
// and sqrt(E) lies within r_x + r_q of sqrt(D) for the reference's E.
__global__ void k_q8_flags(const float *__restrict__ X, int64_t n, int d, int64_t ldx, int32_t *flags) {
  // flags[0]: some x < 0; flags[1]: some x not an integer in [0, 255]
  bool neg = false, nonint = false;
  const int64_t total = n * d;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = g / d, c = g - i * d;
    const float x = X[i * ldx + c];
    neg |= x < 0.f;
    nonint |= !(x >= 0.f && x <= 255.f && rintf(x) == x);
  }
  if (__any_sync(0xffffffffu, neg) && (threadIdx.x & 31) == 0) flags[0] = 1;
  if (__any_sync(0xffffffffu, nonint) && (threadIdx.x & 31) == 0) flags[1] = 1;
}

__global__ void k_quantize_u8(const float *__restrict__ X, int64_t n, int d, int64_t ldx,
                              uint8_t *Xq, int64_t ldq, float *scale, int32_t *norm, float *radius,
                              int integer_mode) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += wstride) {
    const float *xr = X + i * ldx;
    float mx = 0.f;
    for (int c = lane; c < d; c += 32) mx = fmaxf(mx, xr[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float sc = integer_mode ? 1.f : (mx > 0.f ? mx / 255.f : 1.f);
    double r2 = 0.0;
    int nn = 0;
    for (int c = lane; c < ldq; c += 32) {
      const float x = c < d ? xr[c] : 0.f;
      float qv = rintf(x / sc);
      qv = fminf(fmaxf(qv, 0.f), 255.f);
      const int qi = (int)qv;
      Xq[i * ldq + c] = (uint8_t)qi;
      const double e = (double)x - (double)sc * (double)qi;
      r2 = fma(e, e, r2);
      nn += qi * qi;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r2 += __shfl_xor_sync(0xffffffffu, r2, o);
      nn += __shfl_xor_sync(0xffffffffu, nn, o);
    }
    if (lane == 0) {
      scale[i] = sc;
      norm[i] = nn;
      radius[i] = r2 == 0.0 ? 0.f : __double2float_ru(__dsqrt_ru(r2 * (1.0 + 1e-12)));
    }
  }
}

__device__ __forceinline__ void dist_bounds2(float A, float r, float eta, double &L, double &U) {
  const double a = (double)A, e = (double)eta;
  const double slo = fmax(0.0, sqrt(fmax(0.0, a - e)) - (double)r);
  const double shi = sqrt(a + e) + (double)r;
  L = slo * slo * (1.0 - 1e-12);
  U = shi * shi * (1.0 + 1e-12);
}

// admitted iff A <= (sqrt(U_k) + r)^2 + eta, upward rounding: a superset of
// "lower bound <= U_k"
__device__ __forceinline__ bool admit2(float A, float r, float eta, float su) {
  const float t = __fadd_ru(su, r);
  const float rhs = __fadd_ru(__fmul_ru(t, t), __fadd_ru(eta, 1.1754944e-38f));
  return A <= rhs;
}

template <int BUFW>
__device__ int shrink_bounds2(float *ma, float *mr, float *me, int32_t *mi, int cnt, int kk,
                              float *su_scr, int32_t *ix_scr, float *su_out) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < BUFW; i += 32) {
    if (i < cnt) {
      double L, U;
      dist_bounds2(ma[i], mr[i], me[i], L, U);
      su_scr[i] = __double2float_ru(U);
    } else {
      su_scr[i] = __int_as_float(0x7f800000);
    }
    ix_scr[i] = i;
  }
  __syncwarp();
  warp_sort(su_scr, ix_scr, BUFW);
  const double uk = (double)su_scr[kk - 1];
  int keep = 0;
  for (int i0 = 0; i0 < cnt; i0 += 32) {
    const int i = i0 + lane;
    bool in = false;
    float av = 0.f, rv = 0.f, ev = 0.f;
    int32_t iv = 0;
    if (i < cnt) {
      av = ma[i];
      rv = mr[i];
      ev = me[i];
      iv = mi[i];
      double L, U;
      dist_bounds2(av, rv, ev, L, U);
      in = L <= uk;
    }
    const unsigned bm = __ballot_sync(0xffffffffu, in);
    __syncwarp();
    if (in) {
      const int dst = keep + __popc(bm & lanemask_lt());
      ma[dst] = av;
      mr[dst] = rv;
      me[dst] = ev;
      mi[dst] = iv;
    }
    __syncwarp();
    keep += __popc(bm);
  }
  *su_out = uk >= 3.0e38 ? __int_as_float(0x7f800000) : __double2float_ru(sqrt(uk));
  return keep;
}

struct QParams;

struct Q8Rows {
  const uint8_t *X;  // (n, ldq) u8
  int64_t ldq;       // multiple of 16, <= 1024
  const float *scale;
  const int32_t *norm;
  const float *radius;
};

// a: 4 row bytes (u8), b: 4 query bytes (s8 when QS, else u8)
template <bool QS>
__device__ __forceinline__ int dp4a_us(uint32_t a, uint32_t b, int c) {
  int d;
  if (QS)
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  else
    asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// U rows' partial dot products over this lane's 16-byte chunks.  The query's
// signedness is a template parameter: a runtime flag here puts a branch
// around every dp4a (inline asm cannot be predicated).
template <int U, int G, bool QS>
__device__ __forceinline__ void dot_rows_u8(const uint8_t *(&rp)[U], const uint32_t *qb,
                                            int gl, int nchunk, int (&acc)[U]) {
  for (int ch = gl; ch < nchunk; ch += G) {
    const uint4 qv = *reinterpret_cast<const uint4 *>(qb + 4 * ch);
    uint4 xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(reinterpret_cast<const uint4 *>(rp[u] + 16 * ch));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[u] = dp4a_us<QS>(xv[u].x, qv.x, acc[u]);
      acc[u] = dp4a_us<QS>(xv[u].y, qv.y, acc[u]);
      acc[u] = dp4a_us<QS>(xv[u].z, qv.z, acc[u]);
      acc[u] = dp4a_us<QS>(xv[u].w, qv.w, acc[u]);
    }
  }
}

// Per-query quantisation parameters of the u8 filter.
struct QParams {
  float sq;     // query scale (1 for integer-valued queries in [0, 255])
  float rq;     // L2 norm of the query's quantisation error, rounded up
  float t2f;    // sq^2 * ||qq||^2 in float32 (the filter's t2 term)
  int qsigned;  // 1: s8 entries (the query has negatives), 0: u8
  int qsum;     // sum of the quantised entries over ldq (pads are 0)
  int pad;
};

template <int NW>
struct QScratch {
  float mn[NW], mx[NW];
  int isint[NW];
  double r2[NW];
  long long nq[NW];
  int qs[NW];
};

// Block-wide quantisation of one query row into qb (ldq/4 packed words):
// u8 when q >= 0 (exact for integer values <= 255), else s8 with scale
// max|q|/127.  Every thread returns the same parameters.
template <int NT>
__device__ __forceinline__ QParams quantize_query_u8(const float *qrow, int d, int ldq, uint32_t *qb,
                                                     QScratch<NT / 32> &sc) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float mn = 3.4e38f, mx = 0.f;
  int isint = 1;
  for (int c = tid; c < d; c += NT) {
    const float v = qrow[c];
    mn = fminf(mn, v);
    mx = fmaxf(mx, fabsf(v));
    isint &= (v >= 0.f && v <= 255.f && rintf(v) == v) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    isint &= __shfl_xor_sync(0xffffffffu, isint, o);
  }
  if (lane == 0) {
    sc.mn[warp] = mn;
    sc.mx[warp] = mx;
    sc.isint[warp] = isint;
  }
  __syncthreads();
  mn = sc.mn[0];
  mx = sc.mx[0];
  isint = sc.isint[0];
  for (int w = 1; w < NW; ++w) {
    mn = fminf(mn, sc.mn[w]);
    mx = fmaxf(mx, sc.mx[w]);
    isint &= sc.isint[w];
  }
  const bool qsigned = mn < 0.f;
  const float sq = isint ? 1.f : (mx > 0.f ? mx / (qsigned ? 127.f : 255.f) : 1.f);
  double r2 = 0.0;
  long long nq = 0;
  int qs = 0;
  for (int w4 = tid; w4 < ldq / 4; w4 += NT) {
    uint32_t packed = 0u;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = 4 * w4 + b;
      const float v = c < d ? qrow[c] : 0.f;
      float qv = rintf(v / sq);
      qv = qsigned ? fminf(fmaxf(qv, -127.f), 127.f) : fminf(fmaxf(qv, 0.f), 255.f);
      const int qi = (int)qv;
      packed |= ((uint32_t)qi & 0xffu) << (8 * b);
      const double e = (double)v - (double)sq * (double)qi;
      r2 = fma(e, e, r2);
      nq += (long long)qi * qi;
      qs += qi;
    }
    qb[w4] = packed;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    nq += __shfl_xor_sync(0xffffffffu, nq, o);
    qs += __shfl_xor_sync(0xffffffffu, qs, o);
  }
  __syncthreads();  // everyone has read sc.mn/mx before the next query rewrites them
  if (lane == 0) {
    sc.r2[warp] = r2;
    sc.nq[warp] = nq;
    sc.qs[warp] = qs;
  }
  __syncthreads();
  double r2t = 0.0;
  long long nqt = 0;
  int qst = 0;
  for (int w = 0; w < NW; ++w) {
    r2t += sc.r2[w];
    nqt += sc.nq[w];
    qst += sc.qs[w];
  }
  QParams P;
  P.rq = r2t == 0.0 ? 0.f : __double2float_ru(__dsqrt_ru(r2t * (1.0 + 1e-12)));
  P.sq = sq;
  P.t2f = sq * sq * (float)nqt;
  P.qsigned = qsigned ? 1 : 0;
  P.qsum = qst;
  P.pad = 0;
  return P;
}

// One candidate per lane of the u8 filter: float32 bounds of its distance
// (each of t1, t2, t3 carries <= 3 roundings and the sum two more, so
// |A - D| <= 8 * 2^-24 * (t1 + t2 + |t3|)), admission against the warp's
// running k-th upper bound, buffer append, and a shrink when the buffer is
// full; false when it cannot shrink (-> exact fallback).
// su_cta: the smallest sqrt(k-th upper bound) any warp of the CTA has
// established for this query (float bits; every warp's k-th bound bounds the
// query's k-th, so each warp may filter with the smallest).
template <int BUFW, int CPI>
__device__ __forceinline__ bool admit_lane_u8(int32_t myc, int mys, float sx, int nrm, float rad, float sqf,
                                              float t2f, float rq, float &su, int &cnt, float *ma, float *mr,
                                              float *me, int32_t *mi, int kk, float *cu_w, int32_t *cid_w,
                                              unsigned *su_cta) {
  su = fminf(su, __uint_as_float(*reinterpret_cast<volatile unsigned *>(su_cta)));
  float A = 0.f, r = 0.f, eta = 0.f;
  if (myc >= 0) {
    const float t1 = sx * sx * (float)nrm;
    const float t3 = 2.0f * sx * sqf * (float)mys;
    A = (t1 + t2f) - t3;
    eta = __fmul_ru(4.76837158203125e-07f, __fadd_ru(__fadd_ru(t1, t2f), fabsf(t3)));
    r = __fadd_ru(rad, rq);
  }
  const bool take = myc >= 0 && admit2(A, r, eta, su);
  const unsigned tm = __ballot_sync(0xffffffffu, take);
  if (take) {
    const int slot = cnt + __popc(tm & lanemask_lt());
    ma[slot] = A;
    mr[slot] = r;
    me[slot] = eta;
    mi[slot] = myc;
  }
  cnt += __popc(tm);
  if (cnt > BUFW - CPI) {
    __syncwarp();
    cnt = shrink_bounds2<BUFW>(ma, mr, me, mi, cnt, kk, cu_w, cid_w, &su);
    if ((threadIdx.x & 31) == 0) atomicMin(su_cta, __float_as_uint(su));
    if (cnt > BUFW - CPI) return false;
  }
  return true;
}

// G lanes per row (ldq / 16 rounded up to a power of two, <= 32); each warp
// iteration scores (32 / G) * 4 candidates with 16-byte loads.
template <int BUFW, int G>
__global__ void __launch_bounds__(kScanNT, 4) k_scan_topk_u8(TopkArgs a, Q8Rows rows,
                                                             int32_t *fb_list, int32_t *fb_count) {
  extern __shared__ unsigned long long topk_smem[];
  constexpr int NWARP = kScanNT / 32;
  constexpr int R = 32 / G;             // rows per load instruction
  constexpr int U = 4;                  // loads in flight per lane
  constexpr int CPI = R * U;            // candidates per warp iteration (<= 32)
  uint32_t *qb = reinterpret_cast<uint32_t *>(topk_smem);             // 256 words: quantized q
  float *wa = reinterpret_cast<float *>(qb + 256);
  float *wr = wa + NWARP * BUFW;
  float *we = wr + NWARP * BUFW;
  int32_t *wid = reinterpret_cast<int32_t *>(we + NWARP * BUFW);
  unsigned long long *ckey = reinterpret_cast<unsigned long long *>(wid + NWARP * BUFW);
  int32_t *cid = reinterpret_cast<int32_t *>(ckey + NWARP * BUFW);
  float *cu = reinterpret_cast<float *>(cid + NWARP * BUFW);
  float *cl = cu + NWARP * BUFW;
  __shared__ int s_wcnt[NWARP];
  __shared__ int s_bad, s_ns;
  __shared__ unsigned s_su_cta;
  __shared__ QScratch<NWARP> qscr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float *ma = wa + warp * BUFW;
  float *mr = wr + warp * BUFW;
  float *me = we + warp * BUFW;
  int32_t *mi = wid + warp * BUFW;
  const int d = a.d;
  const int ldq = (int)rows.ldq;
  const int nchunk = ldq / 16;
  const int kk = a.k;
  const int grp = lane / G, gl = lane % G;
  for (int64_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
    const float *qrow = a.Q + q * a.ldq;
    if (tid == 0) {
      s_bad = 0;
      s_su_cta = 0x7f800000u;  // +inf
    }
    const QParams P = quantize_query_u8<kScanNT>(qrow, d, ldq, qb, qscr);
    const bool qsigned = P.qsigned != 0;
    const float rq = P.rq;
    const float sqf = P.sq, t2f = P.t2f;
    int64_t m;
    if (a.cand) {
      const int64_t nc = a.ncand[q];
      m = nc < a.cap ? nc : a.cap;
    } else {
      m = a.n;
    }
    const int32_t *qc = a.cand ? a.cand + q * a.cap : nullptr;
    int cnt = 0;
    float su = __int_as_float(0x7f800000);
    bool bad = false;
    // One candidate per lane: bound it, admit it into the warp's buffer, shrink
    // the buffer when full; false when the buffer cannot shrink (-> fallback).
    float *cu_w = cu + warp * BUFW;
    int32_t *cid_w = cid + warp * BUFW;
#define ADMIT_LANE(MYC, MYS, SX, NRM, RAD) \
  admit_lane_u8<BUFW, CPI>((MYC), (MYS), (SX), (NRM), (RAD), sqf, t2f, rq, su, cnt, ma, mr, me, mi, kk, cu_w, cid_w, \
                           &s_su_cta)
    {
    for (int64_t g = (int64_t)warp * CPI; g < m; g += (int64_t)NWARP * CPI) {
      int mys = 0;
      int32_t myc = -1;
      int32_t cidv[U];
      const uint8_t *rp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = g + u * R + grp;
        cidv[u] = j < m ? (qc ? __ldg(qc + j) : (int32_t)j) : -1;
        rp[u] = rows.X + (int64_t)(cidv[u] < 0 ? 0 : cidv[u]) * ldq;
      }
      int acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = 0;
      if (qsigned)
        dot_rows_u8<U, G, true>(rp, qb, gl, nchunk, acc);
      else
        dot_rows_u8<U, G, false>(rp, qb, gl, nchunk, acc);
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
      }
      // group leader of row group grp holds candidates u*R + grp; hand candidate
      // (lane) = u*R + grp' to lane (u*R + grp') for the buffer decision
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = __shfl_sync(0xffffffffu, acc[u], ((lane - u * R) & (R - 1)) * G);
        const int32_t c2 = __shfl_sync(0xffffffffu, cidv[u], ((lane - u * R) & (R - 1)) * G);
        if (lane >= u * R && lane < (u + 1) * R) {
          mys = v;
          myc = c2;
        }
      }
      float sx = 0.f, rad = 0.f;
      int nrm = 0;
      if (lane >= CPI) myc = -1;
      if (myc >= 0) {
        sx = __ldg(rows.scale + myc);
        nrm = __ldg(rows.norm + myc);
        rad = __ldg(rows.radius + myc);
      }
      if (!ADMIT_LANE(myc, mys, sx, nrm, rad)) {
        bad = true;
        cnt = 0;
        break;
      }
    }
    }
    __syncwarp();
    if (lane == 0) {
      s_wcnt[warp] = cnt;
      if (bad) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) {
      if (tid == 0) {
        fb_list[atomicAdd(fb_count, 1)] = (int32_t)q;
        if (a.surv) a.nsurv[q] = -1;
      }
      __syncthreads();
      continue;
    }
    int off = 0, total = 0;
    for (int w = 0; w < NWARP; ++w) {
      off += w < warp ? s_wcnt[w] : 0;
      total += s_wcnt[w];
    }
    for (int i = lane; i < cnt; i += 32) {
      double L, Uu;
      dist_bounds2(ma[i], mr[i], me[i], L, Uu);
      cu[off + i] = __double2float_ru(Uu);
      cl[off + i] = __double2float_rd(L);
      cid[off + i] = mi[i];
    }
    __syncthreads();
    int np2 = 32;
    while (np2 < total) np2 <<= 1;
    float *su2 = wa;
    int32_t *sx = wid;
    for (int i = tid; i < np2; i += kScanNT) {
      su2[i] = i < total ? cu[i] : __int_as_float(0x7f800000);
      sx[i] = i;
    }
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = tid; i < np2 / 2; i += kScanNT) {
          const int lo = 2 * i - (i & (stride - 1));
          const int hi = lo + stride;
          const bool asc = (lo & size) == 0;
          const float ka = su2[lo], kb = su2[hi];
          const int ia = sx[lo], ib = sx[hi];
          if (fpair_less(kb, ib, ka, ia) == asc) {
            su2[lo] = kb;
            su2[hi] = ka;
            sx[lo] = ib;
            sx[hi] = ia;
          }
        }
        __syncthreads();
      }
    }
    const double uk = total >= kk ? (double)su2[kk - 1] : __longlong_as_double(0x7ff0000000000000LL);
    if (tid == 0) s_ns = 0;
    __syncthreads();
    for (int i = tid; i < total; i += kScanNT) {
      if ((double)cl[i] <= uk) sx[atomicAdd(&s_ns, 1)] = cid[i];
    }
    __syncthreads();
    const int ns = s_ns;
    if (a.surv) {
      // hand the survivors to k_rerank (many queries' exact distances in
      // flight at once) unless there are too many
      if (ns <= kSurvCap) {
        for (int i = tid; i < ns; i += kScanNT) a.surv[q * kSurvCap + i] = sx[i];
        if (tid == 0) a.nsurv[q] = ns;
        __syncthreads();
        continue;
      }
      if (tid == 0) a.nsurv[q] = -1;
    }
    int np3 = 1;
    while (np3 < ns) np3 <<= 1;
    for (int i = tid; i < np3; i += kScanNT) {
      if (i < ns) {
        const int32_t id = sx[i];
        const float *xr = a.X + (int64_t)id * a.ldx;
        const double e = exact_dist2(xr, qrow, d, a.vec4 && aligned16_dev(qrow));
        ckey[i] = (unsigned long long)__double_as_longlong(e);
        cid[i] = id;
      } else {
        ckey[i] = ~0ull;
        cid[i] = 0x7fffffff;
      }
    }
    __syncthreads();
    for (int size = 2; size <= np3; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = tid; i < np3 / 2; i += kScanNT) {
          const int lo = 2 * i - (i & (stride - 1));
          const int hi = lo + stride;
          const bool asc = (lo & size) == 0;
          const unsigned long long ka = ckey[lo], kb = ckey[hi];
          const int ia = cid[lo], ib = cid[hi];
          if (pair_less(kb, ib, ka, ia) == asc) {
            ckey[lo] = kb;
            ckey[hi] = ka;
            cid[lo] = ib;
            cid[hi] = ia;
          }
        }
        __syncthreads();
      }
    }
    const int kept = ns < kk ? ns : kk;
    for (int i = tid; i < kk; i += kScanNT) {
      if (i < kept) {
        a.ids[q * a.kstride + i] = cid[i];
        a.dists[q * a.kstride + i] = sqrt(__longlong_as_double((long long)ckey[i]));
      } else {
        a.ids[q * a.kstride + i] = -1;
        a.dists[q * a.kstride + i] = __longlong_as_double(0x7ff0000000000000LL);
      }
    }
    __syncthreads();
  }
}

// exact_dist2 with the query in shared memory and 16 float4 row loads (64
// coordinates) in flight ahead of each run of additions; same terms in the
// same order.
__device__ __forceinline__ double exact_dist2_sq(const float *__restrict__ xr, const float *qs, int d,
                                                 bool vec4) {
  double e = 0.0;
  int c = 0;
  if (vec4) {
    for (; c + 64 <= d; c += 64) {
      float4 xv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) xv[u] = __ldg(reinterpret_cast<const float4 *>(xr + c) + u);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float4 qv = *reinterpret_cast<const float4 *>(qs + c + 4 * u);
        double t;
        t = (double)xv[u].x - (double)qv.x;
        e = __dadd_rn(e, __dmul_rn(t, t));
        t = (double)xv[u].y - (double)qv.y;
        e = __dadd_rn(e, __dmul_rn(t, t));
        t = (double)xv[u].z - (double)qv.z;
        e = __dadd_rn(e, __dmul_rn(t, t));
        t = (double)xv[u].w - (double)qv.w;
        e = __dadd_rn(e, __dmul_rn(t, t));
      }
    }
    for (; c + 4 <= d; c += 4) {
      const float4 xv = __ldg(reinterpret_cast<const float4 *>(xr + c));
      const float4 qv = *reinterpret_cast<const float4 *>(qs + c);
      double t;
      t = (double)xv.x - (double)qv.x;
      e = __dadd_rn(e, __dmul_rn(t, t));
      t = (double)xv.y - (double)qv.y;
      e = __dadd_rn(e, __dmul_rn(t, t));
      t = (double)xv.z - (double)qv.z;
      e = __dadd_rn(e, __dmul_rn(t, t));
      t = (double)xv.w - (double)qv.w;
      e = __dadd_rn(e, __dmul_rn(t, t));
    }
  }
  for (; c < d; ++c) {
    const double t = (double)__ldg(xr + c) - (double)qs[c];
    e = __dadd_rn(e, __dmul_rn(t, t));
  }
  return e;
}

constexpr int kRerankSmemD = 2048;  // query staged in shared memory up to this width

// Exact re-rank of the survivors the u8 filter handed over (a.surv /
// a.nsurv): one warp per query, one lane per survivor (two when > 32), each
// lane summing its row's float64 distance in coordinate order
// (exact_dist2); the (distance, id) order is a rank count over the warp.
// Many queries' rows are in flight at once, instead of a few threads per
// filter CTA waiting out one row each.
__global__ void __launch_bounds__(256) k_rerank(TopkArgs a) {
  extern __shared__ float rr_smem[];
  const int lane = threadIdx.x & 31;
  const bool staged = a.d <= kRerankSmemD;
  float *qs = rr_smem + (threadIdx.x >> 5) * ((a.d + 3) & ~3);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < a.nq; q += nw) {
    const int ns = a.nsurv[q];
    if (ns < 0) continue;
    const float *qrow = a.Q + q * a.ldq;
    if (staged) {
      __syncwarp();
      for (int c = lane; c < a.d; c += 32) qs[c] = __ldg(qrow + c);
      __syncwarp();
    }
    const bool v4 = a.vec4 && aligned16_dev(qrow);
    unsigned long long k0 = ~0ull, k1 = ~0ull;
    int i0 = 0x7fffffff, i1 = 0x7fffffff;
    if (lane < ns) {
      i0 = a.surv[q * kSurvCap + lane];
      const float *xr = a.X + (int64_t)i0 * a.ldx;
      k0 = (unsigned long long)__double_as_longlong(staged ? exact_dist2_sq(xr, qs, a.d, a.vec4)
                                                           : exact_dist2(xr, qrow, a.d, v4));
    }
    if (lane + 32 < ns) {
      i1 = a.surv[q * kSurvCap + 32 + lane];
      const float *xr = a.X + (int64_t)i1 * a.ldx;
      k1 = (unsigned long long)__double_as_longlong(staged ? exact_dist2_sq(xr, qs, a.d, a.vec4)
                                                           : exact_dist2(xr, qrow, a.d, v4));
    }
    int r0 = 0, r1 = 0;
    for (int j = 0; j < 32; ++j) {
      const unsigned long long kj = __shfl_sync(0xffffffffu, k0, j);
      const int ij = __shfl_sync(0xffffffffu, i0, j);
      r0 += pair_less(kj, ij, k0, i0) ? 1 : 0;
      r1 += pair_less(kj, ij, k1, i1) ? 1 : 0;
    }
    if (ns > 32) {
      for (int j = 0; j < 32; ++j) {
        const unsigned long long kj = __shfl_sync(0xffffffffu, k1, j);
        const int ij = __shfl_sync(0xffffffffu, i1, j);
        r0 += pair_less(kj, ij, k0, i0) ? 1 : 0;
        r1 += pair_less(kj, ij, k1, i1) ? 1 : 0;
      }
    }
    int64_t *oid = a.ids + q * a.kstride;
    double *od = a.dists + q * a.kstride;
    if (lane < ns && r0 < a.k) {
      oid[r0] = i0;
      od[r0] = sqrt(__longlong_as_double((long long)k0));
    }
    if (lane + 32 < ns && r1 < a.k) {
      oid[r1] = i1;
      od[r1] = sqrt(__longlong_as_double((long long)k1));
    }
    for (int i = ns + lane; i < a.k; i += 32) {
      oid[i] = -1;
      od[i] = __longlong_as_double(0x7ff0000000000000LL);
    }
  }
}


// GEMM operand of each query: the filter's own quantisation (u8 or s8),
// stored as s8 (u8 entries shifted by -128, i.e. byte ^ 0x80), and its
// parameters.  One CTA per query.
__global__ void __launch_bounds__(kScanNT) k_quantize_q8(const float *__restrict__ Q, int64_t ldqq, int d,
                                                         int ldq, int64_t nq, int8_t *__restrict__ qop,
                                                         QParams *__restrict__ qp) {
  __shared__ uint32_t qb[256];
  __shared__ QScratch<kScanNT / 32> qscr;
  for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
    const QParams P = quantize_query_u8<kScanNT>(Q + q * ldqq, d, ldq, qb, qscr);
    const uint32_t flip = P.qsigned ? 0u : 0x80808080u;
    uint32_t *dst = reinterpret_cast<uint32_t *>(qop + q * (int64_t)ldq);
    for (int w = threadIdx.x; w < ldq / 4; w += kScanNT) dst[w] = qb[w] ^ flip;
    if (threadIdx.x == 0) qp[q] = P;
    __syncthreads();  // qb is rewritten by the next query
  }
}

// s8 copy of the u8 filter rows (byte ^ 0x80) -- the GEMM's row operand --
// and one 16-byte record per row for the filter: {scale, norm, radius, sum of
// the u8 entries (the GEMM's offset correction)}.  One warp per row.
__global__ void k_u8_gemm_rows(const uint8_t *__restrict__ Xq, int64_t n, int ldq, const float *__restrict__ scale,
                               const int32_t *__restrict__ norm, const float *__restrict__ radius,
                               int8_t *__restrict__ Xs, uint4 *__restrict__ info) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += wstride) {
    const uint32_t *src = reinterpret_cast<const uint32_t *>(Xq + r * ldq);
    uint32_t *dst = reinterpret_cast<uint32_t *>(Xs + r * ldq);
    int sum = 0;
    for (int w = lane; w < ldq / 4; w += 32) {
      const uint32_t v = src[w];
      dst[w] = v ^ 0x80808080u;
      sum += (int)(v & 0xffu) + (int)((v >> 8) & 0xffu) + (int)((v >> 16) & 0xffu) + (int)(v >> 24);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0)
      info[r] = make_uint4(__float_as_uint(scale[r]), (uint32_t)norm[r], __float_as_uint(radius[r]), (uint32_t)sum);
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

#include "tc_filter.cuh"

using namespace mrpt;

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Queries handed to each filter route (same slots as g_fallbacks).
static std::atomic<long long> g_route_queries[8];

extern "C" int32_t mrpt_fallback_stats(int64_t *out, int32_t reset) {
  clear_error();
  if (!out) return fail(MRPT_EPARAM, "mrpt_fallback_stats: out is NULL");
  unsigned long long fb[8] = {0};
  if (cudaMemcpyFromSymbol(fb, g_fallbacks, sizeof(fb)) != cudaSuccess)
    return launch_status("mrpt_fallback_stats");
  for (int r = 0; r < 4; ++r) {
    out[2 * r] = g_route_queries[r + 1].load();
    out[2 * r + 1] = (int64_t)fb[r + 1];
  }
  if (reset) {
    const unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_fallbacks, z, sizeof(z));
    for (auto &c : g_route_queries) c.store(0);
  }
  return launch_status("mrpt_fallback_stats");
}

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
  (count_launch(), k_scan<<<grid, kScanNT, smem, s>>>(X, ldx, d, cand, m, q, out, vec4));
  return launch_status("mrpt_scan");
}

typedef void (*topk_fn)(TopkArgs);
typedef void (*topk_fn_f)(TopkArgs, double, double, int32_t *, int32_t *);

template <int FU, int MINB>
static topk_fn_f pick_filter_b(int bufw) {
  return bufw == 64 ? k_scan_topk_filter<64, FU, MINB>
                    : (bufw == 128 ? k_scan_topk_filter<128, FU, MINB> : k_scan_topk_filter<256, FU, MINB>);
}

static topk_fn_f pick_filter(int bufw, int fu, int minb) {
  if (fu == 8) return minb >= 3 ? pick_filter_b<8, 3>(bufw) : pick_filter_b<8, 2>(bufw);
  if (fu == 2) return pick_filter_b<2, 4>(bufw);
  if (minb >= 5) return pick_filter_b<4, 5>(bufw);
  if (minb == 3) return pick_filter_b<4, 3>(bufw);
  return pick_filter_b<4, 4>(bufw);
}

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
  TopkArgs a = {};
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
    keep_pool_warm();
  if (cudaMallocAsync((void **)&a.lb_key, sizeof(unsigned long long) * nq, s) != cudaSuccess ||
        cudaMallocAsync((void **)&a.lb_id, sizeof(int32_t) * nq, s) != cudaSuccess)
      return fail(MRPT_ECUDA, "mrpt_scan_topk: scratch allocation failed");
    // lower bound below every key: (0, -1)
    cudaMemsetAsync(a.lb_key, 0, sizeof(unsigned long long) * nq, s);
    cudaMemsetAsync(a.lb_id, 0xff, sizeof(int32_t) * nq, s);
  }
  const int64_t grid = nq < (int64_t)num_sms() * 8 ? nq : (int64_t)num_sms() * 8;
  a.qlist = nullptr;
  a.qcount = nullptr;
  const bool qvec4 = (ldq % 4 == 0) && aligned16(Q);
  if (a.vec4 && qvec4 && d <= 128 * kFMaxJ && k <= 120) {
    // filter (float32) + exact float64 rerank; exact-tie overflows go to the
    // tiled exact kernel through a device-side query list.
    const int bufw = (2 * k + 16 <= 64) ? 64 : ((2 * k + 16 <= 128) ? 128 : 256);
    const size_t smem = sizeof(float) * 128 * kFMaxJ + (size_t)(kScanNT / 32) * bufw * (4 + 4 + 8 + 4 + 4);
    int32_t *fb = nullptr;
    keep_pool_warm();
  if (cudaMallocAsync((void **)&fb, sizeof(int32_t) * (nq + 1), s) != cudaSuccess)
      return fail(MRPT_ECUDA, "mrpt_scan_topk: scratch allocation failed");
    cudaMemsetAsync(fb, 0, sizeof(int32_t), s);
    const double u = 5.9604644775390625e-08;  // 2^-24
    const double eps = 2.0 * (d + 16) * u;
    const double eta = 2.0 * (d + 16) * 1.401298464324817e-45;  // subnormal float spacing
    const char *var = getenv("MRPT_SCAN_VARIANT");  // experiments: "FU,MINB"
    int fu = 4, minb = 4;
    if (var) sscanf(var, "%d,%d", &fu, &minb);
    topk_fn_f ffn = pick_filter(bufw, fu, minb);
    cudaFuncSetAttribute(ffn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    a.k = k;
    a.ids = ids;
    a.dists = dists;
    (count_launch(), ffn<<<(unsigned)grid, kScanNT, smem, s>>>(a, eps, eta, fb + 1, fb));
    // fallback: exact tiled kernel over the listed queries
    a.qlist = fb + 1;
    a.stat_slot = 1;  // fallback statistics: see mrpt_fallback_stats
    g_route_queries[1] += nq;
    a.qcount = fb;
    const int buf = (k + kScanNT <= 1024) ? 1024 : 2048;
    topk_fn tfn = buf == 1024 ? k_scan_topk_tiled<1024> : k_scan_topk_tiled<2048>;
    const size_t tsmem = (size_t)buf * 12 + sizeof(float) * (kScanNT / 32) * 32 * kTileStride +
                         sizeof(double) * (size_t)d;
    cudaFuncSetAttribute(tfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
    (count_launch(), tfn<<<(unsigned)(grid < 64 ? grid : 64), kScanNT, tsmem, s>>>(a));
    cudaFreeAsync(fb, s);
    return launch_status("mrpt_scan_topk");
  }
  for (int p = 0; p < passes; ++p) {
    const int off = p * chunk_max;
    const int kk = (k - off) < chunk_max ? (k - off) : chunk_max;
    a.k = kk;
    a.ids = ids + off;
    a.dists = dists + off;
    topk_fn fn;
    int buf;
    size_t extra = 0;
    if (a.vec4) {
      // tiled kernel: one 256-candidate round between threshold updates
      buf = (kk + kScanNT <= 1024) ? 1024 : ((kk + kScanNT <= 2048) ? 2048 : 4096);
      fn = buf == 1024 ? k_scan_topk_tiled<1024>
                       : (buf == 2048 ? k_scan_topk_tiled<2048> : k_scan_topk_tiled<4096>);
      extra = sizeof(float) * (kScanNT / 32) * 32 * kTileStride;
    } else if (kk + kScanNT * kScanR <= 2048) {
      fn = k_scan_topk<2048>;
      buf = 2048;
    } else {
      fn = k_scan_topk<4096>;
      buf = 4096;
    }
    const size_t smem = (size_t)buf * 12 + extra + sizeof(double) * (size_t)d;
    if (smem > 220 * 1024) return fail(MRPT_EPARAM, "mrpt_scan_topk: d too large");
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    (count_launch(), fn<<<(unsigned)grid, kScanNT, smem, s>>>(a));
  }
  if (passes > 1) {
    cudaFreeAsync(a.lb_key, s);
    cudaFreeAsync(a.lb_id, s);
  }
  return launch_status("mrpt_scan_topk");
}

extern "C" int32_t mrpt_quantize_fp16(const float *X, int64_t n, int32_t d, int64_t ldx, void *Xh,
                                      int64_t ldh, float *radius, int32_t *bad, void *stream) {
  clear_error();
  if (n < 1 || d < 1 || ldx < d || ldh < d || ldh % 8 != 0)
    return fail(MRPT_ESHAPE, "mrpt_quantize_fp16: bad shape");
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(bad, 0, sizeof(int32_t), s);
  const int64_t blocks = ceil_div<int64_t>(n, 8);
  const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  (count_launch(), k_quantize_fp16<<<grid, 256, 0, s>>>(X, n, d, ldx, reinterpret_cast<__half *>(Xh), ldh, radius, bad));
  return launch_status("mrpt_quantize_fp16");
}

extern "C" int32_t mrpt_scan_topk_fp16(const float *X, int64_t n, int32_t d, int64_t ldx,
                                       const void *Xh, int64_t ldh, const float *radius,
                                       const float *Q, int64_t nq, int64_t ldq, const int32_t *cand,
                                       int64_t cap, const int32_t *ncand, int32_t k, int64_t *ids,
                                       double *dists, void *stream) {
  clear_error();
  if (!Xh || !radius || ldh % 8 != 0 || ldh < d || ldh > 1024 || k > 120 || k < 1 ||
      (ldq % 4) != 0 || !aligned16(Q) || d % 4 != 0 || ldx % 4 != 0 || !aligned16(X))
    return mrpt_scan_topk(X, n, d, ldx, Q, nq, ldq, cand, cap, ncand, k, ids, dists, stream);
  if (n < 1 || n >= (int64_t)1 << 31 || d < 1 || ldx < d || ldq < d || nq < 0)
    return fail(MRPT_ESHAPE, "mrpt_scan_topk_fp16: bad shape");
  if (cand && (cap < 1 || !ncand)) return fail(MRPT_EPARAM, "mrpt_scan_topk_fp16: bad candidate lists");
  if (nq == 0) return MRPT_OK;
  cudaStream_t s = as_stream(stream);
  TopkArgs a = {};
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
  a.k = k;
  a.kstride = k;
  a.ids = ids;
  a.dists = dists;
  a.lb_key = nullptr;
  a.lb_id = nullptr;
  a.vec4 = (d % 4 == 0) && (ldx % 4 == 0) && aligned16(X);
  a.qlist = nullptr;
  a.qcount = nullptr;
  a.Xh = reinterpret_cast<const __half *>(Xh);
  a.ldh = ldh;
  a.radius = radius;
  const int bufw = (2 * k + 16 <= 64) ? 64 : ((2 * k + 16 <= 128) ? 128 : 256);
  const size_t smem = sizeof(float) * 256 * 4 + (size_t)(kScanNT / 32) * bufw * (4 + 4 + 4 + 4 + 4 + 4);
  int32_t *fb = nullptr;
  keep_pool_warm();
  if (cudaMallocAsync((void **)&fb, sizeof(int32_t) * (nq + 1), s) != cudaSuccess)
    return fail(MRPT_ECUDA, "mrpt_scan_topk_fp16: scratch allocation failed");
  cudaMemsetAsync(fb, 0, sizeof(int32_t), s);
  const double u = 5.9604644775390625e-08;  // 2^-24
  const double eps = 2.0 * (ldh + 16) * u;
  const double eta = 2.0 * (ldh + 16) * 1.401298464324817e-45;
  topk_fn_f ffn = bufw == 64 ? k_scan_topk_filter_h<64>
                             : (bufw == 128 ? k_scan_topk_filter_h<128> : k_scan_topk_filter_h<256>);
  cudaFuncSetAttribute(ffn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t grid = nq < (int64_t)num_sms() * 8 ? nq : (int64_t)num_sms() * 8;
  (count_launch(), ffn<<<(unsigned)grid, kScanNT, smem, s>>>(a, eps, eta, fb + 1, fb));
  // fallback: exact tiled kernel over the listed queries
  a.qlist = fb + 1;
  a.stat_slot = 2;  // fallback statistics: see mrpt_fallback_stats
  g_route_queries[2] += nq;
  a.qcount = fb;
  if (a.vec4) {
    const int buf = (k + kScanNT <= 1024) ? 1024 : 2048;
    topk_fn tfn = buf == 1024 ? k_scan_topk_tiled<1024> : k_scan_topk_tiled<2048>;
    const size_t tsmem = (size_t)buf * 12 + sizeof(float) * (kScanNT / 32) * 32 * kTileStride +
                         sizeof(double) * (size_t)d;
    cudaFuncSetAttribute(tfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
    (count_launch(), tfn<<<(unsigned)(grid < 64 ? grid : 64), kScanNT, tsmem, s>>>(a));
  } else {
    return fail(MRPT_EPARAM, "mrpt_scan_topk_fp16: exact fallback needs 16-byte rows");
  }
  cudaFreeAsync(fb, s);
  return launch_status("mrpt_scan_topk_fp16");
}

extern "C" int32_t mrpt_quantize_u8(const float *X, int64_t n, int32_t d, int64_t ldx, void *Xq,
                                    int64_t ldq, float *scale, int32_t *norm, float *radius,
                                    int32_t *flags, void *stream) {
  // flags (device, 2 int32): [0] = 1 if some x < 0 (the u8 shadow is then
  // unusable and left unwritten), [1] = 1 if not integer-valued in [0, 255]
  clear_error();
  if (n < 1 || d < 1 || ldx < d || ldq < d || ldq % 16 != 0 || ldq > 1024)
    return fail(MRPT_ESHAPE, "mrpt_quantize_u8: bad shape");
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(flags, 0, 2 * sizeof(int32_t), s);
  const int64_t total = n * d;
  const int64_t blocks = ceil_div<int64_t>(total, 256 * 8);
  const int g1 = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  (count_launch(), k_q8_flags<<<g1, 256, 0, s>>>(X, n, d, ldx, flags));
  int32_t hflags[2] = {0, 0};
  cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return launch_status("mrpt_quantize_u8");
  if (hflags[0]) return MRPT_OK;
  const int64_t wb = ceil_div<int64_t>(n, 8);
  const int g2 = (int)(wb < (int64_t)num_sms() * 16 ? wb : (int64_t)num_sms() * 16);
  (count_launch(), k_quantize_u8<<<g2, 256, 0, s>>>(X, n, d, ldx, reinterpret_cast<uint8_t *>(Xq), ldq, scale, norm,
                                   radius, hflags[1] ? 0 : 1));
  return launch_status("mrpt_quantize_u8");
}

typedef void (*topk_fn_u8)(TopkArgs, Q8Rows, int32_t *, int32_t *);

template <int G>
static topk_fn_u8 pick_u8_b(int bufw) {
  return bufw == 64 ? k_scan_topk_u8<64, G> : (bufw == 128 ? k_scan_topk_u8<128, G> : k_scan_topk_u8<256, G>);
}

static void launch_rerank(const TopkArgs &a, cudaStream_t s) {
  const int64_t blocks = ceil_div<int64_t>(a.nq, 8);
  const int64_t cap = (int64_t)num_sms() * 16;
  const size_t smem = a.d <= kRerankSmemD ? (size_t)8 * ((a.d + 3) & ~3) * sizeof(float) : 0;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_rerank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  (count_launch(), k_rerank<<<(unsigned)(blocks < cap ? blocks : cap), 256, smem, s>>>(a));
}

static int32_t scan_u8_impl(const float *X, int64_t n, int32_t d, int64_t ldx, const void *Xq, int64_t ldq,
                            const float *scale, const int32_t *norm, const float *radius, const float *Q,
                            int64_t nq, int64_t ldqq, const int32_t *cand, int64_t cap, const int32_t *ncand,
                            int32_t k, int64_t *ids, double *dists, void *stream) {
  if (!Xq || !scale || !norm || !radius || ldq % 16 != 0 || ldq < d || ldq > 1024 || k > 120 || k < 1 ||
      d % 4 != 0 || ldx % 4 != 0 || !aligned16(X))  // the exact fallback needs 16-byte rows
    return mrpt_scan_topk(X, n, d, ldx, Q, nq, ldqq, cand, cap, ncand, k, ids, dists, stream);
  if (n < 1 || n >= (int64_t)1 << 31 || d < 1 || ldx < d || ldqq < d || nq < 0)
    return fail(MRPT_ESHAPE, "mrpt_scan_topk_u8: bad shape");
  if (cand && (cap < 1 || !ncand)) return fail(MRPT_EPARAM, "mrpt_scan_topk_u8: bad candidate lists");
  if (nq == 0) return MRPT_OK;
  cudaStream_t s = as_stream(stream);
  TopkArgs a = {};
  a.X = X;
  a.n = n;
  a.d = d;
  a.ldx = ldx;
  a.Q = Q;
  a.nq = nq;
  a.ldq = ldqq;
  a.cand = cand;
  a.cap = cap;
  a.ncand = ncand;
  a.k = k;
  a.kstride = k;
  a.ids = ids;
  a.dists = dists;
  a.lb_key = nullptr;
  a.lb_id = nullptr;
  a.vec4 = (d % 4 == 0) && (ldx % 4 == 0) && aligned16(X);
  a.qlist = nullptr;
  a.qcount = nullptr;
  a.Xh = nullptr;
  a.ldh = 0;
  a.radius = nullptr;
  a.surv = nullptr;
  a.nsurv = nullptr;
  Q8Rows rows;
  rows.X = reinterpret_cast<const uint8_t *>(Xq);
  rows.ldq = ldq;
  rows.scale = scale;
  rows.norm = norm;
  rows.radius = radius;
  // G lanes per row: 8 for wide rows (16 candidates per warp iteration, several
  // chunk loads in flight per lane); 4 for rows of <= 256 bytes (two or more
  // chunks per lane, 32 candidates per iteration, one shuffle level less).
  // MRPT_U8_G overrides (4, 8, 16, 32).
  static int g_env = -1;
  if (g_env < 0) {
    const char *e = getenv("MRPT_U8_G");
    g_env = e ? atoi(e) : 0;
  }
  int G = (g_env == 4 || g_env == 8 || g_env == 16 || g_env == 32) ? g_env : (ldq <= 256 ? 4 : 8);
  const int cpi = (32 / G) * 4;
  int bufw = 64;
  while (bufw < 2 * k + 2 * cpi) bufw <<= 1;
  if (bufw > 256) return mrpt_scan_topk(X, n, d, ldx, Q, nq, ldqq, cand, cap, ncand, k, ids, dists, stream);
  const size_t smem = 1024 + (size_t)(kScanNT / 32) * bufw * (4 * 4 + 8 + 4 * 3);
  int32_t *fb = nullptr;
  keep_pool_warm();
  // scratch: fallback count + list, survivor counts, survivor lists
  if (cudaMallocAsync((void **)&fb, sizeof(int32_t) * ((nq + 1) + nq * (kSurvCap + 1)), s) != cudaSuccess)
    return fail(MRPT_ECUDA, "mrpt_scan_topk_u8: scratch allocation failed");
  cudaMemsetAsync(fb, 0, sizeof(int32_t), s);
  a.nsurv = fb + 1 + nq;
  a.surv = a.nsurv + nq;
  topk_fn_u8 fn = G == 32 ? pick_u8_b<32>(bufw)
                          : (G == 16 ? pick_u8_b<16>(bufw) : (G == 8 ? pick_u8_b<8>(bufw) : pick_u8_b<4>(bufw)));
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t grid = nq < (int64_t)num_sms() * 8 ? nq : (int64_t)num_sms() * 8;
  (count_launch(), fn<<<(unsigned)grid, kScanNT, smem, s>>>(a, rows, fb + 1, fb));
  a.qlist = fb + 1;
  a.stat_slot = 3;  // fallback statistics: see mrpt_fallback_stats
  g_route_queries[3] += nq;
  a.qcount = fb;
  if (a.vec4) {
    const int buf = (k + kScanNT <= 1024) ? 1024 : 2048;
    topk_fn tfn = buf == 1024 ? k_scan_topk_tiled<1024> : k_scan_topk_tiled<2048>;
    const size_t tsmem = (size_t)buf * 12 + sizeof(float) * (kScanNT / 32) * 32 * kTileStride +
                         sizeof(double) * (size_t)d;
    cudaFuncSetAttribute(tfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
    (count_launch(), tfn<<<(unsigned)(grid < 64 ? grid : 64), kScanNT, tsmem, s>>>(a));
  } else {
    cudaFreeAsync(fb, s);
    return fail(MRPT_EPARAM, "mrpt_scan_topk_u8: exact fallback needs 16-byte rows");
  }
  launch_rerank(a, s);
  cudaFreeAsync(fb, s);
  return launch_status("mrpt_scan_topk_u8");
}

extern "C" int32_t mrpt_scan_topk_u8(const float *X, int64_t n, int32_t d, int64_t ldx,
                                     const void *Xq, int64_t ldq, const float *scale,
                                     const int32_t *norm, const float *radius, const float *Q,
                                     int64_t nq, int64_t ldqq, const int32_t *cand, int64_t cap,
                                     const int32_t *ncand, int32_t k, int64_t *ids, double *dists,
                                     void *stream) {
  clear_error();
  return scan_u8_impl(X, n, d, ldx, Xq, ldq, scale, norm, radius, Q, nq, ldqq, cand, cap, ncand, k, ids, dists,
                      stream);
}

extern "C" int32_t mrpt_u8_gemm_rows(const void *Xq, int64_t n, int64_t ldq, const float *scale,
                                     const int32_t *norm, const float *radius, void *Xs, void *info,
                                     void *stream) {
  // Xs holds round_up(n, 16) rows: the GEMM runs over whole 16-row groups
  // (cuBLASLt's int8 kernels want the row count a multiple of 4); pad rows are 0
  const int64_t n16 = (n + 15) & ~(int64_t)15;
  if (Xs && n16 > n)
    cudaMemsetAsync(reinterpret_cast<int8_t *>(Xs) + n * ldq, 0, (size_t)((n16 - n) * ldq), as_stream(stream));
  clear_error();
  if (!Xq || !Xs || !info || !scale || !norm || !radius || n < 1 || ldq < 16 || ldq % 16 != 0 || ldq > 1024)
    return fail(MRPT_ESHAPE, "mrpt_u8_gemm_rows: bad shape");
  if (reinterpret_cast<uintptr_t>(info) & 15u) return fail(MRPT_EPARAM, "mrpt_u8_gemm_rows: info must be 16-byte aligned");
  const int64_t blocks = ceil_div<int64_t>(n, 8);
  const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  (count_launch(), k_u8_gemm_rows<<<grid, 256, 0, as_stream(stream)>>>(reinterpret_cast<const uint8_t *>(Xq), n, (int)ldq,
                                                       scale, norm, radius, reinterpret_cast<int8_t *>(Xs),
                                                       reinterpret_cast<uint4 *>(info)));
  return launch_status("mrpt_u8_gemm_rows");
}

// ------------------------------------------------------------ K4 tc route --
// The u8 filter fused onto tcgen05 (tc_filter.cuh): no dot-product matrix in
// HBM.  Workspace per query chunk of mc queries: quantised queries, their
// parameters, the row records, per-query entry lists and counts, and the
// survivor / fallback lists the re-rank and the exact fallback read.
static const int kTcCap = tc::kSelCap;
static const int kTcKb = tc::kKbSort;  // per query: the CTAs' k smallest bounds

static int64_t u8tc_bytes(int64_t n, int64_t ldq, int64_t mc, int64_t *off) {
  auto al = [](int64_t x) { return (x + 1023) & ~(int64_t)1023; };
  int64_t o = 0;
  off[0] = o;  // qop (mc x ldq s8)
  o = al(o + mc * ldq);
  off[1] = o;  // qp
  o = al(o + mc * (int64_t)sizeof(QParams));
  off[2] = o;  // rinfo (n x 16 B)
  o = al(o + n * 16);
  off[6] = o;  // row t1 terms (n floats, 16-B padded)
  o = al(o + n * 4 + 16);
  off[3] = o;  // entries (mc x cap x 16 B)
  o = al(o + mc * kTcCap * 16);
  off[4] = o;  // entry counts (mc), shared k-th bounds (mc), bound counts (mc), bounds (mc x kTcKb)
  o = al(o + mc * 12 + mc * kTcKb * 4);
  off[5] = o;  // fallback count + list, survivor counts, survivor lists
  return al(o + ((mc + 1) + mc * (kSurvCap + 1)) * 4) + 1024;  // + base alignment
}

static const int64_t kTcChunk = 16384;  // queries per chunk (entry lists: 8 KB per query)

extern "C" int32_t mrpt_scan_topk_u8tc_workspace_size(int64_t n, int64_t ldq, int64_t nq, int64_t *bytes) {
  clear_error();
  if (n < 1 || ldq < 16 || nq < 0 || !bytes) return fail(MRPT_ESHAPE, "mrpt_scan_topk_u8tc_workspace_size");
  int64_t mc = nq < kTcChunk ? nq : kTcChunk;
  if (mc < 1) mc = 1;
  int64_t off[7];
  *bytes = u8tc_bytes(n, ldq, mc, off);
  return MRPT_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    tried = true;
  }
  return fn;
}

// 2-D u8 tensor map (rows x ldq bytes), boxes of 128 bytes x box_rows rows,
// 128-B swizzle (the UMMA K-major canonical layout); reads past the edges
// fill zeros.
static bool tc_map(CUtensorMap *m, const void *base, int64_t rows, int64_t ldq, int box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 fn = tc_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)ldq, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ldq};
  cuuint32_t box[2] = {(cuuint32_t)tc::kKB, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D u32 tensor map of the candidate bitmaps (rows x bstride words), boxes
// of one row tile's 8 words x 128 queries, no swizzle.
static bool tc_map_words(CUtensorMap *m, const void *base, int64_t rows, int64_t bstride) {
  PFN_cuTensorMapEncodeTiled_v12000 fn = tc_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)bstride, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)bstride * 4};
  cuuint32_t box[2] = {(cuuint32_t)(tc::kN / 32), (cuuint32_t)tc::kM};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

extern "C" int32_t mrpt_scan_topk_u8tc_bits(const float *X, int64_t n, int32_t d, int64_t ldx, const void *Xs,
                                            int64_t ldq, const void *info, const float *Q, int64_t nq,
                                            int64_t ldqq, const uint32_t *cbits, int64_t bstride, int32_t k,
                                            int64_t *ids, double *dists, void *workspace, int64_t ws_bytes,
                                            void *wait_event, void *stream) {
  clear_error();
  if (!cbits || bstride < (n + 31) / 32 || bstride % 4 != 0 || !aligned16(cbits))
    return fail(MRPT_EPARAM, "mrpt_scan_topk_u8tc_bits: bad candidate bitmaps (bstride a multiple of 4 words, "
                             "16-byte aligned)");
  if (!X || !Xs || !info || !Q || n < 1 || n >= (int64_t)1 << 31 || d < 1 || ldx < d || ldqq < d || nq < 0)
    return fail(MRPT_ESHAPE, "mrpt_scan_topk_u8tc_bits: bad shape");
  if (ldq % 16 != 0 || ldq < d || ldq < tc::kKB || ldq > tc::kMaxKB * tc::kKB || k < 1 || k > tc::kTopMax || d % 4 != 0 ||
      ldx % 4 != 0 || !aligned16(X) || !aligned16(Xs) || (reinterpret_cast<uintptr_t>(info) & 15u))
    return fail(MRPT_EPARAM, "mrpt_scan_topk_u8tc_bits: unsupported shape");
  if (nq == 0) return MRPT_OK;
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return fail(MRPT_EWORKSPACE, "mrpt_scan_topk_u8tc_bits: workspace must be 256-byte aligned");
  int64_t off[7];
  int64_t mc = nq < kTcChunk ? nq : kTcChunk;
  while (mc > 0 && u8tc_bytes(n, ldq, mc, off) > ws_bytes) mc = mc > 128 ? mc - 128 : mc - 1;
  if (mc < 1) return fail(MRPT_EWORKSPACE, "mrpt_scan_topk_u8tc_bits: workspace too small for one query");
  u8tc_bytes(n, ldq, mc, off);
  char *w = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(workspace) + 1023) & ~(uintptr_t)1023);
  int8_t *qop = reinterpret_cast<int8_t *>(w + off[0]);
  QParams *qp = reinterpret_cast<QParams *>(w + off[1]);
  uint4 *rinfo = reinterpret_cast<uint4 *>(w + off[2]);
  float *rt1 = reinterpret_cast<float *>(w + off[6]);
  uint4 *ent = reinterpret_cast<uint4 *>(w + off[3]);
  int32_t *ent_cnt = reinterpret_cast<int32_t *>(w + off[4]);
  int32_t *fb = reinterpret_cast<int32_t *>(w + off[5]);
  cudaStream_t s = as_stream(stream);
  CUtensorMap tmB;
  const int mcast = getenv("MRPT_TC_MC") ? (atoi(getenv("MRPT_TC_MC")) == 2 ? 2 : 1) : 2;
  // (a cluster pair loads half a row tile per CTA and multicasts it)
  if (!tc_map(&tmB, Xs, n, ldq, tc::kN / mcast)) return fail(MRPT_ECUDA, "mrpt_scan_topk_u8tc_bits: tensor map (rows)");
  {
    const int64_t g = ceil_div<int64_t>(n, 256);
    (count_launch(), tc::k_tc_rows<<<(unsigned)(g < 4096 ? g : 4096), 256, 0, s>>>(
                         reinterpret_cast<const uint4 *>(info), n, rinfo, rt1));
  }
  // kernel variant per chunk (below): CG column-group warps per query, MC
  // CTAs per cluster sharing the row tiles (multicast)
  typedef void (*tc_fn)(const CUtensorMap, const CUtensorMap, const CUtensorMap, tc::TcArgs);
  auto pick_tc = [&](int cg, int mc, int *threads) -> tc_fn {
    if (cg >= 4) {
      *threads = tc::threads_for<4>();
      return mc == 2 ? tc::k_tc_filter<16, 4, 2> : tc::k_tc_filter<16, 4, 1>;
    }
    if (cg == 2) {
      *threads = tc::threads_for<2>();
      return mc == 2 ? tc::k_tc_filter<16, 2, 2> : tc::k_tc_filter<16, 2, 1>;
    }
    *threads = tc::threads_for<1>();
    return mc == 2 ? tc::k_tc_filter<16, 1, 2> : tc::k_tc_filter<16, 1, 1>;
  };

  const int buf = (k + kScanNT <= 1024) ? 1024 : 2048;
  topk_fn tfn = buf == 1024 ? k_scan_topk_tiled<1024> : k_scan_topk_tiled<2048>;
  const size_t tsmem =
      (size_t)buf * 12 + sizeof(float) * (kScanNT / 32) * 32 * kTileStride + sizeof(double) * (size_t)d;
  cudaFuncSetAttribute(tfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
  const int ntiles = (int)ceil_div<int64_t>(n, tc::kN);
  for (int64_t q0 = 0; q0 < nq; q0 += mc) {
    const int64_t m = nq - q0 < mc ? nq - q0 : mc;
    const int64_t g1 = m < (int64_t)num_sms() * 8 ? m : (int64_t)num_sms() * 8;
    (count_launch(), k_quantize_q8<<<(unsigned)g1, kScanNT, 0, s>>>(Q + q0 * ldqq, ldqq, d, (int)ldq, m, qop, qp));
    CUtensorMap tmA, tmC;
    if (!tc_map(&tmA, qop, m, ldq, tc::kM)) return fail(MRPT_ECUDA, "mrpt_scan_topk_u8tc_bits: tensor map (queries)");
    if (!tc_map_words(&tmC, cbits + q0 * bstride, m, bstride))
      return fail(MRPT_ECUDA, "mrpt_scan_topk_u8tc_bits: tensor map (candidate bitmaps)");
    cudaMemsetAsync(ent_cnt, 0, (size_t)m * 4, s);
    cudaMemsetAsync(ent_cnt + mc, 0x7f, (size_t)m * 4, s);  // 3.4e38: no bound yet
    cudaMemsetAsync(ent_cnt + 2 * mc, 0, (size_t)m * 4, s);
    cudaMemsetAsync(fb, 0, sizeof(int32_t), s);
    if (wait_event && q0 == 0) cudaStreamWaitEvent(s, reinterpret_cast<cudaEvent_t>(wait_event), 0);
    tc::TcArgs ta;
    ta.n = n;
    ta.m = m;
    ta.ntiles = ntiles;
    ta.nqb = (int)ceil_div<int64_t>(m, tc::kM);
    ta.kblocks = (int)ceil_div<int64_t>(ldq, tc::kKB);
    ta.k = k;
    ta.ldq = (int)ldq;
    ta.rinfo = rinfo;
    ta.rt1 = rt1;
    ta.qp = qp;
    ta.cbits = cbits + q0 * bstride;
    ta.bstride = bstride;
    ta.ent = ent;
    ta.ent_cnt = ent_cnt;
    ta.cap = kTcCap;
    ta.su_g = reinterpret_cast<unsigned *>(ent_cnt + mc);
    ta.kb_cnt = ent_cnt + 2 * mc;
    ta.kb = reinterpret_cast<float *>(ent_cnt + 3 * mc);
    ta.kbcap = kTcKb;
    // Every CTA that touches a query runs its own warm-up of the query's
    // k-th bound (>= k admissions; the CTA's column-group warps share one):
    // few query blocks per CTA (small chunks) means many CTAs per query, so
    // at most 8 CTAs per query block (fewer CTAs for tiny chunks).
    // (units: query blocks, or query-block pairs for a cluster pair; groups:
    // CTAs, or clusters)
    const int64_t items = ceil_div<int64_t>(ta.nqb, mcast) * ntiles;
    const int64_t maxg = num_sms() / mcast;
    int groups = (int)(items < maxg ? items : maxg);
    auto cpq = [&](int g) { return (int)ceil_div<int64_t>((int64_t)ntiles * g, items) + 1; };
    int cg = 4;
    while (groups > 1 && cpq(groups) > 8) --groups;
    if (const char *cge = getenv("MRPT_TC_CG")) cg = atoi(cge);
    const int grid = groups * mcast;
    int fthreads = 0;
    const tc_fn fk = pick_tc(cg, mcast, &fthreads);
    cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::kSmemBytes);
    ta.dbgD = nullptr;
    ta.noepi = getenv("MRPT_TC_NOEPI") ? atoi(getenv("MRPT_TC_NOEPI")) : 0;
    const bool dbg = getenv("MRPT_TC_DEBUG") != nullptr;
    int32_t *D1 = nullptr, *D2 = nullptr;
    if (dbg) {
      cudaMalloc(&D1, (size_t)m * n * 4);
      cudaMalloc(&D2, (size_t)m * ((n + 15) & ~15) * 4 + 64);
      ta.dbgD = D1;
    }
    cudaEvent_t kt0;
    ktimer_begin(s, &kt0);
    if (mcast == 2) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)grid);
      cfg.blockDim = dim3((unsigned)fthreads);
      cfg.dynamicSmemBytes = tc::kSmemBytes;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      count_launch();
      cudaLaunchKernelEx(&cfg, fk, tmA, tmB, tmC, ta);
    } else {
      (count_launch(), fk<<<grid, fthreads, tc::kSmemBytes, s>>>(tmA, tmB, tmC, ta));
    }
    ktimer_end(s, kt0);
    if (dbg) {
      const int64_t ldD = (n + 15) & ~(int64_t)15;
      // naive int32 dot products of the same s8 operands (debug reference)
      tc::k_dot_ref<<<dim3((unsigned)((n + 255) / 256), (unsigned)m), 256, 0, s>>>(
          reinterpret_cast<const int8_t *>(Xs), n, qop, ldq, D2, ldD);
      const int32_t st = 0;
      unsigned long long *o = nullptr;
      cudaMalloc(&o, 24);
      cudaMemsetAsync(o, 0, 24, s);
      tc::k_tc_debug<<<1024, 256, 0, s>>>(D1, D2, n, ldD, ent_cnt, m, o);
      unsigned long long h[3];
      cudaMemcpyAsync(h, o, 24, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      int32_t fbc = 0;
      fprintf(stderr, "[tc debug] m=%lld n=%lld gemm_st=%d D mismatches=%llu entries total=%llu max=%llu (cap %d)\n",
              (long long)m, (long long)n, st, h[0], h[1], h[2], kTcCap);
      (void)fbc;
      cudaFree(o);
      cudaFree(D1);
      cudaFree(D2);
    }
    TopkArgs a = {};
    a.X = X;
    a.n = n;
    a.d = d;
    a.ldx = ldx;
    a.Q = Q + q0 * ldqq;
    a.nq = m;
    a.ldq = ldqq;
    a.cbits = ta.cbits;
    a.bstride = bstride;
    a.k = k;
    a.kstride = k;
    a.ids = ids + q0 * k;
    a.dists = dists + q0 * k;
    a.vec4 = true;
    a.nsurv = fb + 1 + mc;
    a.surv = a.nsurv + mc;
    {
      const int64_t g = ceil_div<int64_t>(m, 4);
      (count_launch(), tc::k_tc_select<<<(unsigned)(g < 4096 ? g : 4096), 128, 0, s>>>(
                           ent, ent_cnt, ta.kb, ta.kb_cnt, kTcKb, kTcCap, m, k, a.surv, a.nsurv, fb + 1, fb));
    }
    if (getenv("MRPT_TC_DEBUG")) {
      int32_t fbc = 0;
      cudaMemcpyAsync(&fbc, fb, 4, cudaMemcpyDeviceToHost, s);
      std::vector<int32_t> hs((size_t)m), he((size_t)m);
      cudaMemcpyAsync(hs.data(), a.nsurv, (size_t)m * 4, cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(he.data(), ent_cnt, (size_t)m * 4, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      long long ss = 0, se = 0;
      for (int64_t i = 0; i < m; ++i) {
        ss += hs[i] > 0 ? hs[i] : 0;
        se += he[i];
      }
      fprintf(stderr, "[tc debug] cg=%d grid=%d fallback queries %d of %lld, mean entry slots %.1f, mean survivors %.1f\n",
              cg, grid, fbc, (long long)m, (double)se / m, (double)ss / m);
    }
    a.qlist = fb + 1;
    a.stat_slot = 4;  // fallback statistics: see mrpt_fallback_stats
    g_route_queries[4] += m;
    a.qcount = fb;
    const int64_t tg = m < 64 ? m : 64;
    (count_launch(), tfn<<<(unsigned)tg, kScanNT, tsmem, s>>>(a));
    launch_rerank(a, s);
  }
  return launch_status("mrpt_scan_topk_u8tc_bits");
}
