// Query ordering for the batched path: queries that land in the same leaf of
// tree 0 sit close together in space, so they share most of their leaves in
// the other trees and most of their candidate rows.  Processing a batch in
// that order lets the CTAs running at the same time read the same leaf-id
// pieces (K3) and the same candidate rows (K4) from L2 instead of DRAM.  The
// answers do not depend on the order (every query is independent); the rows
// are gathered into the order before K3/K4 and the results scattered back.
#include "common.cuh"

namespace mrpt {

__global__ void k_order_count(const int32_t *__restrict__ leaves, int64_t nq, int T, int32_t *cnt) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + leaves[q * T], 1);
}

// Exclusive scan of L counters in place (one CTA of 1024 threads).
__global__ void __launch_bounds__(1024) k_order_scan(int32_t *cnt, int L) {
  __shared__ int wsum[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int carry = 0;
  for (int b0 = 0; b0 < L; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    const int v = i < L ? cnt[i] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int c = wsum[lane];
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += u;
      }
      wsum[lane] = x - c;
      if (lane == 31) wsum[32] = x;
    }
    __syncthreads();
    if (i < L) cnt[i] = carry + wsum[warp] + incl - v;
    carry += wsum[32];
    __syncthreads();
  }
}

__global__ void k_order_scatter(const int32_t *__restrict__ leaves, int64_t nq, int T, int32_t *off,
                                int32_t *order) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x)
    order[atomicAdd(off + leaves[q * T], 1)] = (int32_t)q;
}

// dst row i = src row idx[i] (gather) or dst row idx[i] = src row i
// (scatter); rows of `words` 4-byte words.  One warp per row.
__global__ void k_permute_rows(const uint32_t *__restrict__ src, int64_t src_ld, const int32_t *__restrict__ idx,
                               int64_t rows, int64_t words, uint32_t *dst, int64_t dst_ld, int scatter) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < rows; i += nw) {
    const int64_t j = idx[i];
    const uint32_t *s = src + (scatter ? i : j) * src_ld;
    uint32_t *d = dst + (scatter ? j : i) * dst_ld;
    for (int64_t c = lane; c < words; c += 32) d[c] = __ldg(s + c);
  }
}

}  // namespace mrpt

using namespace mrpt;

extern "C" int32_t mrpt_query_order(const int32_t *leaves, int64_t nq, int32_t T, int32_t depth, int32_t *order,
                                    int32_t *ws, void *stream) {
  clear_error();
  if (nq < 0 || T < 1 || depth < 0 || depth > 24 || !order || !ws)
    return fail(MRPT_EPARAM, "mrpt_query_order: bad arguments");
  if (nq == 0) return MRPT_OK;
  cudaStream_t s = as_stream(stream);
  const int L = 1 << depth;
  cudaMemsetAsync(ws, 0, sizeof(int32_t) * (size_t)L, s);
  const int64_t blocks = ceil_div<int64_t>(nq, 256);
  const int grid = (int)(blocks < (int64_t)num_sms() * 8 ? blocks : (int64_t)num_sms() * 8);
  (count_launch(), k_order_count<<<grid, 256, 0, s>>>(leaves, nq, T, ws));
  (count_launch(), k_order_scan<<<1, 1024, 0, s>>>(ws, L));
  (count_launch(), k_order_scatter<<<grid, 256, 0, s>>>(leaves, nq, T, ws, order));
  return launch_status("mrpt_query_order");
}

extern "C" int32_t mrpt_permute_rows(const void *src, int64_t src_ld, const int32_t *idx, int64_t rows,
                                     int64_t words, void *dst, int64_t dst_ld, int32_t scatter, void *stream) {
  clear_error();
  if (rows < 0 || words < 0 || src_ld < words || dst_ld < words) return fail(MRPT_ESHAPE, "mrpt_permute_rows: bad shape");
  if (rows == 0 || words == 0) return MRPT_OK;
  const int64_t blocks = ceil_div<int64_t>(rows, 8);
  const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  (count_launch(), k_permute_rows<<<grid, 256, 0, as_stream(stream)>>>(
                       reinterpret_cast<const uint32_t *>(src), src_ld, idx, rows, words,
                       reinterpret_cast<uint32_t *>(dst), dst_ld, scatter));
  return launch_status("mrpt_permute_rows");
}
