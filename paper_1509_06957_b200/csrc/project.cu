// K1 (sparse projection, fp64-exact) and K2 (routing / fused query descent).
//
// Parity contract (_cy.pyx:27-33, setup.py:37-39): every
// output is a float64 sum of products (double)x * (double)r taken in stored
// CSC order starting from +0.0, rounded once to float32.  A float*float
// product is exact in float64 (24+24 < 53 mantissa bits), so one fused
// multiply-add per term rounds exactly like the reference's separate
// multiply and add -- the chain below is bit-identical to _cy.project.
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"

namespace mrpt {

// ---------------------------------------------------------------- K1 ------
// One CTA owns a tile of `tp` points staged in shared memory (row stride
// `stride`, odd, so lanes reading different points at the same coordinate
// hit distinct banks).  Thread (pg, cg) computes points pg + j*npg for
// j < PPT (independent fp64 chains hide DFMA latency) and columns
// cg, cg+G, ...; consecutive lanes own consecutive points, so column-major
// outputs (the build layout) are written coalesced.  The CSC entry of the
// current column is uniform across the warp (broadcast load).
template <int PPT>
__global__ void __launch_bounds__(256)
k_project_smem(const float *__restrict__ X, int64_t m, int d, int64_t ldx,
               const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ rows,
               const float *__restrict__ vals, int ncols, float *__restrict__ out,
               int64_t ors, int64_t ocs, int tp, int stride) {
  extern __shared__ float xs[];
  const int npg = tp / PPT;
  const int G = blockDim.x / npg;
  const int pg = threadIdx.x % npg, cg = threadIdx.x / npg;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int64_t tile = blockIdx.x; tile * tp < m; tile += gridDim.x) {
    const int64_t i0 = tile * tp;
    const int here = (int)((m - i0) < tp ? (m - i0) : tp);
    __syncthreads();
    for (int r = warp; r < here; r += nwarps) {
      const float *src = X + (i0 + r) * ldx;
      float *dst = xs + r * stride;
      for (int c = lane; c < d; c += 32) dst[c] = __ldg(src + c);
    }
    __syncthreads();
    if (cg >= G) continue;
    for (int c = cg; c < ncols; c += G) {
      const int64_t s0 = __ldg(col_ptr + c), s1 = __ldg(col_ptr + c + 1);
      double acc[PPT];
#pragma unroll
      for (int j = 0; j < PPT; ++j) acc[j] = 0.0;
      for (int64_t s = s0; s < s1; ++s) {
        const int r = __ldg(rows + s);
        const double v = (double)__ldg(vals + s);
#pragma unroll
        for (int j = 0; j < PPT; ++j)
          acc[j] = __fma_rn((double)xs[(pg + j * npg) * stride + r], v, acc[j]);
      }
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const int p = pg + j * npg;
        if (p < here) out[(i0 + p) * ors + (int64_t)c * ocs] = __double2float_rn(acc[j]);
      }
    }
  }
}

// Float64 tile variant (the default where a warp's 32 consecutive points fit
// in shared memory as float64): a CTA of 32 warps stages TP = 32 * PPT
// points converted to float64 once (odd row stride in doubles: the 32 lanes
// of a load hit 32 distinct bank pairs), every warp takes whole columns and
// its lanes take consecutive points (lane + 32 j), so each CSC entry is one
// warp-uniform 8-byte load (packed {row, value}) and each term one
// conflict-free 8-byte shared load and one DFMA -- no per-term conversion.
// Output stores are coalesced (32 consecutive points per column).
template <int PPT>
__global__ void __launch_bounds__(1024, 1)
k_project_d64(const float *__restrict__ X, int64_t m, int d, int64_t ldx,
              const int64_t *__restrict__ col_ptr, const int2 *__restrict__ ent, int64_t ent_cap, int ncols,
              float *__restrict__ out, int64_t ors, int64_t ocs, int stride) {
  extern __shared__ double xd[];
  constexpr int TP = 32 * PPT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t tile = blockIdx.x; tile * TP < m; tile += gridDim.x) {
    const int64_t i0 = tile * TP;
    const int here = (int)((m - i0) < TP ? (m - i0) : TP);
    __syncthreads();
    for (int r = warp; r < TP; r += nw) {
      const float *src = X + (i0 + r) * ldx;
      double *dst = xd + r * stride;
      for (int c = lane; c < d; c += 32) dst[c] = r < here ? (double)__ldg(src + c) : 0.0;
    }
    __syncthreads();
    const double *xb = xd + lane * stride;
    for (int c = warp; c < ncols; c += nw) {
      const int64_t s0 = __ldg(col_ptr + c), s1r = __ldg(col_ptr + c + 1);
      const int64_t s1 = s1r < ent_cap ? s1r : ent_cap;
      double acc[PPT];
#pragma unroll
      for (int j = 0; j < PPT; ++j) acc[j] = 0.0;
#pragma unroll 4
      for (int64_t s = s0; s < s1; ++s) {
        const int2 e = __ldg(ent + s);
        const double v = (double)__int_as_float(e.y);
        const double *xr = xb + e.x;
#pragma unroll
        for (int j = 0; j < PPT; ++j) acc[j] = __fma_rn(xr[j * 32 * stride], v, acc[j]);
      }
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const int p = lane + 32 * j;
        if (p < here) out[(i0 + p) * ors + (int64_t)c * ocs] = __double2float_rn(acc[j]);
      }
    }
  }
}

// Packed float64 tile (PPT = 3 or 5; the default where it fits).  K1 is
// bound by the shared-memory return path (a warp's 8-byte load returns 256
// bytes = 2 cycles per DFMA), so the tile keeps fewer bytes per coordinate.
// (double)x of a float has at most 23 explicit mantissa bits: its high word
// plus the top 3 bits of its low word are the whole value.  Per (coordinate,
// lane) the tile stores the PPT high words of points lane + 32 j and one word
// holding the PPT 3-bit fields -- 16 bytes for 3 points, 24 bytes for 5
// (5.3 / 4.8 bytes per term instead of 8) -- and a term rebuilds its float64
// with one or two integer operations before the same DFMA.  The value is the
// exact float64 the plain tile holds, so the chain is bit-identical.
template <int J>
__device__ __forceinline__ uint32_t h32_lo(uint32_t w) {
  // fields: j=0 bits 0-2, j=1 bits 13-15 (byte 1 otherwise zero), j=2 bits
  // 21-23 (byte 2 otherwise zero), j=3 bits 29-31, j=4 bits 3-5
  if (J == 0) return w << 29;
  if (J == 1) return __byte_perm(w, 0u, 0x1444);
  if (J == 2) return __byte_perm(w, 0u, 0x2444);
  if (J == 3) return w & 0xE0000000u;
  return (w << 26) & 0xE0000000u;
}
__device__ __forceinline__ uint32_t h32_field(int j, double x) {
  const uint32_t l = (uint32_t)__double2loint(x) >> 29;
  return l << (j == 0 ? 0 : (j == 1 ? 13 : (j == 2 ? 21 : (j == 3 ? 29 : 3))));
}

// Stage TP = 32 * PPT rows of X (rows i0 .. i0 + here) into the packed tile:
// a warp takes 4 coordinates at a time, its lanes the points lane + 32 j.
template <int PPT>
__device__ __forceinline__ void h32_stage(const float *__restrict__ X, int64_t ldx, int d, int64_t i0, int here,
                                          uint4 *A, uint2 *B) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int g = warp; 4 * g < d; g += nw) {
    float4 x[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int p = lane + 32 * j;
      x[j] = p < here ? __ldg(reinterpret_cast<const float4 *>(X + (i0 + p) * ldx) + g)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t hi[PPT], w = 0u;
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const float f = u == 0 ? x[j].x : (u == 1 ? x[j].y : (u == 2 ? x[j].z : x[j].w));
        const double xd = (double)f;
        hi[j] = (uint32_t)__double2hiint(xd);
        w |= h32_field(j, xd);
      }
      const int at = (4 * g + u) * 32 + lane;
      A[at] = make_uint4(hi[0], hi[1], hi[2], w);
      if (PPT == 5) B[at] = make_uint2(hi[PPT - 2], hi[PPT - 1]);
    }
  }
}

// One column's chain for the lane's PPT points: acc[j] = fma(x_j[row], value,
// acc[j]) over the column's entries in stored order.  Al / Bl: the tile
// regions offset by the lane.
template <int PPT>
__device__ __forceinline__ void h32_column(const uint4 *Al, const uint2 *Bl, const int2 *__restrict__ ent, int64_t s0,
                                           int64_t s1, double (&acc)[PPT]) {
#pragma unroll 4
  for (int64_t s = s0; s < s1; ++s) {
    const int2 e = __ldg(ent + s);
    const double v = (double)__int_as_float(e.y);
    const uint4 a = Al[e.x * 32];
    acc[0] = __fma_rn(__hiloint2double((int)a.x, (int)h32_lo<0>(a.w)), v, acc[0]);
    acc[1] = __fma_rn(__hiloint2double((int)a.y, (int)h32_lo<1>(a.w)), v, acc[1]);
    acc[2] = __fma_rn(__hiloint2double((int)a.z, (int)h32_lo<2>(a.w)), v, acc[2]);
    if (PPT == 5) {
      const uint2 b = Bl[e.x * 32];
      acc[PPT - 2] = __fma_rn(__hiloint2double((int)b.x, (int)h32_lo<3>(a.w)), v, acc[PPT - 2]);
      acc[PPT - 1] = __fma_rn(__hiloint2double((int)b.y, (int)h32_lo<4>(a.w)), v, acc[PPT - 1]);
    }
  }
}

template <int PPT>
__global__ void __launch_bounds__(1024, 1)
k_project_h32(const float *__restrict__ X, int64_t m, int d, int64_t ldx,
              const int64_t *__restrict__ col_ptr, const int2 *__restrict__ ent, int64_t ent_cap, int ncols,
              float *__restrict__ out, int64_t ors, int64_t ocs) {
  static_assert(PPT == 3 || PPT == 5, "packed tile: 3 or 5 points per lane");
  extern __shared__ uint4 h32_smem[];
  constexpr int TP = 32 * PPT;
  uint4 *A = h32_smem;                                      // [d][32]: hi0, hi1, hi2, fields
  uint2 *B = reinterpret_cast<uint2 *>(h32_smem + 32 * d);  // [d][32]: hi3, hi4 (PPT == 5)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t tile = blockIdx.x; tile * TP < m; tile += gridDim.x) {
    const int64_t i0 = tile * TP;
    const int here = (int)((m - i0) < TP ? (m - i0) : TP);
    __syncthreads();
    h32_stage<PPT>(X, ldx, d, i0, here, A, B);
    __syncthreads();
    const uint4 *Al = A + lane;
    const uint2 *Bl = B + lane;
    for (int c = warp; c < ncols; c += nw) {
      const int64_t s0 = __ldg(col_ptr + c), s1r = __ldg(col_ptr + c + 1);
      const int64_t s1 = s1r < ent_cap ? s1r : ent_cap;
      double acc[PPT];
#pragma unroll
      for (int j = 0; j < PPT; ++j) acc[j] = 0.0;
      h32_column<PPT>(Al, Bl, ent, s0, s1, acc);
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const int p = lane + 32 * j;
        if (p < here) out[(i0 + p) * ors + (int64_t)c * ocs] = __double2float_rn(acc[j]);
      }
    }
  }
}

// K2 on the packed tile (batched queries): a CTA stages 32 * PPT query rows
// like K1 and its warps take whole trees of its share [part T/S, (part+1)
// T/S): per level the column's chain for the lane's PPT queries (the K1
// chain: warp-uniform entries, conflict-free tile loads), then the descent
// _cy.route: node = 2*node + 1 + (p > split[node]).  Against k_query_route
// (thread = tree, query coordinates gathered at per-lane rows: bank
// conflicts on every term) the shared-memory return path carries 4.8 bytes
// per term without conflicts.
template <int PPT>
__global__ void __launch_bounds__(1024, 1)
k_query_route_h32(const float *__restrict__ Q, int64_t nq, int d, int64_t ldq,
                  const int64_t *__restrict__ col_ptr, const int2 *__restrict__ ent, int64_t ent_cap,
                  const float *__restrict__ splits, int T, int depth, int32_t *__restrict__ leaves, int S) {
  static_assert(PPT == 3 || PPT == 5, "packed tile: 3 or 5 points per lane");
  extern __shared__ uint4 h32_smem[];
  constexpr int TP = 32 * PPT;
  uint4 *A = h32_smem;
  uint2 *B = reinterpret_cast<uint2 *>(h32_smem + 32 * d);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int32_t nint = (int32_t)(((int64_t)1 << depth) - 1);
  const int64_t items = ((nq + TP - 1) / TP) * S;
  int64_t staged = -1;
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t tile = item / S;
    const int part = (int)(item - tile * S);
    const int64_t i0 = tile * TP;
    const int here = (int)((nq - i0) < TP ? (nq - i0) : TP);
    if (tile != staged) {  // CTA-uniform
      __syncthreads();
      h32_stage<PPT>(Q, ldq, d, i0, here, A, B);
      __syncthreads();
      staged = tile;
    }
    const uint4 *Al = A + lane;
    const uint2 *Bl = B + lane;
    const int t0 = (int)(((int64_t)part * T) / S), t1 = (int)(((int64_t)(part + 1) * T) / S);
    for (int t = t0 + warp; t < t1; t += nw) {
      const float *tsplit = splits + (int64_t)t * nint;
      int32_t node[PPT];
#pragma unroll
      for (int j = 0; j < PPT; ++j) node[j] = 0;
      for (int lev = 0; lev < depth; ++lev) {
        const int64_t c = (int64_t)t * depth + lev;
        const int64_t s0 = __ldg(col_ptr + c), s1r = __ldg(col_ptr + c + 1);
        const int64_t s1 = s1r < ent_cap ? s1r : ent_cap;
        double acc[PPT];
#pragma unroll
        for (int j = 0; j < PPT; ++j) acc[j] = 0.0;
        h32_column<PPT>(Al, Bl, ent, s0, s1, acc);
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const float p = __double2float_rn(acc[j]);
          node[j] = 2 * node[j] + 1 + (p > __ldg(tsplit + node[j]) ? 1 : 0);
        }
      }
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const int p = lane + 32 * j;
        if (p < here) leaves[(i0 + p) * T + t] = node[j] - nint;
      }
    }
  }
}

// {row, value bits} pairs of a CSC column set (one 8-byte load per entry).
__global__ void k_pack_entries(const int32_t *__restrict__ rows, const float *__restrict__ vals,
                               const int64_t *__restrict__ nnz_ptr, int64_t cap, int2 *ent) {
  const int64_t nnz = *nnz_ptr < cap ? *nnz_ptr : cap;  // cap: ncols * d (rows distinct per column)
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nnz; s += (int64_t)gridDim.x * blockDim.x)
    ent[s] = make_int2(rows[s], __float_as_int(vals[s]));
}

// Fallback for rows too wide to stage (d beyond ~1.6K): one thread per
// (point, column), coordinates read through the read-only path.
__global__ void __launch_bounds__(256)
k_project_global(const float *__restrict__ X, int64_t m, int64_t ldx,
                 const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ rows,
                 const float *__restrict__ vals, int ncols, float *__restrict__ out,
                 int64_t ors, int64_t ocs) {
  const int64_t total = m * ncols;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(g / m);
    const int64_t i = g - (int64_t)c * m;
    const float *xr = X + i * ldx;
    double acc = 0.0;
    for (int64_t s = col_ptr[c]; s < col_ptr[c + 1]; ++s)
      acc = __fma_rn((double)__ldg(xr + rows[s]), (double)vals[s], acc);
    out[i * ors + (int64_t)c * ocs] = __double2float_rn(acc);
  }
}

// ---------------------------------------------------------------- K2 ------
// _cy.route: node = 2*node + 1 + (p > split); leaf = node - n_internal.
__global__ void k_route(const float *__restrict__ proj, int64_t nrows, int depth,
                        const float *__restrict__ splits, int64_t n_internal,
                        int64_t *__restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t node = 0;
    for (int lev = 0; lev < depth; ++lev) {
      const float p = proj[r * depth + lev];
      node = 2 * node + 1 + (p > splits[r * n_internal + node] ? 1 : 0);
    }
    out[r] = node - n_internal;
  }
}

// Fused query projection + descent.  CTA = QB queries x 128 trees; the QB
// query rows are staged in shared memory, each thread walks one tree for all
// QB queries at once (QB independent fp64 chains, CSC entries loaded once).
template <int QB, bool SMEM, typename QT = float>
__global__ void __launch_bounds__(128)
k_query_route(const float *__restrict__ Q, int64_t nq, int d, int64_t ldq,
              const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ rows,
              const float *__restrict__ vals, const float *__restrict__ splits, int T,
              int depth, int32_t *__restrict__ leaves, int stride) {
  extern __shared__ __align__(16) unsigned char qs_raw[];
  QT *qs = reinterpret_cast<QT *>(qs_raw);
  const int64_t q0 = (int64_t)blockIdx.y * QB;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nint = ((int64_t)1 << depth) - 1;
  if (SMEM) {
    for (int qi = 0; qi < QB; ++qi) {
      const bool live = q0 + qi < nq;
      const float *src = Q + (q0 + qi) * ldq;
      for (int c = threadIdx.x; c < d; c += blockDim.x)
        qs[qi * stride + c] = (QT)(live ? __ldg(src + c) : 0.0f);
    }
    __syncthreads();
  }
  if (t >= T) return;
  int64_t node[QB];
#pragma unroll
  for (int qi = 0; qi < QB; ++qi) node[qi] = 0;
  const float *tsplit = splits + (int64_t)t * nint;
  for (int lev = 0; lev < depth; ++lev) {
    const int64_t c = (int64_t)t * depth + lev;
    const int64_t s0 = __ldg(col_ptr + c), s1 = __ldg(col_ptr + c + 1);
    double acc[QB];
#pragma unroll
    for (int qi = 0; qi < QB; ++qi) acc[qi] = 0.0;
    // CSC entries 8 at a time: their loads are independent of the FMA chain,
    // so all 8 (and the query loads they index) are in flight together
    int64_t s = s0;
    for (; s + 8 <= s1; s += 8) {
      int r[8];
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        r[u] = __ldg(rows + s + u);
        v[u] = __ldg(vals + s + u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
#pragma unroll
        for (int qi = 0; qi < QB; ++qi) {
          QT x;
          if (SMEM) {
            x = qs[qi * stride + r[u]];
          } else {
            x = (q0 + qi < nq) ? __ldg(Q + (q0 + qi) * ldq + r[u]) : 0.0f;
          }
          acc[qi] = __fma_rn((double)x, (double)v[u], acc[qi]);
        }
      }
    }
    for (; s < s1; ++s) {
      const int r = __ldg(rows + s);
      const double v = (double)__ldg(vals + s);
#pragma unroll
      for (int qi = 0; qi < QB; ++qi) {
        QT x;
        if (SMEM) {
          x = qs[qi * stride + r];
        } else {
          x = (q0 + qi < nq) ? __ldg(Q + (q0 + qi) * ldq + r) : 0.0f;
        }
        acc[qi] = __fma_rn((double)x, v, acc[qi]);
      }
    }
#pragma unroll
    for (int qi = 0; qi < QB; ++qi) {
      const float p = __double2float_rn(acc[qi]);
      node[qi] = 2 * node[qi] + 1 + (p > __ldg(tsplit + node[qi]) ? 1 : 0);
    }
  }
#pragma unroll
  for (int qi = 0; qi < QB; ++qi)
    if (q0 + qi < nq) leaves[(q0 + qi) * T + t] = (int32_t)(node[qi] - nint);
}

}  // namespace mrpt

using namespace mrpt;

static const int kProjSmemBudget = 100 * 1024;  // two CTAs per SM

extern "C" int32_t mrpt_project(const float *X, int64_t m, int32_t d, int64_t ldx,
                                const int64_t *col_ptr, const int32_t *rows, const float *vals,
                                int32_t ncols, float *out, int64_t out_row_stride,
                                int64_t out_col_stride, void *stream) {
  clear_error();
  if (m < 0 || d < 1 || ldx < d || ncols < 0)
    return fail(MRPT_ESHAPE, "mrpt_project: bad shape");
  if (m == 0 || ncols == 0) return MRPT_OK;
  if (!X || !col_ptr || !out) return fail(MRPT_EPARAM, "mrpt_project: null pointer");
  cudaStream_t s = as_stream(stream);
  const int stride = (d & 1) ? d : d + 1;
  const int64_t row_bytes = (int64_t)stride * 4;
  // float64 tile: as many 32-point groups as fit (PPT 1..6)
  {
    const char *pe = getenv("MRPT_PROJ_D64");  // experiments: 0 disables
    int ppt = (int)((212 * 1024) / ((int64_t)stride * 8 * 32));
    if (ppt > 6) ppt = 6;
    if ((!pe || atoi(pe) != 0) && ppt >= 1 && ncols >= 32) {
      // packed entries: sized by the bound d per column (no host read of
      // col_ptr[ncols], so the call never synchronises)
      const int64_t nnz_bound = (int64_t)ncols * d;
      int2 *ent = nullptr;
      keep_pool_warm();
      if (cudaMallocAsync((void **)&ent, sizeof(int2) * (size_t)nnz_bound, s) != cudaSuccess)
        return fail(MRPT_ECUDA, "mrpt_project: scratch allocation failed");
      {
        const int64_t pb = ceil_div<int64_t>(nnz_bound, 256);
        (count_launch(), k_pack_entries<<<(unsigned)(pb < 4096 ? pb : 4096), 256, 0, s>>>(rows, vals,
                                                                                          col_ptr + ncols, nnz_bound, ent));
      }
      // packed tile (k_project_h32): 5 points per lane in 24 bytes per
      // coordinate, or 3 in 16, where the rows are 16-byte loadable
      {
        const char *ph = getenv("MRPT_PROJ_H32");  // experiments: 0 disables
        const bool vec = d % 4 == 0 && ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
        const int hp = (int64_t)d * 32 * 24 <= 224 * 1024 ? 5 : ((int64_t)d * 32 * 16 <= 224 * 1024 ? 3 : 0);
        if ((!ph || atoi(ph) != 0) && vec && hp) {
          const size_t hsmem = (size_t)d * 32 * (hp == 5 ? 24 : 16);
          void (*hf)(const float *, int64_t, int, int64_t, const int64_t *, const int2 *, int64_t, int, float *,
                     int64_t, int64_t) = hp == 5 ? k_project_h32<5> : k_project_h32<3>;
          cudaFuncSetAttribute(hf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
          const int64_t htiles = ceil_div<int64_t>(m, 32 * hp);
          const int hgrid = (int)(htiles < (int64_t)num_sms() ? htiles : (int64_t)num_sms());
          (count_launch(), hf<<<hgrid, 1024, hsmem, s>>>(X, m, d, ldx, col_ptr, ent, nnz_bound, ncols, out,
                                                       out_row_stride, out_col_stride));
          cudaFreeAsync(ent, s);
          return launch_status("mrpt_project");
        }
      }
      const size_t smem = (size_t)32 * ppt * stride * 8;
      void (*fn)(const float *, int64_t, int, int64_t, const int64_t *, const int2 *, int64_t, int, float *,
                 int64_t, int64_t, int) =
          ppt >= 6 ? k_project_d64<6>
                   : (ppt == 5 ? k_project_d64<5>
                               : (ppt == 4 ? k_project_d64<4>
                                           : (ppt == 3 ? k_project_d64<3> : (ppt == 2 ? k_project_d64<2> : k_project_d64<1>))));
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int64_t tiles = ceil_div<int64_t>(m, 32 * ppt);
      const int grid = (int)(tiles < (int64_t)num_sms() ? tiles : (int64_t)num_sms());
      (count_launch(), fn<<<grid, 1024, smem, s>>>(X, m, d, ldx, col_ptr, ent, nnz_bound, ncols, out, out_row_stride,
                                                out_col_stride, stride));
      cudaFreeAsync(ent, s);
      return launch_status("mrpt_project");
    }
  }
  // tile of 256, 128 or 64 points (point groups must be a power-of-two
  // multiple of the warp so every thread has a column group)
  int tp = 256;
  while (tp >= 64 && (int64_t)tp * row_bytes > kProjSmemBudget) tp >>= 1;
  if (tp >= 64) {
    const size_t smem = (size_t)tp * row_bytes;
    const int64_t tiles = ceil_div<int64_t>(m, tp);
    // as many resident CTAs as shared memory allows (latency hiding)
    int per_sm = (int)((220 * 1024) / (smem + 1024));
    per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
    const int64_t cap = (int64_t)num_sms() * per_sm;
    const int grid = (int)(tiles < cap ? tiles : cap);
    // points per thread: each CSC entry (two warp-uniform loads and a
    // conversion) is shared by PPT independent fp64 chains
    const char *pe = getenv("MRPT_PROJ_PPT");
    int ppt = pe ? atoi(pe) : 4;
    if (ppt != 2 && ppt != 4 && ppt != 8) ppt = 2;
    while (ppt > 2 && tp / ppt < 8) ppt >>= 1;  // >= 8 consecutive points per column write
    void (*fn)(const float *, int64_t, int, int64_t, const int64_t *, const int32_t *, const float *, int,
               float *, int64_t, int64_t, int, int) =
        ppt == 8 ? k_project_smem<8> : (ppt == 4 ? k_project_smem<4> : k_project_smem<2>);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    (count_launch(), fn<<<grid, 256, smem, s>>>(X, m, d, ldx, col_ptr, rows, vals, ncols, out,
                                                out_row_stride, out_col_stride, tp, stride));
  } else if (32 * row_bytes <= 200 * 1024) {
    tp = 32;
    const size_t smem = (size_t)tp * row_bytes;
    const int64_t tiles = ceil_div<int64_t>(m, tp);
    const int grid = (int)(tiles < (int64_t)num_sms() ? tiles : (int64_t)num_sms());
    cudaFuncSetAttribute(k_project_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    (count_launch(), k_project_smem<1><<<grid, 256, smem, s>>>(X, m, d, ldx, col_ptr, rows, vals, ncols, out,
                                               out_row_stride, out_col_stride, tp, stride));
  } else {
    const int64_t total = m * ncols;
    const int64_t blocks = ceil_div<int64_t>(total, 256);
    const int grid = (int)(blocks < (int64_t)num_sms() * 8 ? blocks : (int64_t)num_sms() * 8);
    (count_launch(), k_project_global<<<grid, 256, 0, s>>>(X, m, ldx, col_ptr, rows, vals, ncols, out,
                                          out_row_stride, out_col_stride));
  }
  return launch_status("mrpt_project");
}

extern "C" int32_t mrpt_route(const float *proj, int64_t nrows, int32_t depth, const float *splits,
                              int64_t n_internal, int64_t *out, void *stream) {
  clear_error();
  if (nrows < 0 || depth < 0 || n_internal < 0) return fail(MRPT_ESHAPE, "mrpt_route: bad shape");
  if (nrows == 0) return MRPT_OK;
  cudaStream_t s = as_stream(stream);
  const int64_t blocks = ceil_div<int64_t>(nrows, 128);
  const int grid = (int)(blocks < 65535 ? blocks : 65535);
  (count_launch(), k_route<<<grid, 128, 0, s>>>(proj, nrows, depth, splits, n_internal, out));
  return launch_status("mrpt_route");
}

template <int QB, typename QT = float>
static int32_t query_route_launch(const float *Q, int64_t nq, int32_t d, int64_t ldq, const int64_t *col_ptr,
                                  const int32_t *rows, const float *vals, const float *splits, int32_t T,
                                  int32_t depth, int32_t *leaves, cudaStream_t s) {
  const int stride = (d & 1) ? d : d + 1;
  const size_t smem = (size_t)QB * stride * sizeof(QT);
  const int64_t qblocks = ceil_div<int64_t>(nq, QB);
  if (qblocks > 65535LL * 1024) return fail(MRPT_EPARAM, "mrpt_query_route: too many queries per call");
  int64_t off = 0;
  // gridDim.y is limited to 65535: split very large batches.
  while (off < nq) {
    const int64_t chunk_q = (nq - off) < 65535LL * QB ? (nq - off) : 65535LL * QB;
    dim3 grid((unsigned)ceil_div<int>(T, 128), (unsigned)ceil_div<int64_t>(chunk_q, QB));
    if (smem <= 160 * 1024) {
      cudaFuncSetAttribute(k_query_route<QB, true, QT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      (count_launch(), k_query_route<QB, true, QT><<<grid, 128, smem, s>>>(Q + off * ldq, chunk_q, d, ldq, col_ptr,
                                                                       rows, vals, splits, T, depth,
                                                                       leaves + off * T, stride));
    } else {
      (count_launch(), k_query_route<QB, false><<<grid, 128, 0, s>>>(Q + off * ldq, chunk_q, d, ldq, col_ptr,
                                                                     rows, vals, splits, T, depth,
                                                                     leaves + off * T, stride));
    }
    off += chunk_q;
  }
  return MRPT_OK;
}

extern "C" int32_t mrpt_query_route(const float *Q, int64_t nq, int32_t d, int64_t ldq,
                                    const int64_t *col_ptr, const int32_t *rows,
                                    const float *vals, const float *splits, int32_t T,
                                    int32_t depth, int32_t *leaves, void *stream) {
  clear_error();
  if (nq < 0 || d < 1 || ldq < d || T < 1 || depth < 1 || depth > 30)
    return fail(MRPT_ESHAPE, "mrpt_query_route: bad shape");
  if (nq == 0) return MRPT_OK;
  cudaStream_t s = as_stream(stream);
  // batched queries on the packed tile (k_query_route_h32)
  {
    const char *ph = getenv("MRPT_ROUTE_H32");  // experiments: 0 disables, 1 forces for any batch size
    const bool vec = d % 4 == 0 && ldq % 4 == 0 && (reinterpret_cast<uintptr_t>(Q) & 15) == 0;
    const int hp = (int64_t)d * 32 * 24 <= 224 * 1024 ? 5 : ((int64_t)d * 32 * 16 <= 224 * 1024 ? 3 : 0);
    const bool want = ph ? atoi(ph) != 0 : nq >= 1024;
    if (want && vec && hp && depth <= 30) {
      const int64_t ncols = (int64_t)T * depth, nnz_bound = ncols * d;
      int2 *ent = nullptr;
      keep_pool_warm();
      if (cudaMallocAsync((void **)&ent, sizeof(int2) * (size_t)nnz_bound, s) != cudaSuccess)
        return fail(MRPT_ECUDA, "mrpt_query_route: scratch allocation failed");
      const int64_t pb = ceil_div<int64_t>(nnz_bound, 256);
      (count_launch(), k_pack_entries<<<(unsigned)(pb < 4096 ? pb : 4096), 256, 0, s>>>(rows, vals, col_ptr + ncols,
                                                                                        nnz_bound, ent));
      const size_t hsmem = (size_t)d * 32 * (hp == 5 ? 24 : 16);
      void (*hf)(const float *, int64_t, int, int64_t, const int64_t *, const int2 *, int64_t, const float *, int,
                 int, int32_t *, int) = hp == 5 ? k_query_route_h32<5> : k_query_route_h32<3>;
      cudaFuncSetAttribute(hf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
      const int64_t tiles = ceil_div<int64_t>(nq, 32 * hp);
      // tree shares per tile so that every SM gets ~10 work items or more
      int64_t S = ceil_div<int64_t>(10 * (int64_t)num_sms(), tiles);
      S = S < 1 ? 1 : (S > 8 ? 8 : S);
      if (S > T / 32) S = T / 32 > 0 ? T / 32 : 1;
      const int64_t items = tiles * S;
      const int grid = (int)(items < (int64_t)num_sms() ? items : (int64_t)num_sms());
      (count_launch(), hf<<<grid, 1024, hsmem, s>>>(Q, nq, d, ldq, col_ptr, ent, nnz_bound, splits, T, depth, leaves,
                                                    (int)S));
      cudaFreeAsync(ent, s);
      return launch_status("mrpt_query_route");
    }
  }
  const char *qe = getenv("MRPT_ROUTE_QB");
  const int qbs = qe ? atoi(qe) : 8;
  // 8 queries per thread (8 independent float64 chains per CSC entry load);
  // measured at config 2: 0.27 ms vs 0.30 (4) and 0.46 (2).  A float64 copy
  // of the query rows in shared memory was slower (0.47 ms: 8-byte loads at
  // random coordinates conflict twice as often).
  const int32_t st = qbs == 4
      ? query_route_launch<4>(Q, nq, d, ldq, col_ptr, rows, vals, splits, T, depth, leaves, s)
      : query_route_launch<8>(Q, nq, d, ldq, col_ptr, rows, vals, splits, T, depth, leaves, s);
  if (st) return st;
  return launch_status("mrpt_query_route");
}
