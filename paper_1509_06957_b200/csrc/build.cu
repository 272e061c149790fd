#include <stdlib.h>
// K5: level-synchronous random-projection-tree construction for a batch of
// trees (replaces build_tree / median_split, pkg/src/mrpt/trees.py:33-98).
//
// Per level, every node (segment of the point permutation) of every tree in
// the batch is split at the lower median of its projections -- the
// kth = (m+1)/2-1 smallest value, found EXACTLY by MSD radix select over
// order-preserving uint32 keys -- and stably partitioned (value <= split
// goes left), so leaf slices stay ascending in point id exactly like the
// reference's np.partition + boolean-mask build starting from arange(n).
// m == 0 keeps split 0.0 and sends nothing left (trees.py:84-85).
//
// Segments are classified on the device every level (no host sync):
//   tiny  (m <= 2048)          one CTA, keys+ids staged in 16 KB smem
//   mid   (2048 < m <= 8192)   one CTA, 64 KB smem
//   big   (m > 8192)           chunked over many CTAs: key gather pass,
//                              up to four 8-bit histogram passes with global
//                              histograms, count / scan / stable scatter.
// The radix select first strips the prefix shared by the segment's min and
// max key, so the first histogram already splits the live key range.
#include "common.cuh"

namespace mrpt {

constexpr int kTinyMax = 2048;
constexpr int kMidMax = 8192;
constexpr int kChunk = 8192;  // elements per CTA work item in the big path
constexpr int kNT = 256;      // threads per CTA for all build kernels

struct BigSeg {
  int64_t b, e;
  int64_t chunk_base;
  int32_t t, s;
  int32_t nchunks;
  int32_t nb;  // key bits already determined
  uint32_t kmin, kmax, prefix;
  int32_t done;
  int32_t kth, krem, cnt_last, nle;
};

struct LevelCtl {
  int32_t ntiny, nmid, nbig, pad;
  int64_t nchunks;
};

struct LevelArgs {
  const float *P;
  int64_t n;
  int depth, lev, Tb;
  const int32_t *order_in;
  int32_t *order_out;
  const int64_t *bounds_in;
  int64_t *bounds_out;
  int64_t bstride;  // 2^depth + 1
  float *splits;
  int64_t sstride;  // 2^depth - 1
  uint32_t *keys;   // big path: (Tb, n)
  LevelCtl *ctl;
  int32_t *tiny_list, *mid_list;
  BigSeg *big;
  uint32_t *ghist;  // (maxbig, 256)
  int2 *chunks;
  int32_t *chunk_left, *chunk_off;
  int32_t *tree_nch;   // (Tb) big-path chunks per tree this level
  int64_t *tree_base;  // (Tb) first chunk of each tree (tree-major chunk order)
};

__device__ __forceinline__ void write_node(const LevelArgs &a, int t, int s, int64_t b, int64_t e,
                                           int64_t nle, float split) {
  const int nseg = 1 << a.lev;
  a.splits[(int64_t)t * a.sstride + (nseg - 1) + s] = split;
  int64_t *bo = a.bounds_out + (int64_t)t * a.bstride;
  if (s == 0) bo[0] = 0;
  bo[2 * s + 1] = b + nle;
  bo[2 * s + 2] = e;
}

// Warp-wide search of a 256-bin histogram for the bin holding rank `krem`:
// returns bin, count below it and its count (valid in every lane).
__device__ __forceinline__ void warp_pick(const uint32_t *hist, int krem, int &bin, int &below,
                                          int &cnt) {
  const int lane = threadIdx.x & 31;
  uint32_t h[8];
  int sum = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    h[j] = hist[lane * 8 + j];
    sum += (int)h[j];
  }
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int excl = incl - sum;
  const unsigned hit = __ballot_sync(0xffffffffu, incl > krem);
  const int src = __ffs(hit) - 1;
  int mb = 0, mbel = 0, mc = 0;
  if (lane == src) {
    int c = excl;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (c + (int)h[j] > krem) {
        mb = lane * 8 + j;
        mbel = c;
        mc = (int)h[j];
        break;
      }
      c += (int)h[j];
    }
  }
  bin = __shfl_sync(0xffffffffu, mb, src);
  below = __shfl_sync(0xffffffffu, mbel, src);
  cnt = __shfl_sync(0xffffffffu, mc, src);
}

__device__ __forceinline__ bool prefix_match(uint32_t k, uint32_t prefix, int nb) {
  return nb == 0 || ((k ^ prefix) >> (32 - nb)) == 0u;
}

template <typename T>
__device__ __forceinline__ void block_minmax(T &mn, T &mx, T *red_mn, T *red_mx) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if (lane == 0) {
    red_mn[warp] = mn;
    red_mx[warp] = mx;
  }
  __syncthreads();
  mn = red_mn[0];
  mx = red_mx[0];
  for (int w = 1; w < kNT / 32; ++w) {
    mn = red_mn[w] < mn ? red_mn[w] : mn;
    mx = red_mx[w] > mx ? red_mx[w] : mx;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
__global__ void k_build_init(int32_t *order, int64_t *bounds, int64_t n, int Tb, int64_t bstride) {
  const int64_t total = (int64_t)Tb * n;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = g / n;
    order[g] = (int32_t)(g - t * n);
  }
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < Tb;
       t += (int64_t)gridDim.x * blockDim.x) {
    bounds[t * bstride] = 0;
    bounds[t * bstride + 1] = n;
  }
}

// One thread per segment: classify, allocate big-path work.
__global__ void k_level_plan(LevelArgs a) {
  const int nseg = 1 << a.lev;
  const int64_t total = (int64_t)a.Tb * nseg;
  const int64_t seg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (seg >= total) return;
  const int t = (int)(seg >> a.lev), s = (int)(seg & (nseg - 1));
  const int64_t *B = a.bounds_in + (int64_t)t * a.bstride;
  const int64_t b = B[s], e = B[s + 1], m = e - b;
  if (m > kMidMax) {  // tiny / mid segments are found by k_seg_small itself
    const int slot = atomicAdd(&a.ctl->nbig, 1);
    const int nch = (int)ceil_div<int64_t>(m, kChunk);
    // chunk position within its tree; k_chunk_layout adds the tree's base so
    // the chunk table is tree-major (concurrent CTAs gather from the same
    // tree's projection column, which then stays in L2)
    const int64_t cb = (int64_t)atomicAdd(&a.tree_nch[t], nch);
    BigSeg g;
    g.b = b;
    g.e = e;
    g.chunk_base = cb;
    g.t = t;
    g.s = s;
    g.nchunks = nch;
    g.nb = 0;
    g.kmin = 0xffffffffu;
    g.kmax = 0u;
    g.prefix = 0u;
    g.done = 0;
    g.kth = (int32_t)((m + 1) / 2 - 1);
    g.krem = g.kth;
    g.cnt_last = 0;
    g.nle = 0;
    a.big[slot] = g;
    uint32_t *h = a.ghist + (int64_t)slot * 256;
    for (int i = 0; i < 256; ++i) h[i] = 0u;
  }
}

// Tree-major chunk table: exclusive scan of the per-tree chunk counts (one
// CTA), then one warp per big segment rebases its chunks and writes them.
__global__ void __launch_bounds__(1024) k_chunk_layout(LevelArgs a) {
  __shared__ int64_t wsum[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t carry = 0;
  for (int t0 = 0; t0 < a.Tb; t0 += 1024) {
    const int t = t0 + threadIdx.x;
    const int64_t v = t < a.Tb ? a.tree_nch[t] : 0;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int64_t c = wsum[lane];
      int64_t x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += u;
      }
      wsum[lane] = x - c;
      if (lane == 31) wsum[32] = x;
    }
    __syncthreads();
    if (t < a.Tb) a.tree_base[t] = carry + wsum[warp] + incl - v;
    carry += wsum[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.ctl->nchunks = carry;
}

__global__ void k_chunk_fill(LevelArgs a) {
  const int lane = threadIdx.x & 31;
  const int nbig = a.ctl->nbig;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < nbig; i += wstride) {
    BigSeg *g = a.big + i;
    const int64_t cb = g->chunk_base + a.tree_base[g->t];
    __syncwarp();
    if (lane == 0) g->chunk_base = cb;
    for (int c = lane; c < g->nchunks; c += 32) a.chunks[cb + c] = make_int2((int)i, c);
  }
}

// One CTA per segment with m <= MAXM (keys and ids staged in smem).  CTAs
// walk the segments in tree-major order (segment = t * 2^lev + s) and skip
// those of the other size class, so the CTAs resident at any time gather
// from one or two trees' projection columns, which then stay in L2 (an
// atomically appended work list interleaves all trees of the batch and made
// the gathers read DRAM ~13x the keys' bytes at config 5).
template <int MAXM>
__global__ void __launch_bounds__(kNT) k_seg_small(LevelArgs a, int which) {
  extern __shared__ uint32_t dyn_smem[];
  uint32_t *keys = dyn_smem;                                      // MAXM
  int32_t *ids = reinterpret_cast<int32_t *>(dyn_smem + MAXM);    // MAXM
  __shared__ uint32_t hist[256];
  __shared__ uint32_t red_mn[kNT / 32], red_mx[kNT / 32];
  __shared__ int s_bin, s_below, s_cnt;
  __shared__ int wcnt[kNT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nseg = 1 << a.lev;
  const int64_t total = (int64_t)a.Tb << a.lev;
  for (int64_t seg = blockIdx.x; seg < total; seg += gridDim.x) {
    const int t = (int)(seg >> a.lev), s = (int)(seg & (nseg - 1));
    const int64_t *B = a.bounds_in + (int64_t)t * a.bstride;
    const int64_t b = B[s], e = B[s + 1];
    if (which == 0 ? (e - b > kTinyMax) : (e - b <= kTinyMax || e - b > kMidMax)) continue;  // CTA-uniform
    const int m = (int)(e - b);
    if (m == 0) {
      if (tid == 0) write_node(a, t, s, b, e, 0, 0.0f);
      continue;
    }
    const float *Pc = a.P + ((int64_t)t * a.depth + a.lev) * a.n;
    const int32_t *oin = a.order_in + (int64_t)t * a.n + b;
    int32_t *oout = a.order_out + (int64_t)t * a.n + b;
    uint32_t mn = 0xffffffffu, mx = 0u;
    for (int i = tid; i < m; i += kNT) {
      const int32_t id = oin[i];
      const uint32_t k = f2key(__ldg(Pc + id));
      keys[i] = k;
      ids[i] = id;
      mn = k < mn ? k : mn;
      mx = k > mx ? k : mx;
    }
    block_minmax(mn, mx, red_mn, red_mx);  // includes the barrier publishing keys/ids
    const int kth = (m + 1) / 2 - 1;
    uint32_t K;
    int nle;
    if (mn == mx) {
      K = mn;
      nle = m;
    } else {
      int nb = __clz(mn ^ mx);
      uint32_t prefix = nb ? (mn & (0xffffffffu << (32 - nb))) : 0u;
      int krem = kth, cnt_last = 0;
      while (nb < 32) {
        const int w8 = (32 - nb) < 8 ? (32 - nb) : 8;
        const int shift = 32 - nb - w8;
        const uint32_t dmask = (1u << w8) - 1u;
        hist[tid] = 0u;  // kNT == 256 bins
        __syncthreads();
        for (int i = tid; i < m; i += kNT) {
          const uint32_t k = keys[i];
          if (prefix_match(k, prefix, nb)) atomicAdd(&hist[(k >> shift) & dmask], 1u);
        }
        __syncthreads();
        if (warp == 0) {
          int bin, below, cnt;
          warp_pick(hist, krem, bin, below, cnt);
          if (lane == 0) {
            s_bin = bin;
            s_below = below;
            s_cnt = cnt;
          }
        }
        __syncthreads();
        prefix |= (uint32_t)s_bin << shift;
        krem -= s_below;
        cnt_last = s_cnt;
        nb += w8;
        __syncthreads();
      }
      K = prefix;
      nle = kth - krem + cnt_last;
    }
    // stable partition: rounds of kNT elements, ballot ranks
    int base_left = 0;
    for (int r0 = 0; r0 < m; r0 += kNT) {
      const int i = r0 + tid;
      const bool valid = i < m;
      const bool f = valid && keys[i] <= K;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) wcnt[warp] = __popc(bal);
      __syncthreads();
      int before = 0, tot = 0;
#pragma unroll
      for (int w2 = 0; w2 < kNT / 32; ++w2) {
        const int c = wcnt[w2];
        before += w2 < warp ? c : 0;
        tot += c;
      }
      const int lrank = base_left + before + __popc(bal & lanemask_lt());
      if (valid) oout[f ? lrank : nle + (i - lrank)] = ids[i];
      base_left += tot;
      __syncthreads();
    }
    if (tid == 0) write_node(a, t, s, b, e, nle, key2f(K));
    __syncthreads();
  }
}

// ---- big path -------------------------------------------------------------
__global__ void __launch_bounds__(kNT) k_big_keys(LevelArgs a) {
  __shared__ uint32_t red_mn[kNT / 32], red_mx[kNT / 32];
  const int64_t nch = a.ctl->nchunks;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const int2 ch = a.chunks[c];
    BigSeg *g = a.big + ch.x;
    const int64_t p0 = g->b + (int64_t)ch.y * kChunk;
    const int64_t p1 = (p0 + kChunk) < g->e ? (p0 + kChunk) : g->e;
    const int t = g->t;
    const float *Pc = a.P + ((int64_t)t * a.depth + a.lev) * a.n;
    const int32_t *oin = a.order_in + (int64_t)t * a.n;
    uint32_t *kb = a.keys + (int64_t)t * a.n;
    uint32_t mn = 0xffffffffu, mx = 0u;
    constexpr int U = 8;  // independent gathers in flight per thread
    for (int64_t r0 = p0 + threadIdx.x; r0 < p1; r0 += (int64_t)U * kNT) {
      int32_t id[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int64_t p = r0 + (int64_t)j * kNT;
        id[j] = p < p1 ? __ldg(oin + p) : -1;
      }
      float v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = id[j] >= 0 ? __ldg(Pc + id[j]) : 0.f;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (id[j] >= 0) {
          const uint32_t k = f2key(v[j]);
          kb[r0 + (int64_t)j * kNT] = k;
          mn = k < mn ? k : mn;
          mx = k > mx ? k : mx;
        }
      }
    }
    block_minmax(mn, mx, red_mn, red_mx);
    if (threadIdx.x == 0) {
      atomicMin(&g->kmin, mn);
      atomicMax(&g->kmax, mx);
    }
  }
}

__global__ void k_big_init(LevelArgs a) {
  const int nbig = a.ctl->nbig;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nbig; i += gridDim.x * blockDim.x) {
    BigSeg *g = a.big + i;
    const uint32_t mn = g->kmin, mx = g->kmax;
    if (mn == mx) {
      g->prefix = mn;
      g->nb = 32;
      g->done = 1;
      g->nle = (int32_t)(g->e - g->b);
    } else {
      const int nb = __clz(mn ^ mx);
      g->nb = nb;
      g->prefix = nb ? (mn & (0xffffffffu << (32 - nb))) : 0u;
    }
  }
}

// Calls f(key) for every element of kb[p0, p1) (one chunk, <= kChunk
// elements): the 16-byte-aligned body as uint4 loads, all of a thread's
// loads issued before any key is used (one memory round trip per chunk);
// the unaligned head and tail (< 4 elements each) element-wise.
template <typename F>
__device__ __forceinline__ void for_chunk_keys(const uint32_t *__restrict__ kb, int64_t p0, int64_t p1, F f) {
  const int64_t mis = (int64_t)(((uintptr_t)(kb + p0) >> 2) & 3);
  int64_t a0 = p0 + ((4 - mis) & 3);
  if (a0 > p1) a0 = p1;
  const int64_t a1 = a0 + ((p1 - a0) & ~3LL);
  if (p0 + threadIdx.x < a0) f(__ldg(kb + p0 + threadIdx.x));
  if (a1 + threadIdx.x < p1) f(__ldg(kb + a1 + threadIdx.x));
  const uint4 *k4 = reinterpret_cast<const uint4 *>(kb + a0);
  const int nv = (int)((a1 - a0) >> 2);
  constexpr int U = kChunk / 4 / kNT;
  for (int v0 = threadIdx.x; v0 < nv; v0 += U * kNT) {
    uint4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = v0 + j * kNT;
      r[j] = i < nv ? __ldg(k4 + i) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (v0 + j * kNT < nv) {
        f(r[j].x);
        f(r[j].y);
        f(r[j].z);
        f(r[j].w);
      }
    }
  }
}

__global__ void __launch_bounds__(kNT) k_big_hist(LevelArgs a) {
  __shared__ uint32_t hist[256];
  const int64_t nch = a.ctl->nchunks;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const int2 ch = a.chunks[c];
    const BigSeg *g = a.big + ch.x;
    if (g->done) continue;  // uniform per CTA
    const int nb = g->nb;
    const uint32_t prefix = g->prefix;
    const int w8 = (32 - nb) < 8 ? (32 - nb) : 8;
    const int shift = 32 - nb - w8;
    const uint32_t dmask = (1u << w8) - 1u;
    const int64_t p0 = g->b + (int64_t)ch.y * kChunk;
    const int64_t p1 = (p0 + kChunk) < g->e ? (p0 + kChunk) : g->e;
    const uint32_t *kb = a.keys + (int64_t)g->t * a.n;
    hist[threadIdx.x] = 0u;
    __syncthreads();
    for_chunk_keys(kb, p0, p1, [&](uint32_t k) {
      if (prefix_match(k, prefix, nb)) atomicAdd(&hist[(k >> shift) & dmask], 1u);
    });
    __syncthreads();
    const uint32_t v = hist[threadIdx.x];
    if (v) atomicAdd(a.ghist + (int64_t)ch.x * 256 + threadIdx.x, v);
    __syncthreads();
  }
}

// Stable partition of one chunk with 16-byte loads: thread i of a round
// owns the four consecutive positions of 16-byte group i (groups aligned on
// the address, positions outside [p0, p1) masked), so positions are in
// thread order and a warp scan of the per-thread left counts gives every
// element's rank -- the same ranks as the element-wise k_big_scatter.
__global__ void __launch_bounds__(kNT) k_big_scatter4(LevelArgs a) {
  constexpr int NW = kNT / 32;
  constexpr int SR = 2;  // rounds of kNT groups per barrier pair
  __shared__ int wcnt[SR][NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nch = a.ctl->nchunks;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const int2 ch = a.chunks[c];
    const BigSeg *g = a.big + ch.x;
    const uint32_t K = g->prefix;
    const int64_t b = g->b;
    const int64_t p0 = b + (int64_t)ch.y * kChunk;
    const int64_t p1 = (p0 + kChunk) < g->e ? (p0 + kChunk) : g->e;
    const int64_t nle = g->nle;
    const uint32_t *kb = a.keys + (int64_t)g->t * a.n;
    const int32_t *oin = a.order_in + (int64_t)g->t * a.n;
    int32_t *oout = a.order_out + (int64_t)g->t * a.n;
    const int64_t pa = p0 - (int64_t)(((uintptr_t)(kb + p0) >> 2) & 3);  // first group's position
    int64_t base_left = a.chunk_off[c];
    // software pipelined: the next round's keys and ids are loaded before
    // this round's ranks are published and its ids stored
    uint4 kk[SR];
    int4 id[SR];
#pragma unroll
    for (int j = 0; j < SR; ++j) {
      const int64_t q = pa + ((int64_t)j * kNT + threadIdx.x) * 4;  // group start position
      const bool any = q < p1;
      kk[j] = any ? __ldg(reinterpret_cast<const uint4 *>(kb + q)) : make_uint4(0u, 0u, 0u, 0u);
      id[j] = any ? __ldg(reinterpret_cast<const int4 *>(oin + q)) : make_int4(0, 0, 0, 0);
    }
    for (int64_t r0 = pa; r0 < p1; r0 += (int64_t)SR * kNT * 4) {
      int fl[SR], cl[SR], incl[SR];
#pragma unroll
      for (int j = 0; j < SR; ++j) {
        const int64_t q = r0 + ((int64_t)j * kNT + threadIdx.x) * 4;
        const uint32_t kv[4] = {kk[j].x, kk[j].y, kk[j].z, kk[j].w};
        int f = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (q + e >= p0 && q + e < p1 && kv[e] <= K) f |= 1 << e;
        fl[j] = f;
        cl[j] = __popc(f);
        int x = cl[j];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += u;
        }
        incl[j] = x;
        if (lane == 31) wcnt[j][warp] = x;
      }
      int4 idc[SR];
#pragma unroll
      for (int j = 0; j < SR; ++j) idc[j] = id[j];
      const int64_t rn = r0 + (int64_t)SR * kNT * 4;
#pragma unroll
      for (int j = 0; j < SR; ++j) {
        const int64_t q = rn + ((int64_t)j * kNT + threadIdx.x) * 4;
        const bool any = q < p1;
        kk[j] = any ? __ldg(reinterpret_cast<const uint4 *>(kb + q)) : make_uint4(0u, 0u, 0u, 0u);
        id[j] = any ? __ldg(reinterpret_cast<const int4 *>(oin + q)) : make_int4(0, 0, 0, 0);
      }
      __syncthreads();
      int tot = 0;
#pragma unroll
      for (int j = 0; j < SR; ++j) {
        int bj = tot;
#pragma unroll
        for (int w2 = 0; w2 < NW; ++w2) {
          const int cc = wcnt[j][w2];
          bj += w2 < warp ? cc : 0;
          tot += cc;
        }
        const int64_t q = r0 + ((int64_t)j * kNT + threadIdx.x) * 4;
        int64_t lrank = base_left + bj + incl[j] - cl[j];
        const int iv[4] = {idc[j].x, idc[j].y, idc[j].z, idc[j].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t p = q + e;
          if (p >= p0 && p < p1) {
            const bool left = (fl[j] >> e) & 1;
            oout[left ? b + lrank : b + nle + ((p - b) - lrank)] = iv[e];
            lrank += left ? 1 : 0;
          }
        }
      }
      base_left += tot;
      __syncthreads();
    }
  }
}

// One warp per big segment.
__global__ void k_big_pick(LevelArgs a) {
  const int nbig = a.ctl->nbig;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < nbig; i += gridDim.x * wpb) {
    BigSeg *g = a.big + i;
    if (g->done) continue;
    uint32_t *h = a.ghist + (int64_t)i * 256;
    const int nb = g->nb;
    const int w8 = (32 - nb) < 8 ? (32 - nb) : 8;
    const int shift = 32 - nb - w8;
    int bin, below, cnt;
    warp_pick(h, g->krem, bin, below, cnt);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) h[lane * 8 + j] = 0u;
    if (lane == 0) {
      g->prefix |= (uint32_t)bin << shift;
      g->krem -= below;
      g->cnt_last = cnt;
      g->nb = nb + w8;
      if (nb + w8 == 32) {
        g->done = 1;
        g->nle = g->kth - g->krem + cnt;
      }
    }
  }
}

__global__ void __launch_bounds__(kNT) k_big_count(LevelArgs a) {
  __shared__ int wsum[kNT / 32];
  const int64_t nch = a.ctl->nchunks;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const int2 ch = a.chunks[c];
    const BigSeg *g = a.big + ch.x;
    const uint32_t K = g->prefix;
    const int64_t p0 = g->b + (int64_t)ch.y * kChunk;
    const int64_t p1 = (p0 + kChunk) < g->e ? (p0 + kChunk) : g->e;
    const uint32_t *kb = a.keys + (int64_t)g->t * a.n;
    int cnt = 0;
    for_chunk_keys(kb, p0, p1, [&](uint32_t k) { cnt += k <= K ? 1 : 0; });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < kNT / 32; ++w) tot += wsum[w];
      a.chunk_left[c] = tot;
    }
    __syncthreads();
  }
}

// One warp per big segment: exclusive scan of its chunks' left counts.
__global__ void k_big_scan(LevelArgs a) {
  const int nbig = a.ctl->nbig;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < nbig; i += gridDim.x * wpb) {
    BigSeg *g = a.big + i;
    int run = 0;
    for (int c0 = 0; c0 < g->nchunks; c0 += 32) {
      const int c = c0 + lane;
      const int v = c < g->nchunks ? a.chunk_left[g->chunk_base + c] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (c < g->nchunks) a.chunk_off[g->chunk_base + c] = run + incl - v;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      g->nle = run;  // == kth - krem + cnt_last
      write_node(a, g->t, g->s, g->b, g->e, run, key2f(g->prefix));
    }
  }
}

__global__ void __launch_bounds__(kNT) k_big_scatter(LevelArgs a) {
  // sub-rounds of kNT elements per barrier pair (8 or 16 measured slower:
  // 140 / 242 registers leave one CTA per SM)
  constexpr int SR = 4;
  constexpr int NW = kNT / 32;
  __shared__ int wcnt[SR][NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nch = a.ctl->nchunks;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const int2 ch = a.chunks[c];
    const BigSeg *g = a.big + ch.x;
    const uint32_t K = g->prefix;
    const int64_t b = g->b;
    const int64_t p0 = b + (int64_t)ch.y * kChunk;
    const int64_t p1 = (p0 + kChunk) < g->e ? (p0 + kChunk) : g->e;
    const int64_t nle = g->nle;
    const uint32_t *kb = a.keys + (int64_t)g->t * a.n;
    const int32_t *oin = a.order_in + (int64_t)g->t * a.n;
    int32_t *oout = a.order_out + (int64_t)g->t * a.n;
    int64_t base_left = a.chunk_off[c];
    for (int64_t r0 = p0; r0 < p1; r0 += (int64_t)SR * kNT) {
      uint32_t kk[SR];
      int32_t id[SR];
      bool f[SR];
      unsigned bal[SR];
#pragma unroll
      for (int j = 0; j < SR; ++j) {
        const int64_t p = r0 + (int64_t)j * kNT + threadIdx.x;
        const bool valid = p < p1;
        kk[j] = valid ? __ldg(kb + p) : 0xffffffffu;
        id[j] = valid ? __ldg(oin + p) : 0;
      }
#pragma unroll
      for (int j = 0; j < SR; ++j) {
        const int64_t p = r0 + (int64_t)j * kNT + threadIdx.x;
        f[j] = p < p1 && kk[j] <= K;
        bal[j] = __ballot_sync(0xffffffffu, f[j]);
        if (lane == 0) wcnt[j][warp] = __popc(bal[j]);
      }
      __syncthreads();
      int tot = 0;
      int before[SR];
#pragma unroll
      for (int j = 0; j < SR; ++j) {
        int bj = tot;
#pragma unroll
        for (int w2 = 0; w2 < NW; ++w2) {
          const int cc = wcnt[j][w2];
          bj += w2 < warp ? cc : 0;
          tot += cc;
        }
        before[j] = bj;
      }
#pragma unroll
      for (int j = 0; j < SR; ++j) {
        const int64_t p = r0 + (int64_t)j * kNT + threadIdx.x;
        if (p < p1) {
          const int64_t lrank = base_left + before[j] + __popc(bal[j] & lanemask_lt());
          oout[f[j] ? b + lrank : b + nle + ((p - b) - lrank)] = id[j];
        }
      }
      base_left += tot;
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
struct WsLayout {
  size_t order_tmp, bounds_tmp, keys, ctl, tiny, mid, big, ghist, chunks, cleft, coff, tnch, tbase, total;
};

static size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

static WsLayout layout(int64_t n, int Tb, int depth) {
  WsLayout L;
  const int64_t nleaf = (int64_t)1 << depth;
  const int64_t max_level_segs = (int64_t)Tb * (depth > 0 ? (nleaf >> 1) : 1);
  int64_t big_per_tree = n / (kMidMax + 1);
  if (depth > 0 && big_per_tree > (nleaf >> 1)) big_per_tree = nleaf >> 1;
  const int64_t maxbig = (int64_t)Tb * big_per_tree + 1;
  const int64_t maxchunks = (int64_t)Tb * (n / kChunk + big_per_tree + 1) + 1;
  size_t off = 0;
  L.order_tmp = off; off = align_up(off + sizeof(int32_t) * (size_t)Tb * n);
  L.bounds_tmp = off; off = align_up(off + sizeof(int64_t) * (size_t)Tb * (nleaf + 1));
  L.keys = off; off = align_up(off + sizeof(uint32_t) * (size_t)Tb * n);
  L.ctl = off; off = align_up(off + sizeof(LevelCtl));
  L.tiny = off; off = align_up(off + sizeof(int32_t) * (size_t)max_level_segs);
  L.mid = off; off = align_up(off + sizeof(int32_t) * (size_t)max_level_segs);
  L.big = off; off = align_up(off + sizeof(BigSeg) * (size_t)maxbig);
  L.ghist = off; off = align_up(off + sizeof(uint32_t) * 256 * (size_t)maxbig);
  L.chunks = off; off = align_up(off + sizeof(int2) * (size_t)maxchunks);
  L.cleft = off; off = align_up(off + sizeof(int32_t) * (size_t)maxchunks);
  L.coff = off; off = align_up(off + sizeof(int32_t) * (size_t)maxchunks);
  L.tnch = off; off = align_up(off + sizeof(int32_t) * (size_t)Tb);
  L.tbase = off; off = align_up(off + sizeof(int64_t) * (size_t)Tb);
  L.total = off;
  return L;
}

}  // namespace mrpt

using namespace mrpt;

static int32_t check_build_args(int64_t n, int32_t Tb, int32_t depth) {
  if (n < 1 || n >= (int64_t)1 << 31) return fail(MRPT_ESHAPE, "build: n must lie in [1, 2^31)");
  if (Tb < 1) return fail(MRPT_EPARAM, "build: Tb must be >= 1");
  if (depth < 0 || depth > 24) return fail(MRPT_EPARAM, "build: depth must lie in [0, 24]");
  if ((int64_t)Tb * ((int64_t)1 << depth) >= (int64_t)1 << 31)
    return fail(MRPT_EPARAM, "build: Tb * 2^depth too large for one batch");
  return MRPT_OK;
}

extern "C" int32_t mrpt_build_workspace_size(int64_t n, int32_t Tb, int32_t depth, size_t *bytes) {
  clear_error();
  int32_t st = check_build_args(n, Tb, depth);
  if (st) return st;
  if (!bytes) return fail(MRPT_EPARAM, "build: null bytes");
  *bytes = layout(n, Tb, depth).total;
  return MRPT_OK;
}

extern "C" int32_t mrpt_build_levels(const float *P, int64_t n, int32_t Tb, int32_t depth,
                                     float *splits, int64_t *leaf_offsets, int32_t *leaf_indices,
                                     void *ws, size_t ws_bytes, void *stream) {
  clear_error();
  int32_t st = check_build_args(n, Tb, depth);
  if (st) return st;
  const WsLayout L = layout(n, Tb, depth);
  if (ws_bytes < L.total || !ws) return fail(MRPT_EWORKSPACE, "build: workspace too small");
  cudaStream_t s = as_stream(stream);
  char *w = static_cast<char *>(ws);
  const int64_t nleaf = (int64_t)1 << depth;
  const int64_t bstride = nleaf + 1;
  int32_t *obuf[2];
  int64_t *bbuf[2];
  obuf[depth & 1] = leaf_indices;
  obuf[(depth + 1) & 1] = reinterpret_cast<int32_t *>(w + L.order_tmp);
  bbuf[depth & 1] = leaf_offsets;
  bbuf[(depth + 1) & 1] = reinterpret_cast<int64_t *>(w + L.bounds_tmp);
  {
    const int64_t total = (int64_t)Tb * n;
    const int64_t blocks = ceil_div<int64_t>(total, 256);
    const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
    (count_launch(), k_build_init<<<grid, 256, 0, s>>>(obuf[0], bbuf[0], n, Tb, bstride));
  }
  const int sms = num_sms();
  cudaFuncSetAttribute(k_seg_small<kMidMax>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMidMax * 8);
  for (int lev = 0; lev < depth; ++lev) {
    LevelArgs a;
    a.P = P;
    a.n = n;
    a.depth = depth;
    a.lev = lev;
    a.Tb = Tb;
    a.order_in = obuf[lev & 1];
    a.order_out = obuf[(lev + 1) & 1];
    a.bounds_in = bbuf[lev & 1];
    a.bounds_out = bbuf[(lev + 1) & 1];
    a.bstride = bstride;
    a.splits = splits;
    a.sstride = nleaf - 1;
    a.keys = reinterpret_cast<uint32_t *>(w + L.keys);
    a.ctl = reinterpret_cast<LevelCtl *>(w + L.ctl);
    a.tiny_list = reinterpret_cast<int32_t *>(w + L.tiny);
    a.mid_list = reinterpret_cast<int32_t *>(w + L.mid);
    a.big = reinterpret_cast<BigSeg *>(w + L.big);
    a.ghist = reinterpret_cast<uint32_t *>(w + L.ghist);
    a.chunks = reinterpret_cast<int2 *>(w + L.chunks);
    a.chunk_left = reinterpret_cast<int32_t *>(w + L.cleft);
    a.chunk_off = reinterpret_cast<int32_t *>(w + L.coff);
    a.tree_nch = reinterpret_cast<int32_t *>(w + L.tnch);
    a.tree_base = reinterpret_cast<int64_t *>(w + L.tbase);
    cudaMemsetAsync(a.ctl, 0, sizeof(LevelCtl), s);
    cudaMemsetAsync(a.tree_nch, 0, sizeof(int32_t) * (size_t)Tb, s);
    const int64_t nsegs = (int64_t)Tb << lev;
    (count_launch(), k_level_plan<<<(unsigned)ceil_div<int64_t>(nsegs, 256), 256, 0, s>>>(a));
    // expected per-segment size decides how many CTAs the small paths get
    const int64_t est = n >> lev;
    const int64_t tiny_grid = nsegs < (int64_t)sms * 8 ? nsegs : (int64_t)sms * 8;
    // one CTA per segment for the same L2 locality of the projection gathers
    static const bool small_flat = [] {
      const char *e = getenv("MRPT_BUILD_SMALL_FLAT");  // "0": grid-stride loop
      return !(e && atoi(e) == 0);
    }();
    const unsigned flat_grid = (unsigned)(nsegs < 0x7fffffff ? nsegs : 0x7fffffff);
    (count_launch(), k_seg_small<kTinyMax><<<small_flat ? flat_grid
                                                        : (unsigned)(est <= kTinyMax ? tiny_grid : (tiny_grid < sms ? tiny_grid : sms)),
                             kNT, kTinyMax * 8, s>>>(a, 0));
    const int64_t mid_grid = small_flat ? (int64_t)flat_grid : (nsegs < (int64_t)sms * 3 ? nsegs : (int64_t)sms * 3);
    (count_launch(), k_seg_small<kMidMax><<<(unsigned)mid_grid, kNT, kMidMax * 8, s>>>(a, 1));
    if (est > kMidMax || lev > 0) {
      // the big path may have work whenever a segment can exceed kMidMax;
      // after level 0 ties can make any segment large, so always launch.
      static const int big_per_sm = [] {
        // 8 resident 256-thread CTAs per SM for the streaming passes
        // (config 5 half scale: 549 vs 558 ms for hist + count + scatter + keys)
        const char *e = getenv("MRPT_BUILD_CTAS_PER_SM");  // experiments
        const int v = e ? atoi(e) : 8;
        return v < 1 ? 1 : (v > 8 ? 8 : v);
      }();
      const int big_grid = sms * big_per_sm;
      (count_launch(), k_chunk_layout<<<1, 1024, 0, s>>>(a));
      (count_launch(), k_chunk_fill<<<sms * 2, 256, 0, s>>>(a));
      // The gather P[t][lev][order[i]] re-reads a tree's projection column
      // once per segment; with one CTA per chunk (in-order dispatch keeps the
      // resident chunks within about one tree) those re-reads hit L2 -- a
      // grid-stride loop let CTAs drift over several trees and read DRAM ~2x
      // (config 5 half scale: 1099 -> 602 GB, 229 -> 155 ms).
      static const bool keys_flat = [] {
        const char *e = getenv("MRPT_BUILD_KEYS_FLAT");  // "0": grid-stride loop
        return !(e && atoi(e) == 0);
      }();
      // chunk count bound (device-side count unknown here): big segments hold
      // > kChunk points each, so chunks <= 2 * n * Tb / kChunk
      const int64_t chunk_bound = 2 * ceil_div<int64_t>(a.n * (int64_t)a.Tb, kChunk);
      const int keys_grid = keys_flat ? (int)(chunk_bound < 0x7fffffff ? chunk_bound : 0x7fffffff) : big_grid;
      (count_launch(), k_big_keys<<<keys_grid, kNT, 0, s>>>(a));
      (count_launch(), k_big_init<<<ceil_div<int>(sms, 1), 256, 0, s>>>(a));
      for (int pass = 0; pass < 4; ++pass) {
        (count_launch(), k_big_hist<<<big_grid, kNT, 0, s>>>(a));
        (count_launch(), k_big_pick<<<sms, 256, 0, s>>>(a));
      }
      (count_launch(), k_big_count<<<big_grid, kNT, 0, s>>>(a));
      (count_launch(), k_big_scan<<<sms, 256, 0, s>>>(a));
      static const bool scatter4 = [] {
        const char *e = getenv("MRPT_BUILD_SCATTER4");  // "0": the element-wise scatter
        return !(e && atoi(e) == 0);
      }();
      if (scatter4 && (((uintptr_t)a.keys | (uintptr_t)a.order_in) & 15) == 0)
        (count_launch(), k_big_scatter4<<<big_grid, kNT, 0, s>>>(a));
      else
        (count_launch(), k_big_scatter<<<big_grid, kNT, 0, s>>>(a));
    }
  }
  return launch_status("mrpt_build_levels");
}
