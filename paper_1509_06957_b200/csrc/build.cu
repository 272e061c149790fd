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
//   tiny  (m <= 2048)          one CTA of 128, keys+ids staged in 16 KB smem
//   mid   (2048 < m <= 8192)   one CTA of 256, keys in 32 KB smem (ids re-read)
//   large (8192 < m <= 23552)  one CTA of 1024, keys in 92 KB smem (ids are
//                              re-read for the partition), segments taken
//                              from a tree-major list
//   big   (m > 23552)          chunked over many CTAs: key gather pass,
//                              up to four 8-bit histogram passes with global
//                              histograms, count / scan / stable scatter.
// The radix select first strips the prefix shared by the segment's min and
// max key, so the first histogram already splits the live key range.
#include "common.cuh"

namespace mrpt {

constexpr int kTinyMax = 2048;
constexpr int kMidMax = 8192;
constexpr int kLargeMax = 47104;   // 184 KB of keys + 8 KB of buckets: one CTA per SM
constexpr int kLargeMax2 = 23552;  // 92 KB of keys: two CTAs per SM
constexpr int kLinList = 512;     // bucket members ranked by counting (else: radix select)
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
  int32_t ntiny, nmid, nbig, nlarge;
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
  int32_t *tree_nlg;   // (Tb) large segments per tree this level
  int32_t *tree_lfill; // (Tb) large segments of the tree already listed
  int64_t *tree_lbase; // (Tb) first list slot of each tree
  int32_t *large_list; // tree-major list of this level's large segments
  int large_max;       // upper size of the large class (kMidMax: no large class)
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
  if (m > kMidMax && m <= a.large_max) {
    atomicAdd(&a.tree_nlg[t], 1);  // listed tree-major by k_large_fill
  } else if (m > a.large_max) {  // tiny / mid segments are found by k_seg_cta itself
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

// Exclusive scan of a per-tree count array by one CTA of 1024; returns the
// total in every thread.
__device__ __forceinline__ int64_t scan_trees(const int32_t *cnt, int64_t *base, int Tb, int64_t *wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t carry = 0;
  for (int t0 = 0; t0 < Tb; t0 += 1024) {
    const int t = t0 + threadIdx.x;
    const int64_t v = t < Tb ? cnt[t] : 0;
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
    if (t < Tb) base[t] = carry + wsum[warp] + incl - v;
    carry += wsum[32];
    __syncthreads();
  }
  return carry;
}

// Tree-major tables: the big path's chunk table and the list of large
// segments start, per tree, at the exclusive scan of the per-tree counts.
__global__ void __launch_bounds__(1024) k_chunk_layout(LevelArgs a) {
  __shared__ int64_t wsum[33];
  const int64_t nch = scan_trees(a.tree_nch, a.tree_base, a.Tb, wsum);
  const int64_t nlg = scan_trees(a.tree_nlg, a.tree_lbase, a.Tb, wsum);
  if (threadIdx.x == 0) {
    a.ctl->nchunks = nch;
    a.ctl->nlarge = (int32_t)nlg;
  }
}

// One thread per segment: large segments enter the list at their tree's base
// (any order within a tree; what matters is that consecutive entries gather
// from the same projection column).
__global__ void k_large_fill(LevelArgs a) {
  const int nseg = 1 << a.lev;
  const int64_t total = (int64_t)a.Tb * nseg;
  const int64_t seg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (seg >= total) return;
  const int t = (int)(seg >> a.lev), s = (int)(seg & (nseg - 1));
  const int64_t *B = a.bounds_in + (int64_t)t * a.bstride;
  const int64_t m = B[s + 1] - B[s];
  if (m > kMidMax && m <= a.large_max)
    a.large_list[a.tree_lbase[t] + atomicAdd(&a.tree_lfill[t], 1)] = (int32_t)seg;
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

// Exact rank select over m keys staged in shared memory: K = the kth
// smallest key (0-based), nle = the number of keys <= K; every thread gets
// both.  mn / mx: the calling thread's partial min / max of the keys it
// stored (the first barrier inside also publishes the keys).
template <int NT, int NB>
__device__ __forceinline__ void cta_select(const uint32_t *keys, int m, int kth, uint32_t mn, uint32_t mx,
                                           uint32_t *hist, uint32_t *red, int *sh, uint32_t &Kout, int &nle_out) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // block min / max (the barrier also publishes keys / ids)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint32_t x = __shfl_xor_sync(0xffffffffu, mn, o), y = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = x < mn ? x : mn;
    mx = y > mx ? y : mx;
  }
  if (lane == 0) {
    red[warp] = mn;
    red[NW + warp] = mx;
  }
  __syncthreads();
  {
    uint32_t x = lane < NW ? red[lane] : 0xffffffffu, y = lane < NW ? red[NW + lane] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint32_t x2 = __shfl_xor_sync(0xffffffffu, x, o), y2 = __shfl_xor_sync(0xffffffffu, y, o);
      x = x2 < x ? x2 : x;
      y = y2 > y ? y2 : y;
    }
    mn = x;
    mx = y;
  }
  uint32_t K = mn;
  int nle = m;
  bool solved = mn == mx;
  // Linear buckets first: bucket(v) = min(NB-1, int((v - vmin) * scale))
  // is non-decreasing in v (rounded subtraction, multiplication by a positive
  // constant and truncation all are), so the bucket holding rank kth holds
  // the median, and its few members are ranked exactly by their keys.  The
  // 8-bit digits of a float key put a whole segment into a handful of bins
  // (sign and exponent bits), i.e. thousands of same-address shared atomics.
  if (!solved) {
    const float vmin = key2f(mn), span = key2f(mx) - vmin;
    const float scale = (float)NB / span;
    if (isfinite(span) && isfinite(scale)) {
      constexpr int BPT = NB / NT;  // consecutive buckets per thread
      for (int i = tid; i < NB; i += NT) hist[i] = 0u;
      if (tid == 0) sh[3] = 0;
      __syncthreads();
      for (int i = tid; i < m; i += NT) {
        const int bk = (int)((key2f(keys[i]) - vmin) * scale);
        atomicAdd(&hist[bk < NB - 1 ? bk : NB - 1], 1u);
      }
      __syncthreads();
      uint32_t hv[BPT];
      int sum = 0;
#pragma unroll
      for (int j = 0; j < BPT; ++j) {
        hv[j] = hist[tid * BPT + j];
        sum += (int)hv[j];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      int *wtot = sh + 4;
      if (lane == 31) wtot[warp] = incl;
      __syncthreads();
      int wbase = lane < warp ? wtot[lane] : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wbase += __shfl_xor_sync(0xffffffffu, wbase, o);
      int excl = wbase + incl - sum;
      if (excl <= kth && kth < excl + sum) {  // exactly one thread
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
          if (kth < excl + (int)hv[j]) {
            sh[0] = tid * BPT + j;
            sh[1] = excl;
            sh[2] = (int)hv[j];
            break;
          }
          excl += (int)hv[j];
        }
      }
      __syncthreads();
      const int bsel = sh[0], below = sh[1], cnt = sh[2];
      if (cnt <= kLinList) {
        uint32_t *list = hist;  // the counts are no longer needed
        for (int i = tid; i < m; i += NT) {
          const uint32_t k = keys[i];
          const int bk = (int)((key2f(k) - vmin) * scale);
          if ((bk < NB - 1 ? bk : NB - 1) == bsel) list[atomicAdd(&sh[3], 1)] = k;
        }
        __syncthreads();
        const int r = kth - below;
        for (int j = tid; j < cnt; j += NT) {
          const uint32_t kj = list[j];
          int lt = 0, le = 0;
          for (int i = 0; i < cnt; ++i) {
            const uint32_t ki = list[i];
            lt += ki < kj ? 1 : 0;
            le += ki <= kj ? 1 : 0;
          }
          if (lt <= r && r < le) {  // every holder of the median value writes the same pair
            sh[0] = (int)kj;
            sh[1] = below + le;
          }
        }
        __syncthreads();
        K = (uint32_t)sh[0];
        nle = sh[1];
        solved = true;
      }
      __syncthreads();  // sh / hist are rewritten below
    }
  }
  if (!solved) {
    int nb = __clz(mn ^ mx);
    uint32_t prefix = nb ? (mn & (0xffffffffu << (32 - nb))) : 0u;
    int krem = kth, cnt_last = 0;
    while (nb < 32) {
      const int w8 = (32 - nb) < 8 ? (32 - nb) : 8;
      const int shift = 32 - nb - w8;
      const uint32_t dmask = (1u << w8) - 1u;
      if (tid < 256) hist[tid] = 0u;
      __syncthreads();
      for (int i = tid; i < m; i += NT) {
        const uint32_t k = keys[i];
        if (prefix_match(k, prefix, nb)) atomicAdd(&hist[(k >> shift) & dmask], 1u);
      }
      __syncthreads();
      if (warp == 0) {
        int bin, below, cnt;
        warp_pick(hist, krem, bin, below, cnt);
        if (lane == 0) {
          sh[0] = bin;
          sh[1] = below;
          sh[2] = cnt;
        }
      }
      __syncthreads();
      prefix |= (uint32_t)sh[0] << shift;
      krem -= sh[1];
      cnt_last = sh[2];
      nb += w8;
    }
    K = prefix;
    nle = kth - krem + cnt_last;
  }
  Kout = K;
  nle_out = nle;
}

// One CTA per segment with m <= MAXM: keys (and, with IDS, the ids) staged in
// shared memory, exact radix select there, stable partition by warp ranges.
//  * load: every thread issues U id loads, then U projection gathers, before
//    any key is stored (two memory round trips per U*NT elements);
//  * partition: warp w owns a contiguous range of positions, counts its
//    left-goers by ballots, one barrier publishes the warp totals, then every
//    warp writes its range at its ranks (lanes consecutive: the left and the
//    right runs are both coalesced).
template <int MAXM, int NT, int NB, bool IDS>
__device__ __forceinline__ void seg_cta(const LevelArgs &a, int t, int s, int64_t b, int64_t e,
                                        uint32_t *keys, int32_t *ids, uint32_t *hist,
                                        uint32_t *red, int *sh) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = (int)(e - b);
  const float *Pc = a.P + ((int64_t)t * a.depth + a.lev) * a.n;
  const int32_t *oin = a.order_in + (int64_t)t * a.n + b;
  int32_t *oout = a.order_out + (int64_t)t * a.n + b;
  uint32_t mn = 0xffffffffu, mx = 0u;
  constexpr int U = 8;
  for (int i0 = tid; i0 < m; i0 += U * NT) {
    int32_t id[U];
#pragma unroll
    for (int j = 0; j < U; ++j) id[j] = i0 + j * NT < m ? __ldg(oin + i0 + j * NT) : -1;
    float v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) v[j] = id[j] >= 0 ? __ldg(Pc + id[j]) : 0.f;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (id[j] >= 0) {
        const uint32_t k = f2key(v[j]);
        keys[i0 + j * NT] = k;
        if (IDS) ids[i0 + j * NT] = id[j];
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
      }
    }
  }
  uint32_t K;
  int nle;
  cta_select<NT, NB>(keys, m, (m + 1) / 2 - 1, mn, mx, hist, red, sh, K, nle);
  // stable partition by warp ranges
  int *wtot = sh + 4;
  const int R = ((m + NW - 1) / NW + 31) & ~31;
  const int r0 = warp * R;
  const int r1 = r0 + R < m ? r0 + R : m;
  int c = 0;
  for (int i = r0 + lane; i - lane < r1; i += 32)  // warp-uniform trip count
    c += __popc(__ballot_sync(0xffffffffu, i < r1 && keys[i] <= K));
  if (lane == 0) wtot[warp] = c;
  __syncthreads();
  int base = lane < warp ? wtot[lane] : 0;  // NW <= 32
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) base += __shfl_xor_sync(0xffffffffu, base, o);
  constexpr int PU = IDS ? 1 : 4;  // id re-reads in flight per lane
  for (int i0 = r0; i0 < r1; i0 += 32 * PU) {
    int32_t idv[PU];
#pragma unroll
    for (int j = 0; j < PU; ++j) {
      const int i = i0 + j * 32 + lane;
      idv[j] = i < r1 ? (IDS ? ids[i] : __ldg(oin + i)) : 0;
    }
#pragma unroll
    for (int j = 0; j < PU; ++j) {
      const int i = i0 + j * 32 + lane;
      const bool f = i < r1 && keys[i] <= K;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      const int lrank = base + __popc(bal & lanemask_lt());
      if (i < r1) oout[f ? lrank : nle + (i - lrank)] = idv[j];
      base += __popc(bal);
    }
  }
  if (tid == 0) write_node(a, t, s, b, e, nle, key2f(K));
  __syncthreads();  // keys / hist / sh are reused by the CTA's next segment
}

// Flat mode (list == nullptr): CTA i looks at segment i = t * 2^lev + s and
// returns unless its size lies in (lo, hi] -- in-order dispatch keeps the
// resident CTAs within one or two trees, whose projection columns then stay
// in L2 (an atomically appended work list interleaved all trees of the batch
// and made the gathers read DRAM ~13x the keys' bytes at config 5).  List
// mode: persistent CTAs stride over the tree-major list of large segments.
template <int MAXM, int NT, int NB, bool IDS>
__global__ void __launch_bounds__(NT) k_seg_cta(LevelArgs a, int lo, int hi, bool use_list) {
  extern __shared__ uint32_t dyn_smem[];
  uint32_t *keys = dyn_smem;                                                          // MAXM
  int32_t *ids = reinterpret_cast<int32_t *>(dyn_smem + MAXM);                        // MAXM if IDS
  __shared__ uint32_t hist[NB];
  static_assert(NB % NT == 0 && NB >= kLinList && NB >= 256, "bucket table");
  __shared__ uint32_t red[2 * NT / 32];
  __shared__ int sh[4 + NT / 32];
  const int nseg = 1 << a.lev;
  const int64_t total = use_list ? (int64_t)a.ctl->nlarge : ((int64_t)a.Tb << a.lev);
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
    const int64_t seg = use_list ? (int64_t)a.large_list[w] : w;
    const int t = (int)(seg >> a.lev), s = (int)(seg & (nseg - 1));
    const int64_t *B = a.bounds_in + (int64_t)t * a.bstride;
    const int64_t b = B[s], e = B[s + 1];
    if (e - b <= lo || e - b > hi) continue;  // CTA-uniform
    if (e == b) {
      if (threadIdx.x == 0) write_node(a, t, s, b, e, 0, 0.0f);
      continue;
    }
    seg_cta<MAXM, NT, NB, IDS>(a, t, s, b, e, keys, ids, hist, red, sh);
  }
}

}  // namespace mrpt
#include "build_top.cuh"
namespace mrpt {

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
  size_t order_tmp, bounds_tmp, keys, ctl, tiny, mid, big, ghist, chunks, cleft, coff, tnch, tbase, tlbase, llist;
  size_t tnode, tsize, tk, tinfo, tfill, thist, trange, ttable, total;
};

static size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

// Levels taken by the top path (build_top.cuh), at most kTopMaxLev.
static int top_levels(int64_t n, int depth) {
  if (n <= kLargeMax) return 0;
  int L = 0;
  // A level takes the top path while its expected node size exceeds 4,096: a
  // top level costs ~7 ms per 100 trees of 10M points, a level of
  // one-CTA-per-segment kernels ~15 (config 5: 1.765 -> 1.709 s with level 11
  // on the top path; MRPT_BUILD_TOP_MIN overrides for experiments).
  const char *te = getenv("MRPT_BUILD_TOP_MIN");  // read per call: build_ab switches it between builds
  const int64_t top_min = te ? (int64_t)atoll(te) : (int64_t)4096;
  while (L < depth && L < kTopMaxLev && (n >> L) > top_min) ++L;
  return L;
}

static WsLayout layout(int64_t n, int Tb, int depth) {
  WsLayout L;
  const int64_t nleaf = (int64_t)1 << depth;
  const int64_t max_level_segs = (int64_t)Tb * (depth > 0 ? (nleaf >> 1) : 1);
  int64_t big_per_tree = n / (kMidMax + 1);
  if (depth > 0 && big_per_tree > (nleaf >> 1)) big_per_tree = nleaf >> 1;
  int64_t large_per_tree = n / (kMidMax + 1);
  if (depth > 0 && large_per_tree > (nleaf >> 1)) large_per_tree = nleaf >> 1;
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
  L.tnch = off; off = align_up(off + sizeof(int32_t) * 3 * (size_t)Tb);  // tree_nch, tree_nlg, tree_lfill
  L.tbase = off; off = align_up(off + sizeof(int64_t) * (size_t)Tb);
  L.tlbase = off; off = align_up(off + sizeof(int64_t) * (size_t)Tb);
  L.llist = off; off = align_up(off + sizeof(int32_t) * ((size_t)Tb * large_per_tree + 1));
  const int Lc = top_levels(n, depth);
  const int64_t nrun = ceil_div<int64_t>(n, kTopBlk);
  L.tnode = off; off = align_up(off + (Lc ? sizeof(uint16_t) * (size_t)Tb * n : 0));
  L.tsize = off; off = align_up(off + (Lc ? sizeof(int32_t) * (size_t)Tb * 4 * kTopNodes : 0));
  L.tk = off; off = align_up(off + (Lc ? sizeof(uint32_t) * (size_t)Tb * kTopNodes : 0));
  L.tinfo = off; off = align_up(off + (Lc ? sizeof(int4) * (size_t)Tb * kTopNodes : 0));
  L.tfill = off; off = align_up(off + (Lc ? sizeof(int32_t) * (size_t)Tb * kTopNodes : 0));
  L.thist = off; off = align_up(off + (Lc ? sizeof(uint32_t) * (size_t)Tb * kTopBins : 0));
  L.trange = off; off = align_up(off + (Lc ? sizeof(float2) * (size_t)Tb * depth : 0));
  L.ttable = off; off = align_up(off + (Lc ? sizeof(int32_t) * (size_t)Tb * nrun * ((size_t)1 << kTopDigit) : 0));
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
  const int sms = num_sms();
  int Lc = top_levels(n, depth);
  if (const char *e = getenv("MRPT_BUILD_TOP"))  // experiments: "0" = every level through the permutation
    if (atoi(e) == 0) Lc = 0;
  if (Lc == 0) {
    const int64_t total = (int64_t)Tb * n;
    const int64_t blocks = ceil_div<int64_t>(total, 256);
    const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
    (count_launch(), k_build_init<<<grid, 256, 0, s>>>(obuf[0], bbuf[0], n, Tb, bstride));
  } else {
    TopArgs ta;
    ta.P = P;
    ta.n = n;
    ta.depth = depth;
    ta.Tb = Tb;
    ta.Lc = Lc;
    ta.node = reinterpret_cast<uint16_t *>(w + L.tnode);
    ta.tsize = reinterpret_cast<int32_t *>(w + L.tsize);
    ta.tK = reinterpret_cast<uint32_t *>(w + L.tk);
    ta.tinfo = reinterpret_cast<int4 *>(w + L.tinfo);
    ta.tfill = reinterpret_cast<int32_t *>(w + L.tfill);
    ta.ghist = reinterpret_cast<uint32_t *>(w + L.thist);
    ta.colrange = reinterpret_cast<float2 *>(w + L.trange);
    ta.lists = reinterpret_cast<uint32_t *>(w + L.keys);  // the chunked path's key buffer is free here
    ta.table = reinterpret_cast<int32_t *>(w + L.ttable);
    ta.sid = obuf[(Lc + 1) & 1];                                  // the other order buffer, unused so far
    ta.snode = reinterpret_cast<uint16_t *>(w + L.keys);         // after the last select the lists are dead
    ta.nrun = ceil_div<int64_t>(n, kTopBlk);
    ta.splits = splits;
    ta.sstride = nleaf - 1;
    ta.bounds = bbuf[Lc & 1];
    ta.bstride = bstride;
    ta.order = obuf[Lc & 1];
    ta.lev = 0;
    ta.NB = kTopMaxNB;
    cudaFuncSetAttribute(k_top_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, kTopBins * 4);
    cudaFuncSetAttribute(k_top_select<kTopListLarge, 1024, 2048>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kTopListLarge * 4);
    cudaFuncSetAttribute(k_top_collect, cudaFuncAttributeMaxDynamicSharedMemorySize, kTopBuf * 8);
    const unsigned nchunk = (unsigned)ceil_div<int64_t>(n, kTopChunk);
    (count_launch(), k_top_range<<<(unsigned)(Tb * depth), 256, 0, s>>>(ta));
    (count_launch(), k_top_init<<<(unsigned)ceil_div<int64_t>((int64_t)Tb * kTopBins, 256), 256, 0, s>>>(ta));
    for (int lev = 0; lev < Lc; ++lev) {
      ta.lev = lev;
      ta.NB = (kTopBins >> lev) < kTopMaxNB ? (kTopBins >> lev) : kTopMaxNB;
      const dim3 gchunk(nchunk, (unsigned)Tb), gnode(1u << lev, (unsigned)Tb);
      (count_launch(), k_top_hist<<<gchunk, 1024, (size_t)(ta.NB << lev) * 4, s>>>(ta));
      (count_launch(), k_top_pick<<<(unsigned)Tb, 1024, 0, s>>>(ta));
      (count_launch(), k_top_collect<<<gchunk, 1024, kTopBuf * 8, s>>>(ta));
      (count_launch(), k_top_select<kTopListSmall, 256, 512><<<gnode, 256, kTopListSmall * 4, s>>>(ta, -1, kTopListSmall));
      (count_launch(), k_top_select<kTopListLarge, 1024, 2048><<<gnode, 1024, kTopListLarge * 4, s>>>(
          ta, kTopListSmall, kTopListLarge));
      (count_launch(), k_top_select_huge<<<gnode, 1024, 0, s>>>(ta, kTopListLarge));
    }
    const dim3 grun((unsigned)ta.nrun, (unsigned)Tb);
    const size_t gsmem = (size_t)kTopBlk * 6;
    cudaFuncSetAttribute(k_top_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem);
    cudaFuncSetAttribute(k_top_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem);
    // stable grouping by node: low kTopDigit bits, then the rest
    // (6 + up to 6 bits; 7 + 6 for 13 levels)
    const int bitsA = Lc <= 6 ? Lc : (Lc <= 12 ? 6 : kTopDigit), bitsB = Lc - bitsA;
    (count_launch(), k_top_count<true><<<grun, 512, 0, s>>>(ta, 0, bitsA));
    (count_launch(), k_top_scan<<<(unsigned)Tb, 1 << kTopDigit, 0, s>>>(ta, bitsA));
    (count_launch(), k_top_bounds<<<(unsigned)Tb, 1024, 0, s>>>(ta));
    (count_launch(), k_top_scatter<true><<<grun, 512, gsmem, s>>>(ta, 0, bitsA, bitsB == 0));
    if (bitsB > 0) {
      (count_launch(), k_top_count<false><<<grun, 512, 0, s>>>(ta, bitsA, bitsB));
      (count_launch(), k_top_scan<<<(unsigned)Tb, 1 << kTopDigit, 0, s>>>(ta, bitsB));
      (count_launch(), k_top_scatter<false><<<grun, 512, gsmem, s>>>(ta, bitsA, bitsB, 1));
    }
  }
  cudaFuncSetAttribute(k_seg_cta<kMidMax, 256, 1024, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMidMax * 4);
  cudaFuncSetAttribute(k_seg_cta<kLargeMax, 1024, 2048, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kLargeMax * 4);
  cudaFuncSetAttribute(k_seg_cta<kLargeMax2, 1024, 2048, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kLargeMax2 * 4);
  const int large_max = [] {  // read per call: build_ab switches it between builds
    const char *e = getenv("MRPT_BUILD_LARGE");  // experiments: 0 (no large class), 23552, 47104
    const int v = e ? atoi(e) : kLargeMax;
    return v >= kLargeMax ? kLargeMax : (v >= kLargeMax2 ? kLargeMax2 : kMidMax);
  }();
  for (int lev = Lc; lev < depth; ++lev) {
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
    a.tree_nlg = a.tree_nch + Tb;
    a.tree_lfill = a.tree_nch + 2 * (size_t)Tb;
    a.tree_base = reinterpret_cast<int64_t *>(w + L.tbase);
    a.tree_lbase = reinterpret_cast<int64_t *>(w + L.tlbase);
    a.large_list = reinterpret_cast<int32_t *>(w + L.llist);
    a.large_max = large_max;
    cudaMemsetAsync(a.ctl, 0, sizeof(LevelCtl), s);
    cudaMemsetAsync(a.tree_nch, 0, sizeof(int32_t) * 3 * (size_t)Tb, s);
    const int64_t nsegs = (int64_t)Tb << lev;
    const unsigned seg_blocks = (unsigned)ceil_div<int64_t>(nsegs, 256);
    (count_launch(), k_level_plan<<<seg_blocks, 256, 0, s>>>(a));
    (count_launch(), k_chunk_layout<<<1, 1024, 0, s>>>(a));
    (count_launch(), k_large_fill<<<seg_blocks, 256, 0, s>>>(a));
    // one CTA per segment (flat, in tree-major order) for the L2 locality of
    // the projection gathers; large segments from their tree-major list
    const unsigned flat_grid = (unsigned)(nsegs < 0x7fffffff ? nsegs : 0x7fffffff);
    (count_launch(), k_seg_cta<kTinyMax, 128, 512, true><<<flat_grid, 128, kTinyMax * 8, s>>>(a, -1, kTinyMax, false));
    (count_launch(), k_seg_cta<kMidMax, 256, 1024, false><<<flat_grid, 256, kMidMax * 4, s>>>(a, kTinyMax, kMidMax, false));
    if (large_max > kMidMax) {
      // a level has at most n * Tb / (kMidMax + 1) large segments
      const int64_t bound = (int64_t)Tb * (n / (kMidMax + 1)) + 1;
      const int64_t lg = bound < nsegs ? bound : nsegs;
      if (large_max == kLargeMax)
        (count_launch(), k_seg_cta<kLargeMax, 1024, 2048, false><<<(unsigned)(lg < sms ? lg : sms), 1024, kLargeMax * 4, s>>>(
            a, kMidMax, kLargeMax, true));
      else
        (count_launch(), k_seg_cta<kLargeMax2, 1024, 2048, false><<<(unsigned)(lg < 2 * sms ? lg : 2 * sms), 1024, kLargeMax2 * 4, s>>>(
            a, kMidMax, kLargeMax2, true));
    }
    const int64_t est = n >> lev;
    if (est > large_max || lev > 0) {
      // the big path may have work whenever a segment can exceed the large class;
      // after level 0 ties can make any segment large, so always launch.
      static const int big_per_sm = [] {
        // 8 resident 256-thread CTAs per SM for the streaming passes
        // (config 5 half scale: 549 vs 558 ms for hist + count + scatter + keys)
        const char *e = getenv("MRPT_BUILD_CTAS_PER_SM");  // experiments
        const int v = e ? atoi(e) : 8;
        return v < 1 ? 1 : (v > 8 ? 8 : v);
      }();
      const int big_grid = sms * big_per_sm;
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
