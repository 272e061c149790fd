// K5, top levels: the first Lc levels of every tree of a batch WITHOUT moving
// the point permutation (included by build.cu).
//
// While a tree's nodes are huge, splitting them through the permutation costs
// a gather of the level's projections plus a stable partition of the ids per
// level (~44 bytes per point per level in the chunked path).  Here every point
// keeps a 16-bit node id in point order instead; a level is
//   k_top_hist     node id of the level (from the parent's id and split) and
//                  a per-node histogram of LINEAR buckets of the level's
//                  projection -- all reads sequential (P[lev][i], P[lev-1][i],
//                  node[i]); one CTA per 64K points, 32K shared counters
//                  (2^lev nodes x NB buckets), flushed to the tree's table
//   k_top_pick     per node: the bucket holding the lower median's rank
//   k_top_collect  the members of those buckets (a few per mille to a few per
//                  cent of the points) appended to per-node key lists
//   k_top_select   per node: exact rank select over its list in shared memory
//                  (cta_select) -> split value, child sizes
// (~18 bytes per point per level), and after the last top level the ids are
// grouped by node in ONE stable multi-way split (warp-private counting over
// 16K-point runs: count, scan over runs, scatter), which yields exactly the
// permutation and bounds the per-level stable partitions would have produced:
// ids ascending within every node.  bucket(v) is non-decreasing in v, so the
// bucket holding rank kth holds the kth smallest value; its members are
// ranked by their order-preserving keys (ties and -0.0 as in f2key).
#pragma once

namespace mrpt {

constexpr int kTopMaxLev = 13;      // node ids < 2^13
constexpr int kTopBins = 32768;     // shared counters per CTA: nodes x buckets
constexpr int kTopMaxNB = 2048;     // buckets per node at the first levels
constexpr int kTopChunk = 65536;    // points per histogram / collect CTA
constexpr int kTopBuf = 16384;      // staged list members per collect CTA
constexpr int kTopDigit = 7;        // bits per pass of the final grouping (at most)
constexpr int kTopNodes = 1 << (kTopMaxLev - 1);  // nodes of the last top level
constexpr int kTopListSmall = 4096;
constexpr int kTopListLarge = 47104;

struct TopArgs {
  const float *P;
  int64_t n;
  int depth, Tb, lev, Lc, NB;
  uint16_t *node;      // (Tb, n) node id per point, point order
  int32_t *tsize;      // (Tb, 2 * kTopNodes * 2) heap order: node nd of level L at (1 << L) + nd
  uint32_t *tK;        // (Tb, kTopNodes) split key per node of the level last solved
  int4 *tinfo;         // (Tb, kTopNodes): bucket, count below it, its count, list offset
  int32_t *tfill;      // (Tb, kTopNodes) list fill cursors
  uint32_t *ghist;     // (Tb, kTopBins)
  float2 *colrange;    // (Tb * depth): sample minimum, 1 / sample span
  uint32_t *lists;     // (Tb, n) per-node key lists of the current level
  int32_t *table;      // (Tb, nrun, 2^kTopDigit) per-run digit counts -> output offsets
  int32_t *sid;        // (Tb, n) ids after the first grouping pass
  uint16_t *snode;     // (Tb, n) their node ids
  int64_t nrun;
  float *splits;
  int64_t sstride;
  int64_t *bounds;     // level-Lc bounds out (first 2^Lc + 1 entries per tree)
  int64_t bstride;
  int32_t *order;      // level-Lc permutation out
};

__device__ __forceinline__ int top_bucket(float v, float vmin, float sc, int NB) {
  const int b = __float2int_rz(__fmul_rn(__fsub_rn(v, vmin), sc));
  return b < 0 ? 0 : (b < NB - 1 ? b : NB - 1);
}

// Bucket range per projection column from its first 64K points (values
// outside the sample's range fall into the end buckets, still monotone).
__global__ void __launch_bounds__(256) k_top_range(TopArgs a) {
  __shared__ uint32_t rmn[8], rmx[8];
  const int64_t col = blockIdx.x;  // t * depth + lev
  const float *Pc = a.P + col * a.n;
  const int64_t ns = a.n < 65536 ? a.n : 65536;
  uint32_t mn = 0xffffffffu, mx = 0u;
  for (int64_t i = threadIdx.x; i < ns; i += 256) {
    const uint32_t k = f2key(__ldg(Pc + i));
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint32_t x = __shfl_xor_sync(0xffffffffu, mn, o), y = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = x < mn ? x : mn;
    mx = y > mx ? y : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    rmn[threadIdx.x >> 5] = mn;
    rmx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) {
      mn = rmn[w] < mn ? rmn[w] : mn;
      mx = rmx[w] > mx ? rmx[w] : mx;
    }
    const float vmin = key2f(mn), span = key2f(mx) - vmin;
    const float inv = 1.0f / span;
    const bool ok = isfinite(vmin) && isfinite(span) && span > 0.f && isfinite(inv) &&
                    isfinite(inv * (float)kTopMaxNB);
    a.colrange[col] = ok ? make_float2(vmin, inv) : make_float2(0.f, 0.f);  // all in bucket 0: exact select of the whole node
  }
}

__global__ void k_top_init(TopArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < (int64_t)a.Tb * kTopBins) a.ghist[i] = 0u;
  if (i < a.Tb) a.tsize[i * (4 * kTopNodes) + 1] = (int32_t)a.n;  // the root
}

// Node id of level `lev` for point i (lev >= 1) from the parent level's id
// and split key: right child iff key > K (value <= split goes left).
__device__ __forceinline__ int top_child(int parent, float vprev, const uint32_t *Ks) {
  return 2 * parent + (f2key(vprev) > Ks[parent] ? 1 : 0);
}

__global__ void __launch_bounds__(1024, 1) k_top_hist(TopArgs a) {
  extern __shared__ uint32_t top_smem[];
  uint32_t *hist = top_smem;  // (1 << lev) * NB
  __shared__ uint32_t Ks[kTopNodes / 2];
  const int t = blockIdx.y, lev = a.lev, NB = a.NB;
  const int nbins = NB << lev;
  const int64_t p0 = (int64_t)blockIdx.x * kTopChunk;
  const int64_t p1 = p0 + kTopChunk < a.n ? p0 + kTopChunk : a.n;
  for (int i = threadIdx.x; i < nbins; i += 1024) hist[i] = 0u;
  if (lev >= 1)
    for (int i = threadIdx.x; i < (1 << (lev - 1)); i += 1024) Ks[i] = a.tK[(int64_t)t * kTopNodes + i];
  __syncthreads();
  const float *Pc = a.P + ((int64_t)t * a.depth + lev) * a.n;
  const float *Pp = Pc - a.n;  // level lev - 1
  uint16_t *nd = a.node + (int64_t)t * a.n;
  const float2 cr = a.colrange[(int64_t)t * a.depth + lev];
  const float sc = cr.y * (float)NB;
  constexpr int U = 4;
  if ((a.n & 3) == 0) {
    // four consecutive points per thread: 16-byte projection loads, 8-byte
    // node-id load and store (columns and node rows are 16- / 8-byte aligned
    // when n is a multiple of 4; chunk starts are multiples of 65536)
#pragma unroll 2
    for (int64_t i0 = p0 + 4 * (int64_t)threadIdx.x; i0 < p1; i0 += 4 * 1024) {
      const float4 v4 = __ldg(reinterpret_cast<const float4 *>(Pc + i0));
      float4 vp4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (lev >= 1) vp4 = __ldg(reinterpret_cast<const float4 *>(Pp + i0));
      ushort4 par4 = make_ushort4(0, 0, 0, 0);
      if (lev >= 2) par4 = *reinterpret_cast<const ushort4 *>(nd + i0);
      const float v[4] = {v4.x, v4.y, v4.z, v4.w}, vp[4] = {vp4.x, vp4.y, vp4.z, vp4.w};
      const int par[4] = {par4.x, par4.y, par4.z, par4.w};
      int me[4] = {0, 0, 0, 0};
      if (lev >= 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) me[j] = top_child(par[j], vp[j], Ks);
        *reinterpret_cast<ushort4 *>(nd + i0) =
            make_ushort4((unsigned short)me[0], (unsigned short)me[1], (unsigned short)me[2], (unsigned short)me[3]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) atomicAdd(&hist[me[j] * NB + top_bucket(v[j], cr.x, sc, NB)], 1u);
    }
  } else
  for (int64_t i0 = p0 + threadIdx.x; i0 < p1; i0 += (int64_t)U * 1024) {
    float v[U], vp[U];
    int par[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t i = i0 + (int64_t)j * 1024;
      const bool in = i < p1;
      v[j] = in ? __ldg(Pc + i) : 0.f;
      vp[j] = (in && lev >= 1) ? __ldg(Pp + i) : 0.f;
      par[j] = (in && lev >= 2) ? (int)nd[i] : 0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t i = i0 + (int64_t)j * 1024;
      if (i < p1) {
        int me = 0;
        if (lev >= 1) {
          me = top_child(par[j], vp[j], Ks);
          nd[i] = (uint16_t)me;
        }
        atomicAdd(&hist[me * NB + top_bucket(v[j], cr.x, sc, NB)], 1u);
      }
    }
  }
  __syncthreads();
  uint32_t *gh = a.ghist + (int64_t)t * kTopBins;
  for (int i = threadIdx.x; i < nbins; i += 1024) {
    const uint32_t c = hist[i];
    if (c) atomicAdd(gh + i, c);
  }
}

// Per node: the bucket holding rank kth = (m+1)/2-1, the count below it and
// its count; list offsets = exclusive scan of those counts over the tree's
// nodes.  One CTA per tree; the table is zeroed for the next level.
__global__ void __launch_bounds__(1024) k_top_pick(TopArgs a) {
  __shared__ int s_cnt[kTopNodes];
  const int t = blockIdx.x, lev = a.lev, NB = a.NB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nnode = 1 << lev;
  uint32_t *gh = a.ghist + (int64_t)t * kTopBins;
  const int32_t *sz = a.tsize + (int64_t)t * (4 * kTopNodes) + nnode;
  int4 *info = a.tinfo + (int64_t)t * kTopNodes;
  // buckets per lane; with fewer than 32 buckets per node (level 11 on) the
  // first NB lanes take one each
  const int per = NB >= 32 ? NB / 32 : (lane < NB ? 1 : 0);
  for (int nd = warp; nd < nnode; nd += 32) {
    const int m = sz[nd];
    uint32_t *h = gh + nd * NB + (NB >= 32 ? lane * per : lane);
    int sum = 0;
    for (int j = 0; j < per; ++j) sum += (int)h[j];
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const int kth = (m + 1) / 2 - 1;
    int excl = incl - sum;
    if (m > 0 && excl <= kth && kth < incl) {
      for (int j = 0; j < per; ++j) {
        const int c = (int)h[j];
        if (kth < excl + c) {
          info[nd] = make_int4((NB >= 32 ? lane * per : lane) + j, excl, c, 0);
          s_cnt[nd] = c;
          break;
        }
        excl += c;
      }
    }
    if (m == 0 && lane == 0) {
      info[nd] = make_int4(0, 0, 0, 0);
      s_cnt[nd] = 0;
    }
    __syncwarp();
    for (int j = 0; j < per; ++j) h[j] = 0u;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of s_cnt over the nodes
    int carry = 0;
    for (int b0 = 0; b0 < nnode; b0 += 32) {
      const int nd = b0 + lane;
      const int c = nd < nnode ? s_cnt[nd] : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (nd < nnode) {
        info[nd].w = carry + incl - c;
        a.tfill[(int64_t)t * kTopNodes + nd] = 0;
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// The selected buckets' members go to their node's list.  Appending straight
// to the global lists costs a dependent atomic round trip per member, all on
// the tree's few cursors; a CTA stages its members in shared memory with
// their rank among the CTA's members of the same node, reserves list space
// once per node, and then stores every member at its place.
__global__ void __launch_bounds__(1024, 1) k_top_collect(TopArgs a) {
  extern __shared__ uint32_t top_smem[];
  uint2 *buf = reinterpret_cast<uint2 *>(top_smem);  // kTopBuf x (node | rank << 16, key)
  __shared__ int s_cnt[kTopNodes], s_gb[kTopNodes];
  __shared__ int16_t s_bsel[kTopNodes];  // selected bucket (< kTopMaxNB) or -1; list offsets stay in tinfo
  __shared__ int s_n;
  const int t = blockIdx.y, lev = a.lev, NB = a.NB;
  const int lane = threadIdx.x & 31;
  const int nnode = 1 << lev;
  const int64_t p0 = (int64_t)blockIdx.x * kTopChunk;
  const int64_t p1 = p0 + kTopChunk < a.n ? p0 + kTopChunk : a.n;
  const int4 *info = a.tinfo + (int64_t)t * kTopNodes;
  for (int i = threadIdx.x; i < nnode; i += 1024) {
    const int4 f = info[i];
    s_bsel[i] = (int16_t)(f.z > 0 ? f.x : -1);
    s_cnt[i] = 0;
  }
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  // shared addresses as 32-bit values, kept opaque; the slot counter's one is
  // made lane-dependent (+ 0 ptxas cannot fold) so that its atomic stays a
  // plain per-lane atomic
  uint32_t bsel_s = (uint32_t)__cvta_generic_to_shared(s_bsel), cnt_s = (uint32_t)__cvta_generic_to_shared(s_cnt);
  uint32_t buf_s = (uint32_t)__cvta_generic_to_shared(buf);
  uint32_t lm_eq;
  asm volatile("mov.u32 %0, %%lanemask_eq;" : "=r"(lm_eq));
  uint32_t sn_lane = (uint32_t)__cvta_generic_to_shared(&s_n) + (uint32_t)(__popc(lm_eq) - 1);
  asm volatile("" : "+r"(bsel_s), "+r"(cnt_s), "+r"(buf_s), "+r"(sn_lane));
  const float *Pc = a.P + ((int64_t)t * a.depth + lev) * a.n;
  const uint16_t *nd = a.node + (int64_t)t * a.n;
  const float2 cr = a.colrange[(int64_t)t * a.depth + lev];
  const float sc = cr.y * (float)NB;
  int32_t *fill = a.tfill + (int64_t)t * kTopNodes;
  uint32_t *list = a.lists + (int64_t)t * a.n;
  constexpr int U = kTopBuf / 1024;  // a round stages at most kTopBuf members
  for (int64_t i0 = p0 + threadIdx.x; i0 - threadIdx.x < p1; i0 += (int64_t)U * 1024) {  // CTA-uniform trips
    float v[U];
    int me[U];
    if (i0 - threadIdx.x + (int64_t)U * 1024 <= p1) {  // a whole round (CTA-uniform): no per-element range checks
#pragma unroll
      for (int j = 0; j < U; ++j) {
        v[j] = __ldg(Pc + i0 + j * 1024);
        me[j] = lev >= 1 ? (int)nd[i0 + j * 1024] : 0;
      }
    } else {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int64_t i = i0 + (int64_t)j * 1024;
        const bool in = i < p1;
        v[j] = in ? __ldg(Pc + i) : 0.f;
        me[j] = in ? (lev >= 1 ? (int)nd[i] : 0) : -1;
      }
    }
    // (32-bit shared addresses and PTX atomics: through generic pointers the
    // compiler rebuilds the shared window base per access and wraps the
    // leader's reservation in a second warp aggregation -- 73 instructions
    // per element where most elements of a deep level are hits)
#pragma unroll
    for (int j = 0; j < U; ++j) {
      bool hit = false;
      if (me[j] >= 0) {
        int16_t bs;
        asm volatile("ld.shared.s16 %0, [%1];" : "=h"(bs) : "r"(bsel_s + 2u * (uint32_t)me[j]));
        hit = top_bucket(v[j], cr.x, sc, NB) == (int)bs;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (bal) {
        const int leader = __ffs(bal) - 1;
        uint32_t base = 0;
        if (lane == leader)
          asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(base) : "r"(sn_lane), "r"((uint32_t)__popc(bal)) : "memory");
        base = __shfl_sync(0xffffffffu, base, leader);
        if (hit) {
          uint32_t lr;
          asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(lr) : "r"(cnt_s + 4u * (uint32_t)me[j]), "r"(1u) : "memory");
          const uint32_t at = buf_s + 8u * (base + (uint32_t)__popc(bal & lanemask_lt()));
          asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(at), "r"((uint32_t)me[j] | (lr << 16)), "r"(f2key(v[j]))
                       : "memory");
        }
      }
    }
    __syncthreads();
    const int cnt = s_n;
    if (cnt > 0) {  // CTA-uniform
      for (int i = threadIdx.x; i < nnode; i += 1024) {
        const int c = s_cnt[i];
        if (c) {
          s_gb[i] = info[i].w + atomicAdd(fill + i, c);
          s_cnt[i] = 0;
        }
      }
      __syncthreads();
      for (int e = threadIdx.x; e < cnt; e += 1024) {
        const uint2 en = buf[e];
        list[s_gb[en.x & 0xffffu] + (int)(en.x >> 16)] = en.y;
      }
      __syncthreads();
      if (threadIdx.x == 0) s_n = 0;
      __syncthreads();
    }
  }
}

__device__ __forceinline__ void top_write_node(const TopArgs &a, int t, int nd, int m, int nle, uint32_t K,
                                               float split) {
  const int lev = a.lev;
  a.splits[(int64_t)t * a.sstride + ((1 << lev) - 1) + nd] = split;
  a.tK[(int64_t)t * kTopNodes + nd] = K;
  int32_t *sz = a.tsize + (int64_t)t * (4 * kTopNodes) + (2 << lev);
  sz[2 * nd] = nle;
  sz[2 * nd + 1] = m - nle;
}

// One CTA per node whose list length lies in (lo, hi]: the list is staged in
// shared memory and ranked exactly.  lo < 0 also takes the empty nodes
// (split 0.0, nothing goes anywhere: trees.py:84-85).
template <int MAXM, int NT, int NB>
__global__ void __launch_bounds__(NT) k_top_select(TopArgs a, int lo, int hi) {
  extern __shared__ uint32_t top_smem[];
  uint32_t *keys = top_smem;  // MAXM
  __shared__ uint32_t hist[NB];
  __shared__ uint32_t red[2 * NT / 32];
  __shared__ int sh[4 + NT / 32];
  const int nd = blockIdx.x, t = blockIdx.y;
  const int4 f = a.tinfo[(int64_t)t * kTopNodes + nd];
  const int cnt = f.z;
  if (cnt <= lo || cnt > hi) return;
  const int m = a.tsize[(int64_t)t * (4 * kTopNodes) + (1 << a.lev) + nd];
  if (m == 0) {
    if (threadIdx.x == 0) top_write_node(a, t, nd, 0, 0, 0u, 0.0f);
    return;
  }
  const uint32_t *list = a.lists + (int64_t)t * a.n + f.w;
  uint32_t mn = 0xffffffffu, mx = 0u;
  for (int i = threadIdx.x; i < cnt; i += NT) {
    const uint32_t k = __ldg(list + i);
    keys[i] = k;
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
  }
  uint32_t K;
  int nle;
  cta_select<NT, NB>(keys, cnt, (m + 1) / 2 - 1 - f.y, mn, mx, hist, red, sh, K, nle);
  if (threadIdx.x == 0) top_write_node(a, t, nd, m, f.y + nle, K, key2f(K));
}

// Lists beyond shared memory (a bucket of one value repeated, or a sample
// range that missed the column): 8-bit radix select over the list in global
// memory by one CTA.
__global__ void __launch_bounds__(1024) k_top_select_huge(TopArgs a, int lo) {
  __shared__ uint32_t hist[256];
  __shared__ int s_pick[3];
  const int nd = blockIdx.x, t = blockIdx.y;
  const int4 f = a.tinfo[(int64_t)t * kTopNodes + nd];
  const int cnt = f.z;
  if (cnt <= lo) return;
  const int m = a.tsize[(int64_t)t * (4 * kTopNodes) + (1 << a.lev) + nd];
  const uint32_t *list = a.lists + (int64_t)t * a.n + f.w;
  const int kth = (m + 1) / 2 - 1 - f.y;
  uint32_t prefix = 0u;
  int nb = 0, krem = kth, cnt_last = 0;
  while (nb < 32) {
    const int shift = 24 - nb;
    if (threadIdx.x < 256) hist[threadIdx.x] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += 1024) {
      const uint32_t k = __ldg(list + i);
      if (prefix_match(k, prefix, nb)) atomicAdd(&hist[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      int bin, below, c;
      warp_pick(hist, krem, bin, below, c);
      if (threadIdx.x == 0) {
        s_pick[0] = bin;
        s_pick[1] = below;
        s_pick[2] = c;
      }
    }
    __syncthreads();
    prefix |= (uint32_t)s_pick[0] << shift;
    krem -= s_pick[1];
    cnt_last = s_pick[2];
    nb += 8;
  }
  if (threadIdx.x == 0) top_write_node(a, t, nd, m, f.y + kth - krem + cnt_last, prefix, key2f(prefix));
}

// Final grouping: the ids ordered by their level-Lc node, ascending within a
// node -- a stable sort by the node id, done as one or two stable digit
// passes (kTopDigit low bits, then the rest).  A CTA owns a block of kTopBlk
// consecutive positions (warp w the w-th 1024 of them): a count pass gives
// every (block, digit) its output offset (scan over the blocks); the scatter
// pass ranks the block's elements stably -- per-warp digit counts, prefix
// over the warps, then every warp walks its positions in order, 32 a round,
// equal digits of a round ranked by lane (match_any) -- into a digit-major
// staging buffer in shared memory, which is then copied out: consecutive
// staged elements of a digit go to consecutive addresses, so all global
// stores are coalesced full sectors (scattering straight from the warps
// wrote DRAM 5-10x the ids' bytes in partial sectors).
//
// Pass A reads the node ids in point order (and first derives them from the
// last top level's split), pass B the (node, id) pairs pass A wrote.
constexpr int kTopBlk = 16384;

template <bool PASS_A>
__global__ void __launch_bounds__(512) k_top_count(TopArgs a, int shift, int bits) {
  __shared__ uint32_t Ks[kTopNodes];
  __shared__ int32_t hist[1 << kTopDigit];
  const int t = blockIdx.y, Lc = a.Lc;
  const int nb = 1 << bits, mask = nb - 1;
  if (PASS_A)
    for (int i = threadIdx.x; i < (1 << (Lc - 1)); i += 512) Ks[i] = a.tK[(int64_t)t * kTopNodes + i];
  if (threadIdx.x < nb) hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t p0 = (int64_t)blockIdx.x * kTopBlk;
  const int64_t p1 = p0 + kTopBlk < a.n ? p0 + kTopBlk : a.n;
  const float *Pp = a.P + ((int64_t)t * a.depth + (Lc - 1)) * a.n;
  uint16_t *nd = a.node + (int64_t)t * a.n;
  const uint16_t *sn = a.snode + (int64_t)t * a.n;
  constexpr int U = 8;
  for (int64_t i0 = p0 + threadIdx.x; i0 < p1; i0 += 512 * U) {
    float vp[U];
    int par[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t i = i0 + 512 * j;
      vp[j] = (PASS_A && i < p1) ? __ldg(Pp + i) : 0.f;
      par[j] = i < p1 ? (PASS_A ? (Lc >= 2 ? (int)nd[i] : 0) : (int)sn[i]) : 0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t i = i0 + 512 * j;
      if (i < p1) {
        int me = par[j];
        if (PASS_A) {
          me = top_child(par[j], vp[j], Ks);
          nd[i] = (uint16_t)me;
        }
        atomicAdd(&hist[(me >> shift) & mask], 1);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < nb) a.table[((int64_t)t * a.nrun + blockIdx.x) * nb + threadIdx.x] = hist[threadIdx.x];
}

// Per tree: table[block][digit] -> its output offset (digit-major, blocks in
// order within a digit).  One CTA of 64 threads per tree, thread = digit.
__global__ void __launch_bounds__(1 << kTopDigit) k_top_scan(TopArgs a, int bits) {
  __shared__ int s_tot[1 << kTopDigit];
  const int t = blockIdx.x, nb = 1 << bits, b = threadIdx.x;
  int32_t *col = a.table + (int64_t)t * a.nrun * nb + b;
  int run = 0;
  if (b < nb) {
    for (int64_t r = 0; r < a.nrun; ++r) {
      const int v = col[r * nb];
      col[r * nb] = run;
      run += v;
    }
  }
  s_tot[b] = b < nb ? run : 0;
  __syncthreads();
  int base = 0;
  for (int i = 0; i < b; ++i) base += s_tot[i];
  if (b < nb && base)
    for (int64_t r = 0; r < a.nrun; ++r) col[r * nb] += base;
}

template <bool PASS_A>
__global__ void __launch_bounds__(512) k_top_scatter(TopArgs a, int shift, int bits, int last) {
  extern __shared__ uint32_t top_smem[];
  int32_t *st_id = reinterpret_cast<int32_t *>(top_smem);                 // kTopBlk
  uint16_t *st_node = reinterpret_cast<uint16_t *>(top_smem + kTopBlk);   // kTopBlk
  __shared__ int32_t wcnt[16][1 << kTopDigit];
  __shared__ int32_t lbase[1 << kTopDigit], gbase[1 << kTopDigit];
  const int t = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = 1 << bits, mask = nb - 1;
  const int64_t p0 = (int64_t)blockIdx.x * kTopBlk;
  const int64_t p1 = p0 + kTopBlk < a.n ? p0 + kTopBlk : a.n;
  const int64_t w0 = p0 + (int64_t)warp * 1024;
  const int64_t w1 = w0 + 1024 < p1 ? w0 + 1024 : p1;
  const uint16_t *src_node = (PASS_A ? a.node : a.snode) + (int64_t)t * a.n;
  const int32_t *src_id = a.sid + (int64_t)t * a.n;
  for (int i = lane; i < nb; i += 32) wcnt[warp][i] = 0;
  __syncwarp();
  // this warp's positions stay in registers: 32 rounds of 32
  int me[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const int64_t i = w0 + 32 * r + lane;
    me[r] = i < w1 ? (int)src_node[i] : -1;
    if (me[r] >= 0) atomicAdd(&wcnt[warp][(me[r] >> shift) & mask], 1);
  }
  __syncthreads();
  if (threadIdx.x < nb) {  // prefix over the warps, block totals
    int run = 0;
    for (int w = 0; w < 16; ++w) {
      const int c = wcnt[w][threadIdx.x];
      wcnt[w][threadIdx.x] = run;
      run += c;
    }
    lbase[threadIdx.x] = run;
    gbase[threadIdx.x] = a.table[((int64_t)t * a.nrun + blockIdx.x) * nb + threadIdx.x];
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the totals over the digits (nb <= 2^kTopDigit)
    int carry = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int c = b0 + lane < nb ? lbase[b0 + lane] : 0;
      int inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      if (b0 + lane < nb) lbase[b0 + lane] = carry + inc - c;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const int64_t i = w0 + 32 * r + lane;
    const int dg = me[r] < 0 ? nb : ((me[r] >> shift) & mask);  // nb: the lanes past the end
    const unsigned grp = __match_any_sync(0xffffffffu, dg);
    const int leader = __ffs(grp) - 1;
    int base = 0;
    if (lane == leader && dg < nb) {
      base = wcnt[warp][dg];
      wcnt[warp][dg] = base + __popc(grp);
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    if (dg < nb) {
      const int lp = lbase[dg] + base + __popc(grp & lanemask_lt());
      st_id[lp] = PASS_A ? (int32_t)i : __ldg(src_id + i);
      st_node[lp] = (uint16_t)me[r];
    }
    __syncwarp();
  }
  __syncthreads();
  int32_t *out = a.order + (int64_t)t * a.n;
  int32_t *out_id = a.sid + (int64_t)t * a.n;
  uint16_t *out_node = a.snode + (int64_t)t * a.n;
  const int cnt = (int)(p1 - p0);
  for (int e = threadIdx.x; e < cnt; e += 512) {
    const int node = st_node[e];
    const int dg = (node >> shift) & mask;
    const int64_t gp = (int64_t)gbase[dg] + (e - lbase[dg]);
    if (last) {
      out[gp] = st_id[e];
    } else {
      out_id[gp] = st_id[e];
      out_node[gp] = (uint16_t)node;
    }
  }
}

// Level-Lc bounds: exclusive scan of the node sizes.  One CTA per tree.
__global__ void __launch_bounds__(1024) k_top_bounds(TopArgs a) {
  __shared__ int64_t wsum[33];
  const int t = blockIdx.x, nnode = 1 << a.Lc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t *sz = a.tsize + (int64_t)t * (4 * kTopNodes) + nnode;
  int64_t *bo = a.bounds + (int64_t)t * a.bstride;
  int64_t carry = 0;
  for (int b0 = 0; b0 < nnode; b0 += 1024) {
    const int nd = b0 + threadIdx.x;
    const int64_t v = nd < nnode ? sz[nd] : 0;
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
    if (nd < nnode) bo[nd] = carry + wsum[warp] + incl - v;
    carry += wsum[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) bo[nnode] = carry;
}

}  // namespace mrpt
