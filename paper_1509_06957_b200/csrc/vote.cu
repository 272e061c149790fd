// K3: vote counting over the T leaves each query lands in
// (replaces VoteAccumulator.accumulate + _cy.vote, search.py:75-86,
// _kernels/_cy.pyx:57-78).
//
// One CTA per query.  Vote counters live in shared memory over a tile of W
// point ids, packed 4 (u8), 2 (u16) or 1 (u32) per 32-bit word and bumped
// with atomicAdd(word, 1 << lane_shift); the counter width is chosen so no
// count can overflow into its neighbour.  When n > W the CTA sweeps the id
// tiles in order with one cursor per tree: leaf slices built by K5 are
// ascending, so the part of a slice inside the current tile is the next run
// from the cursor.  The increment that raises a count to v (the reference's
// `counts[idx] == v` test, _cy.pyx:75-77) sets the point's bit in a per-tile
// bitmap; after the tile, the bitmap is compacted in id order, so every
// candidate list comes out ascending (the order candidate_set returns, and
// the order that lets concurrent queries sweep X through L2 together).
// Groups of G lanes share one tree slice (G ~ mean slice length per tile)
// and each lane keeps U loads in flight.
#include <atomic>
#include <stdlib.h>

#include "common.cuh"

namespace mrpt {

struct VoteArgs {
  const int32_t *leaf_indices;
  const int64_t *leaf_offsets;
  int64_t n;
  int T, L;  // L = 2^depth leaves
  const int32_t *leaves;
  int64_t nq;
  int v;
  int32_t *cand;
  int64_t cap;
  int32_t *ncand;
  int W, ntiles;
  const int32_t *qlist;  // optional: only these queries (count *qcount)
  const int32_t *qcount;
  const uint16_t *dir;   // optional tile directory (T, 2^depth, ntiles+1)
  uint32_t *bits_out;    // optional: candidate bitmap per query instead of lists
  int64_t bstride;       // words per query in bits_out
  uint16_t *cnt_out;     // optional: each listed candidate's vote count (saturated), beside cand
  int dbg;               // timing experiments only (MRPT_VOTE_DBG): 1 no bumps, 2 no per-tile clearing
};

// Vote count of tile-local id `local` in the packed counters (code cw).
__device__ __forceinline__ uint32_t counter_read(const uint32_t *cnt, int cw, int local) {
  if (cw == 1) return (cnt[local >> 2] >> ((local & 3) << 3)) & 0xffu;
  if (cw == 3) {
    const int w = local / 3;
    return (cnt[w] >> ((local - 3 * w) * 10)) & 0x3ffu;
  }
  if (cw == 2) return (cnt[local >> 1] >> ((local & 1) << 4)) & 0xffffu;
  return cnt[local];
}

constexpr int kVoteNT = 1024;
constexpr int kVoteU = 8;

// Counter packing codes: 1 = 4 x 8-bit, 3 = 3 x 10-bit, 2 = 2 x 16-bit,
// 4 = 1 x 32-bit lanes per 32-bit word.  A lane never carries into its
// neighbour because the code is chosen from the largest possible count.
template <int CW>
__host__ __device__ __forceinline__ int counter_words(int W) {
  return CW == 1 ? W / 4 : (CW == 2 ? W / 2 : (CW == 3 ? (W + 2) / 3 : W));
}

template <int CW>
__device__ __forceinline__ uint32_t bump(uint32_t *cnt, int local) {
  if (CW == 1) {
    const int sh = (local & 3) << 3;
    const uint32_t old = atomicAdd(cnt + (local >> 2), 1u << sh);
    return ((old >> sh) & 0xffu) + 1u;
  } else if (CW == 3) {
    const int w = local / 3;
    const int sh = (local - 3 * w) * 10;
    const uint32_t old = atomicAdd(cnt + w, 1u << sh);
    return ((old >> sh) & 0x3ffu) + 1u;
  } else if (CW == 2) {
    const int sh = (local & 1) << 4;
    const uint32_t old = atomicAdd(cnt + (local >> 1), 1u << sh);
    return ((old >> sh) & 0xffffu) + 1u;
  } else {
    return atomicAdd(cnt + local, 1u) + 1u;
  }
}

// Append, in id order, the ids whose bit is set in bits[0..nwords) (tile
// origin lo) to out[base..]; returns the new base (block-uniform).  Clears
// the bitmap as it goes.
template <int NT = kVoteNT>
__device__ __forceinline__ int64_t emit_bitmap(uint32_t *bits, int nwords, int32_t lo, int32_t *out,
                                               int64_t base, int64_t cap, int *wsum,
                                               const uint32_t *cntw = nullptr, int cw = 0,
                                               uint16_t *cout = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  for (int r0 = 0; r0 < nwords; r0 += NT) {
    const int i = r0 + threadIdx.x;
    uint32_t word = i < nwords ? bits[i] : 0u;
    if (i < nwords && word) bits[i] = 0u;
    const int pc = __popc(word);
    int incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the per-warp totals, total in wsum[NW]
      const int c = lane < NW ? wsum[lane] : 0;
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += u;
      }
      if (lane < NW) wsum[lane] = x - c;
      if (lane == 31) wsum[NW] = x;
    }
    __syncthreads();
    const int before = wsum[warp], tot = wsum[NW];
    int64_t pos = base + before + incl - pc;
    while (word) {
      const int b = __ffs(word) - 1;
      if (pos < cap) {
        out[pos] = lo + i * 32 + b;
        if (cout) {
          const uint32_t c = counter_read(cntw, cw, i * 32 + b);
          cout[pos] = (uint16_t)(c < 65535u ? c : 65535u);
        }
      }
      ++pos;
      word &= word - 1u;
    }
    base += tot;
    __syncthreads();
  }
  return base;
}

// Bitmap output: copy the tile's "reached v" words to dst (coalesced),
// clearing them; returns their popcount (block-uniform).
template <int NT = kVoteNT>
__device__ __forceinline__ int64_t store_bits(uint32_t *bits, int nwords, uint32_t *dst, int *wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  int c = 0;
  for (int i = threadIdx.x; i < nwords; i += NT) {
    const uint32_t w = bits[i];
    dst[i] = w;
    if (w) bits[i] = 0u;
    c += __popc(w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) wsum[warp] = c;
  __syncthreads();
  int64_t tot = 0;
  for (int w = 0; w < NW; ++w) tot += wsum[w];
  __syncthreads();
  return tot;
}

template <int CW, int G, bool SORTED>
__global__ void __launch_bounds__(kVoteNT, 1) k_vote(VoteArgs a) {
  extern __shared__ uint4 vote_smem[];
  uint32_t *cnt = reinterpret_cast<uint32_t *>(vote_smem);
  const int cwords = (counter_words<CW>(a.W) + 3) & ~3;  // uint4-zeroable
  uint32_t *bits = cnt + cwords;    // W/32 words: "reached v" flags
  const int bwords = a.W / 32;
  int32_t *cur = reinterpret_cast<int32_t *>(bits + bwords);
  int32_t *endp = cur + a.T;
  __shared__ int wsum[kVoteNT / 32 + 1];
  const int tid = threadIdx.x, lane = tid & 31;
  const int gl = lane & (G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  const int gi = tid / G, ngroups = kVoteNT / G;
  const int64_t nwork = a.qlist ? (int64_t)*a.qcount : a.nq;
  for (int64_t wq = blockIdx.x; wq < nwork; wq += gridDim.x) {
    const int64_t q = a.qlist ? (int64_t)a.qlist[wq] : wq;
    for (int t = tid; t < a.T; t += kVoteNT) {
      const int leaf = a.leaves[q * a.T + t];
      const int64_t *o = a.leaf_offsets + (int64_t)t * (a.L + 1);
      cur[t] = (int32_t)o[leaf];
      endp[t] = (int32_t)o[leaf + 1];
    }
    uint4 *c4 = reinterpret_cast<uint4 *>(cnt);
    for (int i = tid; i < cwords / 4; i += kVoteNT) c4[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = tid; i < bwords; i += kVoteNT) bits[i] = 0u;
    __syncthreads();
    int32_t *qcand = a.cand + q * a.cap;
    int64_t ncand = 0;
    for (int tile = 0; tile < a.ntiles; ++tile) {
      const int32_t lo = tile * a.W;
      const int64_t hi64 = (int64_t)lo + a.W < a.n ? (int64_t)lo + a.W : a.n;
      const int32_t hi = (int32_t)hi64;
      for (int t = gi; t < a.T; t += ngroups) {
        const int32_t *Lt = a.leaf_indices + (int64_t)t * a.n;
        const int32_t e = endp[t];
        if (SORTED) {
          int32_t pos = cur[t];
          while (pos < e) {
            int32_t id[kVoteU];
#pragma unroll
            for (int u = 0; u < kVoteU; ++u) {
              const int32_t idx = pos + gl + u * G;
              id[u] = idx < e ? __ldg(Lt + idx) : 0x7fffffff;
            }
            int consumed = 0;
#pragma unroll
            for (int u = 0; u < kVoteU; ++u) {
              const bool in = id[u] < hi;
              if (in) {
                const int local = id[u] - lo;
                if (bump<CW>(cnt, local) == (uint32_t)a.v)
                  atomicOr(bits + (local >> 5), 1u << (local & 31));
              }
              consumed += __popc(__ballot_sync(gmask, in) & gmask);
            }
            pos += consumed;
            if (consumed < kVoteU * G) break;
          }
          if (gl == 0) cur[t] = pos;
        } else {
          // unsorted slices (foreign index): filter the whole slice per tile
          for (int32_t idx = cur[t] + gl; idx < e; idx += G) {
            const int32_t id = __ldg(Lt + idx);
            if (id >= lo && id < hi) {
              const int local = id - lo;
              if (bump<CW>(cnt, local) == (uint32_t)a.v)
                atomicOr(bits + (local >> 5), 1u << (local & 31));
            }
          }
        }
      }
      __syncthreads();
      if (a.bits_out)
        ncand += store_bits(bits, (int)((hi - lo + 31) >> 5), a.bits_out + q * a.bstride + (lo >> 5), wsum);
      else
        ncand = emit_bitmap(bits, (int)((hi - lo + 31) >> 5), lo, qcand, ncand, a.cap, wsum, cnt, CW,
                            a.cnt_out ? a.cnt_out + q * a.cap : nullptr);
      if (tile + 1 < a.ntiles) {
        for (int i = tid; i < cwords / 4; i += kVoteNT) c4[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
      }
    }
    if (tid == 0) a.ncand[q] = (int32_t)ncand;  // > cap means only cap ids were stored
    __syncthreads();
  }
}



// ---------------------------------------------------------------------------
// Tile directory (built once per index): dir[(t*L + leaf)*(ntiles+1) + w] =
// number of ids of that (ascending) leaf slice below w*W, i.e. where the
// slice's part in id tile w starts.  One warp per leaf.
__global__ void k_build_dir(const int32_t *__restrict__ leaf_indices,
                            const int64_t *__restrict__ leaf_offsets, int64_t n, int T, int L, int W,
                            int ntiles, uint16_t *dir) {
  const int lane = threadIdx.x & 31;
  const int64_t nleaves = (int64_t)T * L;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < nleaves; g += wstride) {
    const int64_t t = g / L, leaf = g - t * L;
    const int64_t *o = leaf_offsets + t * (L + 1);
    const int64_t s = o[leaf], e = o[leaf + 1];
    const int32_t *Lt = leaf_indices + t * n;
    uint16_t *d = dir + g * (ntiles + 1);
    int prev_tile = -1;  // tile of the element before this chunk
    for (int64_t p0 = s; p0 < e; p0 += 32) {
      const int64_t p = p0 + lane;
      const int tl = p < e ? (int)(Lt[p] / W) : ntiles;
      int before = __shfl_up_sync(0xffffffffu, tl, 1);
      if (lane == 0) before = prev_tile;
      if (p < e)
        for (int w = before + 1; w <= tl; ++w) d[w] = (uint16_t)(p - s);
      prev_tile = __shfl_sync(0xffffffffu, tl, 31);
      if (p0 + 32 >= e) {
        // the lane holding the last element fills the trailing tiles
        const int64_t last = e - 1;
        if (p == last)
          for (int w = tl + 1; w <= ntiles; ++w) d[w] = (uint16_t)(e - s);
      }
    }
    if (s == e && lane == 0)
      for (int w = 0; w <= ntiles; ++w) d[w] = 0;
  }
}

// Directory-driven vote: per id tile, every tree's slice bounds come from the
// directory, so a warp flattens the slices of its 32 trees and streams them
// with consecutive lanes on consecutive ids.  A flat position is mapped to
// its slice without searching: per 32-wide window one __reduce_or_sync
// collects the slice starts inside the window, and the running count of
// slice starts plus a popcount gives the slice's rank among the non-empty
// slices, looked up in a 32-entry per-warp table.
template <int CW, int NT, bool OFF32 = false>
__global__ void __launch_bounds__(NT, 1024 / NT) k_vote_dir(VoteArgs a) {
  extern __shared__ uint4 vote_smem[];
  uint32_t *cnt = reinterpret_cast<uint32_t *>(vote_smem);
  const int cwords = (counter_words<CW>(a.W) + 3) & ~3;
  uint32_t *bits = cnt + cwords;
  const int bwords = a.W / 32;
  int32_t *sbase = reinterpret_cast<int32_t *>(bits + bwords);  // T: slice start of the leaf
  int32_t *sleaf = sbase + a.T;                                   // T: leaf id
  __shared__ int wsum[NT / 32 + 1];
  constexpr int kWList = 2048;  // bitmap words that became non-zero in this tile
  __shared__ int32_t wlist[kWList];
  __shared__ int s_nw, s_nc;
  constexpr int NW = NT / 32;
  // per warp: where each non-empty slice (by rank) starts -- a global index,
  // or (OFF32, 32 * n < 2^31) an offset from the warp's first tree's row
  __shared__ long long w_base[NW][OFF32 ? 1 : 32];
  __shared__ int32_t w_off[NW][OFF32 ? 32 : 1];
  __shared__ int w_pre[NW][32];         // per warp: flat start of each non-empty slice (by rank)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ngroups = (a.T + 31) >> 5;
  const int64_t dstride = a.ntiles + 1;
  const int64_t nwork = a.qlist ? (int64_t)*a.qcount : a.nq;
  for (int64_t wq = blockIdx.x; wq < nwork; wq += gridDim.x) {
    const int64_t q = a.qlist ? (int64_t)a.qlist[wq] : wq;
    for (int t = tid; t < a.T; t += NT) {
      const int leaf = a.leaves[q * a.T + t];
      sleaf[t] = leaf;
      sbase[t] = (int32_t)a.leaf_offsets[(int64_t)t * (a.L + 1) + leaf];
    }
    uint4 *c4 = reinterpret_cast<uint4 *>(cnt);
    for (int i = tid; i < cwords / 4; i += NT) c4[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = tid; i < bwords; i += NT) bits[i] = 0u;
    if (tid == 0) {
      s_nw = 0;
      s_nc = 0;
    }
    __syncthreads();
    int32_t *qcand = a.cand + q * a.cap;
    int64_t ncand = 0;
    // Work split per tile: with NW <= T <= 32*NW every warp owns a balanced
    // contiguous range of <= 32 trees; with fewer trees several warps share
    // one group, each taking every parts-th 32-wide window; with more, warps
    // loop over 32-tree groups.
    const bool ranged = a.T >= NW && a.T <= 32 * NW;
    const int parts = ranged || ngroups >= NW ? 1 : NW / ngroups;
    const int nvirt = ranged ? NW : ngroups * parts;
    // ranged: each lane owns one tree for the whole query, so its directory
    // entries for the current and next tile stay in registers and the one
    // after is fetched while the current tile is processed
    const uint16_t *dlane = nullptr;
    int dcur = 0, dnxt = 0;
    if (ranged) {
      const int t = (int)(((int64_t)warp * a.T) / NW) + lane;
      if (t < (int)(((int64_t)(warp + 1) * a.T) / NW)) {
        dlane = a.dir + ((int64_t)t * a.L + sleaf[t]) * dstride;
        dcur = dlane[0];
        dnxt = dlane[1];
      }
    }
    for (int tile = 0; tile < a.ntiles; ++tile) {
      const int32_t lo = tile * a.W;
      const int dnn = (dlane && tile + 2 <= a.ntiles) ? (int)__ldg(dlane + tile + 2) : 0;
      for (int vw = warp; vw < nvirt; vw += NW) {
        const int g = ranged ? 0 : vw % ngroups, part = ranged ? 0 : vw / ngroups;
        const int t_lo = ranged ? (int)(((int64_t)vw * a.T) / NW) : g * 32;
        const int t_hi = ranged ? (int)(((int64_t)(vw + 1) * a.T) / NW) : (g * 32 + 32 < a.T ? g * 32 + 32 : a.T);
        const int t = t_lo + lane;
        const int32_t *wrow = a.leaf_indices + (int64_t)t_lo * a.n;  // OFF32 origin
        int len = 0;
        long long base = 0;
        if (t < t_hi) {
          int s0, s1;
          if (ranged) {
            s0 = dcur;
            s1 = dnxt;
          } else {
            const uint16_t *d = a.dir + ((int64_t)t * a.L + sleaf[t]) * dstride + tile;
            s0 = d[0];
            s1 = d[1];
          }
          len = s1 - s0;
          base = OFF32 ? (long long)(t - t_lo) * a.n + sbase[t] + s0 : (long long)t * a.n + sbase[t] + s0;
        }
        int pre = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, pre, o);
          if (lane >= o) pre += u;
        }
        const int total = __shfl_sync(0xffffffffu, pre, 31);
        pre -= len;
        // rank table of the non-empty slices
        const unsigned ne = __ballot_sync(0xffffffffu, len > 0);
        __syncwarp();
        if (len > 0) {
          const int r = __popc(ne & lanemask_lt());
          if (OFF32)
            w_off[warp][r] = (int32_t)base;
          else
            w_base[warp][r] = base;
          w_pre[warp][r] = pre;
        }
        __syncwarp();
        constexpr int UNR = 8;
        const int stride = parts * 32;
        for (int e0 = part * 32; e0 < total; e0 += UNR * stride) {
          int32_t id[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            const int w0 = e0 + u * stride;
            // slice starts inside [w0, w0+32) and before w0
            const int rel = pre - w0;
            const bool inwin = len > 0 && rel >= 0 && rel < 32;
            const unsigned starts = __reduce_or_sync(0xffffffffu, inwin ? (1u << rel) : 0u);
            const int before = __popc(__ballot_sync(0xffffffffu, len > 0 && rel < 0));
            const int e = w0 + lane;
            const int rank = before + __popc(starts & (0xffffffffu >> (31 - lane))) - 1;
            id[u] = -1;
            if (e < total) {
              const int pk = w_pre[warp][rank];
              if (OFF32)
                id[u] = __ldg(wrow + (w_off[warp][rank] + (e - pk)));
              else
                id[u] = __ldg(a.leaf_indices + w_base[warp][rank] + (e - pk));
            }
          }
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            if (id[u] >= 0) {
              const int local = id[u] - lo;
              if (bump<CW>(cnt, local) == (uint32_t)a.v) {
                if (atomicOr(bits + (local >> 5), 1u << (local & 31)) == 0u) {
                  const int wi = atomicAdd(&s_nw, 1);
                  if (wi < kWList) wlist[wi] = local >> 5;
                }
              }
            }
          }
        }
        __syncwarp();
      }
      __syncthreads();
      const int nw = s_nw;
      if (a.bits_out) {
        const int64_t hi = (int64_t)lo + a.W < a.n ? (int64_t)lo + a.W : a.n;
        ncand += store_bits<NT>(bits, (int)((hi - lo + 31) >> 5), a.bits_out + q * a.bstride + (lo >> 5), wsum);
      } else if (nw > kWList) {  // too many words to list: ordered scan of the whole bitmap
        const int64_t hi = (int64_t)lo + a.W < a.n ? (int64_t)lo + a.W : a.n;
        ncand = emit_bitmap<NT>(bits, (int)((hi - lo + 31) >> 5), lo, qcand, ncand, a.cap, wsum, cnt, CW,
                                a.cnt_out ? a.cnt_out + q * a.cap : nullptr);
      } else {
        // listed words only (ids within the tile unordered; tiles ascending)
        for (int i0 = 0; i0 < nw; i0 += NT) {
          const int i = i0 + tid;
          uint32_t word = 0u;
          int wi = 0;
          if (i < nw) {
            wi = wlist[i];
            word = bits[wi];
            bits[wi] = 0u;
          }
          const int pc = __popc(word);
          int incl = pc;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int u2 = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u2;
          }
          int wbase = 0;
          if (lane == 31 && incl) wbase = atomicAdd(&s_nc, incl);
          wbase = __shfl_sync(0xffffffffu, wbase, 31);
          int64_t pos = ncand + wbase + incl - pc;
          while (word) {
            const int b = __ffs(word) - 1;
            if (pos < a.cap) {
              qcand[pos] = lo + wi * 32 + b;
              if (a.cnt_out) {
                const uint32_t c = counter_read(cnt, CW, wi * 32 + b);
                a.cnt_out[q * a.cap + pos] = (uint16_t)(c < 65535u ? c : 65535u);
              }
            }
            ++pos;
            word &= word - 1u;
          }
        }
        __syncthreads();
        ncand += s_nc;
      }
      __syncthreads();
      if (tid == 0) {
        s_nw = 0;
        s_nc = 0;
      }
      dcur = dnxt;
      dnxt = dnn;
      if (tile + 1 < a.ntiles) {
        for (int i = tid; i < cwords / 4; i += NT) c4[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
      }
    }
    if (tid == 0) a.ncand[q] = (int32_t)ncand;
    __syncthreads();
  }
}

// Ordered compaction of a bitmap into out[base..], four words per thread per
// round, clearing it on the way.  Each warp stages its ids in shared memory
// (kUnionStage per warp, in windows if a round yields more) and copies them
// out with consecutive lanes on consecutive positions, so the stores are
// coalesced instead of one 32-byte sector per 4-byte id.
constexpr int kUnionStage = 512;

template <int NT>
__device__ __forceinline__ int64_t emit_bitmap_staged(uint4 *bits4, int nwords4, int32_t *out,
                                                      int64_t cap, int *wsum, int32_t *stage) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  const int capi = cap < 0x7fffffff ? (int)cap : 0x7fffffff;
  int64_t total = 0;
  for (int r0 = 0; r0 < nwords4; r0 += NT) {
    const int i = r0 + threadIdx.x;
    uint4 w4 = i < nwords4 ? bits4[i] : make_uint4(0u, 0u, 0u, 0u);
    const int pc = __popc(w4.x) + __popc(w4.y) + __popc(w4.z) + __popc(w4.w);
    if (pc) bits4[i] = make_uint4(0u, 0u, 0u, 0u);
    int incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int c = lane < NW ? wsum[lane] : 0;
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += u;
      }
      if (lane < NW) wsum[lane] = x - c;
      if (lane == 31) wsum[NW] = x;
    }
    __syncthreads();
    const int tot = wsum[NW];
    const int64_t gbase = total + wsum[warp];  // this warp's first output position
    const int wtot = __shfl_sync(0xffffffffu, incl, 31);
    const int pos0 = incl - pc;  // warp-local
    const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
    for (int c0 = 0; c0 < wtot && gbase + c0 < capi; c0 += kUnionStage) {
      if (pc && pos0 < c0 + kUnionStage && incl > c0) {
        if (pos0 >= c0 && incl <= c0 + kUnionStage) {
          // common case: all of this thread's ids land in the window
          int p = pos0 - c0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t word = wv[j];
            const int32_t id0 = (i * 4 + j) * 32;
            while (word) {
              stage[p++] = id0 + __ffs(word) - 1;
              word &= word - 1u;
            }
          }
        } else {
          int p = pos0 - c0;  // may start below the window
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t word = wv[j];
            const int32_t id0 = (i * 4 + j) * 32;
            while (word) {
              if (p >= 0 && p < kUnionStage) stage[p] = id0 + __ffs(word) - 1;
              ++p;
              word &= word - 1u;
            }
          }
        }
      }
      __syncwarp();
      const int cnt = wtot - c0 < kUnionStage ? wtot - c0 : kUnionStage;
      for (int k = lane; k < cnt; k += 32) {
        const int64_t gp = gbase + c0 + k;
        if (gp < capi) out[gp] = stage[k];
      }
      __syncwarp();
    }
    total += tot;
    __syncthreads();
  }
  return total;
}

// v == 1: the candidate set is the union of the T leaves, so one bit per id
// replaces the counters and the whole id range fits one shared-memory bitmap
// (n <= ~1.3M).  Slices need not be sorted.  The T slice bounds are fetched
// into shared memory in one round trip; groups of G lanes then walk whole
// leaf slices (contiguous runs of leaf_indices) with UNR loads in flight and
// set bits with shared atomicOr; the bitmap is compacted in id order
// (ascending candidate lists, like the counting path) and cleared on the way.
template <int NT>
__global__ void __launch_bounds__(NT, NT <= 256 ? 4 : 1) k_vote_union(VoteArgs a, int G) {
  extern __shared__ uint4 vote_smem[];
  uint32_t *bits = reinterpret_cast<uint32_t *>(vote_smem);
  const int nwords4 = (int)((a.n + 127) >> 7);
  int32_t *stage = reinterpret_cast<int32_t *>(vote_smem + nwords4);  // NW * kUnionStage
  int64_t *s_start = reinterpret_cast<int64_t *>(stage + (NT / 32) * kUnionStage);  // T
  int32_t *s_len = reinterpret_cast<int32_t *>(s_start + a.T);                      // T
  __shared__ int wsum[NT / 32 + 1];
  const int tid = threadIdx.x;
  const int gl = tid & (G - 1), ngroups = NT / G;
  int32_t *my_stage = stage + (tid >> 5) * kUnionStage;
  for (int i = tid; i < nwords4; i += NT) vote_smem[i] = make_uint4(0u, 0u, 0u, 0u);
  const int64_t nwork = a.qlist ? (int64_t)*a.qcount : a.nq;
  for (int64_t wq = blockIdx.x; wq < nwork; wq += gridDim.x) {
    const int64_t q = a.qlist ? (int64_t)a.qlist[wq] : wq;
    for (int t = tid; t < a.T; t += NT) {
      const int leaf = a.leaves[q * a.T + t];
      const int64_t *o = a.leaf_offsets + (int64_t)t * (a.L + 1) + leaf;
      const int64_t s0 = o[0];
      s_start[t] = (int64_t)t * a.n + s0;
      s_len[t] = (int)(o[1] - s0);
    }
    __syncthreads();
    // 16-byte loads: a slice [s, s + len) is covered by the aligned int4
    // groups from s & ~3; lanes keep the components that fall inside it
    for (int t = tid / G; t < a.T; t += ngroups) {
      const int64_t s0 = s_start[t];
      const int len = s_len[t];
      const int64_t a0 = s0 & ~(int64_t)3;
      const int lo = (int)(s0 - a0), hi = lo + len;  // element range within the aligned run
      const int4 *L4 = reinterpret_cast<const int4 *>(a.leaf_indices + a0);
      const int n4 = (hi + 3) >> 2;
      constexpr int UNR = 8;
      for (int p0 = gl; p0 < n4; p0 += UNR * G) {
        int4 v[UNR];
        const int64_t total = (int64_t)a.T * a.n;  // no 16-byte load past the array
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int p = p0 + u * G;
          if (p < n4 && a0 + 4 * (int64_t)p + 4 <= total) {
            v[u] = __ldg(L4 + p);
          } else {
            int w[4];
#pragma unroll
            for (int c = 0; c < 4; ++c)
              w[c] = p < n4 && a0 + 4 * (int64_t)p + c < total ? __ldg(a.leaf_indices + a0 + 4 * p + c) : -1;
            v[u] = make_int4(w[0], w[1], w[2], w[3]);
          }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int e = 4 * (p0 + u * G);
          const int ids[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
          if (e >= lo && e + 4 <= hi) {  // interior group: no per-id range checks
#pragma unroll
            for (int c = 0; c < 4; ++c) atomicOr(bits + (ids[c] >> 5), 1u << (ids[c] & 31));
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (e + c >= lo && e + c < hi) atomicOr(bits + (ids[c] >> 5), 1u << (ids[c] & 31));
          }
        }
      }
    }
    __syncthreads();
    const int64_t nc = a.bits_out
        ? store_bits<NT>(bits, (int)((a.n + 31) >> 5), a.bits_out + q * a.bstride, wsum)
        : emit_bitmap_staged<NT>(vote_smem, nwords4, a.cand + q * a.cap, a.cap, wsum, my_stage);
    if (tid == 0) a.ncand[q] = (int32_t)nc;  // > cap means only cap ids were stored
  }
}

typedef void (*vote_fn)(VoteArgs);
typedef void (*union_fn)(VoteArgs, int);
static inline void k_vote_union_launch(union_fn fn, unsigned grid, int nt, size_t smem, cudaStream_t s,
                                       const VoteArgs &a, int G) {
  (count_launch(), fn<<<grid, nt, smem, s>>>(a, G));
}

template <int CW, bool SORTED>
static vote_fn pick_g(int G) {
  switch (G) {
    case 1: return k_vote<CW, 1, SORTED>;
    case 2: return k_vote<CW, 2, SORTED>;
    case 4: return k_vote<CW, 4, SORTED>;
    case 8: return k_vote<CW, 8, SORTED>;
    case 16: return k_vote<CW, 16, SORTED>;
    default: return k_vote<CW, 32, SORTED>;
  }
}

template <bool SORTED>
static vote_fn pick_cw(int CW, int G) {
  if (CW == 1) return pick_g<1, SORTED>(G);
  if (CW == 2) return pick_g<2, SORTED>(G);
  if (CW == 3) return pick_g<3, SORTED>(G);
  return pick_g<4, SORTED>(G);
}

// Dense counts for one query: one CTA per tree, global atomics.
__global__ void k_vote_dense(const int32_t *__restrict__ leaf_indices,
                             const int64_t *__restrict__ leaf_offsets, int64_t n, int L,
                             const int32_t *__restrict__ leaves, int32_t *counts) {
  const int t = blockIdx.x;
  const int leaf = leaves[t];
  const int64_t *o = leaf_offsets + (int64_t)t * (L + 1);
  const int32_t *Lt = leaf_indices + (int64_t)t * n;
  for (int64_t i = o[leaf] + threadIdx.x; i < o[leaf + 1]; i += blockDim.x) atomicAdd(counts + Lt[i], 1);
}

// Ordered compaction with one CTA of 1024 threads: rounds of 1024 elements,
// ballot ranks, running base.
__global__ void __launch_bounds__(1024) k_select_ge(const int32_t *__restrict__ counts, int64_t n,
                                                    int v, int32_t *out, int64_t *nout) {
  __shared__ int wcnt[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t base = 0;
  for (int64_t r0 = 0; r0 < n; r0 += 1024) {
    const int64_t i = r0 + threadIdx.x;
    const bool f = i < n && counts[i] >= v;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wcnt[warp] = __popc(bal);
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      before += w < warp ? wcnt[w] : 0;
      tot += wcnt[w];
    }
    if (f) out[base + before + __popc(bal & lanemask_lt())] = (int32_t)i;
    base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *nout = base;
}

__global__ void k_mark_ids(const int64_t *__restrict__ cand, int64_t m, int64_t n, uint32_t *bitmap,
                           int32_t *bad) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id = cand[j];
    if (id < 0 || id >= n) {
      *bad = 1;
    } else {
      atomicOr(bitmap + (id >> 5), 1u << (id & 31));
    }
  }
}

__global__ void __launch_bounds__(1024) k_bitmap_compact(const uint32_t *__restrict__ bitmap,
                                                         int64_t nwords, int32_t *out,
                                                         int64_t *nout) {
  __shared__ int wcnt[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t base = 0;
  for (int64_t r0 = 0; r0 < nwords; r0 += 1024) {
    const int64_t i = r0 + threadIdx.x;
    uint32_t word = i < nwords ? bitmap[i] : 0u;
    const int pc = __popc(word);
    int incl = pc;
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wcnt[warp] = incl;
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      before += w < warp ? wcnt[w] : 0;
      tot += wcnt[w];
    }
    int64_t pos = base + before + incl - pc;
    while (word) {
      const int b = __ffs(word) - 1;
      out[pos++] = (int32_t)(i * 32 + b);
      word &= word - 1;
    }
    base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *nout = base;
}

// ---------------------------------------------------------------------------
// Streamed tiled vote (configs 4-5: many id tiles, T <= 1024).  Built once
// per index: for every leaf slice, its part in each id tile ("piece") is
// stored padded to a multiple of 7 entries, pieces in tile order, and each
// entry is pre-decoded into its tile-local counter address -- the counter
// word (16 bits: a tile's counters are < 64K words) and the lane within the
// word (2 bits) -- seven entries per 16-byte "quad":
//     u16[0..6] = counter words of entries 0..6,  u16[7] = 2-bit lanes
// so the vote reads every piece with aligned 16-byte loads (7 ids each, vs
// 4 for 32-bit ids) and bumps a counter with no division by the packing.
// Padding entries address one of 32 spare words past the counters (by slot,
// so the lanes of a load rarely share one): they are bumped like any entry
// (no per-entry test) and never emitted.
// qdir[(t*L + leaf)*(ntiles+1) + w] = start (in quads) of tile w's piece
// within the leaf's padded slice; qbase[t*L + leaf] = the slice's first quad
// within tree t's padded row (tree t's row starts at quad t * tstride).
// The counts are identical to the plain vote's: every occurrence of every id
// is counted once (_cy.pyx:66-77); only the memory layout differs.
constexpr int kQuadIds = 7;

// counter lanes per 32-bit word and their width (bits)
template <int CW>
__host__ __device__ __forceinline__ constexpr int lanes_per_word() {
  return CW == 1 ? 4 : (CW == 3 ? 3 : (CW == 2 ? 2 : 1));
}
template <int CW>
__host__ __device__ __forceinline__ constexpr int lane_bits() {
  return CW == 1 ? 8 : (CW == 3 ? 10 : (CW == 2 ? 16 : 0));
}
// first spare word (padding target) after the counters (rounded up to 4)
template <int CW>
__host__ __device__ __forceinline__ int spare_word0(int W) {
  return (counter_words<CW>(W) + 3) & ~3;
}
// qdir holds, after k_build_dir, the piece start POSITIONS within each leaf
// slice (u16); this turns them into padded quad offsets in place and writes
// each leaf's padded length (quads) to qlen.  One warp per leaf.
__global__ void k_vstream_quads(uint16_t *qdir, int64_t nleaves, int ntiles, int32_t *qlen) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < nleaves; g += wstride) {
    uint16_t *d = qdir + g * (ntiles + 1);
    int carry = 0;
    for (int w0 = 0; w0 < ntiles; w0 += 32) {
      const int w = w0 + lane;
      int q = 0;
      if (w < ntiles) q = ((int)d[w + 1] - (int)d[w] + kQuadIds - 1) / kQuadIds;  // read before any write
      int incl = q;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      __syncwarp();
      if (w < ntiles) d[w] = (uint16_t)(carry + incl - q);
      carry += __shfl_sync(0xffffffffu, incl, 31);
      __syncwarp();
    }
    if (lane == 0) {
      d[ntiles] = (uint16_t)carry;
      qlen[g] = carry;
    }
  }
}

// Per tree: exclusive scan of the leaves' padded lengths -> qbase, total ->
// tree_quads[t].  One CTA (1024 threads) per tree.
__global__ void __launch_bounds__(1024) k_vstream_base(int32_t *qbase, int L, int64_t *tree_quads) {
  __shared__ int wsum[33];
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int32_t *b = qbase + (int64_t)t * L;
  long long carry = 0;
  for (int f0 = 0; f0 < L; f0 += 1024) {
    const int f = f0 + tid;
    const int v = f < L ? b[f] : 0;
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
    if (f < L) b[f] = (int32_t)(carry + wsum[warp] + incl - v);
    carry += wsum[32];
    __syncthreads();
  }
  if (tid == 0) tree_quads[t] = carry;
}

// Fill the padded, pre-decoded slices.  One warp per leaf: the lanes find
// where each tile's run starts in the (ascending) slice by binary search,
// then every lane assembles whole quads (tile of the quad from the quad
// directory, its 7 entries from the run) and stores each with one 16-byte
// store.  Run starts and the leaf's directory row are staged per warp in
// shared memory (ntiles <= kStreamMaxTiles).
constexpr int kStreamMaxTiles = 1024;
template <int CW>
__global__ void __launch_bounds__(256) k_vstream_fill(const int32_t *__restrict__ leaf_indices,
                                                      const int64_t *__restrict__ leaf_offsets, int64_t n, int T, int L,
                                                      int W, int ntiles, const uint16_t *__restrict__ qdir,
                                                      const int32_t *__restrict__ qbase, int64_t tstride, uint32_t *qs) {
  extern __shared__ int32_t fill_smem[];
  constexpr int PER = lanes_per_word<CW>();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t *rs = fill_smem + warp * 2 * (ntiles + 1);  // run start per tile (+ end)
  int32_t *dq = rs + (ntiles + 1);                    // quad offset per tile (+ total)
  const uint32_t spare = (uint32_t)spare_word0<CW>(W);
  const int64_t nleaves = (int64_t)T * L;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; g < nleaves; g += wstride) {
    const int64_t t = g / L, leaf = g - t * L;
    const int64_t *o = leaf_offsets + t * (L + 1);
    const int64_t s0 = o[leaf];
    const int m = (int)(o[leaf + 1] - s0);
    const int32_t *sl = leaf_indices + t * n + s0;
    const uint16_t *d = qdir + g * (ntiles + 1);
    __syncwarp();
    for (int w = lane; w <= ntiles; w += 32) {
      dq[w] = d[w];
      int lo = 0, hi = m;  // first position with id >= w * W
      const int64_t key = (int64_t)w * W;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int64_t)sl[mid] < key) lo = mid + 1;
        else hi = mid;
      }
      rs[w] = w == ntiles ? m : lo;
    }
    __syncwarp();
    const int nquads = dq[ntiles];
    uint4 *out = reinterpret_cast<uint4 *>(qs) + (t * tstride + qbase[g]);
    for (int q = lane; q < nquads; q += 32) {
      int lo = 0, hi = ntiles - 1;  // tile of quad q: last w with dq[w] <= q
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (dq[mid] <= q) lo = mid;
        else hi = mid - 1;
      }
      const int w = lo;
      const int j0 = rs[w] + kQuadIds * (q - dq[w]);
      const int rend = rs[w + 1];
      uint32_t wd[kQuadIds], fb = 0u;
#pragma unroll
      for (int i = 0; i < kQuadIds; ++i) {
        const int p = j0 + i;
        if (p < rend) {
          const int local = sl[p] - w * W;
          const int word = local / PER;
          wd[i] = (uint32_t)word;
          fb |= (uint32_t)(local - word * PER) << (2 * i);
        } else {
          wd[i] = spare + (uint32_t)((q * kQuadIds + i) & 31);
        }
      }
      out[q] = make_uint4(wd[0] | (wd[1] << 16), wd[2] | (wd[3] << 16), wd[4] | (wd[5] << 16), wd[6] | (fb << 16));
    }
  }
}

// Shared-memory atomic add at a 32-bit shared address; returns the old word.
__device__ __forceinline__ uint32_t atom_add_shared(uint32_t saddr, uint32_t inc) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(saddr), "r"(inc) : "memory");
  return old;
}

// 16-byte load that bypasses L1 allocation and asks L2 to fetch the whole
// 256-byte block around it from DRAM: a leaf slice stores its per-tile pieces
// back to back, so the pieces of the next tiles arrive with this one and are
// found in L2 later, and DRAM serves 256-byte bursts instead of scattered
// 32-byte sectors (random 32-byte reads reach 0.6 TB/s, random 256-byte
// blocks 3 TB/s, tools/micro/rand_mlp.cu).
__device__ __forceinline__ uint4 ld_quad_l2_256(const uint4 *p) {
  uint4 v;
  asm volatile("ld.global.cg.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Per-warp window source of the streamed vote: the warp's pieces of one id
// tile flattened into 32-quad windows; next() returns this lane's quad of
// the next window (padding past the end).  Windows must be taken in order.
struct StreamWindows {
  int pre, len, total, before, next_w;
  int pf;  // experiment: 1 prefetch the 1 KB region a quad opens, 2 the next one, 3 the next 2 KB
  __device__ __forceinline__ void begin(int len_, uint32_t lbase_minus, uint32_t *w_off_row) {
    const int lane = threadIdx.x & 31;
    len = len_;
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    total = __shfl_sync(0xffffffffu, incl, 31);
    pre = incl - len;
    const unsigned ne = __ballot_sync(0xffffffffu, len > 0);
    __syncwarp();  // the previous tile's rank table has been read by every lane
    if (len > 0) w_off_row[__popc(ne & lanemask_lt())] = lbase_minus - (uint32_t)pre;
    __syncwarp();
    before = 0;
    next_w = 0;
  }
  __device__ __forceinline__ int windows() const { return (total + 31) >> 5; }
  template <bool CG>
  __device__ __forceinline__ uint4 next(unsigned long long wb, const uint32_t *w_off_row, uint4 padq) {
    const int lane = threadIdx.x & 31;
    const int w0 = 32 * next_w++;
    const int rel = pre - w0;
    const bool inwin = len > 0 && (unsigned)rel < 32u;
    const unsigned starts = __reduce_or_sync(0xffffffffu, inwin ? (1u << rel) : 0u);
    const int rank = before + __popc(starts & (0xffffffffu >> (31 - lane))) - 1;
    before += __popc(starts);
    const int e = w0 + lane;
    // .cg: the quads are read once; with the counters taking most of the
    // shared/L1 carve-out, allocating them in L1 only throttles the loads
    if (e >= total) return padq;
    const uint4 *src = reinterpret_cast<const uint4 *>(wb) + (w_off_row[rank] + (uint32_t)e);
    if (pf && (reinterpret_cast<uintptr_t>(src) & 1023u) == 0) {
      const char *r = reinterpret_cast<const char *>(src) + (pf >= 2 ? 1024 : 0);
      if (pf == 3)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], 2048;" ::"l"(r) : "memory");
      else
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], 1024;" ::"l"(r) : "memory");
    }
    if (CG) return ld_quad_l2_256(src);
    return __ldg(src);
  }
};

// The streamed vote: one CTA (1024 threads, one per SM) per query at a time;
// warp w owns the contiguous tree range [w*T/32, (w+1)*T/32) (<= 32 trees,
// one per lane).  Per id tile, the warp flattens its trees' pieces (quads)
// into 32-quad windows: a lane finds the piece holding its quad from the
// piece starts inside the window (__reduce_or_sync) and a 32-entry rank
// table, loads the quad with one 16-byte load and bumps its 4 counters.
// Loads run P windows ahead of the bumps (a register ring), across tile
// boundaries: the next tile's first windows are loaded before the barrier
// that separates the tiles.  The increment that lifts a count to v appends
// the id to the query's list (the reference's `counts[idx] == v` emission,
// _cy.pyx:75-77; order within a tile is not kept).  ncand may exceed cap
// (only cap ids stored).
template <int CW, int P, bool CG>
__global__ void __launch_bounds__(1024, 1) k_vote_stream(VoteArgs a, const uint4 *__restrict__ qs,
                                                         const int32_t *__restrict__ qbase, int64_t tstride) {
  extern __shared__ uint4 vote_smem[];
  uint32_t *cnt = reinterpret_cast<uint32_t *>(vote_smem);
  uint32_t cnt_s = (uint32_t)__cvta_generic_to_shared(cnt);
  asm volatile("" : "+r"(cnt_s));  // computed once, not re-derived per bump
  const int cwords = spare_word0<CW>(a.W);  // + 32 spare words (padding targets)
  const uint32_t pad_word = (uint32_t)cwords;  // entries addressing words >= pad_word are padding
  constexpr int NW = 32;
  __shared__ uint32_t w_off[NW][32];
  __shared__ int s_nc;
  constexpr uint32_t MASK = CW == 1 ? 0xffu : (CW == 3 ? 0x3ffu : (CW == 2 ? 0xffffu : 0xffffffffu));
  const uint32_t vm1 = (uint32_t)(a.v - 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t nc_s = (uint32_t)__cvta_generic_to_shared(&s_nc);
  asm volatile("" : "+r"(nc_s));
  const int cap32 = a.cap < 0x7fffffff ? (int)a.cap : 0x7fffffff;
  const int64_t dstride = a.ntiles + 1;
  const int t_lo = (int)(((int64_t)warp * a.T) / NW);
  const int t_hi = (int)(((int64_t)(warp + 1) * a.T) / NW);
  const int t = t_lo + lane;
  const bool has = t < t_hi;
  // the warp's first tree row, kept in a register (opaque to the compiler,
  // which would otherwise re-derive it from the kernel parameters per load)
  unsigned long long wb = reinterpret_cast<unsigned long long>(qs + (int64_t)t_lo * tstride);
  asm volatile("" : "+l"(wb));
  uint32_t *woff = w_off[warp];
  uint4 *c4 = reinterpret_cast<uint4 *>(cnt);
  // window tails: 7 padding entries on this lane's own spare word
  const uint32_t pw = pad_word + (uint32_t)lane;
  const uint4 padq = make_uint4(pw | (pw << 16), pw | (pw << 16), pw | (pw << 16), pw);
  constexpr int PER = lanes_per_word<CW>();
  constexpr int LB = lane_bits<CW>();
  for (int64_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
    const uint16_t *dl = nullptr;
    uint32_t lbase = 0;
    int dcur = 0, dnxt = 0, dnn = 0;
    if (has) {
      const int64_t g = (int64_t)t * a.L + a.leaves[q * a.T + t];
      dl = a.dir + g * dstride;
      lbase = (uint32_t)((int64_t)lane * tstride + qbase[g]);
      dcur = dl[0];
      dnxt = dl[1];
      dnn = a.ntiles >= 2 ? (int)__ldg(dl + 2) : 0;
    }
    int32_t *qcand = a.cand + q * a.cap;
    // tile 0's windows start loading before the counters are cleared
    StreamWindows sw;
    sw.pf = (a.dbg >> 2) & 3;
    sw.begin(dnxt - dcur, lbase + (uint32_t)dcur, woff);
    uint4 ring[P];
#pragma unroll
    for (int i = 0; i < P; ++i) ring[i] = i < sw.windows() ? sw.template next<CG>(wb, woff, padq) : padq;
    for (int i = tid; i < cwords / 4; i += 1024) c4[i] = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) s_nc = 0;
    __syncthreads();
    for (int tile = 0; tile < a.ntiles; ++tile) {
      const int32_t lo = tile * a.W;
      const int nwin = sw.windows();
      for (int w0 = 0; w0 < nwin; w0 += P) {
#pragma unroll
        for (int i = 0; i < P; ++i) {
          if (w0 + i < nwin) {  // warp-uniform
            const uint4 cur = ring[i];
            if (w0 + i + P < nwin) ring[i] = sw.template next<CG>(wb, woff, padq);
            const uint32_t wd[kQuadIds] = {cur.x & 0xffffu, cur.x >> 16, cur.y & 0xffffu, cur.y >> 16,
                                           cur.z & 0xffffu, cur.z >> 16, cur.w & 0xffffu};
            const uint32_t fb = cur.w >> 16;
            uint32_t old[kQuadIds];
#pragma unroll
            for (int c = 0; c < kQuadIds; ++c) {
              const uint32_t sh = ((fb >> (2 * c)) & 3u) * LB;
              old[c] = (a.dbg & 1) ? 0u : atom_add_shared(cnt_s + 4u * wd[c], 1u << sh);
            }
#pragma unroll
            for (int c = 0; c < kQuadIds; ++c) {
              const uint32_t f = (fb >> (2 * c)) & 3u;
              if (((old[c] >> (f * LB)) & MASK) == vm1 && wd[c] < pad_word) {  // lifted a count to v
                const int pos = (int)atom_add_shared(nc_s, 1u);
                if (pos < cap32) qcand[pos] = lo + (int)(wd[c] * PER + f);
              }
            }
          }
        }
      }
      // the next tile's windows start loading before the tile barrier
      if (tile + 1 < a.ntiles) {
        dcur = dnxt;
        dnxt = dnn;
        dnn = (has && tile + 3 <= a.ntiles) ? (int)__ldg(dl + tile + 3) : 0;
        sw.begin(dnxt - dcur, lbase + (uint32_t)dcur, woff);
#pragma unroll
        for (int i = 0; i < P; ++i) ring[i] = i < sw.windows() ? sw.template next<CG>(wb, woff, padq) : padq;
        __syncthreads();
        if (!(a.dbg & 2))
          for (int i = tid; i < cwords / 4; i += 1024) c4[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
      }
    }
    __syncthreads();
    if (tid == 0) a.ncand[q] = s_nc;  // > cap means only cap ids were stored
    __syncthreads();
  }
}

// ------------------------------------------------------ paired streamed vote --
// Pair layout: the id tiles are taken two at a time ("super-tile" j = tiles
// 2j and 2j+1).  Per leaf slice, super-piece j holds max(qa, qb) 32-byte
// PAIRS, pair k = {quad k of tile 2j's piece, quad k of tile 2j+1's piece}
// (the shorter side padded with padding quads), so one 32-byte load brings a
// quad of both tiles and a query's slices are read with half as many
// (twice as long) requests as with one piece per tile.
// pdir[(t*L + leaf)*(nsup+1) + j] = first pair of super-piece j within the
// slice; pbase[t*L + leaf] = the slice's first pair within tree t's row
// (tree t's row starts at pair t * pstride).

// Per leaf: super-piece lengths from the per-tile run starts (k_build_dir),
// exclusive scan -> pdir, total -> plen.  One warp per leaf.
__global__ void k_vpair_dir(const uint16_t *__restrict__ pos, uint16_t *pdir, int64_t nleaves, int ntiles,
                            int nsup, int32_t *plen) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < nleaves; g += wstride) {
    const uint16_t *p = pos + g * (ntiles + 1);
    uint16_t *d = pdir + g * (nsup + 1);
    int carry = 0;
    for (int j0 = 0; j0 < nsup; j0 += 32) {
      const int j = j0 + lane;
      int len = 0;
      if (j < nsup) {
        const int qa = ((int)p[2 * j + 1] - (int)p[2 * j] + kQuadIds - 1) / kQuadIds;
        const int qb = 2 * j + 1 < ntiles ? ((int)p[2 * j + 2] - (int)p[2 * j + 1] + kQuadIds - 1) / kQuadIds : 0;
        len = qa > qb ? qa : qb;
      }
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (j < nsup) d[j] = (uint16_t)(carry + incl - len);
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      d[nsup] = (uint16_t)carry;
      plen[g] = carry;
    }
  }
}

// quad k of tile w's piece of a slice: 7 pre-decoded entries (padding past
// the run end addresses spare words by position)
template <int CW>
__device__ __forceinline__ uint4 vpair_quad(const int32_t *sl, const int32_t *rs, int w, int ntiles, int k, int W,
                                            uint32_t spare) {
  constexpr int PER = lanes_per_word<CW>();
  uint32_t wd[kQuadIds], fb = 0u;
  const int j0 = w < ntiles ? rs[w] + kQuadIds * k : 0;
  const int rend = w < ntiles ? rs[w + 1] : 0;
#pragma unroll
  for (int i = 0; i < kQuadIds; ++i) {
    const int p = j0 + i;
    if (p < rend) {
      const int local = sl[p] - w * W;
      const int word = local / PER;
      wd[i] = (uint32_t)word;
      fb |= (uint32_t)(local - word * PER) << (2 * i);
    } else {
      wd[i] = spare + (uint32_t)((k * kQuadIds + i) & 31);
    }
  }
  return make_uint4(wd[0] | (wd[1] << 16), wd[2] | (wd[3] << 16), wd[4] | (wd[5] << 16), wd[6] | (fb << 16));
}

// Fill the pair layout.  One warp per leaf; run starts and the super-piece
// directory row staged per warp in shared memory.
template <int CW>
__global__ void __launch_bounds__(256) k_vpair_fill(const int32_t *__restrict__ leaf_indices,
                                                    const int64_t *__restrict__ leaf_offsets, int64_t n, int T, int L,
                                                    int W, int ntiles, int nsup, const uint16_t *__restrict__ pos,
                                                    const uint16_t *__restrict__ pdir,
                                                    const int32_t *__restrict__ pbase, int64_t pstride, uint4 *out) {
  extern __shared__ int32_t fill_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t *rs = fill_smem + warp * (ntiles + 1 + nsup + 1);  // run start per tile (+ end)
  int32_t *dp = rs + (ntiles + 1);                           // pair offset per super-tile (+ total)
  const uint32_t spare = (uint32_t)spare_word0<CW>(W);
  const int64_t nleaves = (int64_t)T * L;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; g < nleaves; g += wstride) {
    const int64_t t = g / L, leaf = g - t * L;
    const int32_t *sl = leaf_indices + t * n + leaf_offsets[t * (L + 1) + leaf];
    __syncwarp();
    for (int w = lane; w <= ntiles; w += 32) rs[w] = pos[g * (ntiles + 1) + w];
    for (int j = lane; j <= nsup; j += 32) dp[j] = pdir[g * (nsup + 1) + j];
    __syncwarp();
    const int npairs = dp[nsup];
    uint4 *o = out + 2 * (t * pstride + pbase[g]);
    for (int pp = lane; pp < npairs; pp += 32) {
      int lo = 0, hi = nsup - 1;  // super-piece of pair pp: last j with dp[j] <= pp
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (dp[mid] <= pp) lo = mid;
        else hi = mid - 1;
      }
      const int j = lo, k = pp - dp[j];
      o[2 * pp] = vpair_quad<CW>(sl, rs, 2 * j, ntiles, k, W, spare);
      o[2 * pp + 1] = vpair_quad<CW>(sl, rs, 2 * j + 1, ntiles, k, W, spare);
    }
  }
}

__device__ __forceinline__ void ld_pair_l2_256(const uint4 *p, uint4 &a, uint4 &b) {
  asm volatile("ld.global.cg.L2::256B.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

// Bump the 7 counters of one quad; the increment that lifts a count to v
// appends the id (_cy.pyx:75-77).  The returned counts are tested into one
// predicate per quad (events are rare per id), and only a quad holding an
// event walks its 7 entries again.
// Saturating 8-bit counters (SAT): counts above 255 are possible (T up to
// 1024) but only the crossing of v matters.  The counters are BIASED: they
// are cleared to kSatCross + 1 - v (v <= kSatMaxV = 128), so the increment
// that lifts a count to v is the one that reads kSatCross = 127, and a
// counter that reaches 192 is pulled back by 64 -- by the one increment that
// read 191 -- so it cycles in [128, 192]: above kSatCross, no id is listed
// twice.  Every event value (63: nothing, 127: crossing, 191: pull-back, 255:
// about to wrap) has its low six bits set, so the test per id is one masked
// compare, the same cost as the plain counters'.  Should increments outrun a
// pull-back and wrap a counter, the increment that wraps it reads 255 and
// raises the query's overflow flag; the query is then redone by
// vote_pair_careful.  Either way every id whose count reaches v is listed
// exactly once (_cy.pyx:75-77).
// Queries redone by vote_pair_careful (mrpt_vote_stats; measurement only).
__device__ unsigned long long g_vote_sat_redos;

constexpr uint32_t kSatCross = 127, kSatPull = 191, kSatSub = 64;
constexpr int kSatMaxV = 128;

// Append one id to the query's candidate list.  nc_lane is the list counter's
// shared address made lane-dependent on purpose (see k_vote_pair): with a
// provably uniform address ptxas wraps the atomic in an 11-instruction
// warp-aggregation sequence, which loses when one or two lanes emit; qcand is
// kept opaque so its 64-bit base is not recomputed per emission.
__device__ __forceinline__ void pair_emit(uint32_t nc_lane, int32_t *qcand, int cap32, int32_t id) {
  const int pos = (int)atom_add_shared(nc_lane, 1u);
  if (pos < cap32)
    asm volatile("{ .reg .u64 a; mad.wide.u32 a, %1, 4, %0; st.global.u32 [a], %2; }" ::"l"(qcand), "r"(pos), "r"(id)
                 : "memory");
}

template <int CW, bool SAT = false>
__device__ __forceinline__ void pair_bump(uint4 cur, uint32_t cnt_s, uint32_t nc_s, uint32_t pad_word, uint32_t vm1,
                                          int32_t lo, int32_t *qcand, int cap32, uint32_t ovf_s = 0) {
  constexpr uint32_t MASK = CW == 1 ? 0xffu : (CW == 3 ? 0x3ffu : (CW == 2 ? 0xffffu : 0xffffffffu));
  constexpr int PER = lanes_per_word<CW>();
  constexpr int LB = lane_bits<CW>();
  const uint32_t wd[kQuadIds] = {cur.x & 0xffffu, cur.x >> 16, cur.y & 0xffffu, cur.y >> 16,
                                 cur.z & 0xffffu, cur.z >> 16, cur.w & 0xffffu};
  const uint32_t fb = cur.w >> 16;
  uint32_t old[kQuadIds];
  // an all-padding quad (pieces pad at their end; window tails): its lane sits
  // out, so the others' atomics meet fewer bank conflicts
  if (wd[0] >= pad_word) return;
#pragma unroll
  for (int c = 0; c < kQuadIds; ++c) old[c] = atom_add_shared(cnt_s + 4u * wd[c], 1u << (((fb >> (2 * c)) & 3u) * LB));
  // per-id event predicates, kept for the second walk
  bool ev[kQuadIds], any = false;
#pragma unroll
  for (int c = 0; c < kQuadIds; ++c) {
    const uint32_t fld = (old[c] >> (((fb >> (2 * c)) & 3u) * LB)) & MASK;
    ev[c] = SAT ? ((fld & 63u) == 63u) : (fld == vm1);
    any |= ev[c];
  }
  if (!any) return;
#pragma unroll
  for (int c = 0; c < kQuadIds; ++c) {
    if (!ev[c]) continue;
    const uint32_t f = (fb >> (2 * c)) & 3u;
    if (SAT) {
      // Padding entries are not excluded up front: their spare words are
      // pulled back like any counter (tested for padding inside instead).
      const uint32_t fld = (old[c] >> (f * LB)) & MASK;
      if (fld == kSatCross) {
        if (wd[c] < pad_word) pair_emit(nc_s, qcand, cap32, lo + (int)(wd[c] * PER + f));  // lifted a count to v
      } else if (fld == kSatPull) {
        atom_add_shared(cnt_s + 4u * wd[c], 0u - (kSatSub << (f * LB)));
      } else if (fld == MASK && wd[c] < pad_word) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(ovf_s), "r"(1u) : "memory");
      }
    } else if (wd[c] < pad_word) {
      pair_emit(nc_s, qcand, cap32, lo + (int)(wd[c] * PER + f));  // lifted a count to v
    }
  }
}

// The exact redo of one query after a counter overflow of the saturating
// vote (never seen on the benchmark configurations; MRPT_VOTE_DBG=8 forces
// it for the tests).  Warp 0 alone bumps, every lane walking its own tree's
// piece, and an increment is made only while the counter read just before is
// below v: between that read and the increment at most the other 31 lanes
// of the same instruction add to the counter, so it stays below v + 32 <= 160
// and cannot wrap.  The other warps only help clearing.
// It runs in its own kernel (k_vote_pair_redo) over the queries the main
// kernel listed, so the main kernel carries no call and no stack frame.
__device__ __forceinline__ void vote_pair_careful(const VoteArgs &a, const uint4 *__restrict__ ps,
                                               const int32_t *__restrict__ pbase, int64_t pstride, int64_t q,
                                               uint32_t *cnt, int cwords, int *s_nc) {
  constexpr int PER = 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nsup = (a.ntiles + 1) >> 1;
  const int64_t dstride = nsup + 1;
  const uint32_t pad_word = (uint32_t)cwords, v = (uint32_t)a.v;
  const int cap32 = a.cap < 0x7fffffff ? (int)a.cap : 0x7fffffff;
  int32_t *qcand = a.cand + q * a.cap;
  uint4 *c4 = reinterpret_cast<uint4 *>(cnt);
  if (tid == 0) *s_nc = 0;
  for (int w = 0; w < a.ntiles; ++w) {
    __syncthreads();
    for (int i = tid; i < cwords / 4; i += 1024) c4[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    if (warp != 0) continue;
    const int j = w >> 1, side = w & 1;
    const int32_t lo = w * a.W;
    for (int g = 0; g < 32; ++g) {
      const int t_lo = (int)(((int64_t)g * a.T) / 32), t_hi = (int)(((int64_t)(g + 1) * a.T) / 32);
      const int t = t_lo + lane;
      int len = 0;
      const uint4 *src = nullptr;
      if (t < t_hi) {
        const int64_t gl = (int64_t)t * a.L + a.leaves[q * a.T + t];
        const uint16_t *dl = a.dir + gl * dstride;
        const int start = dl[j];
        len = (int)dl[j + 1] - start;
        src = ps + 2 * ((int64_t)t * pstride + pbase[gl] + start) + side;
      }
      const int maxlen = __reduce_max_sync(0xffffffffu, len);
      for (int p = 0; p < maxlen; ++p) {
        uint4 cur = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0x0000ffffu);  // all padding
        if (p < len) cur = __ldg(src + 2 * p);
        const uint32_t wd[kQuadIds] = {cur.x & 0xffffu, cur.x >> 16, cur.y & 0xffffu, cur.y >> 16,
                                       cur.z & 0xffffu, cur.z >> 16, cur.w & 0xffffu};
        const uint32_t fb = cur.w >> 16;
#pragma unroll 1
        for (int c = 0; c < kQuadIds; ++c) {
          __syncwarp();  // the previous round's increments are visible to every lane
          const uint32_t sh = ((fb >> (2 * c)) & 3u) * 8u;
          if (wd[c] < pad_word) {
            volatile uint32_t *word = cnt + wd[c];
            if (((*word >> sh) & 0xffu) < v) {
              const uint32_t old = atomicAdd(const_cast<uint32_t *>(word), 1u << sh);
              if (((old >> sh) & 0xffu) == v - 1u) {
                const int pos = atomicAdd(s_nc, 1);
                if (pos < cap32) qcand[pos] = lo + (int)(wd[c] * PER + (sh >> 3));
              }
            }
          }
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint4 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 tmem_ld4(uint32_t taddr) {
  uint4 v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return v;
}

constexpr int kPairSlots = 16;  // stashed windows per warp (4 TMEM columns each; 8 warps share a lane quarter)

// The paired streamed vote: one CTA (1024 threads, one per SM) per query at
// a time, warp w owning trees [w*T/32, (w+1)*T/32) (one per lane).  Per
// super-tile the warp flattens its trees' super-pieces into 32-pair windows
// (one pair per lane, one 32-byte load, loaded one window ahead of the
// bumps).  Phase A bumps each pair's first quad into tile 2j's counters and
// parks the second quad in tensor memory (the SM's 256 KB of TMEM, unused
// otherwise: warp w's lanes own columns [64*(w/4), +64) of lane quarter w%4,
// 16 windows of 4 columns); after the tile barrier and clearing, phase B
// bumps the parked quads into tile 2j+1's counters.  Windows past the 16th
// re-read their pair in phase B.  The counts are those of k_vote_stream.
template <int CW, bool SAT = false>
__global__ void __launch_bounds__(1024, 1) k_vote_pair(VoteArgs a, const uint4 *__restrict__ ps,
                                                       const int32_t *__restrict__ pbase, int64_t pstride,
                                                       int32_t *redo /* SAT: count, then queries */) {
  extern __shared__ uint4 vote_smem[];
  uint32_t *cnt = reinterpret_cast<uint32_t *>(vote_smem);
  uint32_t cnt_s = (uint32_t)__cvta_generic_to_shared(cnt);
  asm volatile("" : "+r"(cnt_s));
  const int cwords = spare_word0<CW>(a.W);
  const uint32_t pad_word = (uint32_t)cwords;
  constexpr int NW = 32;
  __shared__ uint32_t w_off[NW][32];
  __shared__ int s_nc;
  __shared__ uint32_t s_tmem, s_ovf;
  const uint32_t vm1 = (uint32_t)(a.v - 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // + 0 in a form ptxas cannot fold: the address stays per-lane (pair_emit)
  uint32_t lm_eq;
  asm volatile("mov.u32 %0, %%lanemask_eq;" : "=r"(lm_eq));
  uint32_t nc_s = (uint32_t)__cvta_generic_to_shared(&s_nc) + (uint32_t)(__popc(lm_eq) - 1);
  asm volatile("" : "+r"(nc_s));
  uint32_t ovf_s = (uint32_t)__cvta_generic_to_shared(&s_ovf);
  asm volatile("" : "+r"(ovf_s));
  const int cap32 = a.cap < 0x7fffffff ? (int)a.cap : 0x7fffffff;
  const int nsup = (a.ntiles + 1) >> 1;
  const int64_t dstride = nsup + 1;
  const int t_lo = (int)(((int64_t)warp * a.T) / NW);
  const int t_hi = (int)(((int64_t)(warp + 1) * a.T) / NW);
  const int t = t_lo + lane;
  const bool has = t < t_hi;
  // pairs addressed as uint4 index 2*p from the warp's first tree row
  unsigned long long wb = reinterpret_cast<unsigned long long>(ps + 2 * (int64_t)t_lo * pstride);
  asm volatile("" : "+l"(wb));
  uint32_t *woff = w_off[warp];
  uint4 *c4 = reinterpret_cast<uint4 *>(cnt);
  const uint32_t pw = pad_word + (uint32_t)lane;
  const uint4 padq = make_uint4(pw | (pw << 16), pw | (pw << 16), pw | (pw << 16), pw);
  // SAT: counters start at kSatCross + 1 - v (see pair_bump).  The clear
  // value comes back from shared memory as one register quad per clear (ptxas
  // otherwise copies it into a fresh quad for every 16-byte store); written
  // here, before the barrier below.
  __shared__ uint4 s_cz;
  if (SAT && tid == 32) {
    const uint32_t c0 = (kSatCross - vm1) * 0x01010101u;
    s_cz = make_uint4(c0, c0, c0, c0);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tslot = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
  auto clear_counters = [&]() {
    uint4 cz = make_uint4(0u, 0u, 0u, 0u);
    if (SAT)
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(cz.x), "=r"(cz.y), "=r"(cz.z), "=r"(cz.w)
                   : "r"((uint32_t)__cvta_generic_to_shared(&s_cz)));
    for (int i = tid; i < cwords / 4; i += 1024) c4[i] = cz;
  };
  for (int64_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
    const uint16_t *dl = nullptr;
    uint32_t lbase = 0;
    int dcur = 0, dnxt = 0, dnn = 0;
    if (has) {
      const int64_t g = (int64_t)t * a.L + a.leaves[q * a.T + t];
      dl = a.dir + g * dstride;
      lbase = (uint32_t)((int64_t)lane * pstride + pbase[g]);
      dcur = dl[0];
      dnxt = dl[1];
      dnn = nsup >= 2 ? (int)__ldg(dl + 2) : 0;
    }
    int32_t *qcand = a.cand + q * a.cap;
    asm volatile("" : "+l"(qcand));
    StreamWindows sw;
    sw.pf = 0;
    sw.begin(dnxt - dcur, lbase + (uint32_t)dcur, woff);
    // next pair of the flattened window sequence: its index (uint4 units / 2)
    // or ~0 past the end
    auto next_pair = [&](uint4 &A, uint4 &B) {
      const int w0 = 32 * sw.next_w++;
      const int rel = sw.pre - w0;
      const bool inwin = sw.len > 0 && (unsigned)rel < 32u;
      const unsigned starts = __reduce_or_sync(0xffffffffu, inwin ? (1u << rel) : 0u);
      const int rank = sw.before + __popc(starts & (0xffffffffu >> (31 - lane))) - 1;
      sw.before += __popc(starts);
      const int e = w0 + lane;
      if (e >= sw.total) {
        A = padq;
        B = padq;
      } else {
        ld_pair_l2_256(reinterpret_cast<const uint4 *>(wb) + 2 * (size_t)(woff[rank] + (uint32_t)e), A, B);
      }
    };
    uint4 rA, rB;
    if (sw.windows() > 0) next_pair(rA, rB);
    clear_counters();
    if (tid == 0) {
      s_nc = 0;
      s_ovf = (SAT && (a.dbg & 8)) ? 1u : 0u;
    }
    __syncthreads();
    for (int j = 0; j < nsup; ++j) {
      const bool hasB = 2 * j + 1 < a.ntiles;
      const int32_t loA = 2 * j * a.W, loB = loA + a.W;
      const int nwin = sw.windows();
      // phase A: tile 2j
      for (int i = 0; i < nwin; ++i) {
        const uint4 cA = rA, cB = rB;
        if (i + 1 < nwin) next_pair(rA, rB);
        if (hasB && i < kPairSlots) tmem_st4(tslot + 4u * (uint32_t)i, cB);
        pair_bump<CW, SAT>(cA, cnt_s, nc_s, pad_word, vm1, loA, qcand, cap32, ovf_s);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      __syncthreads();
      clear_counters();
      __syncthreads();
      // phase B: tile 2j+1 from the parked quads (windows past the parked
      // ones re-read from the stream)
      if (hasB) {
        const int nst = nwin < kPairSlots ? nwin : kPairSlots;
        for (int i = 0; i < nst; ++i) pair_bump<CW, SAT>(tmem_ld4(tslot + 4u * (uint32_t)i), cnt_s, nc_s, pad_word, vm1, loB, qcand, cap32, ovf_s);
        if (nwin > kPairSlots) {
          sw.begin(dnxt - dcur, lbase + (uint32_t)dcur, woff);  // same super-tile again
          for (int i = 0; i < nwin; ++i) {
            uint4 xA, xB;
            next_pair(xA, xB);
            if (i >= kPairSlots) pair_bump<CW, SAT>(xB, cnt_s, nc_s, pad_word, vm1, loB, qcand, cap32, ovf_s);
          }
        }
      }
      // the next super-tile's first window starts loading before the barrier
      if (j + 1 < nsup) {
        dcur = dnxt;
        dnxt = dnn;
        dnn = (has && j + 3 <= nsup) ? (int)__ldg(dl + j + 3) : 0;
        sw.begin(dnxt - dcur, lbase + (uint32_t)dcur, woff);
        if (sw.windows() > 0) next_pair(rA, rB);
      }
      if (hasB) {
        __syncthreads();
        if (j + 1 < nsup)
          clear_counters();
        __syncthreads();
      }
    }
    __syncthreads();
    if (tid == 0) {
      a.ncand[q] = s_nc;  // > cap means only cap ids were stored
      // a counter wrapped: the query is listed for the exact redo kernel
      if (SAT && s_ovf) redo[1 + atomicAdd(redo, 1)] = (int32_t)q;
    }
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
  }
}

// The queries the saturating vote listed (a counter wrapped), redone exactly.
__global__ void __launch_bounds__(1024, 1) k_vote_pair_redo(VoteArgs a, const uint4 *__restrict__ ps,
                                                            const int32_t *__restrict__ pbase, int64_t pstride,
                                                            const int32_t *__restrict__ redo) {
  extern __shared__ uint4 vote_smem[];
  uint32_t *cnt = reinterpret_cast<uint32_t *>(vote_smem);
  __shared__ int s_nc;
  const int cwords = spare_word0<1>(a.W);
  const int m = redo[0];
  for (int i = blockIdx.x; i < m; i += gridDim.x) {
    const int64_t q = redo[1 + i];
    if (threadIdx.x == 0) atomicAdd(&g_vote_sat_redos, 1ull);
    vote_pair_careful(a, ps, pbase, pstride, q, cnt, cwords, &s_nc);
    if (threadIdx.x == 0) a.ncand[q] = s_nc;
    __syncthreads();
  }
}
}  // namespace mrpt

using namespace mrpt;

static const int kVoteSmemSingle = 110 * 1024;  // single tile
static const int kVoteSmemTiled = 196 * 1024;   // tiled sweep: one big CTA per SM (+ static tables)
static const int kVoteSmemUnion = 222 * 1024;   // v == 1 bitmap over all ids + staging

// Tile geometry shared by mrpt_vote, mrpt_vote_plan and the directory.
// Smem per tile: the packed counters, a 1-bit "reached v" flag per id, and
// 8 bytes per tree (cursors / slice bases).
static size_t vote_smem_bytes(int CW, int64_t W, int32_t T) {
  const int64_t words = CW == 1 ? W / 4 : (CW == 2 ? W / 2 : (CW == 3 ? (W + 2) / 3 : W));
  return (size_t)((words + 3) & ~3LL) * 4 + (size_t)W / 8 + (size_t)8 * T;
}

static int64_t counter_words_host(int CW, int64_t W) {
  return CW == 1 ? W / 4 : (CW == 2 ? W / 2 : (CW == 3 ? (W + 2) / 3 : W));
}

static int vote_dir_threads() {
  const char *e = getenv("MRPT_VOTE_NT");  // experiments: 512 = two CTAs per SM
  return (e && atoi(e) == 512) ? 512 : 1024;
}

static int32_t vote_geometry(int64_t n, int32_t T, int64_t max_count, int *CWo, int64_t *Wo,
                             int *ntiles_o) {
  const size_t tiled_budget = vote_dir_threads() == 512 ? 96 * 1024 : kVoteSmemTiled;
  const int CW = max_count <= 255 ? 1 : (max_count <= 1023 ? 3 : (max_count <= 65535 ? 2 : 4));
  const int64_t single = ceil_div<int64_t>(n, 192) * 192;
  int64_t W;
  if (vote_smem_bytes(CW, single, T) <= (size_t)kVoteSmemSingle) {
    W = single;
  } else {
    // largest multiple of 192 ids (bitmap words x 10-bit triples) in budget
    int64_t lo = 0, hi = single / 192;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (vote_smem_bytes(CW, mid * 192, T) <= tiled_budget) lo = mid; else hi = mid - 1;
    }
    if (lo == 0) return fail(MRPT_EPARAM, "mrpt_vote: too many trees for shared cursors");
    W = lo * 192;
  }
  *CWo = CW;
  *Wo = W;
  *ntiles_o = (int)ceil_div<int64_t>(n, W);
  return MRPT_OK;
}

extern "C" int32_t mrpt_vote_plan(int64_t n, int32_t T, int32_t depth, int64_t max_count,
                                  int32_t *ntiles, int64_t *dir_entries) {
  clear_error();
  if (n < 1 || n >= (int64_t)1 << 31 || T < 1 || depth < 0 || depth > 30 || !ntiles || !dir_entries)
    return fail(MRPT_ESHAPE, "mrpt_vote_plan: bad arguments");
  int CW, nt;
  int64_t W;
  int32_t st = vote_geometry(n, T, max_count, &CW, &W, &nt);
  if (st) return st;
  *ntiles = nt;
  *dir_entries = nt > 1 ? (int64_t)T * ((int64_t)1 << depth) * (nt + 1) : 0;
  return MRPT_OK;
}

extern "C" int32_t mrpt_vote_build_dir(const int32_t *leaf_indices, const int64_t *leaf_offsets,
                                       int64_t n, int32_t T, int32_t depth, int64_t max_count,
                                       uint16_t *dir, void *stream) {
  clear_error();
  int CW, nt;
  int64_t W;
  int32_t st = vote_geometry(n, T, max_count, &CW, &W, &nt);
  if (st) return st;
  if (nt <= 1) return MRPT_OK;
  cudaStream_t s = as_stream(stream);
  const int64_t nleaves = (int64_t)T << depth;
  const int64_t blocks = ceil_div<int64_t>(nleaves, 8);
  const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  (count_launch(), k_build_dir<<<grid, 256, 0, s>>>(leaf_indices, leaf_offsets, n, T, 1 << depth, (int)W, nt, dir));
  return launch_status("mrpt_vote_build_dir");
}

static int32_t vote_impl(const int32_t *leaf_indices, const int64_t *leaf_offsets, int64_t n, int32_t T,
                         int32_t depth, const int32_t *leaves, int64_t nq, int32_t v, int32_t leaves_sorted,
                         int64_t max_count, const uint16_t *dir, int32_t *cand, int64_t cap,
                         uint32_t *bits_out, int64_t bstride, int32_t *ncand, void *stream,
                         uint16_t *cnt_out = nullptr) {
  if (n < 1 || n >= (int64_t)1 << 31 || T < 1 || depth < 0 || depth > 30 || nq < 0)
    return fail(MRPT_ESHAPE, "mrpt_vote: bad shape");
  if (v < 1 || v > max_count) return fail(MRPT_EPARAM, "mrpt_vote: vote threshold out of range");
  if (!bits_out && cap < 1) return fail(MRPT_EPARAM, "mrpt_vote: cap must be >= 1");
  if (bits_out && bstride < (n + 31) / 32) return fail(MRPT_EPARAM, "mrpt_vote_bitmap: bstride < ceil(n/32)");
  if (nq == 0) return MRPT_OK;
  cudaStream_t s = as_stream(stream);
  int CW, ntiles;
  int64_t W;
  int32_t st = vote_geometry(n, T, max_count, &CW, &W, &ntiles);
  if (st) return st;
  const bool sorted = leaves_sorted != 0 || ntiles == 1;
  // lanes per tree slice for the cursor sweep (pow2 in [1, 32])
  const double mean_leaf = (double)n / (double)((int64_t)1 << depth);
  const double per_tile = mean_leaf / ntiles;
  int G = 1;
  while (G < 32 && G * kVoteU < per_tile) G <<= 1;
  if (const char *env = getenv("MRPT_VOTE_G")) G = atoi(env);  // experiments
  VoteArgs a = {};
  a.leaf_indices = leaf_indices;
  a.leaf_offsets = leaf_offsets;
  a.n = n;
  a.T = T;
  a.L = 1 << depth;
  a.leaves = leaves;
  a.nq = nq;
  a.v = v;
  a.cand = cand;
  a.cap = cap;
  a.ncand = ncand;
  a.W = (int)W;
  a.ntiles = ntiles;
  a.qlist = nullptr;
  a.qcount = nullptr;
  a.dir = dir;
  a.bits_out = bits_out;
  a.bstride = bstride;
  a.cnt_out = cnt_out;
  const size_t smem = vote_smem_bytes(CW, W, T);
  const int64_t grid = nq < (int64_t)num_sms() * 4 ? nq : (int64_t)num_sms() * 4;
  // v == 1: bitmap + per-warp staging + slice table
  const size_t ubits = (size_t)((n + 127) >> 7) * 16;
  const size_t usmem512 = ubits + 16 * kUnionStage * 4 + (size_t)12 * T;
  const size_t usmem1024 = ubits + 32 * kUnionStage * 4 + (size_t)12 * T;
  // (only where the counting path needs several id tiles: with one tile the
  // counting kernel is as fast)
  const char *uenv = getenv("MRPT_VOTE_UNION");  // "0": never, "1": whenever it fits
  // bitmap hand-over: the union kernel also for a single id tile (measured
  // 0.43 vs 0.58 ms per 10k queries at config 2)
  const bool want_union = uenv ? atoi(uenv) != 0 : (ntiles > 1 || bits_out != nullptr);
  const size_t usmem256 = ubits + 8 * kUnionStage * 4 + (size_t)12 * T;
  if (v == 1 && want_union && !cnt_out && usmem1024 <= (size_t)kVoteSmemUnion && !getenv("MRPT_VOTE_NO_UNION")) {
    // small bitmaps: NT=256 with four or more queries in flight per SM (the
    // per-query slice fetches and tree walks are latency chains); else
    // NT=512 when two CTAs fit per SM (one query's compaction overlaps the
    // other's atomics), else one CTA of 1024 threads
    const bool four = usmem256 + 1024 <= (size_t)kVoteSmemUnion / 4;
    const bool two = usmem512 + 4 * 1024 <= (size_t)kVoteSmemUnion / 2;
    const int nt = four ? 256 : (two ? 512 : 1024);
    const size_t usmem = four ? usmem256 : (two ? usmem512 : usmem1024);
    union_fn fn = four ? k_vote_union<256> : (two ? k_vote_union<512> : k_vote_union<1024>);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usmem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, usmem);
    if (per_sm < 1) per_sm = 1;
    const int64_t g = (int64_t)num_sms() * per_sm;
    // lanes per leaf slice: enough for UNR=8 loads each over a mean slice
    const double mean_slice = (double)n / (double)((int64_t)1 << depth);
    int Gu = 4;  // lanes per slice: enough for 8 int4 loads each over a mean slice
    while (Gu < 32 && Gu * 32 < mean_slice) Gu <<= 1;
    if (const char *ge = getenv("MRPT_VOTE_GU")) Gu = atoi(ge);
    k_vote_union_launch(fn, (unsigned)(nq < g ? nq : g), nt, usmem, s, a, Gu);
    return launch_status("mrpt_vote");
  }
  if (dir && ntiles > 1 && sorted) {
    const int nt = vote_dir_threads();
    vote_fn fn;
    if (nt == 512)
      fn = CW == 1 ? k_vote_dir<1, 512>
                   : (CW == 2 ? k_vote_dir<2, 512> : (CW == 3 ? k_vote_dir<3, 512> : k_vote_dir<4, 512>));
    else if (n * 32 < (1LL << 31) && !(getenv("MRPT_VOTE_OFF32") && atoi(getenv("MRPT_VOTE_OFF32")) == 0))
      // 32-bit slice offsets from each warp's first tree (<= 32 trees per warp)
      fn = CW == 1 ? k_vote_dir<1, 1024, true>
                   : (CW == 2 ? k_vote_dir<2, 1024, true>
                              : (CW == 3 ? k_vote_dir<3, 1024, true> : k_vote_dir<4, 1024, true>));
    else
      fn = CW == 1 ? k_vote_dir<1, 1024>
                   : (CW == 2 ? k_vote_dir<2, 1024> : (CW == 3 ? k_vote_dir<3, 1024> : k_vote_dir<4, 1024>));
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t g2 = nt == 512 ? (nq < (int64_t)num_sms() * 8 ? nq : (int64_t)num_sms() * 8) : grid;
    (count_launch(), fn<<<(unsigned)g2, nt, smem, s>>>(a));
  } else {
    vote_fn fn = sorted ? pick_cw<true>(CW, G) : pick_cw<false>(CW, G);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    (count_launch(), fn<<<(unsigned)grid, kVoteNT, smem, s>>>(a));
  }
  return launch_status("mrpt_vote");
}

extern "C" int32_t mrpt_vote(const int32_t *leaf_indices, const int64_t *leaf_offsets, int64_t n,
                             int32_t T, int32_t depth, const int32_t *leaves, int64_t nq, int32_t v,
                             int32_t leaves_sorted, int64_t max_count, const uint16_t *dir,
                             int32_t *cand, int64_t cap, int32_t *ncand, void *stream) {
  clear_error();
  return vote_impl(leaf_indices, leaf_offsets, n, T, depth, leaves, nq, v, leaves_sorted, max_count, dir, cand,
                   cap, nullptr, 0, ncand, stream);
}

extern "C" int32_t mrpt_vote_bitmap(const int32_t *leaf_indices, const int64_t *leaf_offsets, int64_t n,
                                    int32_t T, int32_t depth, const int32_t *leaves, int64_t nq, int32_t v,
                                    int32_t leaves_sorted, int64_t max_count, const uint16_t *dir,
                                    uint32_t *bits, int64_t bstride, int32_t *ncand, void *stream) {
  clear_error();
  if (!bits) return fail(MRPT_EPARAM, "mrpt_vote_bitmap: bits is NULL");
  return vote_impl(leaf_indices, leaf_offsets, n, T, depth, leaves, nq, v, leaves_sorted, max_count, dir,
                   nullptr, 1, bits, bstride, ncand, stream);
}

extern "C" int32_t mrpt_vote_counted(const int32_t *leaf_indices, const int64_t *leaf_offsets, int64_t n,
                                     int32_t T, int32_t depth, const int32_t *leaves, int64_t nq, int32_t v,
                                     int32_t leaves_sorted, int64_t max_count, const uint16_t *dir,
                                     int32_t *cand, uint16_t *cand_counts, int64_t cap, int32_t *ncand,
                                     void *stream) {
  clear_error();
  if (!cand_counts) return fail(MRPT_EPARAM, "mrpt_vote_counted: cand_counts is NULL");
  return vote_impl(leaf_indices, leaf_offsets, n, T, depth, leaves, nq, v, leaves_sorted, max_count, dir, cand,
                   cap, nullptr, 0, ncand, stream, cand_counts);
}

// One warp per query: keep the listed candidates whose count is >= v, in
// list order (ballot compaction).
__global__ void k_filter_counts(const int32_t *__restrict__ cand, const uint16_t *__restrict__ cnts, int64_t cap,
                                const int32_t *__restrict__ ncand, int64_t nq, int32_t v, int32_t *cand_out,
                                int64_t cap_out, int32_t *ncand_out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < nq; q += nw) {
    const int64_t m = ncand[q] < cap ? ncand[q] : cap;
    const int32_t *c = cand + q * cap;
    const uint16_t *k = cnts + q * cap;
    int32_t *o = cand_out + q * cap_out;
    int64_t outn = 0;
    for (int64_t i0 = 0; i0 < m; i0 += 32) {
      const int64_t i = i0 + lane;
      const bool keep = i < m && (int32_t)k[i] >= v;
      const unsigned bm = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int64_t pos = outn + __popc(bm & lanemask_lt());
        if (pos < cap_out) o[pos] = c[i];
      }
      outn += __popc(bm);
    }
    if (lane == 0) ncand_out[q] = (int32_t)outn;
  }
}

extern "C" int32_t mrpt_filter_counts(const int32_t *cand, const uint16_t *cand_counts, int64_t cap,
                                      const int32_t *ncand, int64_t nq, int32_t v, int32_t *cand_out,
                                      int64_t cap_out, int32_t *ncand_out, void *stream) {
  clear_error();
  if (cap < 1 || cap_out < 1 || nq < 0 || v < 1) return fail(MRPT_EPARAM, "mrpt_filter_counts: bad arguments");
  if (nq == 0) return MRPT_OK;
  const int64_t blocks = ceil_div<int64_t>(nq, 8);
  const int64_t capb = (int64_t)num_sms() * 16;
  (count_launch(), k_filter_counts<<<(unsigned)(blocks < capb ? blocks : capb), 256, 0, as_stream(stream)>>>(
      cand, cand_counts, cap, ncand, nq, v, cand_out, cap_out, ncand_out));
  return launch_status("mrpt_filter_counts");
}

extern "C" int32_t mrpt_vote_counts(const int32_t *leaf_indices, const int64_t *leaf_offsets,
                                    int64_t n, int32_t T, int32_t depth, const int32_t *leaves,
                                    int32_t *counts, void *stream) {
  clear_error();
  if (n < 1 || T < 1 || depth < 0 || depth > 30) return fail(MRPT_ESHAPE, "mrpt_vote_counts: bad shape");
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * n, s);
  (count_launch(), k_vote_dense<<<T, 256, 0, s>>>(leaf_indices, leaf_offsets, n, 1 << depth, leaves, counts));
  return launch_status("mrpt_vote_counts");
}

extern "C" int32_t mrpt_select_ge(const int32_t *counts, int64_t n, int32_t v, int32_t *out,
                                  int64_t *nout, void *stream) {
  clear_error();
  if (n < 0) return fail(MRPT_ESHAPE, "mrpt_select_ge: bad shape");
  cudaStream_t s = as_stream(stream);
  (count_launch(), k_select_ge<<<1, 1024, 0, s>>>(counts, n, v, out, nout));
  return launch_status("mrpt_select_ge");
}

extern "C" int32_t mrpt_unique_ids(const int64_t *cand, int64_t m, int64_t n, uint32_t *bitmap,
                                   int32_t *out, int64_t *nout, int32_t *bad, void *stream) {
  clear_error();
  if (m < 0 || n < 1 || n >= (int64_t)1 << 31) return fail(MRPT_ESHAPE, "mrpt_unique_ids: bad shape");
  cudaStream_t s = as_stream(stream);
  const int64_t nwords = ceil_div<int64_t>(n, 32);
  cudaMemsetAsync(bitmap, 0, sizeof(uint32_t) * nwords, s);
  cudaMemsetAsync(bad, 0, sizeof(int32_t), s);
  if (m > 0) {
    const int64_t blocks = ceil_div<int64_t>(m, 256);
    const int grid = (int)(blocks < (int64_t)num_sms() * 8 ? blocks : (int64_t)num_sms() * 8);
    (count_launch(), k_mark_ids<<<grid, 256, 0, s>>>(cand, m, n, bitmap, bad));
  }
  (count_launch(), k_bitmap_compact<<<1, 1024, 0, s>>>(bitmap, nwords, out, nout));
  return launch_status("mrpt_unique_ids");
}

// ------------------------------------------------------------ streamed vote --
static const int kVoteSmemStream = 218 * 1024;  // counters only (the rank tables are static)

// sat_ok (the paired vote): counts above 255 still use 8-bit counters, which
// then saturate instead of counting on (k_vote_pair, SAT) -- a quarter fewer
// id tiles than 10-bit counters.  MRPT_VOTE_SAT=0 keeps the wide counters.
static bool vote_sat_enabled() {
  const char *e = getenv("MRPT_VOTE_SAT");
  return !(e && e[0] == '0');
}

static int32_t stream_geometry(int64_t n, int32_t T, int64_t max_count, int *CWo, int64_t *Wo, int *ntiles_o,
                               bool sat_ok = false, bool *sat_o = nullptr) {
  if (T < 1 || T > 1024) return fail(MRPT_EPARAM, "streamed vote: needs 1 <= T <= 1024");
  int CW = max_count <= 255 ? 1 : (max_count <= 1023 ? 3 : (max_count <= 65535 ? 2 : 4));
  const int64_t words0 = ((kVoteSmemStream - 128) / 4) & ~3LL;
  // saturating 8-bit counters only where they save super-tiles (pairs of id tiles)
  const int64_t nsup_wide = (ceil_div<int64_t>(n, words0 * (CW == 3 ? 3 : (CW == 2 ? 2 : 1))) + 1) / 2;
  const int64_t nsup_sat = (ceil_div<int64_t>(n, words0 * 4) + 1) / 2;
  const bool sat = sat_ok && CW != 1 && vote_sat_enabled() && nsup_sat < nsup_wide;
  if (sat) CW = 1;
  if (sat_o) *sat_o = sat;
  const int per = CW == 1 ? 4 : (CW == 3 ? 3 : (CW == 2 ? 2 : 1));
  const int64_t words = ((kVoteSmemStream - 128) / 4) & ~3LL;
  int64_t W = words * per;
  if (W >= n) W = n;
  *CWo = CW;
  *Wo = W;
  *ntiles_o = (int)ceil_div<int64_t>(n, W);
  if (*ntiles_o > kStreamMaxTiles) return fail(MRPT_EPARAM, "streamed vote: too many id tiles");
  return MRPT_OK;
}

extern "C" int32_t mrpt_vote_stream_plan(int64_t n, int32_t T, int32_t depth, int64_t max_count,
                                         int32_t *ntiles, int64_t *dir_entries) {
  clear_error();
  if (n < 1 || n >= (int64_t)1 << 31 || depth < 0 || depth > 30 || !ntiles || !dir_entries)
    return fail(MRPT_ESHAPE, "mrpt_vote_stream_plan: bad arguments");
  int CW, nt;
  int64_t W;
  const int32_t st = stream_geometry(n, T, max_count, &CW, &W, &nt);
  if (st) return st;
  *ntiles = nt;
  *dir_entries = (int64_t)T * ((int64_t)1 << depth) * (nt + 1);
  return MRPT_OK;
}

extern "C" int32_t mrpt_vote_stream_layout(const int32_t *leaf_indices, const int64_t *leaf_offsets, int64_t n,
                                           int32_t T, int32_t depth, int64_t max_count, uint16_t *qdir,
                                           int32_t *qbase, int64_t *tree_quads, void *stream) {
  clear_error();
  int CW, nt;
  int64_t W;
  const int32_t st = stream_geometry(n, T, max_count, &CW, &W, &nt);
  if (st) return st;
  cudaStream_t s = as_stream(stream);
  const int64_t nleaves = (int64_t)T << depth;
  const int64_t blocks = ceil_div<int64_t>(nleaves, 8);
  const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  (count_launch(), k_build_dir<<<grid, 256, 0, s>>>(leaf_indices, leaf_offsets, n, T, 1 << depth, (int)W, nt, qdir));
  (count_launch(), k_vstream_quads<<<grid, 256, 0, s>>>(qdir, nleaves, nt, qbase));
  (count_launch(), k_vstream_base<<<T, 1024, 0, s>>>(qbase, 1 << depth, tree_quads));
  return launch_status("mrpt_vote_stream_layout");
}

extern "C" int32_t mrpt_vote_stream_fill(const int32_t *leaf_indices, const int64_t *leaf_offsets, int64_t n,
                                         int32_t T, int32_t depth, int64_t max_count, const uint16_t *qdir,
                                         const int32_t *qbase, int64_t tstride, uint32_t *qs, void *stream) {
  clear_error();
  int CW, nt;
  int64_t W;
  const int32_t st = stream_geometry(n, T, max_count, &CW, &W, &nt);
  if (st) return st;
  if (tstride < 0 || 32 * tstride >= ((int64_t)1 << 31))
    return fail(MRPT_EPARAM, "mrpt_vote_stream_fill: tree stride too large");
  cudaStream_t s = as_stream(stream);
  const int64_t nleaves = (int64_t)T << depth;
  const int64_t blocks = ceil_div<int64_t>(nleaves, 8);
  const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  auto fn = CW == 1 ? k_vstream_fill<1> : (CW == 3 ? k_vstream_fill<3> : (CW == 2 ? k_vstream_fill<2> : k_vstream_fill<4>));
  const size_t fsmem = sizeof(int32_t) * 2 * (size_t)(nt + 1) * 8;  // 8 warps
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
  (count_launch(), fn<<<grid, 256, fsmem, s>>>(leaf_indices, leaf_offsets, n, T, 1 << depth, (int)W, nt, qdir,
                                               qbase, tstride, qs));
  return launch_status("mrpt_vote_stream_fill");
}

extern "C" int32_t mrpt_vote_stream(const uint32_t *qs, int64_t tstride, const uint16_t *qdir, const int32_t *qbase,
                                    int64_t n, int32_t T, int32_t depth, int64_t max_count, const int32_t *leaves,
                                    int64_t nq, int32_t v, int32_t *cand, int64_t cap, int32_t *ncand,
                                    void *stream) {
  clear_error();
  if (n < 1 || n >= (int64_t)1 << 31 || depth < 0 || depth > 30 || nq < 0)
    return fail(MRPT_ESHAPE, "mrpt_vote_stream: bad shape");
  if (v < 1 || v > max_count) return fail(MRPT_EPARAM, "mrpt_vote_stream: vote threshold out of range");
  if (cap < 1) return fail(MRPT_EPARAM, "mrpt_vote_stream: cap must be >= 1");
  if (32 * tstride >= ((int64_t)1 << 31)) return fail(MRPT_EPARAM, "mrpt_vote_stream: tree stride too large");
  int CW, nt;
  int64_t W;
  const int32_t st = stream_geometry(n, T, max_count, &CW, &W, &nt);
  if (st) return st;
  if (nq == 0) return MRPT_OK;
  VoteArgs a = {};
  a.n = n;
  a.T = T;
  a.L = 1 << depth;
  a.leaves = leaves;
  a.nq = nq;
  a.v = v;
  a.cand = cand;
  a.cap = cap;
  a.ncand = ncand;
  a.W = (int)W;
  a.ntiles = nt;
  a.dir = qdir;
  a.dbg = getenv("MRPT_VOTE_DBG") ? atoi(getenv("MRPT_VOTE_DBG")) : 0;
  const size_t smem = (size_t)((counter_words_host(CW, W) + 3) & ~3LL) * 4 + 128;  // + 32 spare words
  typedef void (*sfn_t)(VoteArgs, const uint4 *, const int32_t *, int64_t);
  static int unr = -1;  // experiments: MRPT_VSTREAM_P (1, 2, 4): windows loaded ahead
  if (unr < 0) {
    const char *e1 = getenv("MRPT_VSTREAM_P");
    unr = e1 ? atoi(e1) : 1;  // 2 and 4 measured slower (364, 404 vs 357 ms at config 5)
  }
  static const bool cg = !(getenv("MRPT_VSTREAM_CG") && atoi(getenv("MRPT_VSTREAM_CG")) == 0);
#define VS_PICK(C)                                                                              \
  (cg ? (unr == 2 ? k_vote_stream<C, 2, true> : (unr == 4 ? k_vote_stream<C, 4, true> : k_vote_stream<C, 1, true>)) \
      : (unr == 2 ? k_vote_stream<C, 2, false> : (unr == 4 ? k_vote_stream<C, 4, false> : k_vote_stream<C, 1, false>)))
  sfn_t fn = CW == 1 ? VS_PICK(1) : (CW == 3 ? VS_PICK(3) : (CW == 2 ? VS_PICK(2) : VS_PICK(4)));
#undef VS_PICK
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t ctas = num_sms();
  if (const char *ge = getenv("MRPT_VSTREAM_GRID")) ctas = atoi(ge) > 0 ? atoi(ge) : ctas;  // experiments
  const int64_t grid = nq < ctas ? nq : ctas;
  cudaStream_t s = as_stream(stream);
  (count_launch(), fn<<<(unsigned)grid, 1024, smem, s>>>(a, reinterpret_cast<const uint4 *>(qs), qbase, tstride));
  return launch_status("mrpt_vote_stream");
}

// ------------------------------------------------------- paired vote (host) --
// Queries voted with saturating counters (host count; redone ones: g_vote_sat_redos).
static std::atomic<long long> g_vote_sat_queries{0};

extern "C" int32_t mrpt_vote_pair_max_votes(int64_t n, int32_t T, int64_t max_count, int32_t *max_votes) {
  clear_error();
  if (!max_votes) return fail(MRPT_EPARAM, "mrpt_vote_pair_max_votes: NULL output");
  int CW, nt;
  int64_t W;
  bool sat = false;
  const int32_t st = stream_geometry(n, T, max_count, &CW, &W, &nt, true, &sat);
  if (st) return st;
  *max_votes = sat ? kSatMaxV : (int32_t)(max_count < 0x7fffffff ? max_count : 0x7fffffff);
  return MRPT_OK;
}

extern "C" int32_t mrpt_vote_stats(int64_t *out, int32_t reset) {
  clear_error();
  if (!out) return fail(MRPT_EPARAM, "mrpt_vote_stats: out is NULL");
  unsigned long long redo = 0;
  if (cudaMemcpyFromSymbol(&redo, g_vote_sat_redos, sizeof(redo)) != cudaSuccess)
    return launch_status("mrpt_vote_stats");
  out[0] = g_vote_sat_queries.load();
  out[1] = (int64_t)redo;
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(g_vote_sat_redos, &z, sizeof(z));
    g_vote_sat_queries.store(0);
  }
  return launch_status("mrpt_vote_stats");
}

extern "C" int32_t mrpt_vote_pair_plan(int64_t n, int32_t T, int32_t depth, int64_t max_count, int32_t *ntiles,
                                       int64_t *pos_entries, int64_t *dir_entries) {
  clear_error();
  if (n < 1 || n >= (int64_t)1 << 31 || depth < 0 || depth > 30 || !ntiles || !pos_entries || !dir_entries)
    return fail(MRPT_ESHAPE, "mrpt_vote_pair_plan: bad arguments");
  int CW, nt;
  int64_t W;
  bool sat = false;
  const int32_t st = stream_geometry(n, T, max_count, &CW, &W, &nt, true, &sat);
  if (st) return st;
  *ntiles = nt;
  *pos_entries = (int64_t)T * ((int64_t)1 << depth) * (nt + 1);
  *dir_entries = (int64_t)T * ((int64_t)1 << depth) * ((nt + 1) / 2 + 1);
  return MRPT_OK;
}

extern "C" int32_t mrpt_vote_pair_layout(const int32_t *leaf_indices, const int64_t *leaf_offsets, int64_t n,
                                         int32_t T, int32_t depth, int64_t max_count, uint16_t *pos, uint16_t *pdir,
                                         int32_t *pbase, int64_t *tree_pairs, void *stream) {
  clear_error();
  int CW, nt;
  int64_t W;
  bool sat = false;
  const int32_t st = stream_geometry(n, T, max_count, &CW, &W, &nt, true, &sat);
  if (st) return st;
  cudaStream_t s = as_stream(stream);
  const int64_t nleaves = (int64_t)T << depth;
  const int64_t blocks = ceil_div<int64_t>(nleaves, 8);
  const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  (count_launch(), k_build_dir<<<grid, 256, 0, s>>>(leaf_indices, leaf_offsets, n, T, 1 << depth, (int)W, nt, pos));
  (count_launch(), k_vpair_dir<<<grid, 256, 0, s>>>(pos, pdir, nleaves, nt, (nt + 1) / 2, pbase));
  (count_launch(), k_vstream_base<<<T, 1024, 0, s>>>(pbase, 1 << depth, tree_pairs));
  return launch_status("mrpt_vote_pair_layout");
}

extern "C" int32_t mrpt_vote_pair_fill(const int32_t *leaf_indices, const int64_t *leaf_offsets, int64_t n, int32_t T,
                                       int32_t depth, int64_t max_count, const uint16_t *pos, const uint16_t *pdir,
                                       const int32_t *pbase, int64_t pstride, uint32_t *ps, void *stream) {
  clear_error();
  int CW, nt;
  int64_t W;
  bool sat = false;
  const int32_t st = stream_geometry(n, T, max_count, &CW, &W, &nt, true, &sat);
  if (st) return st;
  if (pstride < 0 || 64 * pstride >= ((int64_t)1 << 31))
    return fail(MRPT_EPARAM, "mrpt_vote_pair_fill: tree stride too large");
  cudaStream_t s = as_stream(stream);
  const int64_t nleaves = (int64_t)T << depth;
  const int64_t blocks = ceil_div<int64_t>(nleaves, 8);
  const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  const int nsup = (nt + 1) / 2;
  auto fn = CW == 1 ? k_vpair_fill<1> : (CW == 3 ? k_vpair_fill<3> : (CW == 2 ? k_vpair_fill<2> : k_vpair_fill<4>));
  const size_t fsmem = sizeof(int32_t) * (size_t)(nt + 1 + nsup + 1) * 8;  // 8 warps
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
  (count_launch(), fn<<<grid, 256, fsmem, s>>>(leaf_indices, leaf_offsets, n, T, 1 << depth, (int)W, nt, nsup, pos,
                                               pdir, pbase, pstride, reinterpret_cast<uint4 *>(ps)));
  return launch_status("mrpt_vote_pair_fill");
}

extern "C" int32_t mrpt_vote_pair(const uint32_t *ps, int64_t pstride, const uint16_t *pdir, const int32_t *pbase,
                                  int64_t n, int32_t T, int32_t depth, int64_t max_count, const int32_t *leaves,
                                  int64_t nq, int32_t v, int32_t *cand, int64_t cap, int32_t *ncand, void *stream) {
  clear_error();
  if (n < 1 || n >= (int64_t)1 << 31 || depth < 0 || depth > 30 || nq < 0)
    return fail(MRPT_ESHAPE, "mrpt_vote_pair: bad shape");
  if (v < 1 || v > max_count) return fail(MRPT_EPARAM, "mrpt_vote_pair: vote threshold out of range");
  if (cap < 1) return fail(MRPT_EPARAM, "mrpt_vote_pair: cap must be >= 1");
  if (64 * pstride >= ((int64_t)1 << 31)) return fail(MRPT_EPARAM, "mrpt_vote_pair: tree stride too large");
  int CW, nt;
  int64_t W;
  bool sat = false;
  const int32_t st = stream_geometry(n, T, max_count, &CW, &W, &nt, true, &sat);
  if (st) return st;
  if (sat && v > kSatMaxV)
    return fail(MRPT_EPARAM, "mrpt_vote_pair: saturating counters need v <= 128 (see mrpt_vote_pair_max_votes)");
  if (nq == 0) return MRPT_OK;
  VoteArgs a = {};
  a.n = n;
  a.T = T;
  a.L = 1 << depth;
  a.leaves = leaves;
  a.nq = nq;
  a.v = v;
  a.cand = cand;
  a.cap = cap;
  a.ncand = ncand;
  a.W = (int)W;
  a.ntiles = nt;
  a.dir = pdir;
  a.dbg = getenv("MRPT_VOTE_DBG") ? atoi(getenv("MRPT_VOTE_DBG")) : 0;
  const size_t smem = (size_t)((counter_words_host(CW, W) + 3) & ~3LL) * 4 + 128;  // + 32 spare words
  typedef void (*pfn_t)(VoteArgs, const uint4 *, const int32_t *, int64_t, int32_t *);
  pfn_t fn = sat ? k_vote_pair<1, true>
                 : (CW == 1 ? k_vote_pair<1> : (CW == 3 ? k_vote_pair<3> : (CW == 2 ? k_vote_pair<2> : k_vote_pair<4>)));
  cudaStream_t s = as_stream(stream);
  int32_t *redo = nullptr;
  if (sat) {  // the list of queries to redo exactly (count first)
    if (nq >= (int64_t)1 << 31) return fail(MRPT_ESHAPE, "mrpt_vote_pair: too many queries in one call");
    g_vote_sat_queries += nq;
    keep_pool_warm();
    if (cudaMallocAsync((void **)&redo, sizeof(int32_t) * (size_t)(nq + 1), s) != cudaSuccess)
      return fail(MRPT_ECUDA, "mrpt_vote_pair: scratch allocation failed");
    cudaMemsetAsync(redo, 0, sizeof(int32_t), s);
  }
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t grid = nq < (int64_t)num_sms() ? nq : (int64_t)num_sms();
  (count_launch(), fn<<<(unsigned)grid, 1024, smem, s>>>(a, reinterpret_cast<const uint4 *>(ps), pbase, pstride, redo));
  if (sat) {
    cudaFuncSetAttribute(k_vote_pair_redo, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    (count_launch(), k_vote_pair_redo<<<(unsigned)grid, 1024, smem, s>>>(a, reinterpret_cast<const uint4 *>(ps), pbase,
                                                                          pstride, redo));
    cudaFreeAsync(redo, s);
  }
  return launch_status("mrpt_vote_pair");
}
