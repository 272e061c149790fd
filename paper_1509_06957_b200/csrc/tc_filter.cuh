// K4 "tc" route: the u8 filter fused onto the 5th-generation tensor cores.
//
// Included by scan.cu (it shares QParams, dist_bounds2, admit2, warp_sort and
// the survivor hand-over with the other u8 routes).
//
// The GEMM route (gemm.cu + k_scan_topk_u8<DM>) forms every (query, row)
// dot product of the u8 shadow with a library int8 GEMM, writes the s32
// matrix D to HBM and reads it back in a separate filter pass (config 2:
// 2.4 GB written + 2.4 GB read per 10k queries).  This kernel never
// materialises D:
//
//   * clusters of 2 persistent CTAs (one per SM) walk contiguous ranges of
//     (pair of 128-query blocks, 256-row tile) items in lockstep;
//   * a 4-stage TMA ring (128-B swizzle, 48 KB per stage) streams each
//     CTA's query-block K block (A, s8, K-major) and the row tile's K block
//     (B, the s8 shadow): each CTA loads half of B and multicasts it to both
//     CTAs of the pair; a stage is refilled once both CTAs' MMAs committed it;
//   * one thread issues tcgen05.mma.cta_group::1.kind::i8 (s8 x s8 -> s32,
//     M=128, N=256, K=32 per instruction) into a double-buffered TMEM
//     accumulator (2 x 256 columns);
//   * 16 epilogue warps read the accumulator with tcgen05.ld (one TMEM lane
//     = one query, 4 column-group warps per lane quarter) and run a 3-op
//     pre-test (a superset of the u8 filter's admission rule) on every
//     column; columns whose candidate bit (K3's bitmap, TMA-staged per tile)
//     is set and that pass are admitted: their raw bound terms go to the
//     query's entry list in global memory, and the query's k smallest upper
//     bounds (shared in shared memory by its 4 column-group warps, across
//     CTAs through a global atomicMin of the k-th) tighten the pre-test;
//   * k_tc_select takes the k-th smallest upper bound from the union of the
//     CTAs' k smallest and hands the survivors (L <= U_k) to k_rerank, the
//     exact float64 re-rank every u8 route shares.
//
// D values are the same exact int32 dot products as the library GEMM's
// (MRPT_TC_DEBUG compares them element for element), so the admitted sets
// are supersets of the exact top-k and the results are bit-identical to the
// reference's.
#pragma once
#include <cuda.h>

namespace mrpt {
namespace tc {

constexpr int kM = 128;         // queries per block = TMEM lanes
constexpr int kN = 256;         // rows per tile = TMEM columns per accumulator
constexpr int kKB = 128;        // K bytes per block (one 128-B swizzle row)
constexpr int kMaxKB = 8;       // ldq <= 1024 (the route's u8 shadow limit)
constexpr int kStages = 4;      // ring of (query block, row tile) K-block pairs: 192 KB in flight per SM
constexpr int kTopMax = 16;     // k <= 16: a query's k smallest upper bounds in shared memory
// epilogue: 4 lane quarters x CG column groups (template); + TMA + MMA warps
template <int CG>
constexpr int threads_for() {
  return (4 * CG + 2) * 32;
}
constexpr uint32_t kABytes = kM * kKB;    // 16 KB per K block
constexpr uint32_t kBBytes = kN * kKB;    // 32 KB per stage
constexpr uint32_t kInfoBytes = kN * 20;  // per tile: 256 x 16-B pre-test records + 256 x t1 (5 KB)

// shared-memory carve-up (offsets from a 1024-B aligned base)
// stage s: the query block's K block (16 KB) then the row tile's (32 KB);
// both streamed by TMA (the queries re-read from L2 every tile: more bytes in
// flight beats a resident query block, the feed is latency-bound)
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr uint32_t kOffStage = 0;
constexpr uint32_t kOffInfo = kOffStage + kStages * kStageBytes;
constexpr uint32_t kBitsBytes = kM * (kN / 32) * 4;  // the block's candidate words of one tile (4 KB)
constexpr uint32_t kOffBits = kOffInfo + 2 * kInfoBytes;
constexpr uint32_t kOffBar = kOffBits + 2 * kBitsBytes;
// barriers: fullB[kStages], emptyB[kStages], (2 unused), tmem_full[2], epi_empty[2], info_full[2]
constexpr int kNumBars = 2 * kStages + 2 + 6;
constexpr uint32_t kOffTmemSlot = kOffBar + 8 * kNumBars;
constexpr uint32_t kOffSu = kOffTmemSlot + 16;
// per query of the block: the k smallest upper bounds its column-group warps
// have found (unsorted, -inf fillers past k), their max and its slot, a lock
constexpr uint32_t kOffTop = kOffSu + 4 * kM;
constexpr uint32_t kOffTopMax = kOffTop + 4 * kM * kTopMax;
constexpr uint32_t kOffTopIdx = kOffTopMax + 4 * kM;
constexpr uint32_t kOffLock = kOffTopIdx + 4 * kM;
constexpr uint32_t kSmemBytes = kOffLock + 4 * kM + 1024;  // + alignment slack

struct TcArgs {
  int64_t n;            // data rows
  int64_t m;            // queries of this chunk
  int ntiles;           // ceil(n / kN)
  int nqb;              // ceil(m / kM)
  int kblocks;          // ceil(ldq / kKB)
  int k;                // neighbours
  int ldq;              // shadow row bytes (the unsigned-query offset term)
  const uint4 *rinfo;   // per row {P (f32), 2 sx (f32), radius (f32), 128 * sum(u8) (s32)}, see k_tc_rows
  const float *rt1;     // per row t1 = sx^2 * nrm (the exact admission rule's row term)
  const QParams *qp;    // per query of the chunk
  const uint32_t *cbits;
  int64_t bstride;
  uint4 *ent;           // (m, cap) entries {L (f32, rounded down), U (f32, rounded up), id, 0}
  int32_t *ent_cnt;     // (m) entries appended (may exceed cap: overflow -> exact fallback)
  int cap;
  unsigned *su_g;       // (m) per-query sqrt(k-th upper bound) as float bits, shared by all CTAs
  float *kb;            // (m, kbcap) every stream's k smallest upper bounds (their union holds the query's k smallest)
  int32_t *kb_cnt;      // (m) values appended to kb
  int kbcap;
  int32_t *dbgD;        // optional (MRPT_TC_DEBUG): every dot product, (m, n)
  int noepi;            // experiment (MRPT_TC_NOEPI): skip the epilogue work (MMA + TMA pipeline only)
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

// Producer / MMA waits: back off between polls so a single-thread role
// spinning on a barrier does not take issue slots from the epilogue warps
// that share its scheduler.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(64);
  }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
// B-tile half loaded once and written to both CTAs of a cluster pair (same
// shared-memory offset, each CTA's barrier at that offset gets the bytes)
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap *map, uint32_t bar, int x, int y,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 128-B swizzle (8 rows x 128 B
// atoms, 1024 B apart), Blackwell descriptor version 1.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;            // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // stride byte offset: next 8-row group
  d |= (uint64_t)1 << 46;            // version
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

// instruction descriptor: s8 x s8 -> s32, K-major A and B, M=128, N=256
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kN >> 3) << 17) |
                            ((uint32_t)(kM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(dtmem), "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accum));
}
// commit arriving on the barrier at this offset in every CTA of the mask
__device__ __forceinline__ void mma_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(bar), "h"(mask)
               : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
        "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Per-query state of one epilogue thread.
template <int KT>
struct EpiState {
  float su;        // sqrt(k-th smallest U) rounded up (+inf until k bounds exist)
  int base, left;  // current block of reserved entry slots: next = base + (kEntBlock - left)
};

// The query's shared k smallest upper bounds (one set per CTA and query,
// merged over its column-group warps): replace the largest under the
// query's lock, find the new largest.  Returns the new k-th bound.
template <int KT>
__device__ __forceinline__ float top_insert(float *top, float *tmax, int *tidx, int *lock, float U) {
  while (atomicCAS(lock, 0, 1) != 0) {
  }
  __threadfence_block();
  float m = *reinterpret_cast<volatile float *>(tmax);
  if (U < m) {
    const int ix = *reinterpret_cast<volatile int *>(tidx);
    reinterpret_cast<volatile float *>(top)[ix] = U;
    float mv[KT];
    int mi[KT];
#pragma unroll
    for (int i = 0; i < KT; i += 4) {
      asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(mv[i]), "=f"(mv[i + 1]), "=f"(mv[i + 2]), "=f"(mv[i + 3])
                   : "r"(smem_u32(top + i)));
      mi[i] = i, mi[i + 1] = i + 1, mi[i + 2] = i + 2, mi[i + 3] = i + 3;
    }
#pragma unroll
    for (int w = KT / 2; w >= 1; w >>= 1) {
#pragma unroll
      for (int i = 0; i < w; ++i) {
        const bool gt = mv[i + w] > mv[i];
        mv[i] = gt ? mv[i + w] : mv[i];
        mi[i] = gt ? mi[i + w] : mi[i];
      }
    }
    m = mv[0];
    *reinterpret_cast<volatile float *>(tmax) = m;
    *reinterpret_cast<volatile int *>(tidx) = mi[0];
  }
  __threadfence_block();
  atomicExch(lock, 0);
  return m;
}

constexpr int kEntBlock = 32;  // entry slots a thread reserves at a time (one atomic per block)

// End of a thread's share of a query: mark the unused tail of its reserved
// block (A = NaN: never a survivor).
template <int KT>
__device__ __forceinline__ void tc_flush(EpiState<KT> &st, int64_t q, const TcArgs &a) {
  for (; st.left > 0; --st.left) {
    const int slot = st.base + (kEntBlock - st.left);
    if (slot < a.cap) a.ent[q * a.cap + slot] = make_uint4(0x7fc00000u, 0u, 0u, 0u);  // A = NaN: no entry
  }
}

// Rigorous float32 bounds of the exact squared distance from the filter's
// (A, r, eta) (same quantities as dist_bounds2, every operation rounded
// toward the safe side instead of float64 plus a relative margin).
__device__ __forceinline__ void dist_bounds_f(float A, float r, float eta, float &L, float &U) {
  const float slo = fmaxf(0.f, __fsub_rd(__fsqrt_rd(fmaxf(0.f, __fsub_rd(A, eta))), r));
  const float shi = __fadd_ru(__fsqrt_ru(__fadd_ru(A, eta)), r);
  L = __fmul_rd(slo, slo);
  U = __fmul_ru(shi, shi);
}

// An admitted candidate: its raw (A, r, eta) go to the entry list (k_tc_select
// turns them into bounds); only a candidate that can enter the k smallest
// upper bounds (U >= A, so A < umax is necessary) pays for its bound here.
template <int KT>
__device__ __forceinline__ void tc_admit(EpiState<KT> &st, float A, float r, float eta, int32_t col, int64_t q,
                                      const TcArgs &a, unsigned *su_slot, float *top, float *tmax, int *tidx,
                                      int *lock) {
  if (st.left == 0) {
    st.base = atomicAdd(a.ent_cnt + q, kEntBlock);
    st.left = kEntBlock;
  }
  const int slot = st.base + (kEntBlock - st.left--);
  if (slot < a.cap)
    a.ent[q * a.cap + slot] =
        make_uint4(__float_as_uint(A), __float_as_uint(r), __float_as_uint(eta), (uint32_t)col);
  if (A >= *reinterpret_cast<volatile float *>(tmax)) return;
  float Lf, Uf;
  dist_bounds_f(A, r, eta, Lf, Uf);
  if (Uf < *reinterpret_cast<volatile float *>(tmax)) {
    const float uk = top_insert<KT>(top, tmax, tidx, lock, Uf);
    if (uk < 3.0e38f) {
      const float s = __fsqrt_ru(uk);
      if (s < st.su) {
        st.su = s;
        atomicMin(su_slot, __float_as_uint(s));
        atomicMin(a.su_g + q, __float_as_uint(s));
      }
    }
  }
}

// MC = 2: launched as clusters of 2 CTAs working on two query blocks over
// the same row tiles in lockstep; each CTA TMA-loads half of every B tile and
// multicasts it to both, so each SM pulls half the row bytes from L2 (the
// MMA feed, not HBM, is the floor of this kernel).  A stage is refilled only
// after both CTAs' MMAs committed it (multicast commits, count-2 barriers).
template <int KT, int CG, int MC>
__global__ void __launch_bounds__(threads_for<CG>(), 1)
    k_tc_filter(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, TcArgs a) {
  extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sStage = sbase + kOffStage, sInfo = sbase + kOffInfo, sBits = sbase + kOffBits;
  const uint32_t bar0 = sbase + kOffBar;
  auto fullB = [&](int s) { return bar0 + 8u * s; };
  auto emptyB = [&](int s) { return bar0 + 8u * (kStages + s); };
  const uint32_t fullA = bar0 + 8u * (2 * kStages), emptyA = fullA + 8u;
  auto tmemFull = [&](int b) { return bar0 + 8u * (2 * kStages + 2 + b); };
  auto epiEmpty = [&](int b) { return bar0 + 8u * (2 * kStages + 4 + b); };
  auto infoFull = [&](int b) { return bar0 + 8u * (2 * kStages + 6 + b); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + kOffTmemSlot);
  unsigned *su_s = reinterpret_cast<unsigned *>(smem + kOffSu);

  constexpr int kEpiWarps = 4 * CG, kColsPerWarp = kN / CG;
  constexpr int kProdWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // work units: query blocks (MC = 1) or query-block pairs (MC = 2, one per
  // cluster); each CTA (cluster) walks a contiguous range of (unit, tile)
  const int rank = MC > 1 ? (int)cluster_rank() : 0;
  const int64_t units = (a.nqb + MC - 1) / MC;
  const int64_t W = units * a.ntiles;
  const int64_t grp = blockIdx.x / MC, ngrp = gridDim.x / MC;
  const int64_t it0 = W * grp / ngrp, it1 = W * (grp + 1) / ngrp;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(fullB(s), 1);
      mbar_init(emptyB(s), MC);
    }
    mbar_init(fullA, 1);
    mbar_init(emptyA, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(tmemFull(b), 1);
      mbar_init(epiEmpty(b), kEpiWarps);
      mbar_init(infoFull(b), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == kProdWarp && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmC)) : "memory");
  }
  if (tid < kM) su_s[tid] = 0x7f800000u;
  tc_fence_before();
  __syncthreads();
  if (MC > 1) cluster_sync_all();  // the partner's barriers exist before any multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == kProdWarp) {
    if (lane == 0) {
      uint32_t g = 0;
      int qb = (int)(it0 / a.ntiles) * MC + rank, tile = (int)(it0 % a.ntiles);
      for (int64_t it = it0; it < it1; ++it, ++tile) {
        if (tile == a.ntiles) {
          tile = 0;
          qb += MC;
        }
        for (int kb = 0; kb < a.kblocks; ++kb, ++g) {
          const int s = (int)(g % kStages);
          mbar_wait_sleep(emptyB(s), ((g / kStages) & 1u) ^ 1u);
          mbar_expect_tx(fullB(s), kStageBytes);
          const uint32_t st = sStage + s * kStageBytes;
          tma_load_2d(st, &tmA, fullB(s), kb * kKB, qb * kM);
          if (MC > 1)
            tma_load_2d_mc(st + kABytes + rank * (kBBytes / 2), &tmB, fullB(s), kb * kKB,
                           tile * kN + rank * (kN / 2), (uint16_t)0x3);
          else
            tma_load_2d(st + kABytes, &tmB, fullB(s), kb * kKB, tile * kN);
        }
      }
      if (MC > 1) {
        // both CTAs' last commits of every stage have arrived here before the
        // cluster may exit (so the partner's commits into this CTA are done)
        for (uint32_t gg = g > (uint32_t)kStages ? g - kStages : 0; gg < g; ++gg)
          mbar_wait_sleep(emptyB((int)(gg % kStages)), (gg / kStages) & 1u);
      }
    } else if (lane == 1) {
      // the tile's row records and candidate words, on their own thread: a
      // buffer is refilled as soon as the epilogue released it, not after the
      // row-tile loads of the item (which wait for the MMA)
      int qb = (int)(it0 / a.ntiles) * MC + rank, tile = (int)(it0 % a.ntiles);
      for (int64_t it = it0; it < it1; ++it, ++tile) {
        if (tile == a.ntiles) {
          tile = 0;
          qb += MC;
        }
        const uint32_t li = (uint32_t)(it - it0), b = li & 1u;
        mbar_wait_sleep(epiEmpty(b), ((li >> 1) & 1u) ^ 1u);
        const int64_t rows = a.n - (int64_t)tile * kN < kN ? a.n - (int64_t)tile * kN : kN;
        const uint32_t t1b = ((uint32_t)rows * 4u + 15u) & ~15u;  // (rt1 is padded to 16 B)
        mbar_expect_tx(infoFull(b), (uint32_t)rows * 16u + t1b + kBitsBytes);
        bulk_load(sInfo + b * kInfoBytes, a.rinfo + (int64_t)tile * kN, (uint32_t)rows * 16u, infoFull(b));
        bulk_load(sInfo + b * kInfoBytes + kN * 16, a.rt1 + (int64_t)tile * kN, t1b, infoFull(b));
        // the block's candidate words for this tile: 128 queries x 8 words
        tma_load_2d(sBits + b * kBitsBytes, &tmC, infoFull(b), tile * (kN / 32), qb * kM);
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      uint32_t g = 0;
      int qb = (int)(it0 / a.ntiles) * MC + rank, tile = (int)(it0 % a.ntiles);
      for (int64_t it = it0; it < it1; ++it, ++tile) {
        if (tile == a.ntiles) {
          tile = 0;
          qb += MC;
        }
        const uint32_t li = (uint32_t)(it - it0), b = li & 1u;
        mbar_wait_sleep(epiEmpty(b), ((li >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dt = tmem_base + b * kN;
        for (int kb = 0; kb < a.kblocks; ++kb, ++g) {
          const int s = (int)(g % kStages);
          mbar_wait_sleep(fullB(s), (g / kStages) & 1u);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kKB / 32; ++kk) {
            const uint64_t ad = sw128_desc(sStage + s * kStageBytes + kk * 32);
            const uint64_t bd = sw128_desc(sStage + s * kStageBytes + kABytes + kk * 32);
            mma_i8(dt, ad, bd, (kb | kk) != 0 ? 1u : 0u);
          }
          if (MC > 1)
            mma_commit_mc(emptyB(s), (uint16_t)0x3);
          else
            mma_commit(emptyB(s));
        }
        mma_commit(tmemFull(b));

      }
    }
  } else {
    // ---------------- epilogue warps ----------------
    const int lq = warp & 3, cg = warp >> 2;
    const int qloc = lq * 32 + lane;
    const uint32_t trow = tmem_base + ((uint32_t)(lq * 32) << 16);
    const float4 *info4 = reinterpret_cast<const float4 *>(smem + kOffInfo);  // [2][kInfoBytes / 16]
    float *top = reinterpret_cast<float *>(smem + kOffTop) + qloc * kTopMax;
    float *tmax = reinterpret_cast<float *>(smem + kOffTopMax) + qloc;
    int *tidx = reinterpret_cast<int *>(smem + kOffTopIdx) + qloc;
    int *tlock = reinterpret_cast<int *>(smem + kOffLock) + qloc;
    EpiState<KT> st;
    int64_t cur_qb = -1, q = 0;
    bool valid = false;
    float sqf = 0.f, t2f = 0.f, rq = 0.f;
    int corr = 0, sel = 0;
    // the CTA's k smallest bounds of its query go to the query's bound list
    // (their union over CTAs holds the query's k smallest)
    auto publish = [&]() {
      const int o = atomicAdd(a.kb_cnt + q, a.k);
      for (int i = 0; i < a.k; ++i)
        if (o + i < a.kbcap) a.kb[q * a.kbcap + o + i] = top[i];
    };
    constexpr int NWD = kColsPerWarp / 32;
    const uint32_t *bits_s = reinterpret_cast<const uint32_t *>(smem + kOffBits);  // [2][kM][8]
    int qb = (int)(it0 / a.ntiles) * MC + rank, tile = (int)(it0 % a.ntiles) - 1;
    float sunext = __int_as_float(0x7f800000);
    for (int64_t it = it0; it < it1; ++it) {
      if (++tile == a.ntiles) {
        tile = 0;
        qb += MC;
      }
      if (qb != cur_qb) {
        if (valid) tc_flush<KT>(st, q, a);
        // new query block: every epilogue warp is past the old one before
        // the shared k-th bounds are reset
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        if (cg == 0) {
          if (valid) publish();
          su_s[qloc] = 0x7f800000u;
          for (int i = 0; i < KT; ++i) top[i] = i < a.k ? __int_as_float(0x7f800000) : -__int_as_float(0x7f800000);
          *tmax = __int_as_float(0x7f800000);
          *tidx = 0;
          *tlock = 0;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        cur_qb = qb;
        q = (int64_t)qb * kM + qloc;
        valid = q < a.m;
        st.su = __int_as_float(0x7f800000);
        sunext = __int_as_float(0x7f800000);  // (a bound of the previous query)
        st.left = 0;
        st.base = 0;
        if (valid) {
          const QParams P = a.qp[q];
          sqf = P.sq;
          t2f = P.t2f;
          rq = P.rq;
          // x.qq = D + 128 sum(qq) (+ 128 sum(x) - 16384 ldq for u8 queries), as k_scan_topk_u8
          corr = 128 * P.qsum - (P.qsigned ? 0 : 16384 * a.ldq);
          sel = P.qsigned ? 0 : 1;
        }
      }
      // the other CTAs' bound for this query, loaded a tile earlier
      st.su = fminf(st.su, sunext);
      if (valid) sunext = __uint_as_float(__ldcg(a.su_g + q));
      const uint32_t li = (uint32_t)(it - it0), b = li & 1u;
      mbar_wait(infoFull(b), (li >> 1) & 1u);
      mbar_wait(tmemFull(b), (li >> 1) & 1u);
      tc_fence_after();
      // candidate words of this warp's columns (TMA-staged with the row records)
      uint32_t wd[NWD];
#pragma unroll
      for (int c = 0; c < NWD; ++c) {
        wd[c] = bits_s[(b * kM + qloc) * (kN / 32) + cg * NWD + c];
        const int64_t col0 = (int64_t)tile * kN + cg * kColsPerWarp + c * 32;
        if (a.n - col0 < 32) wd[c] &= a.n - col0 <= 0 ? 0u : (1u << (a.n - col0)) - 1u;
      }
      if (a.noepi == 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(epiEmpty(b));
        continue;
      }
      // 16 columns per TMEM load (register budget: 18 warps per SM)
#pragma unroll 1
      for (int c = 0; c < kColsPerWarp / 16; ++c) {
        uint32_t v[16];
        const int cofs = cg * kColsPerWarp + c * 16;
        tmem_ld16(trow + b * kN + cofs, v);
        tmem_wait_ld();
        const uint32_t wc = (wd[c >> 1] >> (16 * (c & 1))) & 0xffffu;
        if (a.dbgD && valid) {
          for (int j = 0; j < 16; ++j) {
            const int64_t col = (int64_t)tile * kN + cofs + j;
            if (col < a.n) a.dbgD[q * a.n + col] = (int32_t)v[j];
          }
        }
        if (__any_sync(0xffffffffu, wc != 0u)) {
          st.su = fminf(st.su, __uint_as_float(*reinterpret_cast<volatile unsigned *>(su_s + qloc)));
          const float4 *ri = info4 + b * (kInfoBytes / 16) + cofs;
          const float *rt = reinterpret_cast<const float *>(info4 + b * (kInfoBytes / 16) + kN) + cofs;
          const int32_t colb = tile * kN + cofs;
          // Pre-test, a superset of admit2: admit2 implies
          //   t3 + 2 S (1+2^-16) rad >= [t1 (1-k) - rad^2 (1+2^-16)] + [t2 (1-k) - S^2 (1+2^-16)]
          // with S = su + rq, k = 2^-18 (|t3| <= T, admit2's eta <= 4.8e-7
          // (T + |t3|), and every rounding of both forms is far inside the
          // margins): per column one row record (P = the first bracket) and
          // three float ops.  Columns that pass run the exact rule below
          // (their admissions are rare after the warm-up).
          float s2e = 0.f, nqq = 3.4028235e38f;  // no k-th bound yet: everything passes
          if (st.su < 1.0e18f) {
            const float S = __fadd_ru(st.su, rq);
            s2e = __fmul_ru(2.0f * S, 1.0000153f);
            nqq = -__fsub_rd(__fmul_rd(t2f, 0.99999619f), __fmul_ru(__fmul_ru(S, S), 1.0000153f));
          }
          uint32_t take = 0u;
          if (__all_sync(0xffffffffu, sel == 1)) {  // unsigned queries (the common case)
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float4 r4 = ri[j];
              const float f = (float)((int)v[j] + __float_as_int(r4.w) + corr);
              const float lhs = fmaf(r4.y * sqf, f, fmaf(s2e, r4.z, nqq));
              take |= (lhs >= r4.x ? 1u : 0u) << j;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float4 r4 = ri[j];
              const float f = (float)((int)v[j] + sel * __float_as_int(r4.w) + corr);
              const float lhs = fmaf(r4.y * sqf, f, fmaf(s2e, r4.z, nqq));
              take |= (lhs >= r4.x ? 1u : 0u) << j;
            }
          }
          take &= wc;
          if (a.noepi == 2) take = 0u;  // experiment: bounds without admissions
          while (take) {
            const int j = __ffs(take) - 1;
            take &= take - 1u;
            // v[j] by a depth-4 select tree
            int d8[8], d4[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) d8[i] = (j & 1) ? (int)v[2 * i + 1] : (int)v[2 * i];
#pragma unroll
            for (int i = 0; i < 4; ++i) d4[i] = (j & 2) ? d8[2 * i + 1] : d8[2 * i];
            const int d2a = (j & 4) ? d4[1] : d4[0], d2b = (j & 4) ? d4[3] : d4[2];
            const int dv = (j & 8) ? d2b : d2a;
            const float4 r4 = ri[j];
            const int mys = dv + corr + sel * __float_as_int(r4.w);
            const float t1 = rt[j];
            const float t3 = (r4.y * sqf) * (float)mys;
            const float A = (t1 + t2f) - t3;
            const float eta = __fmul_ru(4.76837158203125e-07f, __fadd_ru(__fadd_ru(t1, t2f), fabsf(t3)));
            const float r = __fadd_ru(r4.z, rq);
            tc_admit<KT>(st, A, r, eta, colb + j, q, a, su_s + qloc, top, tmax, tidx, tlock);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(epiEmpty(b));
    }
    if (valid) tc_flush<KT>(st, q, a);
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
    if (cg == 0 && valid) publish();
  }
  __syncthreads();
  if (MC > 1) cluster_sync_all();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

// Row records of the fused filter, from the GEMM route's {scale, norm,
// radius, sum}: t1 = scale^2 * norm exactly as k_scan_topk_u8 forms it,
// 2 * scale, radius, 128 * sum (the unsigned-query offset term).
__global__ void k_tc_rows(const uint4 *__restrict__ info, int64_t n, uint4 *__restrict__ rinfo, float *rt1) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = info[i];
    const float sx = __uint_as_float(v.x);
    const float t1 = sx * sx * (float)(int)v.y;
    const float rad = __uint_as_float(v.z);
    // pre-test row term P = t1 (1 - 2^-18) - rad^2 (1 + 2^-16), rounded down
    const float P = __fsub_rd(__fmul_rd(t1, 0.99999619f), __fmul_ru(__fmul_ru(rad, rad), 1.0000153f));
    rinfo[i] = make_uint4(__float_as_uint(P), __float_as_uint(2.0f * sx), v.z, (uint32_t)(128 * (int)v.w));
    rt1[i] = t1;
  }
}

// Per query (one warp): bounds of the entries' (A, r, eta), the k-th smallest
// upper bound U_k, survivors L <= U_k to k_rerank's lists; list overflow or
// too many survivors -> exact fallback.
constexpr int kSelCap = 2048;  // entry slots per query
constexpr int kKbSort = 256;   // bounds per query in the union of the CTAs' k smallest (kTcKb)
__global__ void __launch_bounds__(128) k_tc_select(const uint4 *__restrict__ ent, const int32_t *__restrict__ ent_cnt,
                                                   const float *__restrict__ kb, const int32_t *__restrict__ kb_cnt,
                                                   int kbcap, int cap, int64_t m, int k, int32_t *surv, int32_t *nsurv,
                                                   int32_t *fb_list, int32_t *fb_count) {
  __shared__ float sk[4][kKbSort];
  __shared__ int32_t si[4][kKbSort];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float *kk = sk[w];
  int32_t *ii = si[w];
  for (int64_t q = (int64_t)blockIdx.x * 4 + w; q < m; q += (int64_t)gridDim.x * 4) {
    const int cnt = ent_cnt[q];
    const uint4 *e = ent + q * cap;
    const int nb = kb_cnt[q];
    // overflowing entry or bound lists (not reached with <= 8 CTAs per query
    // block): the exact fallback
    if (cnt > cap || nb > kbcap || nb > kKbSort) {
      if (lane == 0) {
        nsurv[q] = -1;
        fb_list[atomicAdd(fb_count, 1)] = (int32_t)q;
      }
      continue;
    }
    // the query's k-th smallest upper bound: the union of the CTAs' k
    // smallest bounds holds it (a short sort)
    int np2 = 32;
    while (np2 < nb) np2 <<= 1;
    for (int i = lane; i < np2; i += 32) {
      kk[i] = i < nb ? kb[q * kbcap + i] : __int_as_float(0x7f800000);
      ii[i] = i;
    }
    __syncwarp();
    warp_sort(kk, ii, np2);
    const double uk = nb >= k ? (double)kk[k - 1] : __longlong_as_double(0x7ff0000000000000LL);
    __syncwarp();
    int ns = 0;
    for (int i0 = 0; i0 < cnt; i0 += 32) {
      const int i = i0 + lane;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      bool in = false;
      if (i < cnt) {
        v = e[i];
        float L, U;
        dist_bounds_f(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), L, U);
        const float A = __uint_as_float(v.x);
        in = A == A && (double)L <= uk;  // an empty slot holds A = NaN
      }
      const unsigned bm = __ballot_sync(0xffffffffu, in);
      const int dst = ns + __popc(bm & lanemask_lt());
      if (in && dst < kSurvCap) surv[q * kSurvCap + dst] = (int32_t)v.w;
      ns += __popc(bm);
    }
    if (lane == 0) {
      if (ns <= kSurvCap) {
        nsurv[q] = ns;
      } else {
        nsurv[q] = -1;
        fb_list[atomicAdd(fb_count, 1)] = (int32_t)q;
      }
    }
    __syncwarp();
  }
}

}  // namespace tc
}  // namespace mrpt

namespace mrpt {
namespace tc {
// debug: compare two (m, n) s32 matrices, count mismatches; entry stats
// Debug reference (MRPT_TC_DEBUG): D[q * ldD + r] = sum_c Xs[r][c] * Qop[q][c]
// over the s8 operands, one thread per (row, query).
__global__ void k_dot_ref(const int8_t *__restrict__ Xs, int64_t n, const int8_t *__restrict__ Qop, int64_t ldq,
                          int32_t *D, int64_t ldD) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t q = blockIdx.y;
  if (r >= n) return;
  int acc = 0;
  for (int64_t c = 0; c < ldq; ++c) acc += (int)Xs[r * ldq + c] * (int)Qop[q * ldq + c];
  D[q * ldD + r] = acc;
}

__global__ void k_tc_debug(const int32_t *A, const int32_t *B, int64_t n, int64_t ldb, const int32_t *ent_cnt,
                           int64_t m, unsigned long long *out) {
  // A: (m, n) dense; B: (m, ldb) library GEMM output
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m * n; i += (int64_t)gridDim.x * blockDim.x)
    if (A[i] != B[(i / n) * ldb + i % n]) atomicAdd(out, 1ull);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(out + 1, (unsigned long long)ent_cnt[i]);
    atomicMax(out + 2, (unsigned long long)ent_cnt[i]);
  }
}
}  // namespace tc
}  // namespace mrpt
