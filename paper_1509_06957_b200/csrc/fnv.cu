// K6: 64-bit FNV-1a of the dataset bytes in parallel (Dataset.checksum,
// pkg/src/mrpt/core.py:77-82 -> _cy.fnv1a64, _kernels/_cy.pyx:100-106).
//
// h' = (h ^ b) * P mod 2^64 is serial, but its low byte evolves on its own:
// low8(h') = ((low8(h) ^ b) * 0xB3) & 0xFF.  Writing l = low8(h) and
// x = l ^ b, h' = (h - l + x) * P, so over a chunk of m bytes starting from
// state h0 with low byte L the result is h0 * P^m + C(L), where C(L) only
// depends on the chunk and L.  Three passes:
//   A  per chunk, the 256 -> 256 low-byte permutation (128 starts walked,
//      two per thread, 1.5 integer ops per start and byte, bytes broadcast
//      from shared memory);
//   S  a serial walk over the permutations gives each chunk's true L;
//   B  one thread per chunk computes C(L) for that L only;
// then h <- h * P^m + C_chunk composes the chunks in order.
#include "common.cuh"

namespace mrpt {

constexpr unsigned long long kFnvOffset = 0xCBF29CE484222325ull;
constexpr unsigned long long kFnvPrime = 0x100000001B3ull;
constexpr int kFnvStage = 4096;  // bytes staged in smem per step (pass A)
constexpr int kStartBlock = 64;   // chunk tables staged per step of the serial walk

// Pass A: the chunk's low-byte permutation.  Two facts cut the work 4x:
//  * the top bit rides along: (l ^ 0x80) ^ b = (l ^ b) ^ 0x80, and since
//    0xB3 is odd, ((x ^ 0x80) * 0xB3) & 0xFF = ((x * 0xB3) & 0xFF) ^ 0x80,
//    so perm(L ^ 0x80) = perm(L) ^ 0x80 and only L < 128 is walked;
//  * two starts share a 32-bit register as 16-bit lanes: per byte one PRMT
//    (the byte into both lanes), one LOP3 ((l & 0x00FF00FF) ^ bb) and one
//    IMAD (x * 0xB3: the low lane's product stays below 2^16).
// 64 threads per chunk, each walking starts 2t and 2t+1.
constexpr int kFnvThreads = 64;
__global__ void __launch_bounds__(kFnvThreads) k_fnv_perm(const uint8_t *__restrict__ buf, int64_t nbytes,
                                                          int64_t chunk, uint8_t *perm) {
  __shared__ uint4 stage[kFnvStage / 16];
  const int64_t c = blockIdx.x;
  const int64_t b0 = c * chunk;
  const int64_t b1 = (b0 + chunk) < nbytes ? (b0 + chunk) : nbytes;
  const uint32_t t = threadIdx.x;
  uint32_t l = (2 * t) | ((2 * t + 1) << 16);
  constexpr uint32_t M = 0x00FF00FFu;
  const bool al = ((reinterpret_cast<uintptr_t>(buf + b0) & 15u) == 0);
  for (int64_t s0 = b0; s0 < b1; s0 += kFnvStage) {
    const int len = (int)((b1 - s0) < kFnvStage ? (b1 - s0) : kFnvStage);
    __syncthreads();
    if (al) {
      const uint4 *src = reinterpret_cast<const uint4 *>(buf + s0);
      for (int i = t; i < len / 16; i += kFnvThreads) stage[i] = __ldg(src + i);
    } else {
      uint8_t *st8 = reinterpret_cast<uint8_t *>(stage);
      for (int i = t; i < (len & ~15); i += kFnvThreads) st8[i] = buf[s0 + i];
    }
    __syncthreads();
    const int nv = len / 16;
#pragma unroll 2
    for (int i = 0; i < nv; ++i) {
      const uint4 v = stage[i];
      const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        l = ((l & M) ^ __byte_perm(ws[q], 0u, 0x4040u)) * 0xB3u;
        l = ((l & M) ^ __byte_perm(ws[q], 0u, 0x4141u)) * 0xB3u;
        l = ((l & M) ^ __byte_perm(ws[q], 0u, 0x4242u)) * 0xB3u;
        l = ((l & M) ^ __byte_perm(ws[q], 0u, 0x4343u)) * 0xB3u;
      }
    }
    for (int j = nv * 16; j < len; ++j) {
      const uint32_t b = buf[s0 + j];
      l = ((l & M) ^ (b | (b << 16))) * 0xB3u;
    }
  }
  const uint8_t p0 = (uint8_t)(l & 0xffu), p1 = (uint8_t)((l >> 16) & 0xffu);
  uint8_t *pc = perm + c * 256;
  pc[2 * t] = p0;
  pc[2 * t + 1] = p1;
  pc[2 * t + 128] = p0 ^ 0x80u;
  pc[2 * t + 129] = p1 ^ 0x80u;
}

// Serial walk over the chunk permutations: the true low byte at each chunk
// start.  Tables are staged kStartBlock at a time so the dependent lookups
// hit shared memory.
__global__ void __launch_bounds__(256) k_fnv_starts(const uint8_t *__restrict__ perm, int64_t nchunks,
                                                    uint8_t *starts) {
  __shared__ uint32_t tabs[kStartBlock * 256 / 4];
  uint32_t l = (uint32_t)(kFnvOffset & 0xffull);
  for (int64_t c0 = 0; c0 < nchunks; c0 += kStartBlock) {
    const int nb = (int)((nchunks - c0) < kStartBlock ? (nchunks - c0) : kStartBlock);
    __syncthreads();
    const uint32_t *src = reinterpret_cast<const uint32_t *>(perm + c0 * 256);
    for (int i = threadIdx.x; i < nb * 64; i += blockDim.x) tabs[i] = src[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint8_t *t8 = reinterpret_cast<const uint8_t *>(tabs);
      for (int j = 0; j < nb; ++j) {
        starts[c0 + j] = (uint8_t)l;
        l = t8[j * 256 + l];
      }
    }
  }
}

// Pass B: the affine offset C of each chunk for its true starting low byte
// (one thread per chunk): h_end = h_start * P^m + C.
__global__ void __launch_bounds__(128) k_fnv_offsets(const uint8_t *__restrict__ buf, int64_t nbytes,
                                                     int64_t chunk, int64_t nchunks,
                                                     const uint8_t *__restrict__ starts,
                                                     unsigned long long *coff) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const int64_t b0 = c * chunk;
  const int64_t b1 = (b0 + chunk) < nbytes ? (b0 + chunk) : nbytes;
  uint32_t l = starts[c];
  unsigned long long C = 0ull;
  int64_t i = b0;
  if ((reinterpret_cast<uintptr_t>(buf + b0) & 15u) == 0) {
    for (; i + 16 <= b1; i += 16) {
      const uint4 v = __ldg(reinterpret_cast<const uint4 *>(buf + i));
      const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t w = ws[q];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t x = (l ^ w) & 0xffu;
          C = (C + (unsigned long long)x - (unsigned long long)l) * kFnvPrime;
          l = (x * 0xB3u) & 0xffu;
          w >>= 8;
        }
      }
    }
  }
  for (; i < b1; ++i) {
    const uint32_t x = l ^ buf[i];
    C = (C + (unsigned long long)x - (unsigned long long)l) * kFnvPrime;
    l = (x * 0xB3u) & 0xffu;
  }
  coff[c] = C;
}

__global__ void k_fnv_combine(const unsigned long long *__restrict__ coff, int64_t nchunks,
                              unsigned long long pm_full, unsigned long long pm_last,
                              unsigned long long *out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long h = kFnvOffset;
  for (int64_t c = 0; c < nchunks; ++c) {
    const unsigned long long pm = (c + 1 == nchunks) ? pm_last : pm_full;
    h = h * pm + coff[c];
  }
  *out = h;
}

static unsigned long long pow_mod64(unsigned long long base, int64_t e) {
  unsigned long long r = 1ull;
  while (e > 0) {
    if (e & 1) r *= base;
    base *= base;
    e >>= 1;
  }
  return r;
}

// Chunk size: enough chunks to fill the GPU in both passes.
static int64_t fnv_chunk(int64_t nbytes) {
  int64_t c = nbytes / ((int64_t)num_sms() * 256);
  c = (c + 15) / 16 * 16;
  if (c < 4096) c = 4096;
  return c;
}

static size_t fnv_ws(int64_t nch) {
  return (size_t)nch * 256 + (size_t)nch + 16 + (size_t)nch * sizeof(unsigned long long) + 64;
}

}  // namespace mrpt

using namespace mrpt;

extern "C" int32_t mrpt_fnv1a64_workspace_size(int64_t nbytes, size_t *bytes) {
  clear_error();
  if (nbytes < 0 || !bytes) return fail(MRPT_EPARAM, "mrpt_fnv1a64_workspace_size: bad arguments");
  const int64_t nch = nbytes == 0 ? 0 : ceil_div<int64_t>(nbytes, fnv_chunk(nbytes));
  *bytes = fnv_ws(nch);
  return MRPT_OK;
}

extern "C" int32_t mrpt_fnv1a64(const uint8_t *buf, int64_t nbytes, uint64_t *out, void *ws,
                                size_t ws_bytes, void *stream) {
  clear_error();
  if (nbytes < 0 || !out) return fail(MRPT_EPARAM, "mrpt_fnv1a64: bad arguments");
  cudaStream_t s = as_stream(stream);
  unsigned long long *o = reinterpret_cast<unsigned long long *>(out);
  if (nbytes == 0) {  // empty input hashes to the offset basis
    (count_launch(), k_fnv_combine<<<1, 32, 0, s>>>(nullptr, 0, 1ull, 1ull, o));
    return launch_status("mrpt_fnv1a64");
  }
  const int64_t chunk = fnv_chunk(nbytes);
  const int64_t nch = ceil_div<int64_t>(nbytes, chunk);
  if (ws_bytes < fnv_ws(nch) || !ws) return fail(MRPT_EWORKSPACE, "mrpt_fnv1a64: workspace too small");
  if (nch > 0x7fffffff) return fail(MRPT_EPARAM, "mrpt_fnv1a64: input too large");
  uint8_t *perm = reinterpret_cast<uint8_t *>(ws);
  uint8_t *starts = perm + (size_t)nch * 256;
  unsigned long long *coff = reinterpret_cast<unsigned long long *>(
      (reinterpret_cast<uintptr_t>(starts + nch) + 15) & ~uintptr_t(15));
  (count_launch(), k_fnv_perm<<<(unsigned)nch, kFnvThreads, 0, s>>>(buf, nbytes, chunk, perm));
  (count_launch(), k_fnv_starts<<<1, 256, 0, s>>>(perm, nch, starts));
  (count_launch(), k_fnv_offsets<<<(unsigned)ceil_div<int64_t>(nch, 128), 128, 0, s>>>(buf, nbytes, chunk, nch, starts,
                                                                      coff));
  const int64_t last = nbytes - (nch - 1) * chunk;
  (count_launch(), k_fnv_combine<<<1, 32, 0, s>>>(coff, nch, pow_mod64(kFnvPrime, chunk), pow_mod64(kFnvPrime, last), o));
  return launch_status("mrpt_fnv1a64");
}
