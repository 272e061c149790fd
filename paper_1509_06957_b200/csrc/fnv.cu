// K6: 64-bit FNV-1a of the dataset bytes in parallel (Dataset.checksum,
// pkg/src/mrpt/core.py:77-82 -> _cy.fnv1a64, _kernels/_cy.pyx:100-106).
//
// h' = (h ^ b) * P mod 2^64 is serial, but its low byte evolves on its own:
// low8(h') = ((low8(h) ^ b) * 0xB3) & 0xFF.  Writing l = low8(h) and
// x = l ^ b, h' = (h - l + x) * P, so over a chunk of m bytes starting from
// state h0 with low byte L the result is h0 * P^m + C(L), where C(L) only
// depends on the chunk and L.  One CTA per chunk computes C for all 256
// values of L (one thread each, bytes broadcast from shared memory); a
// final pass composes the chunks in order: h <- h * P^m + C_chunk[low8(h)].
#include "common.cuh"

namespace mrpt {

constexpr unsigned long long kFnvOffset = 0xCBF29CE484222325ull;
constexpr unsigned long long kFnvPrime = 0x100000001B3ull;
constexpr int kFnvStage = 16384;  // bytes staged in smem per step

__global__ void __launch_bounds__(256) k_fnv_chunks(const uint8_t *__restrict__ buf, int64_t nbytes,
                                                    int64_t chunk, unsigned long long *tab) {
  __shared__ uint32_t stage[kFnvStage / 4];
  const int64_t c = blockIdx.x;
  const int64_t b0 = c * chunk;
  const int64_t b1 = (b0 + chunk) < nbytes ? (b0 + chunk) : nbytes;
  uint32_t l = threadIdx.x;
  unsigned long long C = 0ull;
  const bool al = ((reinterpret_cast<uintptr_t>(buf + b0) & 3u) == 0);
  for (int64_t s0 = b0; s0 < b1; s0 += kFnvStage) {
    const int len = (int)((b1 - s0) < kFnvStage ? (b1 - s0) : kFnvStage);
    __syncthreads();
    if (al) {
      const uint32_t *src = reinterpret_cast<const uint32_t *>(buf + s0);
      for (int i = threadIdx.x; i < len / 4; i += blockDim.x) stage[i] = __ldg(src + i);
      if (threadIdx.x == 0) {
        uint32_t tail = 0;
        for (int j = len & ~3; j < len; ++j) tail |= (uint32_t)buf[s0 + j] << (8 * (j & 3));
        if (len & 3) stage[len / 4] = tail;
      }
    } else {
      uint8_t *st8 = reinterpret_cast<uint8_t *>(stage);
      for (int i = threadIdx.x; i < len; i += blockDim.x) st8[i] = buf[s0 + i];
    }
    __syncthreads();
    const int nw = len / 4;
    for (int i = 0; i < nw; ++i) {
      uint32_t w = stage[i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t x = l ^ (w & 0xffu);
        C = (C + (unsigned long long)x - (unsigned long long)l) * kFnvPrime;
        l = (x * 0xB3u) & 0xffu;
        w >>= 8;
      }
    }
    const uint8_t *st8 = reinterpret_cast<const uint8_t *>(stage);
    for (int j = nw * 4; j < len; ++j) {
      const uint32_t x = l ^ st8[j];
      C = (C + (unsigned long long)x - (unsigned long long)l) * kFnvPrime;
      l = (x * 0xB3u) & 0xffu;
    }
  }
  tab[c * 256 + threadIdx.x] = C;
}

__global__ void k_fnv_combine(const unsigned long long *__restrict__ tab, int64_t nchunks,
                              unsigned long long pm_full, unsigned long long pm_last,
                              unsigned long long *out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long h = kFnvOffset;
  for (int64_t c = 0; c < nchunks; ++c) {
    const unsigned long long pm = (c + 1 == nchunks) ? pm_last : pm_full;
    h = h * pm + tab[c * 256 + (h & 0xffull)];
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

static int64_t fnv_chunk(int64_t nbytes) {
  int64_t c = nbytes / ((int64_t)num_sms() * 8);
  c = (c + 15) / 16 * 16;
  if (c < 4096) c = 4096;
  if (c > (1 << 20)) c = 1 << 20;
  return c;
}

}  // namespace mrpt

using namespace mrpt;

extern "C" int32_t mrpt_fnv1a64_workspace_size(int64_t nbytes, size_t *bytes) {
  clear_error();
  if (nbytes < 0 || !bytes) return fail(MRPT_EPARAM, "mrpt_fnv1a64_workspace_size: bad arguments");
  const int64_t nch = nbytes == 0 ? 0 : ceil_div<int64_t>(nbytes, fnv_chunk(nbytes));
  *bytes = (size_t)nch * 256 * sizeof(unsigned long long) + 256;
  return MRPT_OK;
}

extern "C" int32_t mrpt_fnv1a64(const uint8_t *buf, int64_t nbytes, uint64_t *out, void *ws,
                                size_t ws_bytes, void *stream) {
  clear_error();
  if (nbytes < 0 || !out) return fail(MRPT_EPARAM, "mrpt_fnv1a64: bad arguments");
  cudaStream_t s = as_stream(stream);
  unsigned long long *o = reinterpret_cast<unsigned long long *>(out);
  if (nbytes == 0) {  // empty input hashes to the offset basis
    k_fnv_combine<<<1, 32, 0, s>>>(nullptr, 0, 1ull, 1ull, o);
    return launch_status("mrpt_fnv1a64");
  }
  const int64_t chunk = fnv_chunk(nbytes);
  const int64_t nch = ceil_div<int64_t>(nbytes, chunk);
  if (ws_bytes < (size_t)nch * 256 * sizeof(unsigned long long) || !ws)
    return fail(MRPT_EWORKSPACE, "mrpt_fnv1a64: workspace too small");
  if (nch > 0x7fffffff) return fail(MRPT_EPARAM, "mrpt_fnv1a64: input too large");
  unsigned long long *tab = reinterpret_cast<unsigned long long *>(ws);
  k_fnv_chunks<<<(unsigned)nch, 256, 0, s>>>(buf, nbytes, chunk, tab);
  const int64_t last = nbytes - (nch - 1) * chunk;
  k_fnv_combine<<<1, 32, 0, s>>>(tab, nch, pow_mod64(kFnvPrime, chunk), pow_mod64(kFnvPrime, last), o);
  return launch_status("mrpt_fnv1a64");
}
