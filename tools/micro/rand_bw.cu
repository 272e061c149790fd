// Random-read throughput of HBM by access size: each warp reads one random,
// size-aligned block of S bytes (S/16 lanes' worth of 16-byte loads, looped),
// from a 32 GB buffer (far beyond L2).  Shows what scattered piece reads
// can reach.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rand_bw rand_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) k(const uint4 *buf, unsigned long long nblk, int S16, int iters,
                                             unsigned *out) {
  const int lane = threadIdx.x & 31;
  unsigned long long x = (blockIdx.x * 32ull + (threadIdx.x >> 5)) * 0x9E3779B97F4A7C15ull + 7;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const unsigned long long b = x % nblk;
    const uint4 *p = buf + b * S16;
    for (int j = lane; j < S16; j += 32) {
      const uint4 v = __ldcg(p + j);
      acc += v.x ^ v.w;
    }
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *out;
  cudaMalloc(&out, 64);
  const size_t bytes = 32ull << 30;
  uint4 *buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int S : {64, 128, 256, 512, 1024, 2048, 4096, 16384}) {
    const int S16 = S / 16;
    const unsigned long long nblk = bytes / S;
    const int iters = (int)(((size_t)2 << 30) / ((size_t)sms * 32 * S)) + 1;
    k<<<sms, 1024>>>(buf, nblk, S16, 4, out);
    cudaEventRecord(e0);
    k<<<sms, 1024>>>(buf, nblk, S16, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tot = (double)sms * 32 * iters * S;
    printf("block %6d B: %7.0f GB/s\n", S, tot / (ms * 1e-3) / 1e9);
  }
  return 0;
}
