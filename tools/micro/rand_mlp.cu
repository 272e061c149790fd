// Random-read throughput of HBM by access size AND requests in flight: each
// warp instruction reads 32/(S/16) random, size-aligned blocks of S bytes
// (S <= 512), K independent instructions are issued before any result is
// used, so a warp has K*32*16 bytes in flight.  rand_bw.cu keeps one block
// per warp in flight and so measures latency, not the DRAM limit; this one
// separates the two.  32 GB buffer (far beyond L2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rand_mlp rand_mlp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void __launch_bounds__(1024, 1) k(const uint4 *buf, unsigned long long nblk, int S16, int iters,
                                             unsigned *out) {
  const int lane = threadIdx.x & 31;
  const int per = 32 / S16;  // blocks per instruction
  const int sub = lane / S16, q = lane % S16;
  unsigned long long x = ((blockIdx.x * 1024ull + threadIdx.x) / S16 * 0x9E3779B97F4A7C15ull) + 7;
  (void)per;
  (void)sub;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint4 v[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      x ^= x << 13;
      x ^= x >> 7;
      x ^= x << 17;
      const unsigned long long b = x % nblk;
      v[j] = __ldcg(buf + b * S16 + q);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) acc += v[j].x ^ v[j].w;
  }
  if (acc == 0x12345) out[0] = acc;
}

template <int K>
static void run(const uint4 *buf, size_t bytes, int sms, unsigned *out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int S : {32, 64, 128, 256, 512}) {
    const int S16 = S / 16 < 1 ? 1 : S / 16;
    const unsigned long long nblk = bytes / (16ull * S16);
    const size_t per_iter = (size_t)sms * 1024 * 16 * K;  // bytes per iteration over the grid
    const int iters = (int)(((size_t)4 << 30) / per_iter) + 1;
    k<K><<<sms, 1024>>>(buf, nblk, S16, 2, out);
    cudaEventRecord(e0);
    k<K><<<sms, 1024>>>(buf, nblk, S16, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tot = (double)per_iter * iters;
    const double acc = tot / (16.0 * S16);
    printf("K=%d block %4d B: %7.0f GB/s  %6.2f G blocks/s\n", K, 16 * S16, tot / (ms * 1e-3) / 1e9,
           acc / (ms * 1e-3) / 1e9);
  }
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
  run<1>(buf, bytes, sms, out);
  run<2>(buf, bytes, sms, out);
  run<4>(buf, bytes, sms, out);
  run<8>(buf, bytes, sms, out);
  return 0;
}
