// Random 16-byte loads (4 consecutive quads per lane from a random spot, one
// spot per lane) over buffers of growing size: the vote's access shape
// without its counting.  A drop in throughput with the footprint beyond L2
// points at address translation (TLB reach), not DRAM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tlb_bench tlb_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) k_rand(const uint4 *buf, unsigned long long nquads, int iters,
                                                  unsigned *out) {
  unsigned long long x = (blockIdx.x * 1024ull + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const unsigned long long q = (x % (nquads - 4)) & ~3ull;
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldcg(buf + q + j);
#pragma unroll
    for (int j = 0; j < 4; ++j) acc += v[j].x ^ v[j].w;
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *out;
  cudaMalloc(&out, 64);
  const size_t max_bytes = 48ull << 30;
  uint4 *buf;
  if (cudaMalloc(&buf, max_bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 1, max_bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t gb : {1, 4, 16, 48}) {
    const unsigned long long nq = (gb << 30) / 16;
    const int iters = 2048;
    k_rand<<<sms, 1024>>>(buf, nq, 16, out);
    cudaEventRecord(e0);
    k_rand<<<sms, 1024>>>(buf, nq, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)sms * 1024 * iters * 64;
    printf("footprint %3zu GB: %.0f GB/s of 64-byte random reads\n", gb, bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
