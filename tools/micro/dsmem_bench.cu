// Microbenchmark: shared-memory atomicAdd throughput, local vs remote
// (distributed shared memory within a thread-block cluster), random words.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int CLUSTER>
__global__ void __cluster_dims__(CLUSTER, 1, 1) k_dsm(int iters, int words, unsigned *out, int remote) {
  extern __shared__ unsigned sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = 0;
  cl.sync();
  const unsigned rank = cl.block_rank();
  unsigned x = threadIdx.x * 2654435761u + blockIdx.x * 97u;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const unsigned target = remote ? (x >> 4) % CLUSTER : rank;
    unsigned *base = cl.map_shared_rank(sm, target);
    atomicAdd(base + ((x >> 8) % words), 1u);
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

template <int C>
void run(int sms, unsigned *out, int remote) {
  const int words = 40 * 1024, threads = 1024, iters = 2048;
  cudaFuncSetAttribute(k_dsm<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = (sms / C) * C;
  k_dsm<C><<<grid, threads, words * 4>>>(16, words, out, remote);
  cudaEventRecord(e0);
  k_dsm<C><<<grid, threads, words * 4>>>(iters, words, out, remote);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  printf("cluster=%d remote=%d: %.2f atomics/clk/SM  (%s)\n", C, remote,
         (double)grid * threads * iters / (ms * 1e-3) / 1.965e9 / grid, cudaGetErrorString(err));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *out; cudaMalloc(&out, 1 << 20);
  run<1>(sms, out, 0);
  run<2>(sms, out, 1);
  run<4>(sms, out, 1);
  run<8>(sms, out, 1);
  return 0;
}
