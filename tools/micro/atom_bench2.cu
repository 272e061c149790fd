// Shared-memory atomics on random words of a 55.8K-word (218 KB) array, one
// 1024-thread CTA per SM (the vote's shape): returning atomicAdd (result
// used), non-returning atomicAdd (RED), RED + read-back LDS of the same word,
// and plain LDS.  Reports lanes per clock per SM at 1965 MHz.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ab2 atom_bench2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(int iters, unsigned *out, int words) {
  extern __shared__ unsigned sm[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u + blockIdx.x * 97u;
  unsigned acc = 0;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const unsigned w = (x >> 7) % words, sh = (x & 3) * 10;
    if (MODE == 0) {  // returning
      const unsigned old = atomicAdd(&sm[w], 1u << sh);
      acc += ((old >> sh) & 1023u) == 9u;
    } else if (MODE == 1) {  // RED
      atomicAdd(&sm[w], 1u << sh);
    } else if (MODE == 2) {  // RED + read back
      atomicAdd(&sm[w], 1u << sh);
      acc += ((sm[w] >> sh) & 1023u) >= 10u;
    } else {  // plain loads
      acc += (sm[w] >> sh) & 1u;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0] + acc;
  else if (acc == 12345) out[blockIdx.x] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int words = 55808;
  const char *names[4] = {"returning atomicAdd", "RED (non-returning)", "RED + LDS read-back", "LDS only"};
  void (*fns[4])(int, unsigned *, int) = {k<0>, k<1>, k<2>, k<3>};
  for (int m = 0; m < 4; ++m) {
    cudaFuncSetAttribute(fns[m], cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4);
    fns[m]<<<sms, 1024, words * 4>>>(64, out, words);
    const int iters = 8192;
    cudaEventRecord(e0);
    fns[m]<<<sms, 1024, words * 4>>>(iters, out, words);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-24s %.2f lanes/clk/SM\n", names[m], 1024.0 * iters / (ms * 1e-3) / 1.965e9);
  }
  return 0;
}
