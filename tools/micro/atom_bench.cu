// Microbenchmark: shared-memory atomicAdd throughput on distinct random words,
// and F2F.F64.F32 / DADD throughput, per SM.  nvcc -arch=sm_100a atom_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_atom(int iters, unsigned *out, int words) {
  extern __shared__ unsigned sm[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    atomicAdd(&sm[(x >> 8) % words], 1u << ((x & 1) * 16));
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

__global__ void k_f2f(int iters, double *out, const float *in) {
  float a = in[threadIdx.x & 31], b = a + 1.f, c = a + 2.f, d = a + 3.f;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; ++i) {
    s0 += (double)a; s1 += (double)b; s2 += (double)c; s3 += (double)d;
    a += 1.0f; b += 1.0f; c += 1.0f; d += 1.0f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *out; cudaMalloc(&out, 1 << 20);
  double *dout; cudaMalloc(&dout, 64 << 20);
  float *in; cudaMalloc(&in, 1024); cudaMemset(in, 0, 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int words = 48 * 1024;
  cudaFuncSetAttribute(k_atom, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4);
  for (int threads : {256, 512, 1024}) {
    int iters = 4096;
    k_atom<<<sms, threads, words * 4>>>(16, out, words);
    cudaEventRecord(e0);
    k_atom<<<sms, threads, words * 4>>>(iters, out, words);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double per_sm = (double)threads * iters / (ms * 1e-3) / 1.965e9;
    printf("smem atomicAdd random u16-lane: threads=%d  %.2f atomics/clk/SM (at 1965 MHz)\n", threads, per_sm);
  }
  {
    int iters = 1 << 16, threads = 1024, blocks = sms * 2;
    k_f2f<<<blocks, threads>>>(16, dout, in);
    cudaEventRecord(e0);
    k_f2f<<<blocks, threads>>>(iters, dout, in);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double per_sm = (double)blocks * threads * iters * 4 / (ms * 1e-3) / 1.965e9 / sms;
    printf("F2F.F64.F32 + DADD pairs: %.2f /clk/SM\n", per_sm);
  }
  return 0;
}
