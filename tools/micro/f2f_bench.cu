// K1 inner-loop variants: what a warp can sustain per SM for one float64
// FMA per term when the point's coordinate comes from shared memory as
//   a) float64 (LDS.64, the current K1),
//   b) float32 + conversion (LDS.32 + F2F.F64.F32),
//   c) two points' float32 in one LDS.64 + two conversions.
// 32 warps per SM, coefficient warp-uniform from a register.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f2f_bench f2f_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(const float *src, double *out, int iters) {
  extern __shared__ double xd[];  // 32 * 257 doubles, or 64 * 257 floats
  float *xf = reinterpret_cast<float *>(xd);
  if (MODE == 0)
    for (int i = threadIdx.x; i < 32 * 257; i += 1024) xd[i] = src[i % 1024];
  else
    for (int i = threadIdx.x; i < 64 * 257; i += 1024) xf[i] = src[i % 1024];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  double v = 1.0 + threadIdx.x * 1e-9;
  int r = (threadIdx.x >> 5) * 7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
      r = (r + 37) & 255;
      if (MODE == 0) {
        acc0 = __fma_rn(xd[lane * 257 + r], v, acc0);
        acc1 = __fma_rn(xd[lane * 257 + ((r + 1) & 255)], v, acc1);
      } else if (MODE == 1) {
        acc0 = __fma_rn((double)xf[lane * 257 + r], v, acc0);
        acc1 = __fma_rn((double)xf[lane * 257 + ((r + 1) & 255)], v, acc1);
      } else {
        const float2 f = *reinterpret_cast<const float2 *>(&xf[(2 * lane) * 257 + 2 * (r >> 1)]);
        acc0 = __fma_rn((double)f.x, v, acc0);
        acc1 = __fma_rn((double)f.y, v, acc1);
      }
    }
  }
  out[blockIdx.x * 1024 + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *src;
  double *out;
  cudaMalloc(&src, 4096 * 4);
  cudaMemset(src, 0, 4096 * 4);
  cudaMalloc(&out, (size_t)sms * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      const int sm = 32 * 257 * 8;
      cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      if (mode == 0) k<0><<<sms, 1024, sm>>>(src, out, iters);
      if (mode == 1) k<1><<<sms, 1024, sm>>>(src, out, iters);
      if (mode == 2) k<2><<<sms, 1024, sm>>>(src, out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fmas = (double)sms * 1024 * iters * 32 * 2;
      if (rep) printf("mode %d: %.1f GFMA/s  %.1f FMA/clk/SM (at 1.965 GHz)\n", mode, fmas / ms / 1e6,
                      fmas / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  return 0;
}
