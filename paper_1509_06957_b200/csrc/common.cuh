// Shared helpers for libmrpt_cuda.so (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/mrpt_cuda.h"

namespace mrpt {

// Thread-local error text behind mrpt_last_error().
void set_error(const char *fmt, ...);
void clear_error();

inline int32_t fail(int32_t code, const char *what) {
  set_error("%s", what);
  return code;
}

// Kernels this library has launched (all devices, all threads): the bench's
// gpu_launches evidence, read through mrpt_launch_count().
void count_launch();

// Optional CUDA-event bracket around the dominant kernel of a call (the
// fused tcgen05 filter), read by mrpt_kernel_timer_read: the bench's live
// per-launch duration for the roofline.  No-ops unless mrpt_kernel_timer(1).
void ktimer_begin(cudaStream_t s, cudaEvent_t *e0);
void ktimer_end(cudaStream_t s, cudaEvent_t e0);

// Report the launch status of the kernels just enqueued.
inline int32_t launch_status(const char *where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", where, cudaGetErrorString(e));
    return MRPT_ECUDA;
  }
  return MRPT_OK;
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Small stream-ordered scratch (fallback lists) comes from the device's
// default memory pool; keep freed blocks cached in the pool instead of
// returning them to the driver at every synchronisation, so per-call scratch
// never costs a host-side remap.  Idempotent, per device.
inline void keep_pool_warm() {
  static int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = 64ull << 20;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done_dev = dev;
}

inline int num_sms() {
  static int sms = 0;  // benign race: every thread computes the same value
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms = v > 0 ? v : 148;
  }
  return sms;
}

// Order-preserving float -> uint32 key (a < b  <=>  key(a) < key(b) for
// non-NaN floats).  -0.0 is folded onto +0.0 so that equal values share a
// key, matching float `<=` in median_split (trees.py:48-50).
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t b = __float_as_uint(f);
  if (b == 0x80000000u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(b);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__host__ __device__ __forceinline__ T ceil_div(T a, T b) {
  return (a + b - 1) / b;
}

}  // namespace mrpt
