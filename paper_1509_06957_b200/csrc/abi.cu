// Error plumbing and small validation kernels of libmrpt_cuda.so.
#include <stdarg.h>

#include <atomic>

#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"

namespace mrpt {

static thread_local char g_err[512] = {0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void clear_error() { g_err[0] = 0; }

static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// core.py:63 -- np.isfinite(arr).all()
__global__ void k_check_finite(const float *__restrict__ X, int64_t count, int32_t *bad) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool ok = true;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < count; i += stride) ok &= isfinite(X[i]);
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) *bad = 1;
}

// Leaf audit for foreign (hand-built / loaded) indexes: one thread per
// stored id; its leaf is found by binary search over the tree's offsets.
__global__ void k_audit_leaves(const int32_t *__restrict__ leaf_indices,
                               const int64_t *__restrict__ leaf_offsets, int64_t n, int32_t T,
                               int32_t nleaves, int32_t *flags) {
  int64_t total = (int64_t)T * n;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += stride) {
    int64_t t = g / n, pos = g - t * n;
    int32_t id = leaf_indices[g];
    if (id < 0 || (int64_t)id >= n) flags[1] = 1;
    if (pos + 1 < n) {
      // is pos+1 the start of a new leaf?  offsets are non-decreasing.
      const int64_t *o = leaf_offsets + t * (int64_t)(nleaves + 1);
      int lo = 0, hi = nleaves;  // find any j with o[j] == pos+1
      bool boundary = false;
      while (lo <= hi) {
        int mid = (lo + hi) >> 1;
        int64_t v = o[mid];
        if (v == pos + 1) { boundary = true; break; }
        if (v < pos + 1) lo = mid + 1; else hi = mid - 1;
      }
      if (!boundary && leaf_indices[g + 1] <= id) flags[0] = 1;
    }
  }
}

}  // namespace mrpt

using namespace mrpt;

extern "C" const char *mrpt_last_error(void) { return g_err; }

extern "C" int32_t mrpt_abi_version(void) { return 101; }

extern "C" int64_t mrpt_launch_count(void) { return mrpt::g_launches.load(std::memory_order_relaxed); }

// ---- event timer around the dominant kernel (bench roofline evidence) ----
namespace mrpt {
static std::mutex g_kt_mu;
static bool g_kt_on = false;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_kt;

void ktimer_begin(cudaStream_t s, cudaEvent_t *e0) {
  *e0 = nullptr;
  std::lock_guard<std::mutex> lock(g_kt_mu);
  if (!g_kt_on) return;
  if (cudaEventCreate(e0) != cudaSuccess) {
    *e0 = nullptr;
    return;
  }
  cudaEventRecord(*e0, s);
}

void ktimer_end(cudaStream_t s, cudaEvent_t e0) {
  if (!e0) return;
  cudaEvent_t e1;
  if (cudaEventCreate(&e1) != cudaSuccess) return;
  cudaEventRecord(e1, s);
  std::lock_guard<std::mutex> lock(g_kt_mu);
  g_kt.emplace_back(e0, e1);
}
}  // namespace mrpt

extern "C" int32_t mrpt_kernel_timer(int32_t enable) {
  std::lock_guard<std::mutex> lock(mrpt::g_kt_mu);
  mrpt::g_kt_on = enable != 0;
  for (auto &p : mrpt::g_kt) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  mrpt::g_kt.clear();
  return MRPT_OK;
}

extern "C" int32_t mrpt_kernel_timer_read(double *ms, int64_t *launches) {
  std::lock_guard<std::mutex> lock(mrpt::g_kt_mu);
  double tot = 0.0;
  for (auto &p : mrpt::g_kt) {
    float x = 0.f;
    if (cudaEventSynchronize(p.second) != cudaSuccess || cudaEventElapsedTime(&x, p.first, p.second) != cudaSuccess)
      return mrpt::fail(MRPT_ECUDA, "mrpt_kernel_timer_read: event");
    tot += x;
  }
  if (ms) *ms = tot;
  if (launches) *launches = (int64_t)mrpt::g_kt.size();
  return MRPT_OK;
}

extern "C" int32_t mrpt_check_finite(const float *X, int64_t count, int32_t *bad, void *stream) {
  clear_error();
  if (count < 0 || !bad) return fail(MRPT_EPARAM, "mrpt_check_finite: bad arguments");
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(bad, 0, sizeof(int32_t), s);
  if (count == 0) return launch_status("mrpt_check_finite");
  int64_t blocks = ceil_div<int64_t>(count, 256 * 8);
  int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  (count_launch(), k_check_finite<<<grid, 256, 0, s>>>(X, count, bad));
  return launch_status("mrpt_check_finite");
}

extern "C" int32_t mrpt_audit_leaves(const int32_t *leaf_indices, const int64_t *leaf_offsets,
                                     int64_t n, int32_t T, int32_t depth, int32_t *flags,
                                     void *stream) {
  clear_error();
  if (n < 1 || T < 1 || depth < 0 || depth > 30 || !flags)
    return fail(MRPT_EPARAM, "mrpt_audit_leaves: bad arguments");
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(flags, 0, 2 * sizeof(int32_t), s);
  int64_t total = (int64_t)T * n;
  int64_t blocks = ceil_div<int64_t>(total, 256);
  int grid = (int)(blocks < (int64_t)num_sms() * 32 ? blocks : (int64_t)num_sms() * 32);
  (count_launch(), k_audit_leaves<<<grid, 256, 0, s>>>(leaf_indices, leaf_offsets, n, T, 1 << depth, flags));
  return launch_status("mrpt_audit_leaves");
}
