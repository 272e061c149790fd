# Cython declarations of include/mrpt_cuda.h for a reference-side build
# (cimport from a .pyx next to pkg/src/mrpt/_kernels/_cy.pyx).  Generated from
# the header by hand; tests/test_abi.py checks every parameter list below
# against the header.
from libc.stdint cimport int32_t, int64_t, uint8_t, uint16_t, uint32_t, uint64_t

cdef extern from "mrpt_cuda.h":
    int32_t mrpt_project(const float* X, int64_t m, int32_t d, int64_t ldx,
                         const int64_t* col_ptr, const int32_t* rows, const float* vals,
                         int32_t ncols, float* out, int64_t out_row_stride,
                         int64_t out_col_stride, void* stream)
    int32_t mrpt_query_route(const float* Q, int64_t nq, int32_t d, int64_t ldq,
                             const int64_t* col_ptr, const int32_t* rows, const float* vals,
                             const float* splits, int32_t T, int32_t depth, int32_t* leaves,
                             void* stream)
    int32_t mrpt_vote(const int32_t* leaf_indices, const int64_t* leaf_offsets, int64_t n,
                      int32_t T, int32_t depth, const int32_t* leaves, int64_t nq, int32_t v,
                      int32_t leaves_sorted, int64_t max_count, const uint16_t* dir,
                      int32_t* cand, int64_t cap, int32_t* ncand, void* stream)
    int32_t mrpt_scan_topk(const float* X, int64_t n, int32_t d, int64_t ldx, const float* Q,
                           int64_t nq, int64_t ldq, const int32_t* cand, int64_t cap,
                           const int32_t* ncand, int32_t k, int64_t* ids, double* dists,
                           void* stream)
    int32_t mrpt_fnv1a64(const uint8_t* buf, int64_t nbytes, uint64_t* out, void* ws,
                         size_t ws_bytes, void* stream)
    const char* mrpt_last_error()
