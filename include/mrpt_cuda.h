/*
 * mrpt_cuda.h — C ABI of libmrpt_cuda.so, the sm_100a implementation of the
 * MRPT (arXiv 1509.06957) batched index-build and k-NN query hot path.
 *
 * The reference plugs its hot kernels in at `mrpt._kernels`
 * (pkg/src/mrpt/_kernels/__init__.py:71-88), one call per tree / per query,
 * implemented by pkg/src/mrpt/_kernels/_cy.pyx:18-106.  Each entry point below
 * replaces one of those kernels (or the numpy code around them) for a whole
 * BATCH of trees or queries; the replaced interface is cited per function.
 *
 * Conventions (all functions):
 *   - return an int32 status: MRPT_OK (0) or a negative MRPT_E* code; the
 *     message for the calling thread is available from mrpt_last_error();
 *   - every pointer argument is caller-owned DEVICE memory unless the comment
 *     says "host"; the library never allocates or frees caller memory (its
 *     own scratch: small stream-ordered pool allocations);
 *   - work is enqueued on `stream` (a cudaStream_t, NULL = legacy default) and
 *     the call returns without synchronising; host-side argument validation
 *     fails fast before anything is enqueued;
 *   - calls are reentrant and keep no global mutable state besides
 *     measurement counters (launch count, fallback statistics, the optional
 *     kernel timer); every kernel is this library's own (no library GEMM);
 *   - leaf ids of tree t live at leaf_indices[t*n + off] (64-bit addressing,
 *     T*n reaches 1e10 at the largest configuration).
 * Status codes map onto the reference exception taxonomy
 * (pkg/src/mrpt/exceptions.py:1-29) in the Python layer.
 */
#ifndef MRPT_CUDA_H
#define MRPT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MRPT_OK = 0,
  MRPT_EPARAM = -1,     /* -> ParameterError  */
  MRPT_ESHAPE = -2,     /* -> ShapeError      */
  MRPT_EINTEGRITY = -3, /* -> IntegrityError  */
  MRPT_EWORKSPACE = -4, /* workspace too small */
  MRPT_ECUDA = -10,     /* CUDA launch / runtime failure */
  MRPT_ENCCL = -11
};

/* Thread-local text of the last failing call on this thread ("" if none). */
const char *mrpt_last_error(void);
/* ABI version (major*100 + minor). */
int32_t mrpt_abi_version(void);
/* Kernels this library has launched so far (process-wide; library GEMMs of
 * cuBLASLt are not counted). */
int64_t mrpt_launch_count(void);

/* ------------------------------------------------------------------ K1 --
 * Sparse projection with float64 accumulation in stored CSC order and one
 * final rounding to float32; bit-identical to _cy.project
 * (pkg/src/mrpt/_kernels/_cy.pyx:18-34) and to core.project_dataset /
 * project_query (pkg/src/mrpt/core.py:235-260).
 *   out[i*out_row_stride + c*out_col_stride] =
 *       (float) sum_{s in [col_ptr[c], col_ptr[c+1])} (double)X[i*ldx+rows[s]] * (double)vals[s]
 * A batch of trees is one call: concatenate their CSC columns (col_ptr holds
 * global offsets).  Reference layout (m, ncols) row-major: row stride ncols,
 * col stride 1; the build's level-major layout: row stride 1, col stride n. */
int32_t mrpt_project(const float *X, int64_t m, int32_t d, int64_t ldx,
                     const int64_t *col_ptr, const int32_t *rows,
                     const float *vals, int32_t ncols, float *out,
                     int64_t out_row_stride, int64_t out_col_stride,
                     void *stream);

/* ------------------------------------------------------------------ K2 --
 * Heap descent: replaces _cy.route (pkg/src/mrpt/_kernels/_cy.pyx:37-54).
 * proj (nrows, depth) row-major, splits (nrows, n_internal) row-major,
 * out (nrows) int64 leaf ids; p <= split goes left. */
int32_t mrpt_route(const float *proj, int64_t nrows, int32_t depth,
                   const float *splits, int64_t n_internal, int64_t *out,
                   void *stream);

/* Fused query projection + descent over all T trees for nq queries:
 * replaces search._route_all (pkg/src/mrpt/search.py:116-120), i.e. T calls
 * of project_query (core.py:247-260) followed by _cy.route.
 * Q (nq, d) with row stride ldq; CSC of all trees concatenated (tree t owns
 * columns t*depth .. t*depth+depth-1); splits (T, 2^depth-1);
 * leaves (nq, T) int32. */
int32_t mrpt_query_route(const float *Q, int64_t nq, int32_t d, int64_t ldq,
                         const int64_t *col_ptr, const int32_t *rows,
                         const float *vals, const float *splits, int32_t T,
                         int32_t depth, int32_t *leaves, void *stream);

/* ------------------------------------------------------------------ K5 --
 * Level-synchronous construction of Tb trees at once: per level, per node,
 * the lower median (kth = (m+1)/2-1 smallest) of the node's projections by
 * exact radix select, then a stable partition (value <= split goes left);
 * replaces build_tree / median_split (pkg/src/mrpt/trees.py:33-98).
 *   P:            (Tb, depth, n) float32, P[(t*depth+lev)*n + i]
 *   splits:       (Tb, 2^depth-1) float32, heap order
 *   leaf_offsets: (Tb, 2^depth+1) int64
 *   leaf_indices: (Tb, n) int32 (leaf slices ascending point ids)
 * Workspace: query its size first. */
int32_t mrpt_build_workspace_size(int64_t n, int32_t Tb, int32_t depth,
                                  size_t *bytes /* host */);
int32_t mrpt_build_levels(const float *P, int64_t n, int32_t Tb,
                          int32_t depth, float *splits, int64_t *leaf_offsets,
                          int32_t *leaf_indices, void *ws, size_t ws_bytes,
                          void *stream);

/* ------------------------------------------------------------------ K3 --
 * Vote counting for nq queries; replaces VoteAccumulator.accumulate +
 * _cy.vote (pkg/src/mrpt/search.py:75-86, _kernels/_cy.pyx:57-78).
 * Every occurrence of a point id in the query's T leaves counts one vote;
 * cand[q*cap ..] receives the ids with >= v votes (unordered), ncand[q]
 * their number.  leaves_sorted != 0 promises every leaf slice is ascending
 * (true for indexes built by mrpt_build_levels) and enables the id-tiled
 * sweep; max_count bounds any point's vote count (T for strictly ascending
 * slices) and picks the counter width.  cap should bound the candidate count
 * (min(n, sum of the query's leaf sizes / v) is always safe): ncand[q] is the
 * true count, and when it exceeds cap only cap ids were stored -- the caller
 * must treat that as an error (consumers clamp to cap). */
int32_t mrpt_vote(const int32_t *leaf_indices, const int64_t *leaf_offsets,
                  int64_t n, int32_t T, int32_t depth, const int32_t *leaves,
                  int64_t nq, int32_t v, int32_t leaves_sorted,
                  int64_t max_count, const uint16_t *dir, int32_t *cand,
                  int64_t cap, int32_t *ncand, void *stream);

/* mrpt_vote with the candidates returned as bitmaps instead of lists:
 * bits (nq, bstride) uint32, bit i of query q set iff point i has >= v votes
 * (bstride >= ceil(n/32)); ncand[q] = number of set bits.  No ordered
 * compaction: pays when candidate sets are a sizeable share of the points. */
int32_t mrpt_vote_bitmap(const int32_t *leaf_indices, const int64_t *leaf_offsets,
                         int64_t n, int32_t T, int32_t depth, const int32_t *leaves,
                         int64_t nq, int32_t v, int32_t leaves_sorted,
                         int64_t max_count, const uint16_t *dir, uint32_t *bits,
                         int64_t bstride, int32_t *ncand, void *stream);

/* mrpt_vote that also stores each listed candidate's vote count
 * (cand_counts (nq, cap) uint16, saturated at 65535): one K2/K3 pass at the
 * smallest threshold of a sweep serves every larger v through
 * mrpt_filter_counts (vote counts do not depend on v). */
int32_t mrpt_vote_counted(const int32_t *leaf_indices, const int64_t *leaf_offsets,
                          int64_t n, int32_t T, int32_t depth, const int32_t *leaves,
                          int64_t nq, int32_t v, int32_t leaves_sorted,
                          int64_t max_count, const uint16_t *dir, int32_t *cand,
                          uint16_t *cand_counts, int64_t cap, int32_t *ncand,
                          void *stream);

/* Keep, per query and in list order, the candidates of a counted vote whose
 * count is >= v: cand_out (nq, cap_out), ncand_out (nq) (true count). */
int32_t mrpt_filter_counts(const int32_t *cand, const uint16_t *cand_counts,
                           int64_t cap, const int32_t *ncand, int64_t nq, int32_t v,
                           int32_t *cand_out, int64_t cap_out, int32_t *ncand_out,
                           void *stream);

/* Vote geometry: number of id tiles the vote sweeps for this index shape and
 * the uint16 entries of its tile directory (0 when one tile suffices).
 * The directory (optional `dir` of mrpt_vote, built once per index by
 * mrpt_vote_build_dir from ascending leaf slices of at most 65535 ids) holds,
 * per (tree, leaf), where the slice's part in each id tile starts, so the
 * multi-tile vote streams every slice without cursor walks. */
int32_t mrpt_vote_plan(int64_t n, int32_t T, int32_t depth, int64_t max_count,
                       int32_t *ntiles /* host */, int64_t *dir_entries /* host */);
int32_t mrpt_vote_build_dir(const int32_t *leaf_indices,
                            const int64_t *leaf_offsets, int64_t n, int32_t T,
                            int32_t depth, int64_t max_count, uint16_t *dir,
                            void *stream);

/* Dense per-point vote counts for one query (VoteAccumulator.counts(),
 * pkg/src/mrpt/search.py:68-73): counts (n) int32 is zeroed then filled. */
int32_t mrpt_vote_counts(const int32_t *leaf_indices,
                         const int64_t *leaf_offsets, int64_t n, int32_t T,
                         int32_t depth, const int32_t *leaves, int32_t *counts,
                         void *stream);

/* Ordered compaction: out receives, ascending, the i with counts[i] >= v;
 * *nout (device) their number.  (np.flatnonzero(counts >= v), _py.py:93) */
int32_t mrpt_select_ge(const int32_t *counts, int64_t n, int32_t v,
                       int32_t *out, int64_t *nout, void *stream);

/* ------------------------------------------------------------------ K4 --
 * Squared distances in float64 with the reference's sequential summation
 * order: replaces _cy.scan (pkg/src/mrpt/_kernels/_cy.pyx:81-97).
 * out[j] = sum_c ((double)X[cand[j]*ldx+c] - (double)q[c])^2, c ascending. */
int32_t mrpt_scan(const float *X, int64_t n, int32_t d, int64_t ldx,
                  const int64_t *cand, int64_t m, const float *q,
                  double *out, void *stream);

/* Exact k-NN over per-query candidate lists: replaces exact_knn_in_set's
 * scan + lexsort + sqrt (pkg/src/mrpt/search.py:146-172) for nq queries.
 * cand (nq, cap) int32 ids (unique per query), ncand (nq) int32, or
 * cand == NULL to scan all n points (brute force, evaluation.py:28-47).
 * Output per query, ascending (d^2, id): ids (nq, k) int64 padded with -1,
 * dists (nq, k) float64 = sqrt(d^2) padded with +inf. */
int32_t mrpt_scan_topk(const float *X, int64_t n, int32_t d, int64_t ldx,
                       const float *Q, int64_t nq, int64_t ldq,
                       const int32_t *cand, int64_t cap, const int32_t *ncand,
                       int32_t k, int64_t *ids, double *dists, void *stream);

/* fp16 shadow rows for the filter pass of mrpt_scan_topk_fp16: Xh (n, ldh)
 * halves (ldh % 8 == 0, zero padded), radius[i] >= ||X_i - fp16(X_i)||_2.
 * *bad (device int32) = 1 if some |x| exceeds the fp16 range. */
int32_t mrpt_quantize_fp16(const float *X, int64_t n, int32_t d, int64_t ldx,
                           void *Xh, int64_t ldh, float *radius, int32_t *bad,
                           void *stream);

/* mrpt_scan_topk with its float32 filter pass reading the fp16 shadow rows:
 * per candidate the filter bounds the reference distance E within
 * [(sqrt(D)-r)^2, (sqrt(D)+r)^2] (D the filter's value, r the row radius,
 * plus float32 rounding terms) and keeps it while that lower bound is <= the
 * running k-th smallest upper bound; survivors are reranked from X in float64
 * exactly as mrpt_scan_topk, so results are identical.  Falls back to
 * mrpt_scan_topk when Xh is NULL or the shape is unsupported. */
int32_t mrpt_scan_topk_fp16(const float *X, int64_t n, int32_t d, int64_t ldx,
                            const void *Xh, int64_t ldh, const float *radius,
                            const float *Q, int64_t nq, int64_t ldq,
                            const int32_t *cand, int64_t cap,
                            const int32_t *ncand, int32_t k, int64_t *ids,
                            double *dists, void *stream);

/* u8 shadow rows for non-negative data: Xq (n, ldq) bytes (ldq % 16 == 0,
 * <= 1024), X_i = rint(x_i / scale[i]) (scale = 1 when the whole dataset is
 * integer-valued in [0, 255], which makes the shadow exact), norm[i] =
 * sum X_i^2, radius[i] >= ||x_i - scale[i] X_i||_2.  flags (device, 2 int32):
 * [0] = 1 if some x < 0 (nothing written), [1] = 1 if not integer-valued.
 * Synchronises the stream once (index preparation, not the query path). */
int32_t mrpt_quantize_u8(const float *X, int64_t n, int32_t d, int64_t ldx,
                         void *Xq, int64_t ldq, float *scale, int32_t *norm,
                         float *radius, int32_t *flags, void *stream);

/* mrpt_scan_topk whose filter pass scores candidates on the u8 shadow with
 * exact integer dot products (dp4a): D = s_x^2 N_x + s_q^2 N_q - 2 s_x s_q X.Q
 * in float64, sqrt(E) within r_x + r_q of sqrt(D); kept while the lower bound
 * is <= the running k-th smallest upper bound, then the same float64 rerank
 * from X -- identical results.  Falls back to mrpt_scan_topk for unsupported
 * shapes. */
int32_t mrpt_scan_topk_u8(const float *X, int64_t n, int32_t d, int64_t ldx,
                          const void *Xq, int64_t ldq, const float *scale,
                          const int32_t *norm, const float *radius,
                          const float *Q, int64_t nq, int64_t ldqq,
                          const int32_t *cand, int64_t cap,
                          const int32_t *ncand, int32_t k, int64_t *ids,
                          double *dists, void *stream);

/* Tensor-core operands of the u8 shadow for mrpt_scan_topk_u8tc_bits:
 * Xs = Xq ^ 0x80 (s8, row stride ldq, room for round_up(n, 16) rows -- the
 * rows past n are zeroed here) and info (n x 16 bytes, 16-byte aligned): per
 * row {scale (f32), norm (s32), radius (f32), sum of the u8 entries (s32)}. */
int32_t mrpt_u8_gemm_rows(const void *Xq, int64_t n, int64_t ldq, const float *scale,
                          const int32_t *norm, const float *radius, void *Xs,
                          void *info, void *stream);

/* The u8 filter over candidate bitmaps fused onto the tcgen05 tensor cores
 * (replaces the _cy.scan + lexsort step of exact_knn_in_set,
 * pkg/src/mrpt/search.py:146-172, like every K4 route): a persistent kernel
 * streams the s8 shadow rows Xs (mrpt_u8_gemm_rows) through TMA into
 * shared memory, forms each 128-query x 256-row block of dot products with
 * tcgen05.mma.kind::i8 into TMEM and bounds every candidate straight out of
 * TMEM (no dot-product matrix in HBM); survivors get the exact float64
 * re-rank.  cbits: (nq, bstride) candidate bitmaps from mrpt_vote_bitmap;
 * wait_event (a cudaEvent_t, or NULL): the filter waits for it after the
 * query quantisation, so the bitmaps may come from another stream.
 * 128 <= ldq <= 1024, k <= 16; bstride a multiple of 4 words (the bitmaps are
 * TMA-staged per row tile).  workspace: 256-byte aligned, sized by
 * mrpt_scan_topk_u8tc_workspace_size (smaller workspaces run smaller query
 * chunks). */
int32_t mrpt_scan_topk_u8tc_workspace_size(int64_t n, int64_t ldq, int64_t nq,
                                           int64_t *bytes /* host */);
int32_t mrpt_scan_topk_u8tc_bits(const float *X, int64_t n, int32_t d, int64_t ldx,
                                 const void *Xs, int64_t ldq, const void *info,
                                 const float *Q, int64_t nq, int64_t ldqq,
                                 const uint32_t *cbits, int64_t bstride, int32_t k,
                                 int64_t *ids, double *dists, void *workspace,
                                 int64_t ws_bytes, void *wait_event, void *stream);

/* Measurement support: how often the exact fallback ran.  out (host, 8
 * int64): for the routes fp32 filter, fp16 filter, u8 filter and tcgen05
 * filter in that order, [queries handed to the route, queries that took the
 * exact tiled fallback].  Synchronises the device; reset != 0 clears. */
int32_t mrpt_fallback_stats(int64_t *out /* host */, int32_t reset);

/* Measurement support (not part of the reference interface): when enabled,
 * the fused filter launch of mrpt_scan_topk_u8tc_bits is bracketed by CUDA
 * events on its stream; _read synchronises them and returns the summed
 * milliseconds and the number of bracketed launches.  Enabling (or
 * disabling) clears the record. */
int32_t mrpt_kernel_timer(int32_t enable);
int32_t mrpt_kernel_timer_read(double *ms /* host */, int64_t *launches /* host */);

/* Sorted de-duplication of arbitrary candidate ids (np.unique,
 * search.py:157) through an n-bit bitmap.  ids outside [0, n) set
 * *bad (device int32) to 1 (IntegrityError, search.py:158-162).
 * bitmap: ceil(n/32) uint32 of workspace. */
int32_t mrpt_unique_ids(const int64_t *cand, int64_t m, int64_t n,
                        uint32_t *bitmap, int32_t *out, int64_t *nout,
                        int32_t *bad, void *stream);

/* ------------------------------------------------------------------ K6 --
 * 64-bit FNV-1a over nbytes raw bytes (Dataset.checksum / _cy.fnv1a64,
 * pkg/src/mrpt/core.py:77-82, _kernels/_cy.pyx:100-106), computed in
 * parallel: per chunk a 256-entry table of (low-byte out, affine offset),
 * composed in order.  *out (device uint64). */
int32_t mrpt_fnv1a64_workspace_size(int64_t nbytes, size_t *bytes /* host */);
int32_t mrpt_fnv1a64(const uint8_t *buf, int64_t nbytes, uint64_t *out,
                     void *ws, size_t ws_bytes, void *stream);

/* Streamed tiled vote (configs with many id tiles, T <= 1024): the same
 * counts and the same candidate set as mrpt_vote (replaces
 * VoteAccumulator.accumulate / _cy.vote, pkg/src/mrpt/search.py:75-86,
 * _kernels/_cy.pyx:57-78) over a per-index layout built once:
 * every ascending leaf slice is split into its parts per id tile, each part
 * padded to a multiple of 7 entries, each entry pre-decoded into its
 * tile-local counter address (16-bit counter word, 2-bit lane), 7 entries
 * per 16-byte quad: u16[0..6] = words, u16[7] = the 7 lanes (2 bits each);
 * padding entries address the 32 spare words after the counters.
 *   _plan:   ntiles and the entries of qdir (T * 2^depth * (ntiles + 1) u16);
 *            fails with MRPT_EPARAM where the layout does not apply
 *            (T > 1024 or more than 1024 id tiles).
 *   _layout: qdir (quad offset of each tile's part within its leaf's padded
 *            slice), qbase (T * 2^depth int32: the slice's first quad within
 *            its tree row) and tree_quads (T int64: quads per tree row).
 *   _fill:   qs (T * tstride quads of 4 uint32), tstride >= max tree_quads,
 *            32 * tstride < 2^31.
 *   mrpt_vote_stream: candidate lists like mrpt_vote (cand (nq, cap), ncand
 *            may exceed cap; ids within one id tile in no particular order).
 * Leaf slices must be ascending (as mrpt_build_levels writes them). */
int32_t mrpt_vote_stream_plan(int64_t n, int32_t T, int32_t depth, int64_t max_count,
                              int32_t *ntiles /* host */, int64_t *dir_entries /* host */);
int32_t mrpt_vote_stream_layout(const int32_t *leaf_indices, const int64_t *leaf_offsets,
                                int64_t n, int32_t T, int32_t depth, int64_t max_count,
                                uint16_t *qdir, int32_t *qbase, int64_t *tree_quads,
                                void *stream);
int32_t mrpt_vote_stream_fill(const int32_t *leaf_indices, const int64_t *leaf_offsets,
                              int64_t n, int32_t T, int32_t depth, int64_t max_count,
                              const uint16_t *qdir, const int32_t *qbase, int64_t tstride,
                              uint32_t *qs, void *stream);
int32_t mrpt_vote_stream(const uint32_t *qs, int64_t tstride, const uint16_t *qdir,
                         const int32_t *qbase, int64_t n, int32_t T, int32_t depth,
                         int64_t max_count, const int32_t *leaves, int64_t nq, int32_t v,
                         int32_t *cand, int64_t cap, int32_t *ncand, void *stream);

/* Paired streamed vote (same counts and candidate sets as mrpt_vote_stream;
 * replaces the same reference code, _cy.pyx:57-78 via search.py:130-172).
 * The id tiles are taken two at a time: per leaf slice, super-piece j holds
 * 32-byte pairs {quad k of tile 2j's piece, quad k of tile 2j+1's piece},
 * so one load brings a quad of both tiles; the kernel bumps the first now
 * and parks the second in tensor memory for the next tile.
 *   _plan:   ntiles, pos_entries = T*2^depth*(ntiles+1) (u16 scratch of
 *            _layout and _fill), dir_entries = T*2^depth*(ceil(ntiles/2)+1).
 *   _layout: pos (scratch), pdir (pair offset of each super-piece within its
 *            slice), pbase (T*2^depth int32: slice's first pair within its
 *            tree row), tree_pairs (T int64: pairs per tree row).
 *   _fill:   ps (T * pstride pairs of 8 uint32), pstride >= max tree_pairs,
 *            64 * pstride < 2^31.
 *   mrpt_vote_pair: candidate lists like mrpt_vote_stream.
 * Counter width: where max_count > 255 and 8-bit counters need fewer pairs
 * of id tiles than 10/16-bit ones (large n), the counters are 8 bits wide
 * and SATURATE: they start at 128 - v (so the increment lifting a count to v
 * is the one that reads 127) and a counter reaching 192 is pulled back by 64
 * by the increment that read 191, so it never returns to 127 (v <= 128
 * required, see mrpt_vote_pair_max_votes; larger v is served by mrpt_vote)
 * and each id reaching v votes is still listed exactly once
 * (_cy.pyx:75-77).  An
 * increment that would wrap a counter (it read 255) flags its query, which
 * the same launch then redoes with check-before-increment bumps that cannot
 * wrap -- results are exact either way; mrpt_vote_stats counts the redos.
 * MRPT_VOTE_SAT=0 (environment, read per call; set before the layout is
 * built) keeps 10/16-bit counters instead. */
int32_t mrpt_vote_pair_max_votes(int64_t n, int32_t T, int64_t max_count,
                                 int32_t *max_votes /* host */);
/* out (host, 2 int64): queries voted with saturating counters, queries
 * redone exactly after a counter wrapped.  Synchronises; reset != 0 clears. */
int32_t mrpt_vote_stats(int64_t *out /* host */, int32_t reset);
int32_t mrpt_vote_pair_plan(int64_t n, int32_t T, int32_t depth, int64_t max_count,
                            int32_t *ntiles /* host */, int64_t *pos_entries /* host */,
                            int64_t *dir_entries /* host */);
int32_t mrpt_vote_pair_layout(const int32_t *leaf_indices, const int64_t *leaf_offsets,
                              int64_t n, int32_t T, int32_t depth, int64_t max_count,
                              uint16_t *pos, uint16_t *pdir, int32_t *pbase, int64_t *tree_pairs,
                              void *stream);
int32_t mrpt_vote_pair_fill(const int32_t *leaf_indices, const int64_t *leaf_offsets,
                            int64_t n, int32_t T, int32_t depth, int64_t max_count,
                            const uint16_t *pos, const uint16_t *pdir, const int32_t *pbase,
                            int64_t pstride, uint32_t *ps, void *stream);
int32_t mrpt_vote_pair(const uint32_t *ps, int64_t pstride, const uint16_t *pdir,
                       const int32_t *pbase, int64_t n, int32_t T, int32_t depth,
                       int64_t max_count, const int32_t *leaves, int64_t nq, int32_t v,
                       int32_t *cand, int64_t cap, int32_t *ncand, void *stream);

/* Query ordering for a batch (no reference counterpart: the reference
 * answers one query per call, search.py:175-184).  order (nq int32) lists
 * the queries grouped by their leaf in tree 0 (leaves: (nq, T) int32 from
 * mrpt_query_route); ws: 2^depth int32 scratch.  Processing the batch in
 * this order lets concurrent CTAs share leaf slices and candidate rows in
 * L2; answers do not depend on it. */
int32_t mrpt_query_order(const int32_t *leaves, int64_t nq, int32_t T, int32_t depth,
                         int32_t *order, int32_t *ws, void *stream);

/* Row permutation of a (rows, words) array of 4-byte words (leading
 * dimensions in words): scatter == 0 gathers dst[i] = src[idx[i]],
 * scatter != 0 scatters dst[idx[i]] = src[i]. */
int32_t mrpt_permute_rows(const void *src, int64_t src_ld, const int32_t *idx, int64_t rows,
                          int64_t words, void *dst, int64_t dst_ld, int32_t scatter,
                          void *stream);

/* ------------------------------------------------------------------ f3 --
 * Exact brute-force k-NN (ground truth): replaces evaluation.brute_force_knn
 * and compute_ground_truth (pkg/src/mrpt/evaluation.py:28-81).  Q (nq, ldq)
 * float64 query rows (the reference converts the query to float64,
 * evaluation.py:37); d2 per (query, row) summed in numpy's pairwise order
 * (the reference's ((X - q)**2).sum(axis=1)), ordered by (d2, id) like
 * np.lexsort((ids, d2)).  Output (nq, min(k, n)) row-major: ids int64,
 * dists float64 = sqrt(d2).  d <= 4096.  Workspace from
 * mrpt_brute_force_workspace_size (device bytes). */
int32_t mrpt_brute_force_workspace_size(int64_t n, int32_t d, int64_t nq, int32_t k,
                                        int64_t *bytes /* host */);
int32_t mrpt_brute_force_knn(const float *X, int64_t n, int32_t d, int64_t ldx,
                             const double *Q, int64_t nq, int64_t ldq, int32_t k,
                             int64_t *ids, double *dists, void *ws, int64_t ws_bytes,
                             void *stream);

/* ------------------------------------------------------------- helpers --
 * Dataset validation (core.py:63): *bad (device int32) = 1 if any element of
 * X (m*d float32) is not finite. */
int32_t mrpt_check_finite(const float *X, int64_t count, int32_t *bad,
                          void *stream);

/* Leaf-slice audit for indexes not built by mrpt_build_levels (hand-built or
 * loaded): flags[0] = 1 if some slice is not strictly ascending, flags[1] =
 * 1 if some id is outside [0, n).  flags: 2 int32, zeroed by the call. */
int32_t mrpt_audit_leaves(const int32_t *leaf_indices,
                          const int64_t *leaf_offsets, int64_t n, int32_t T,
                          int32_t depth, int32_t *flags, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MRPT_CUDA_H */
