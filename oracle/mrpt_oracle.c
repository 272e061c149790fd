/*
 * mrpt_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the MRPT reference hot path
 * (arXiv 1509.06957, /root/reference/pkg), used as the parity checker for the
 * CUDA implementation.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product never does.
 *
 * Built with -ffp-contract=off (as the reference, pkg/setup.py:37-39) so the
 * float64 multiply and add stay separate operations.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* _cy.project (pkg/src/mrpt/_kernels/_cy.pyx:18-34): out (m, ncols) row-major,
 * float64 accumulation in stored order from +0.0, one rounding to float32. */
void oracle_project(const float *X, int64_t m, int32_t d, const int64_t *col_ptr,
                    const int32_t *rows, const float *vals, int32_t ncols, float *out) {
  for (int64_t i = 0; i < m; ++i) {
    const float *x = X + i * (int64_t)d;
    for (int32_t j = 0; j < ncols; ++j) {
      double acc = 0.0;
      for (int64_t s = col_ptr[j]; s < col_ptr[j + 1]; ++s) {
        double prod = (double)x[rows[s]] * (double)vals[s];
        acc = acc + prod;
      }
      out[i * ncols + j] = (float)acc;
    }
  }
}

/* _cy.route (_cy.pyx:37-54): left when p <= split. */
void oracle_route(const float *proj, int64_t nrows, int32_t depth, const float *splits,
                  int64_t n_internal, int64_t *out) {
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t node = 0;
    for (int32_t lev = 0; lev < depth; ++lev) {
      if (proj[r * depth + lev] <= splits[r * n_internal + node])
        node = 2 * node + 1;
      else
        node = 2 * node + 2;
    }
    out[r] = node - n_internal;
  }
}

static int cmp_float(const void *a, const void *b) {
  float x = *(const float *)a, y = *(const float *)b;
  return (x > y) - (x < y);
}

/* build_tree (pkg/src/mrpt/trees.py:54-98) with median_split (33-51):
 * per node the kth = (m+1)/2-1 smallest value (here by sorting a copy), the
 * left child takes values <= split in their current order, the right child
 * the rest.  m == 0: split 0.0, nothing left; m == 1: split = its value.
 * P is (n, ldp) row-major, column `level` used at each level. */
void oracle_build_tree(const float *P, int64_t n, int32_t ldp, int32_t depth, float *splits,
                       int64_t *bounds_out, int32_t *order) {
  int64_t nleaf = (int64_t)1 << depth;
  int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (nleaf + 1));
  int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (nleaf + 1));
  float *vals = (float *)malloc(sizeof(float) * (n > 0 ? n : 1));
  float *sorted = (float *)malloc(sizeof(float) * (n > 0 ? n : 1));
  int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) order[i] = (int32_t)i;
  for (int64_t i = 0; i < nleaf - 1; ++i) splits[i] = 0.0f;
  bounds[0] = 0;
  bounds[1] = n;
  int64_t pos = 0;
  for (int32_t level = 0; level < depth; ++level) {
    int64_t nnodes = (int64_t)1 << level;
    next[0] = 0;
    for (int64_t node = 0; node < nnodes; ++node) {
      int64_t start = bounds[node], stop = bounds[node + 1], m = stop - start;
      int64_t n_left;
      if (m == 0) {
        n_left = 0;
      } else if (m == 1) {
        splits[pos] = P[(int64_t)order[start] * ldp + level];
        n_left = 1;
      } else {
        for (int64_t i = 0; i < m; ++i) {
          vals[i] = P[(int64_t)order[start + i] * ldp + level];
          sorted[i] = vals[i];
        }
        qsort(sorted, (size_t)m, sizeof(float), cmp_float);
        float split = sorted[(m + 1) / 2 - 1];
        int64_t l = 0, r = 0;
        for (int64_t i = 0; i < m; ++i)
          if (vals[i] <= split) tmp[l++] = order[start + i];
        n_left = l;
        for (int64_t i = 0; i < m; ++i)
          if (!(vals[i] <= split)) tmp[n_left + r++] = order[start + i];
        memcpy(order + start, tmp, sizeof(int32_t) * (size_t)m);
        splits[pos] = split;
      }
      next[2 * node + 1] = start + n_left;
      next[2 * node + 2] = stop;
      ++pos;
    }
    int64_t *sw = bounds;
    bounds = next;
    next = sw;
  }
  memcpy(bounds_out, bounds, sizeof(int64_t) * (nleaf + 1));
  free(bounds);
  free(next);
  free(vals);
  free(sorted);
  free(tmp);
}

/* Dense vote counts (VoteAccumulator.counts(), search.py:68-73 with
 * _cy.vote's per-occurrence increments, _cy.pyx:71-78). */
void oracle_vote_counts(const int32_t *leaf_indices, const int64_t *leaf_offsets, int64_t n,
                        int32_t T, int64_t nleaf, const int64_t *leaves, int32_t *counts) {
  memset(counts, 0, sizeof(int32_t) * (size_t)n);
  for (int32_t t = 0; t < T; ++t) {
    const int64_t *o = leaf_offsets + (int64_t)t * (nleaf + 1);
    for (int64_t p = o[leaves[t]]; p < o[leaves[t] + 1]; ++p) counts[leaf_indices[t * n + p]]++;
  }
}

/* _cy.scan (_cy.pyx:81-97): float64 squared distances, coordinates in order. */
void oracle_scan(const float *X, int32_t d, const int64_t *cand, int64_t m, const float *q,
                 double *out) {
  for (int64_t i = 0; i < m; ++i) {
    const float *x = X + cand[i] * (int64_t)d;
    double acc = 0.0;
    for (int32_t c = 0; c < d; ++c) {
      double diff = (double)x[c] - (double)q[c];
      double sq = diff * diff;
      acc = acc + sq;
    }
    out[i] = acc;
  }
}

/* _cy.fnv1a64 (_cy.pyx:100-106). */
uint64_t oracle_fnv1a64(const uint8_t *buf, int64_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (int64_t i = 0; i < n; ++i) h = (h ^ (uint64_t)buf[i]) * 0x100000001B3ull;
  return h;
}
