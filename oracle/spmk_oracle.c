/* TEST INFRASTRUCTURE ONLY — CPU oracle (checker) for the spmk hot path.
 * See spmk_oracle.h for the contract and how it is pinned against the
 * reference.  Compiled with -ffp-contract=off (reference: no -march). */
#include "spmk_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define PAD_ROW INT64_MAX /* reduction.hpp:15 kPadRow */

/* ---------------------------------------------------------------- rng */
/* rmat.hpp:20-26 */
uint64_t so_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
/* rmat.hpp:28 */
double so_next_unit(uint64_t* state) {
  return (double)(so_splitmix_next(state) >> 11) * 0x1.0p-53;
}

/* ---------------------------------------------------------------- csr */
void so_csr_free(so_csr* a) {
  free(a->row_ptr);
  free(a->col_idx);
  free(a->val);
  memset(a, 0, sizeof(*a));
}

/* LSD radix sort of (key, payload index) on 64-bit keys; stable. */
static void radix_sort_u64(uint64_t* key, int64_t* idx, int64_t n,
                           int key_bits) {
  uint64_t* k2 = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n ? n : 1));
  int64_t* i2 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int shift = 0; shift < key_bits; shift += 16) {
    int64_t cnt[65537];
    memset(cnt, 0, sizeof(cnt));
    for (int64_t i = 0; i < n; ++i) cnt[((key[i] >> shift) & 0xFFFF) + 1]++;
    for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
    for (int64_t i = 0; i < n; ++i) {
      int64_t d = cnt[(key[i] >> shift) & 0xFFFF]++;
      k2[d] = key[i];
      i2[d] = idx[i];
    }
    memcpy(key, k2, sizeof(uint64_t) * (size_t)n);
    memcpy(idx, i2, sizeof(int64_t) * (size_t)n);
  }
  free(k2);
  free(i2);
}

static int bits_for(int64_t v) {
  int b = 0;
  while (b < 63 && ((int64_t)1 << b) < v) ++b;
  return b;
}

/* csr.hpp:123-164: sort by (row, col), sum duplicates, prefix row_ptr. */
int so_csr_from_coo(int64_t m, int64_t k, int64_t count, const int64_t* rows,
                    const int64_t* cols, const float* vals, so_csr* out) {
  memset(out, 0, sizeof(*out));
  if (m < 0 || k < 0) return -1;
  for (int64_t i = 0; i < count; ++i) {
    if (rows[i] < 0 || rows[i] >= m || cols[i] < 0 || cols[i] >= k) return -1;
  }
  const int cb = bits_for(k), rb = bits_for(m);
  uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(count ? count : 1));
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(count ? count : 1));
  for (int64_t i = 0; i < count; ++i) {
    key[i] = ((uint64_t)rows[i] << cb) | (uint64_t)cols[i];
    idx[i] = i;
  }
  int kb = cb + rb;
  if (kb < 1) kb = 1;
  radix_sort_u64(key, idx, count, kb);
  out->m = m;
  out->k = k;
  out->row_ptr = (int64_t*)calloc((size_t)m + 1, sizeof(int64_t));
  out->col_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(count ? count : 1));
  out->val = (float*)malloc(sizeof(float) * (size_t)(count ? count : 1));
  int64_t nnz = 0, i = 0;
  while (i < count) {
    const int64_t r = rows[idx[i]], c = cols[idx[i]];
    float sum = vals[idx[i]];
    ++i;
    while (i < count && rows[idx[i]] == r && cols[idx[i]] == c) {
      sum += vals[idx[i]];
      ++i;
    }
    out->col_idx[nnz] = c;
    out->val[nnz] = sum;
    ++nnz;
    out->row_ptr[r + 1] = nnz;
  }
  for (int64_t r = 0; r < m; ++r) {
    if (out->row_ptr[r + 1] < out->row_ptr[r]) out->row_ptr[r + 1] = out->row_ptr[r];
  }
  out->nnz = nnz;
  free(key);
  free(idx);
  return 0;
}

/* csr.hpp:95-119 */
int so_validate(const so_csr* a) {
  if (a->m < 0 || a->k < 0) return -1;
  if (a->row_ptr[0] != 0 || a->row_ptr[a->m] != a->nnz) return -1;
  for (int64_t i = 0; i < a->m; ++i) {
    if (a->row_ptr[i] > a->row_ptr[i + 1]) return -1;
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) {
      if (a->col_idx[e] < 0 || a->col_idx[e] >= a->k) return -1;
      if (e > a->row_ptr[i] && a->col_idx[e] <= a->col_idx[e - 1]) return -1;
    }
  }
  return 0;
}

/* rmat.hpp:46-59 validate + rmat.hpp:61-88 generate_rmat */
int so_generate_rmat(uint32_t scale, uint64_t edge_factor, double a, double b,
                     double c, double d, uint64_t seed, so_csr* out) {
  if (scale < 1 || scale > 30 || edge_factor < 1) return -1;
  const double pr[4] = {a, b, c, d};
  double s = 0.0;
  for (int i = 0; i < 4; ++i) {
    if (pr[i] < 0.0 || pr[i] > 1.0) return -1;
    s += pr[i];
  }
  if (fabs(s - 1.0) > 1e-9) return -1;
  const int64_t dim = (int64_t)1 << scale;
  const uint64_t edges = edge_factor << scale;
  const double t_a = a, t_ab = a + b, t_abc = a + b + c;
  uint64_t st = seed;
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * edges);
  int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * edges);
  float* vals = (float*)malloc(sizeof(float) * edges);
  for (uint64_t e = 0; e < edges; ++e) {
    int64_t row = 0, col = 0;
    for (uint32_t lvl = 0; lvl < scale; ++lvl) {
      const double u = so_next_unit(&st);
      const int rbit = u >= t_ab;
      const int cbit = (u >= t_a && u < t_ab) || u >= t_abc;
      row = (row << 1) | rbit;
      col = (col << 1) | cbit;
    }
    rows[e] = row;
    cols[e] = col;
    vals[e] = 1.0f;
  }
  int rc = so_csr_from_coo(dim, dim, (int64_t)edges, rows, cols, vals, out);
  for (int64_t e = 0; e < out->nnz; ++e) out->val[e] = 1.0f; /* rmat.hpp:85-86 */
  free(rows);
  free(cols);
  free(vals);
  return rc;
}

/* corpus.hpp:15-32, 35-54 (grid via rmat.hpp:93-117), 58-105 (edge cases) */
int so_full_corpus(uint64_t seed, so_csr* out, char (*names)[64]) {
  static const uint32_t scales[3] = {8, 10, 12};
  static const uint64_t efs[3] = {4, 8, 16};
  static const char* skew_names[3] = {"uniform", "mild", "heavy"};
  static const double skews[3][4] = {{0.25, 0.25, 0.25, 0.25},
                                     {0.45, 0.22, 0.22, 0.11},
                                     {0.57, 0.19, 0.19, 0.05}};
  uint64_t seed_stream = seed;
  int n = 0;
  for (int si = 0; si < 3; ++si)
    for (int ei = 0; ei < 3; ++ei)
      for (int ki = 0; ki < 3; ++ki) {
        const uint64_t cell_seed = so_splitmix_next(&seed_stream);
        so_generate_rmat(scales[si], efs[ei], skews[ki][0], skews[ki][1],
                         skews[ki][2], skews[ki][3], cell_seed, &out[n]);
        snprintf(names[n], 64, "rmat_s%u_e%llu_%s", scales[si],
                 (unsigned long long)efs[ei], skew_names[ki]);
        ++n;
      }
  uint64_t rng = 0xEDCE;
  /* empty 64x64 */
  memset(&out[n], 0, sizeof(so_csr));
  out[n].m = out[n].k = 64;
  out[n].row_ptr = (int64_t*)calloc(65, sizeof(int64_t));
  out[n].col_idx = (int64_t*)malloc(8);
  out[n].val = (float*)malloc(4);
  snprintf(names[n++], 64, "empty");
  {
    int64_t r[1000], c[1000];
    float v[1000];
    for (int64_t j = 0; j < 1000; ++j) {
      r[j] = 0;
      c[j] = 2 * j;
      v[j] = (float)(2.0 * so_next_unit(&rng) - 1.0);
    }
    so_csr_from_coo(1, 2048, 1000, r, c, v, &out[n]);
    snprintf(names[n++], 64, "single_long_row");
  }
  {
    int64_t r[1024], c[1024];
    float v[1024];
    for (int64_t i = 0; i < 1024; ++i) {
      r[i] = i;
      c[i] = (i * 7 + 3) % 1024;
      v[i] = (float)(2.0 * so_next_unit(&rng) - 1.0);
    }
    so_csr_from_coo(1024, 1024, 1024, r, c, v, &out[n]);
    snprintf(names[n++], 64, "singleton_rows");
  }
  {
    int64_t r[1000], c[1000];
    float v[1000];
    int64_t t = 0;
    for (int64_t i = 0; i < 512; i += 3)
      for (int64_t j = 0; j < 5; ++j) {
        r[t] = i;
        c[t] = (i + 31 * j) % 512;
        v[t] = (float)(2.0 * so_next_unit(&rng) - 1.0);
        ++t;
      }
    so_csr_from_coo(512, 512, t, r, c, v, &out[n]);
    snprintf(names[n++], 64, "empty_row_riddled");
  }
  {
    int64_t r[48 * 48], c[48 * 48];
    float v[48 * 48];
    int64_t t = 0;
    for (int64_t i = 0; i < 48; ++i)
      for (int64_t j = 0; j < 48; ++j) {
        r[t] = i;
        c[t] = j;
        v[t] = (float)(2.0 * so_next_unit(&rng) - 1.0);
        ++t;
      }
    so_csr_from_coo(48, 48, t, r, c, v, &out[n]);
    snprintf(names[n++], 64, "dense_block");
  }
  return n;
}

/* corpus.hpp:116-122 */
void so_make_dense(int64_t rows, int64_t cols, uint64_t seed, float* out) {
  uint64_t st = seed;
  const int64_t total = rows * cols;
  for (int64_t i = 0; i < total; ++i) {
    out[i] = (float)(2.0 * so_next_unit(&st) - 1.0);
  }
}

/* ---------------------------------------------------------------- features */
/* csr.hpp:166-181 */
int so_extract_features(const int64_t* row_ptr, int64_t m, double* out3) {
  if (m < 1) return -1;
  const int64_t nnz = row_ptr[m];
  const double avg = (double)nnz / (double)m;
  double ss = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    const double d = (double)(row_ptr[i + 1] - row_ptr[i]) - avg;
    ss += d * d;
  }
  const double stdv = sqrt(ss / (double)m);
  out3[0] = avg;
  out3[1] = stdv;
  out3[2] = avg == 0.0 ? 0.0 : stdv / avg;
  return 0;
}

/* selector.hpp:28-34 */
int so_select_kernel(double avg_row, double cv, uint64_t n,
                     uint64_t n_parallel_max, double t_parallel_avg,
                     double t_cv) {
  if (n <= n_parallel_max) return avg_row < t_parallel_avg ? 1 : 0;
  return cv > t_cv ? 3 : 2;
}

/* kernels.hpp:133-149 */
int64_t so_plan_balanced(const int64_t* row_ptr, int64_t m, int64_t nnz,
                         int64_t chunk, int64_t* elem_row,
                         int64_t* chunk_first_row) {
  if (chunk < 1) return -1;
  const int64_t chunks = (nnz + chunk - 1) / chunk;
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      if (elem_row) elem_row[e] = i;
      if (chunk_first_row && e % chunk == 0) chunk_first_row[e / chunk] = i;
    }
  }
  return chunks;
}

/* kernels.hpp:124-129 */
void so_partition(int64_t items, int64_t parts, int64_t w, int64_t* lo,
                  int64_t* hi) {
  *lo = items * w / parts;
  *hi = items * (w + 1) / parts;
}

static int64_t lower_bound64(const int64_t* a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

void so_row_slices(const int64_t* row_ptr, int64_t m, int64_t nnz,
                   int64_t parts, int64_t* bounds) {
  bounds[0] = 0;
  for (int64_t g = 1; g < parts; ++g) {
    int64_t lo, hi;
    so_partition(nnz, parts, g, &lo, &hi);
    bounds[g] = lower_bound64(row_ptr, m + 1, lo);
    if (bounds[g] > m) bounds[g] = m;
    if (bounds[g] < bounds[g - 1]) bounds[g] = bounds[g - 1];
  }
  bounds[parts] = m;
}

/* ---------------------------------------------------------------- scan */
/* reduction.hpp:75-86: lockstep Hillis-Steele, top-down in place. */
void so_conditional_scan(int64_t width, int64_t comps, const int64_t* rows,
                         float* vals) {
  for (int64_t off = 1; off < width; off <<= 1) {
    for (int64_t i = width - 1; i >= off; --i) {
      if (rows[i] == rows[i - off]) {
        for (int64_t c = 0; c < comps; ++c) {
          vals[i * comps + c] += vals[(i - off) * comps + c];
        }
      }
    }
  }
}

/* ---------------------------------------------------------------- kernels */
static int is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

/* kernels.hpp:91-100 */
int so_check_config(int64_t lane_width, int64_t vdl_group, int64_t seq_chunk) {
  if (!is_pow2(lane_width) || lane_width < 2 || lane_width > 64) return -1;
  if (vdl_group != 0 && vdl_group != 1 && vdl_group != 2 && vdl_group != 4)
    return -1;
  if (seq_chunk < 1) return -1;
  return 0;
}

/* kernels.hpp:157-224, one output column at a time (per-column arithmetic is
 * independent of the VDL group C). */
static void par_rowsplit(const so_csr* a, int64_t w, const float* x, int64_t n,
                         float* y) {
  float* acc = (float*)malloc(sizeof(float) * (size_t)w);
  for (int64_t i = 0; i < a->m; ++i) {
    const int64_t begin = a->row_ptr[i], end = a->row_ptr[i + 1];
    if (begin == end) continue; /* :211 (Y pre-zeroed) */
    for (int64_t j = 0; j < n; ++j) {
      for (int64_t l = 0; l < w; ++l) acc[l] = 0.0f;
      for (int64_t base = begin; base < end; base += w) { /* :179-188 */
        const int64_t lanes = (end - base) < w ? (end - base) : w;
        for (int64_t l = 0; l < lanes; ++l) {
          const float p = a->val[base + l] * x[a->col_idx[base + l] * n + j];
          acc[l] += p;
        }
      }
      for (int64_t len = w; len > 1; len >>= 1) /* :193-199 */
        for (int64_t l = 0; l < len / 2; ++l) acc[l] = acc[2 * l + 1] + acc[2 * l];
      y[i * n + j] = acc[0];
    }
  }
  free(acc);
}

/* kernels.hpp:232-330 (+ reduction.hpp:75-86), per column. */
static void par_balanced(const so_csr* a, int64_t w, const float* x, int64_t n,
                         float* y) {
  const int64_t nnz = a->nnz;
  const int64_t chunks = (nnz + w - 1) / w;
  int64_t* elem_row = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz ? nnz : 1));
  so_plan_balanced(a->row_ptr, a->m, nnz, w, elem_row, NULL);
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)w);
  float* vals = (float*)malloc(sizeof(float) * (size_t)w);
  int64_t* hrow = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * chunks + 1));
  float* hval = (float*)malloc(sizeof(float) * (size_t)(2 * chunks + 1));
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t q = 0; q < 2 * chunks; ++q) hrow[q] = -1;
    for (int64_t q = 0; q < chunks; ++q) {
      const int64_t e0 = q * w, e1 = (e0 + w < nnz) ? e0 + w : nnz;
      const int64_t real = e1 - e0;
      int any_run = 0;
      for (int64_t l = 0; l < real; ++l) { /* :271-278 */
        const int64_t e = e0 + l;
        rows[l] = elem_row[e];
        any_run |= l > 0 && rows[l] == rows[l - 1];
        vals[l] = a->val[e] * x[a->col_idx[e] * n + j];
      }
      for (int64_t l = real; l < w; ++l) { /* :279-282 */
        rows[l] = PAD_ROW;
        vals[l] = 0.0f;
      }
      if (any_run) so_conditional_scan(w, 1, rows, vals); /* :290-293 */
      for (int64_t l = 0; l < w; ++l) { /* :296-309 */
        if (l + 1 < w && rows[l + 1] == rows[l]) continue;
        const int64_t r = rows[l];
        if (r == PAD_ROW) continue;
        const int complete = a->row_ptr[r] >= e0 && a->row_ptr[r + 1] <= e1;
        if (complete) {
          y[r * n + j] = vals[l];
        } else {
          const int64_t slot = 2 * q + (a->row_ptr[r] < e0 ? 0 : 1);
          hrow[slot] = r;
          hval[slot] = vals[l];
        }
      }
    }
    for (int64_t s = 0; s < 2 * chunks; ++s) /* :316-323 */
      if (hrow[s] >= 0) y[hrow[s] * n + j] += hval[s];
  }
  free(elem_row);
  free(rows);
  free(vals);
  free(hrow);
  free(hval);
}

/* kernels.hpp:339-376 */
static void seq_rowsplit(const so_csr* a, const float* x, int64_t n, float* y) {
  for (int64_t i = 0; i < a->m; ++i) {
    const int64_t begin = a->row_ptr[i], end = a->row_ptr[i + 1];
    if (begin == end) continue;
    for (int64_t j = 0; j < n; ++j) {
      float acc = 0.0f;
      for (int64_t e = begin; e < end; ++e) {
        const float p = a->val[e] * x[a->col_idx[e] * n + j];
        acc += p;
      }
      y[i * n + j] = acc;
    }
  }
}

/* kernels.hpp:384-455 */
static void seq_balanced(const so_csr* a, int64_t chunk, const float* x,
                         int64_t n, float* y) {
  const int64_t nnz = a->nnz;
  const int64_t chunks = (nnz + chunk - 1) / chunk;
  int64_t* elem_row = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz ? nnz : 1));
  so_plan_balanced(a->row_ptr, a->m, nnz, chunk, elem_row, NULL);
  int64_t* brow = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * chunks + 1));
  float* bval = (float*)calloc((size_t)(2 * chunks + 1) * (size_t)n, sizeof(float));
  float* acc = (float*)malloc(sizeof(float) * (size_t)n);
  for (int64_t s = 0; s < 2 * chunks; ++s) brow[s] = -1;
  for (int64_t q = 0; q < chunks; ++q) {
    const int64_t e0 = q * chunk, e1 = (e0 + chunk < nnz) ? e0 + chunk : nnz;
    int64_t cur = elem_row[e0];
    for (int64_t j = 0; j < n; ++j) acc[j] = 0.0f;
    for (int64_t e = e0; e <= e1; ++e) {
      if (e == e1 || elem_row[e] != cur) { /* flush, :415-425 */
        const int64_t r = cur;
        const int complete = a->row_ptr[r] >= e0 && a->row_ptr[r + 1] <= e1;
        float* dst;
        if (complete) {
          dst = y + r * n;
        } else {
          const int64_t slot = 2 * q + (a->row_ptr[r] < e0 ? 0 : 1);
          brow[slot] = r;
          dst = bval + slot * n;
        }
        for (int64_t j = 0; j < n; ++j) dst[j] = acc[j];
        if (e == e1) break;
        for (int64_t j = 0; j < n; ++j) acc[j] = 0.0f;
        cur = elem_row[e];
      }
      const float v = a->val[e];
      const float* xr = x + a->col_idx[e] * n;
      for (int64_t j = 0; j < n; ++j) { /* :439-441 */
        const float p = v * xr[j];
        acc[j] += p;
      }
    }
  }
  for (int64_t s = 0; s < 2 * chunks; ++s) /* :448-453 */
    if (brow[s] >= 0)
      for (int64_t j = 0; j < n; ++j) y[brow[s] * n + j] += bval[s * n + j];
  free(elem_row);
  free(brow);
  free(bval);
  free(acc);
}

/* kernels.hpp:457-464 dispatcher; Y zero-allocated (csr.hpp:66-72). */
int so_spmm(const so_csr* a, int kernel, int64_t lane_width, int64_t vdl_group,
            int64_t seq_chunk, const float* x, int64_t n, float* y) {
  if (so_check_config(lane_width, vdl_group, seq_chunk) != 0) return -1;
  memset(y, 0, sizeof(float) * (size_t)(a->m * n));
  if (n == 0) return 0;
  switch (kernel) {
    case 0: par_rowsplit(a, lane_width, x, n, y); break;
    case 1: if (a->nnz) par_balanced(a, lane_width, x, n, y); break;
    case 2: seq_rowsplit(a, x, n, y); break;
    default: if (a->nnz) seq_balanced(a, seq_chunk, x, n, y); break;
  }
  return 0;
}

static int64_t effective_group(int64_t vdl_group, int64_t n) {
  if (vdl_group != 0) return vdl_group; /* kernels.hpp:116-121 */
  if (n >= 4) return 4;
  if (n >= 2) return 2;
  return 1;
}

void so_kernel_stats(const so_csr* a, int kernel, int64_t w, int64_t vdl_group,
                     int64_t n, uint64_t* lane_multiplies, uint64_t* scan_ops) {
  *lane_multiplies = 0;
  *scan_ops = 0;
  if (n == 0 || kernel >= 2) return;
  int64_t levels = 0;
  for (int64_t off = 1; off < w; off <<= 1) ++levels;
  int64_t group = effective_group(vdl_group, n);
  if (group > n) group = n;
  /* column-group widths: n/group groups of `group`, then n%group singles */
  const uint64_t wc_sum = (uint64_t)((n / group) * group + (n % group));
  if (kernel == 0) { /* :187, :200-201 per non-empty row per group */
    for (int64_t i = 0; i < a->m; ++i) {
      const int64_t len = a->row_ptr[i + 1] - a->row_ptr[i];
      if (len == 0) continue;
      *lane_multiplies += (uint64_t)((len + w - 1) / w) * (uint64_t)w * wc_sum;
      *scan_ops += (uint64_t)levels * (uint64_t)w * wc_sum;
    }
  } else { /* :283-285 per chunk per group */
    if (a->nnz == 0) return;
    const uint64_t chunks = (uint64_t)((a->nnz + w - 1) / w);
    *lane_multiplies = chunks * (uint64_t)w * wc_sum;
    *scan_ops = chunks * (uint64_t)levels * (uint64_t)w * wc_sum;
  }
}

/* kernels.hpp:468-472 */
double so_kernel_tolerance(int64_t max_row_nnz) {
  return 1e-5 * log2((double)max_row_nnz + 2.0);
}

int64_t so_max_row_nnz(const int64_t* row_ptr, int64_t m) {
  int64_t mx = 0;
  for (int64_t i = 0; i < m; ++i)
    if (row_ptr[i + 1] - row_ptr[i] > mx) mx = row_ptr[i + 1] - row_ptr[i];
  return mx;
}

/* ---------------------------------------------------------------- fp64 oracle */
typedef struct {
  const so_csr* a;
  const float* x;
  int64_t n;
  const int64_t* rows;
  int64_t lo, hi;
  double* y;
  double* absb;
} oracle_job;

static void* oracle_worker(void* p) {
  oracle_job* jb = (oracle_job*)p;
  const so_csr* a = jb->a;
  const int64_t n = jb->n;
  for (int64_t t = jb->lo; t < jb->hi; ++t) {
    const int64_t i = jb->rows ? jb->rows[t] : t;
    double* yr = jb->y + t * n;
    double* br = jb->absb ? jb->absb + t * n : NULL;
    for (int64_t j = 0; j < n; ++j) {
      yr[j] = 0.0;
      if (br) br[j] = 0.0;
    }
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) { /* csr.hpp:193-202 */
      const double v = (double)a->val[e];
      const float* xr = jb->x + a->col_idx[e] * n;
      for (int64_t j = 0; j < n; ++j) {
        const double p = v * (double)xr[j];
        yr[j] += p;
        if (br) br[j] += fabs(p);
      }
    }
  }
  return NULL;
}

void so_oracle_rows(const so_csr* a, const float* x, int64_t n,
                    const int64_t* rows, int64_t count, double* y,
                    double* absbound, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  oracle_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t].a = a;
    jobs[t].x = x;
    jobs[t].n = n;
    jobs[t].rows = rows;
    jobs[t].lo = count * t / threads;
    jobs[t].hi = count * (t + 1) / threads;
    jobs[t].y = y;
    jobs[t].absb = absbound;
    if (t > 0) pthread_create(&th[t], NULL, oracle_worker, &jobs[t]);
  }
  oracle_worker(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------- row-subset exact kernels */
/* The four fp32 kernels (kernels.hpp:157-464) evaluated for a list of rows
 * only.  A row's result in every variant depends only on its own nonzeros and
 * on where the global chunk boundaries (q*seq_chunk for seq-ws, q*lane_width
 * for par-ws) cut it, so each listed row is recomputed here in exactly the
 * order the full kernel uses, without touching the rest of the matrix:
 *   par-rs  kernels.hpp:179-199  lanes restart at the row start, pairwise tree
 *   par-ws  kernels.hpp:262-323  per chunk: rounded products, the lockstep
 *           conditional scan (reduction.hpp:75-86) over the row's lanes only
 *           (the scan never adds across rows), the run's last lane emitted;
 *           complete rows store it, rows crossing chunks add the per-chunk
 *           emissions to Y = +0 in ascending slot order (:316-323)
 *   seq-rs  kernels.hpp:360-371  one sequential chain per column
 *   seq-ws  kernels.hpp:410-453  per chunk a chain from +0; complete rows
 *           store it, crossing rows add the partials to +0 in chunk order
 * col_idx is int32 (the device layout) so full-size matrices fit host memory.
 * tests/test_oracle.py checks this against so_spmm on the whole corpus. */
typedef struct {
  const int64_t* row_ptr;
  const int32_t* col;
  const float* val;
  int kernel;
  int64_t w, chunk, n;
  const float* x;
  const int64_t* rows;
  int64_t lo, hi;
  float* y;
} rows_job;

static void row_par_rs(const rows_job* jb, int64_t s, int64_t e, float* yr, float* acc) {
  const int64_t w = jb->w, n = jb->n;
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t l = 0; l < w; ++l) acc[l] = 0.0f;
    for (int64_t base = s; base < e; base += w) {
      const int64_t lanes = (e - base) < w ? (e - base) : w;
      for (int64_t l = 0; l < lanes; ++l) {
        const float p = jb->val[base + l] * jb->x[(int64_t)jb->col[base + l] * n + j];
        acc[l] += p;
      }
    }
    for (int64_t len = w; len > 1; len >>= 1)
      for (int64_t l = 0; l < len / 2; ++l) acc[l] = acc[2 * l + 1] + acc[2 * l];
    yr[j] = acc[0];
  }
}

static void row_par_ws(const rows_job* jb, int64_t s, int64_t e, float* yr, float* lanev) {
  const int64_t w = jb->w, n = jb->n;
  const int64_t q0 = s / w, q1 = (e - 1) / w;
  for (int64_t j = 0; j < n; ++j) {
    float out = 0.0f;
    for (int64_t q = q0; q <= q1; ++q) {
      const int64_t a = s > q * w ? s : q * w;
      const int64_t b = e < (q + 1) * w ? e : (q + 1) * w;
      const int64_t la = a - q * w, lb = b - q * w; /* run lanes [la, lb) */
      for (int64_t l = la; l < lb; ++l)
        lanev[l] = jb->val[q * w + l] * jb->x[(int64_t)jb->col[q * w + l] * n + j];
      for (int64_t off = 1; off < w; off <<= 1)
        for (int64_t i = lb - 1; i >= la + off; --i) lanev[i] += lanev[i - off];
      const float h = lanev[lb - 1];
      if (q0 == q1) out = h;      /* complete: stored */
      else out += h;              /* partial slots, ascending (Y starts at +0) */
    }
    yr[j] = out;
  }
}

static void row_seq(const rows_job* jb, int64_t s, int64_t e, float* yr, int ws) {
  const int64_t n = jb->n;
  const int64_t c = ws ? jb->chunk : (e - s + 1);
  const int64_t q0 = ws ? s / c : 0, q1 = ws ? (e - 1) / c : 0;
  for (int64_t j = 0; j < n; ++j) {
    float out = 0.0f;
    for (int64_t q = q0; q <= q1; ++q) {
      const int64_t a = ws ? (s > q * c ? s : q * c) : s;
      const int64_t b = ws ? (e < (q + 1) * c ? e : (q + 1) * c) : e;
      float acc = 0.0f;
      for (int64_t p = a; p < b; ++p) {
        const float pr = jb->val[p] * jb->x[(int64_t)jb->col[p] * n + j];
        acc += pr;
      }
      if (q0 == q1) out = acc;
      else out += acc;
    }
    yr[j] = out;
  }
}

static void* rows_worker(void* p) {
  rows_job* jb = (rows_job*)p;
  float* tmp = (float*)malloc(sizeof(float) * (size_t)(jb->w > 0 ? jb->w : 1));
  for (int64_t t = jb->lo; t < jb->hi; ++t) {
    const int64_t r = jb->rows[t];
    const int64_t s = jb->row_ptr[r], e = jb->row_ptr[r + 1];
    float* yr = jb->y + t * jb->n;
    if (s == e) {
      for (int64_t j = 0; j < jb->n; ++j) yr[j] = 0.0f;
      continue;
    }
    switch (jb->kernel) {
      case 0: row_par_rs(jb, s, e, yr, tmp); break;
      case 1: row_par_ws(jb, s, e, yr, tmp); break;
      case 2: row_seq(jb, s, e, yr, 0); break;
      default: row_seq(jb, s, e, yr, 1); break;
    }
  }
  free(tmp);
  return NULL;
}

int so_spmm_rows32(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                   int kernel, int64_t lane_width, int64_t seq_chunk, const float* x,
                   int64_t n, const int64_t* rows, int64_t count, float* y, int threads) {
  if (so_check_config(lane_width, 0, seq_chunk) != 0) return -1;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  rows_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    rows_job* jb = &jobs[t];
    memset(jb, 0, sizeof(*jb));
    jb->row_ptr = row_ptr;
    jb->col = col_idx;
    jb->val = val;
    jb->kernel = kernel;
    jb->w = lane_width;
    jb->chunk = seq_chunk;
    jb->n = n;
    jb->x = x;
    jb->rows = rows;
    jb->lo = count * t / threads;
    jb->hi = count * (t + 1) / threads;
    jb->y = y;
    if (t > 0) pthread_create(&th[t], NULL, rows_worker, jb);
  }
  rows_worker(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* csr.hpp:185-205 (fp64 oracle + Σ|a·x|) for listed rows, int32 columns. */
typedef struct {
  const int64_t* row_ptr;
  const int32_t* col;
  const float* val;
  const float* x;
  int64_t n;
  const int64_t* rows;
  int64_t lo, hi;
  double* y;
  double* absb;
} oracle32_job;

static void* oracle32_worker(void* p) {
  oracle32_job* jb = (oracle32_job*)p;
  const int64_t n = jb->n;
  for (int64_t t = jb->lo; t < jb->hi; ++t) {
    const int64_t i = jb->rows[t];
    double* yr = jb->y + t * n;
    double* br = jb->absb + t * n;
    for (int64_t j = 0; j < n; ++j) yr[j] = br[j] = 0.0;
    for (int64_t e = jb->row_ptr[i]; e < jb->row_ptr[i + 1]; ++e) {
      const double v = (double)jb->val[e];
      const float* xr = jb->x + (int64_t)jb->col[e] * n;
      for (int64_t j = 0; j < n; ++j) {
        const double pr = v * (double)xr[j];
        yr[j] += pr;
        br[j] += fabs(pr);
      }
    }
  }
  return NULL;
}

void so_oracle_rows32(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                      const float* x, int64_t n, const int64_t* rows, int64_t count,
                      double* y, double* absbound, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  oracle32_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    oracle32_job* jb = &jobs[t];
    jb->row_ptr = row_ptr;
    jb->col = col_idx;
    jb->val = val;
    jb->x = x;
    jb->n = n;
    jb->rows = rows;
    jb->lo = count * t / threads;
    jb->hi = count * (t + 1) / threads;
    jb->y = y;
    jb->absb = absbound;
    if (t > 0) pthread_create(&th[t], NULL, oracle32_worker, jb);
  }
  oracle32_worker(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
}
