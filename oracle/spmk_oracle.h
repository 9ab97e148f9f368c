/* TEST INFRASTRUCTURE ONLY — the CPU oracle (checker), never the product.
 *
 * Plain-C restatement of the reference algorithm for the adaptive SpMV/SpMM
 * hot path (arxiv 2106.16064 artifact `spmk`, /root/reference/proj/include).
 * Every function cites the reference file:line it follows.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Pinned: tests/test_oracle.py checks every function here bit-for-bit against
 * the reference itself (oracle/_ref/libspmk_ref.so, built from the reference
 * headers by oracle/Makefile) on the pinned corpus, and against the golden
 * vectors under tests/golden/ (generated from the reference by
 * tests/golden/make_golden.py).
 *
 * Value type is fp32 (the device path's type); indices are int64 (Index).
 * Build with -ffp-contract=off: the reference is compiled without -march, so
 * its `acc += v * x` keeps two roundings.
 */
#ifndef SPMK_ORACLE_H
#define SPMK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t m, k, nnz;
  int64_t* row_ptr; /* m+1 */
  int64_t* col_idx; /* nnz */
  float* val;       /* nnz */
} so_csr;

/* rmat.hpp:15-29 SplitMix64 */
uint64_t so_splitmix_next(uint64_t* state);
double so_next_unit(uint64_t* state);

void so_csr_free(so_csr* a);
/* csr.hpp:123-164 csr_from_coo (stable order for duplicate sums; the
 * reference's std::sort is unstable, so duplicates with unequal values are
 * outside the bit-exact contract). Returns 0 or -1 (out-of-range coordinate). */
int so_csr_from_coo(int64_t m, int64_t k, int64_t count, const int64_t* rows,
                    const int64_t* cols, const float* vals, so_csr* out);
/* csr.hpp:95-119 validate: 0 ok, -1 malformed */
int so_validate(const so_csr* a);
/* rmat.hpp:61-88 generate_rmat<float> */
int so_generate_rmat(uint32_t scale, uint64_t edge_factor, double a, double b,
                     double c, double d, uint64_t seed, so_csr* out);
/* rmat.hpp:93-117 + corpus.hpp:35-113: fills up to 32 matrices, returns count.
 * names receive "rmat_s8_e4_uniform" ... "dense_block" (64 bytes each). */
int so_full_corpus(uint64_t seed, so_csr* out, char (*names)[64]);
/* corpus.hpp:116-122 make_dense<float> (row-major) */
void so_make_dense(int64_t rows, int64_t cols, uint64_t seed, float* out);

/* csr.hpp:166-181.  out3 = {avg_row, stdv_row, cv}; -1 when m < 1 */
int so_extract_features(const int64_t* row_ptr, int64_t m, double* out3);
/* selector.hpp:28-34 -> kernel_index (0 par-rs, 1 par-ws, 2 seq-rs, 3 seq-ws) */
int so_select_kernel(double avg_row, double cv, uint64_t n,
                     uint64_t n_parallel_max, double t_parallel_avg,
                     double t_cv);
/* kernels.hpp:133-149.  Returns num_chunks (-1 if chunk < 1).  elem_row (nnz)
 * and chunk_first_row (num_chunks; = elem_row[q*chunk]) may be NULL. */
int64_t so_plan_balanced(const int64_t* row_ptr, int64_t m, int64_t nnz,
                         int64_t chunk, int64_t* elem_row,
                         int64_t* chunk_first_row);
/* kernels.hpp:124-129 */
void so_partition(int64_t items, int64_t parts, int64_t w, int64_t* lo,
                  int64_t* hi);
/* Multi-GPU equal-nnz row slices: bounds[g] =
 * lower_bound(row_ptr, partition(nnz, G, g).lo), bounds[0]=0, bounds[G]=m. */
void so_row_slices(const int64_t* row_ptr, int64_t m, int64_t nnz,
                   int64_t parts, int64_t* bounds);

/* reduction.hpp:75-86 (kPadRow = INT64_MAX) */
void so_conditional_scan(int64_t width, int64_t comps, const int64_t* rows,
                         float* vals);

/* kernels.hpp:91-100 check_config: 0 ok, -1 invalid */
int so_check_config(int64_t lane_width, int64_t vdl_group, int64_t seq_chunk);
/* kernels.hpp:157-464: the four fp32 kernels in the reference's exact
 * summation order.  y is M x n row-major, fully overwritten.  Returns 0, or -1
 * on a bad config. kernel = kernel_index. */
int so_spmm(const so_csr* a, int kernel, int64_t lane_width, int64_t vdl_group,
            int64_t seq_chunk, const float* x, int64_t n, float* y);
/* kernels.hpp:67-79,187,200-201,283-285: analytic KernelStats */
void so_kernel_stats(const so_csr* a, int kernel, int64_t lane_width,
                     int64_t vdl_group, int64_t n, uint64_t* lane_multiplies,
                     uint64_t* scan_ops);
/* kernels.hpp:468-472 (fp32) */
double so_kernel_tolerance(int64_t max_row_nnz);
int64_t so_max_row_nnz(const int64_t* row_ptr, int64_t m);

/* csr.hpp:185-205 oracle_spmm, fp64, per-row ascending e, for the listed rows
 * only (rows == NULL: all rows).  y and absbound (Σ_j |a_ij x_jc|, may be NULL)
 * are (count x n).  Row-parallel over `threads` pthreads; bit-identical to the
 * single-thread reference since every row keeps its own order. */
void so_oracle_rows(const so_csr* a, const float* x, int64_t n,
                    const int64_t* rows, int64_t count, double* y,
                    double* absbound, int threads);

/* kernels.hpp:157-464 restricted to the listed rows (exact reference order,
 * global chunk boundaries), int32 columns; y is (count x n).  Returns 0, or
 * -1 on a bad config.  Row-parallel over `threads` pthreads. */
int so_spmm_rows32(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                   int kernel, int64_t lane_width, int64_t seq_chunk, const float* x,
                   int64_t n, const int64_t* rows, int64_t count, float* y, int threads);
/* so_oracle_rows with int32 columns; y and absbound are (count x n). */
void so_oracle_rows32(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                      const float* x, int64_t n, const int64_t* rows, int64_t count,
                      double* y, double* absbound, int threads);

#ifdef __cplusplus
}
#endif
#endif
