/* spmk_capi.h — C ABI of the B200-native adaptive SpMV/SpMM engine.
 *
 * Drop-in boundary for the reference's hot path (arxiv 2106.16064 artifact
 * `spmk`, /root/reference/proj/include/spmk).  Every entry point below names
 * the reference interface it replaces.  Plain C types only (no torch, no STL):
 * host pointers are `const int64_t*`/`const float*`, device pointers are
 * `d_`-prefixed, streams are passed as `void*` (a cudaStream_t).
 *
 * Value type: fp32 only (the reference's `T=float` instantiation).  T=double is
 * SPMK_EUNSUPPORTED — there is no CPU fallback.  Indices are narrowed to int32
 * on the device (every BASELINE config has nnz < 2^31; larger is
 * SPMK_EUNSUPPORTED).
 *
 * Errors: every call returns spmk_status; the message of the last failure on
 * the calling thread is spmk_last_error().  The C++ drop-in headers
 * (include/spmk/*.hpp) rethrow it as spmk::Error (error.hpp:10-13).
 *
 * Threading: calls are thread-safe on distinct handles; a handle is bound to
 * the CUDA device it was created on.
 */
#ifndef SPMK_CAPI_H
#define SPMK_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPMK_CAPI_VERSION 1

typedef enum {
  SPMK_OK = 0,
  SPMK_EINVAL = 1,       /* bad argument / config (kernels.hpp:91-100)      */
  SPMK_EDIM = 2,         /* dimension mismatch (kernels.hpp:103-109)         */
  SPMK_ECUDA = 3,        /* CUDA runtime error                               */
  SPMK_ENOMEM = 4,       /* device allocation failed                         */
  SPMK_ENCCL = 5,        /* NCCL missing or a collective failed (spmk_mg_*)  */
  SPMK_EUNSUPPORTED = 6  /* valid for the reference, not on this device path */
} spmk_status;

/* kernel_index numbering, kernels.hpp:47-50: 2*seq + ws.
 * Names kernels.hpp:40-45: "par-rs", "par-ws", "seq-rs", "seq-ws". */
typedef enum {
  SPMK_PAR_ROWSPLIT = 0, /* kParRowSplit kernels.hpp:29  (north_star b) */
  SPMK_PAR_BALANCED = 1, /* kParBalanced kernels.hpp:31  (north_star d, VSR) */
  SPMK_SEQ_ROWSPLIT = 2, /* kSeqRowSplit kernels.hpp:33  (north_star a, CSC) */
  SPMK_SEQ_BALANCED = 3  /* kSeqBalanced kernels.hpp:35  (north_star c) */
} spmk_kernel_id;

/* KernelConfig, kernels.hpp:81-87 — same fields, same order, same defaults.
 * worker_count is accepted and ignored on the device (the CUDA grid replaces
 * the ThreadPool); stats are computed analytically (spmk_kernel_stats). */
typedef struct {
  uint64_t lane_width;   /* W: power of two in [2, 64]; default 32          */
  uint64_t vdl_group;    /* C in {0 (auto), 1, 2, 4}; default 0             */
  uint64_t seq_chunk;    /* nonzeros per seq-ws chunk (>= 1); default 256   */
  uint64_t worker_count; /* ignored on device                               */
} spmk_kernel_config;

/* SelectorThresholds, selector.hpp:16-22 */
typedef struct {
  uint64_t n_parallel_max; /* default 4    */
  double t_parallel_avg;   /* default 32.0 */
  double t_cv;             /* default 1.0  */
} spmk_thresholds;

/* MatrixFeatures, csr.hpp:86-92 */
typedef struct {
  double avg_row;
  double stdv_row;
  double cv;
  int64_t num_rows;
  int64_t nnz;
} spmk_features;

typedef struct spmk_csr_s* spmk_csr_t;

/* ------------------------------------------------------------ library */
const char* spmk_last_error(void);
int spmk_version(void);
void spmk_default_config(spmk_kernel_config* cfg);   /* KernelConfig{}       */
void spmk_default_thresholds(spmk_thresholds* t);    /* SelectorThresholds{} */
/* kernels.hpp:91-100 check_config */
spmk_status spmk_check_config(const spmk_kernel_config* cfg);
/* kernels.hpp:40-45 kernel_name / :52-57 parse_kernel */
const char* spmk_kernel_name(spmk_kernel_id id);
spmk_status spmk_parse_kernel(const char* name, spmk_kernel_id* out);

/* ------------------------------------------------------------ operand A */
/* Replaces CsrMatrix<float> (csr.hpp:24-57) + validate (csr.hpp:95-119):
 * validates the HOST arrays (int64, reference layout), uploads them to
 * `device`, narrows indices to int32 and builds the handle's resident row
 * metadata (non-empty row compaction, empty-row list). */
spmk_status spmk_csr_create(int64_t num_rows, int64_t num_cols, int64_t nnz,
                            const int64_t* row_ptr, const int64_t* col_idx,
                            const float* values, int device, spmk_csr_t* out);
/* Same, from int32 DEVICE arrays already in HBM (e.g. the device generator);
 * the call synchronizes the device first, so producers on any stream are done.
 * copy=0 borrows the arrays (caller keeps them alive), copy=1 duplicates.
 * Validation is done on the device (row_ptr shape, column bounds). */
spmk_status spmk_csr_create_device(int64_t num_rows, int64_t num_cols,
                                   int64_t nnz, const int32_t* d_row_ptr,
                                   const int32_t* d_col_idx,
                                   const float* d_values, int copy,
                                   spmk_csr_t* out);
/* Row slice [row_begin, row_end) of `a` as a standalone rebased CSR on
 * `device` (multi-GPU equal-nnz slices). */
spmk_status spmk_csr_slice(spmk_csr_t a, int64_t row_begin, int64_t row_end,
                           int device, spmk_csr_t* out);
/* |A|: a new handle with the same structure and |values| (the north-star
 * tolerance scale sum_j |a_ij x_j| is then one spmm with |X|). */
spmk_status spmk_csr_abs_copy(spmk_csr_t a, spmk_csr_t* out);
spmk_status spmk_csr_destroy(spmk_csr_t a);
spmk_status spmk_csr_info(spmk_csr_t a, int64_t* num_rows, int64_t* num_cols,
                          int64_t* nnz, int64_t* max_row_nnz,
                          int64_t* empty_rows);
/* Device pointers of the resident int32 CSR (rowPtr, colIdx, values). */
spmk_status spmk_csr_device_arrays(spmk_csr_t a, const int32_t** d_row_ptr,
                                   const int32_t** d_col_idx,
                                   const float** d_values);
/* validate (csr.hpp:95-119) of the resident CSR.  Handle creation checks what
 * the device path needs for safety (row_ptr shape, column range: SPMK_EINVAL
 * otherwise) but, like the reference's spmm_* (kernels.hpp:157-455, which
 * never call validate), accepts rows whose columns are not strictly
 * increasing and computes in position order; this call reports that case as
 * SPMK_EINVAL with the reference's message. */
spmk_status spmk_csr_validate(spmk_csr_t a);
/* Per-handle performance knobs (no effect on any result bit):
 * "seq_tile_nnz", "seq_ext", "parws_ext", "parws_t", "parrs_vl", "hub_nnz",
 * "hub_two_pass", "hub_smem", "l2_persist".  Initialised at creation from the
 * environment (SPMK_<KEY upper-case>), read by every later spmm on the handle;
 * a changed knob takes effect on the next call (plans are cached per shape). */
spmk_status spmk_csr_set_tuning(spmk_csr_t a, const char* key, int64_t value);
spmk_status spmk_csr_get_tuning(spmk_csr_t a, const char* key, int64_t* value);
/* Download back to the reference layout (int64 indices). */
spmk_status spmk_csr_download(spmk_csr_t a, int64_t* row_ptr, int64_t* col_idx,
                              float* values);

/* ------------------------------------------------------------ selection */
/* extract_features (csr.hpp:166-181): device reduction of exact integer
 * row-length moments, host finalize.  avg_row is bit-identical to the
 * reference; stdv_row/cv agree to ~1e-12 relative (SURVEY §8a tie-guard). */
spmk_status spmk_features_compute(spmk_csr_t a, spmk_features* out);
/* The same on host row_ptr, in the reference's exact sequential order. */
spmk_status spmk_features_host(int64_t num_rows, const int64_t* row_ptr,
                               spmk_features* out);
/* select_kernel (selector.hpp:28-34).  t may be NULL (defaults). */
spmk_kernel_id spmk_select(const spmk_features* f, uint64_t n,
                           const spmk_thresholds* t);
/* features + select on the handle, with the tie-guard: when cv (or avg_row)
 * lies within 1e-9 relative of its threshold, features are recomputed in the
 * reference's sequential order so the choice is bit-exact. */
spmk_status spmk_select_for(spmk_csr_t a, uint64_t n, const spmk_thresholds* t,
                            spmk_kernel_id* out);

/* ------------------------------------------------------------ partition */
/* plan_balanced (kernels.hpp:133-149) without the COO expansion: computed on
 * the device as upper_bound(rowPtr, q*chunk)-1.  chunk_first_row (host, may be
 * NULL) receives elem_row[q*chunk] for every chunk q; num_chunks =
 * ceil(nnz/chunk). */
spmk_status spmk_plan(spmk_csr_t a, int64_t chunk, int64_t* chunk_first_row,
                      int64_t* num_chunks);
/* Full elem_row expansion (host out, nnz entries) for parity tests. */
spmk_status spmk_plan_elem_row(spmk_csr_t a, int64_t* elem_row);
/* detail::partition (kernels.hpp:124-129) */
void spmk_partition(int64_t items, int64_t parts, int64_t w, int64_t* lo,
                    int64_t* hi);
/* Equal-nnz row slices for `parts` devices: bounds[parts+1] (host), bounds[g] =
 * lower_bound(rowPtr, partition(nnz, parts, g).lo); computed on the device. */
spmk_status spmk_row_slices(spmk_csr_t a, int64_t parts, int64_t* bounds);

/* ------------------------------------------------------------ SpMM */
/* spmm(KernelId, A, X, cfg) (kernels.hpp:457-464) on resident operands:
 * Y (num_rows x n, row-major, fp32, DEVICE) = A * X (num_cols x n, DEVICE).
 * Y is fully overwritten (empty rows get 0).  cfg may be NULL (defaults).
 * Asynchronous on `stream` (NULL = legacy default stream).  Results are
 * bit-identical to the reference's fp32 kernel of the same KernelId at the
 * same lane_width / seq_chunk (same partials, same summation order).
 * A handle's calls on different streams are ordered (a call waits for the
 * previous call's kernels when it arrives on another stream: they share the
 * handle's partial-slot scratch and side stream); calls captured into a CUDA
 * graph are not, so replay such a graph on the capturing stream. */
spmk_status spmk_spmm(spmk_csr_t a, spmk_kernel_id id,
                      const spmk_kernel_config* cfg, const float* d_x,
                      int64_t n, float* d_y, void* stream);
/* Rule-selected variant (select_for + spmm).  chosen may be NULL. */
spmk_status spmk_spmm_auto(spmk_csr_t a, const spmk_thresholds* t,
                           const spmk_kernel_config* cfg, const float* d_x,
                           int64_t n, float* d_y, void* stream,
                           spmk_kernel_id* chosen);
/* Host X in, host Y out (h2d, kernel, d2h on `stream`, then synchronize):
 * the value-returning reference call shape.  Staging buffers are cached in
 * the handle. */
spmk_status spmk_spmm_host(spmk_csr_t a, spmk_kernel_id id,
                           const spmk_kernel_config* cfg, const float* x,
                           int64_t n, float* y, void* stream);
/* The same without the final synchronize: H2D(x) -> kernels -> D2H(y) are
 * enqueued on `stream` and the call returns.  x and y must stay valid (pinned
 * for overlap) until the stream passes the call.  The handle rotates two
 * device staging slots, so consecutive calls on two streams overlap one
 * call's D2H with the next call's H2D (full-duplex PCIe); a slot's reuse
 * waits on the device for its previous call. */
spmk_status spmk_spmm_host_async(spmk_csr_t a, spmk_kernel_id id,
                                 const spmk_kernel_config* cfg, const float* x,
                                 int64_t n, float* y, void* stream);
/* One-shot drop-in for `spmm(id, CsrMatrix, DenseMatrix, cfg)` with every
 * operand on the host (create handle on `device`, run, download, destroy). */
spmk_status spmk_spmm_csr_host(int64_t num_rows, int64_t num_cols, int64_t nnz,
                               const int64_t* row_ptr, const int64_t* col_idx,
                               const float* values, spmk_kernel_id id,
                               const spmk_kernel_config* cfg, const float* x,
                               int64_t n, float* y, int device);

/* KernelStats (kernels.hpp:67-79), computed analytically with the reference's
 * lockstep formulas (:187, :200-201, :283-285). */
spmk_status spmk_kernel_stats(spmk_csr_t a, spmk_kernel_id id,
                              const spmk_kernel_config* cfg, int64_t n,
                              uint64_t* lane_multiplies, uint64_t* scan_ops);
/* kernel_tolerance<float> (kernels.hpp:468-472) */
double spmk_kernel_tolerance(int64_t max_row_nnz);

/* Pin X in L2 for subsequent spmk_spmm calls on `stream`: an access-policy
 * window over d_x (persisting hits, streaming misses), clamped to the
 * device's max window / persisting-L2 size.  bytes=0 clears the window. */
spmk_status spmk_l2_persist_x(void* stream, const float* d_x, size_t bytes);

/* ------------------------------------------------------------ measurement */
/* Kernel launches issued by this library since load (all entry points). */
uint64_t spmk_launch_count(void);
/* When enabled, spmk_spmm records CUDA events on its stream around the
 * dominant (variant) kernel and around the whole call (one event set per call,
 * the last 256 calls kept); spmk_timing_last synchronizes on the last call's
 * events and returns milliseconds, spmk_timing_summary the totals over the
 * calls kept since spmk_timing_enable (no host sync between the calls needed).
 * For bench.py's roofline; no reference counterpart. */
spmk_status spmk_timing_enable(int on);
spmk_status spmk_timing_last(float* main_kernel_ms, float* whole_call_ms);
spmk_status spmk_timing_summary(float* main_kernel_ms, float* whole_call_ms, int* calls);
/* Which device path spmk_spmm takes for (a, id, cfg, n) with 16-byte aligned
 * operands: *path = 1 for seq-ws through the lane-per-job sweep + fold pass
 * (sell_kernels.cuh; empty rows written in the sweep), 0 for the tile /
 * row-split kernels (empty rows zero-filled by a side-stream kernel).  For
 * bench.py's roofline bookkeeping (no reference counterpart). */
spmk_status spmk_spmm_path(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg, int64_t n,
                           int* path);

/* ------------------------------------------------------------ iterative SpMV */
/* PageRank-style driver support (BASELINE cfg5; no reference counterpart —
 * the reference has no iterative driver).  With M == K the
 * column counts are the out-degrees of the transposed graph. */
/* d_counts[K] = nonzeros per column (deterministic integer atomics). */
spmk_status spmk_column_counts(spmk_csr_t a, int32_t* d_counts, void* stream);
/* values[e] = 1 / d_counts[col[e]] (column-stochastic A); the handle must own
 * its values. */
spmk_status spmk_csr_values_inv_column_counts(spmk_csr_t a, const int32_t* d_counts,
                                              void* stream);
/* doubles of d_scratch the two calls below need */
int64_t spmk_pagerank_scratch_doubles(void);
/* d_state[3] = {base, 0, dangling mass of d_r[0..m)} with
 * base = (1-alpha)/m_total + alpha*dangling/m_total. */
spmk_status spmk_pagerank_init(const float* d_r, const int32_t* d_counts, int64_t m,
                               int64_t m_total, double alpha, double* d_state,
                               double* d_scratch, void* stream);
/* r[i] = alpha*y[i] + d_state[0] for i < m; then d_state = {next base (from the
 * local dangling mass), sum|r_new - r_old|, dangling mass}; d_hist[t] = l1
 * when d_hist is not NULL.  Reductions are fixed-order (bit-reproducible). */
spmk_status spmk_pagerank_step(const float* d_y, float* d_r, const int32_t* d_counts,
                               int64_t m, int64_t m_total, double alpha, double* d_state,
                               double* d_scratch, double* d_hist, int32_t t, void* stream);

/* Fused update + exchange for the row-partitioned iterative SpMV (one rank
 * of a multi-GPU run): for i < m, x_next[row0 + i] = alpha*y[i] + d_state[0]
 * is stored into every buffer of peer_x_next[0..npeers) (HOST array of device
 * pointers: this GPU's own x_next and its peers' buffers mapped with
 * spmk_ipc_open, written with P2P stores over NVLink), with the same
 * fixed-order reductions as spmk_pagerank_step (residual against d_x_cur,
 * dangling mass; d_counts and both x vectors are indexed globally).  npeers
 * <= 8.  The replicas are complete once every rank's call has finished. */
spmk_status spmk_pagerank_step_p2p(const float* d_y, const float* d_x_cur,
                                   float* const* peer_x_next, int32_t npeers,
                                   const int32_t* d_counts, int64_t row0, int64_t m,
                                   int64_t m_total, double alpha, double* d_state,
                                   double* d_scratch, void* stream);
/* CUDA IPC for the peer buffers above: 64-byte handle of a device
 * allocation, open a peer's handle (lazy peer access), close it. */
spmk_status spmk_ipc_handle(const void* d_ptr, void* handle64);
spmk_status spmk_ipc_open(const void* handle64, void** d_ptr);
spmk_status spmk_ipc_close(void* d_ptr);

/* ------------------------------------------------------------ multi-GPU */
/* One process (or thread) per GPU over NCCL (NVLink 5 / NVSwitch), for the
 * row-partitioned configs.  Replaces the reference's
 * single-process parallel substrate (ThreadPool, thread_pool.hpp:51-76, whose
 * static partition kernels.hpp:124-129 is applied here to nonzeros): A is cut
 * into equal-nnz row slices (spmk_row_slices), X is replicated once, every
 * rank computes its own Y slice with the per-slice rule — no collective in
 * the SpMM — and only the iterative driver exchanges Y.  NCCL is loaded at
 * run time (libnccl.so.2); without it these calls return SPMK_ENCCL and the
 * rest of the library is unaffected.  Collectives are enqueued on `stream`
 * (asynchronous) and must be issued in the same order on every rank. */
typedef struct spmk_mg_s* spmk_mg_t;
#define SPMK_MG_UNIQUE_ID_BYTES 128
/* NCCL present?  nccl_version (may be NULL) receives ncclGetVersion. */
spmk_status spmk_mg_available(int* nccl_version);
/* Rank 0 creates the id and ships it to the others out of band. */
spmk_status spmk_mg_unique_id(void* id128);
/* Collective over all ranks (ncclCommInitRank), bound to `device`. */
spmk_status spmk_mg_init(const void* id128, int nranks, int rank, int device,
                         spmk_mg_t* out);
spmk_status spmk_mg_destroy(spmk_mg_t mg);
spmk_status spmk_mg_info(spmk_mg_t mg, int* rank, int* nranks, int* device);
/* This rank's equal-nnz row slice of `full` (bounds = spmk_row_slices(full,
 * nranks)) as a rebased handle on the communicator's device; row_begin /
 * row_end (may be NULL) receive its global rows. */
spmk_status spmk_mg_slice(spmk_mg_t mg, spmk_csr_t full, spmk_csr_t* slice,
                          int64_t* row_begin, int64_t* row_end);
/* In-place broadcast of `count` floats from `root` (X replication). */
spmk_status spmk_mg_broadcast(spmk_mg_t mg, float* d_buf, int64_t count,
                              int root, void* stream);
/* In-place all-gather of X cut into nranks equal chunks of `chunk` floats
 * (rank g owns d_x[g*chunk, (g+1)*chunk)): each rank uploads 1/nranks of a
 * host X over its own PCIe link, NVLink assembles the rest.  d_x holds
 * nranks*chunk floats (pad the tail). */
spmk_status spmk_mg_allgather_x(spmk_mg_t mg, float* d_x, int64_t chunk,
                                void* stream);
/* Y exchange of the iterative driver: rank g's rows
 * [row_bounds[g], row_bounds[g+1]) of the row-major (rows x n) d_y are
 * broadcast from g to all ranks, in place, as ONE NCCL group (unequal
 * slices: no padded all-gather).  row_bounds is a HOST array of nranks+1. */
spmk_status spmk_mg_allgather_rows(spmk_mg_t mg, float* d_y,
                                   const int64_t* row_bounds, int64_t n,
                                   void* stream);
/* In-place sum all-reduces (PageRank residual / dangling mass; counts). */
spmk_status spmk_mg_allreduce_f64(spmk_mg_t mg, double* d_buf, int64_t count,
                                  void* stream);
spmk_status spmk_mg_allreduce_i32(spmk_mg_t mg, int32_t* d_buf, int64_t count,
                                  void* stream);
/* Device barrier (a 4-byte all-reduce), then synchronizes `stream`. */
spmk_status spmk_mg_barrier(spmk_mg_t mg, void* stream);
/* This rank's SpMM: spmk_spmm_auto on its slice (per-slice features and
 * rule); no collective — X must already be replicated. */
spmk_status spmk_mg_spmm(spmk_mg_t mg, spmk_csr_t slice, const spmk_thresholds* t,
                         const spmk_kernel_config* cfg, const float* d_x,
                         int64_t n, float* d_y, void* stream,
                         spmk_kernel_id* chosen);

/* ------------------------------------------------------------ generators */
/* generate_rmat<float> (rmat.hpp:61-88 + csr.hpp:123-164) on the device,
 * bit-identical to the reference (counter form of SplitMix64): returns a
 * handle owning int32 rowPtr/colIdx and values = 1. */
spmk_status spmk_generate_rmat(uint32_t scale, uint64_t edge_factor, double a,
                               double b, double c, double d, uint64_t seed,
                               int device, spmk_csr_t* out);
/* make_dense<float> (corpus.hpp:116-122) on the device: d_out[rows*cols]. */
spmk_status spmk_make_dense(int64_t rows, int64_t cols, uint64_t seed,
                            float* d_out, void* stream);
/* The same into HOST memory (generated on `device`, copied back). */
spmk_status spmk_make_dense_host(int64_t rows, int64_t cols, uint64_t seed,
                                 float* out, int device);

/* ------------------------------------------------------------ harness */
/* measure_kernel (bench.hpp:65-98) on the device: X = make_dense(num_cols, n,
 * x_seed) in HBM, `warmup` untimed calls, then `repeats` calls each bracketed
 * by CUDA events (a 256 MiB buffer written before each when flush_l2), median
 * seconds; `correct` (may be NULL) = matches_oracle (bench.hpp:47-58): every
 * |y - o| <= kernel_tolerance(max_row_nnz) * max(1, |o|) against the fp64
 * product o computed by an independent row-parallel device kernel. */
spmk_status spmk_measure_kernel(spmk_csr_t a, spmk_kernel_id id,
                                const spmk_kernel_config* cfg, int64_t n,
                                uint64_t x_seed, int64_t repeats, int64_t warmup,
                                int flush_l2, double* median_seconds,
                                int* correct);

#ifdef __cplusplus
}
#endif
#endif /* SPMK_CAPI_H */
