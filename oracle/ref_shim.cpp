// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/spmk/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libspmk_ref.so.  Used by tests/ (as a checker), by
// tests/golden/make_golden.py (to pin golden vectors) and by bench.py's
// cpu_baseline / --impl reference leg (the reference's own multithreaded CPU
// path, timed).  Nothing here is reached from paper_2106_16064_b200/.
//
// Build flags follow proj/CMakeLists.txt:1-17 (C++20, Release, no -march), so
// the reference's fp32 kernels keep separate mul/add roundings (no FMA
// contraction) — SURVEY.md §8c "Build-flag pin".
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "spmk/spmk.hpp"

using namespace spmk;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

struct RefCsr {
  CsrMatrix<float> a;
  std::string name;
};

KernelId id_of(int idx) {
  // kernel_index numbering, kernels.hpp:47-50: 2*seq + ws
  switch (idx) {
    case 0: return kParRowSplit;
    case 1: return kParBalanced;
    case 2: return kSeqRowSplit;
    default: return kSeqBalanced;
  }
}

KernelConfig cfg_of(int64_t lane_width, int64_t vdl_group, int64_t seq_chunk,
                    int64_t worker_count) {
  KernelConfig c;
  c.lane_width = static_cast<std::size_t>(lane_width);
  c.vdl_group = static_cast<std::size_t>(vdl_group);
  c.seq_chunk = static_cast<std::size_t>(seq_chunk);
  c.worker_count = static_cast<std::size_t>(worker_count);
  return c;
}

std::vector<RefCsr*>* g_corpus = nullptr;
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// rmat.hpp:61-88
void* ref_generate_rmat(uint32_t scale, uint64_t edge_factor, double a,
                        double b, double c, double d, uint64_t seed) {
  try {
    RmatParams p;
    p.scale = scale;
    p.edge_factor = edge_factor;
    p.skew = {a, b, c, d};
    p.seed = seed;
    auto* h = new RefCsr;
    h->a = generate_rmat<float>(p);
    return h;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// csr.hpp:123-164 (sort + duplicate sum), from COO triples.
void* ref_csr_from_coo(int64_t m, int64_t k, int64_t count, const int64_t* rows,
                       const int64_t* cols, const float* vals) {
  try {
    std::vector<Triple<float>> t(static_cast<std::size_t>(count));
    for (int64_t i = 0; i < count; ++i) t[i] = {rows[i], cols[i], vals[i]};
    auto* h = new RefCsr;
    h->a = csr_from_coo<float>(std::move(t), m, k);
    return h;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// Wrap existing canonical CSR arrays (validated with csr.hpp:95-119).
void* ref_csr_from_arrays(int64_t m, int64_t k, int64_t nnz,
                          const int64_t* row_ptr, const int64_t* col_idx,
                          const float* val, int do_validate) {
  try {
    auto* h = new RefCsr;
    h->a.num_rows = m;
    h->a.num_cols = k;
    h->a.row_ptr.assign(row_ptr, row_ptr + m + 1);
    h->a.col_idx.assign(col_idx, col_idx + nnz);
    h->a.values.assign(val, val + nnz);
    if (do_validate) validate(h->a);
    return h;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// Same, from the device format (int32 indices), widening to Index=int64.
void* ref_csr_from_arrays32(int64_t m, int64_t k, int64_t nnz,
                            const int32_t* row_ptr, const int32_t* col_idx,
                            const float* val) {
  auto* h = new RefCsr;
  h->a.num_rows = m;
  h->a.num_cols = k;
  h->a.row_ptr.assign(row_ptr, row_ptr + m + 1);
  h->a.col_idx.assign(col_idx, col_idx + nnz);
  h->a.values.assign(val, val + nnz);
  return h;
}

void ref_csr_free(void* h) { delete static_cast<RefCsr*>(h); }
int64_t ref_csr_rows(void* h) { return static_cast<RefCsr*>(h)->a.num_rows; }
int64_t ref_csr_cols(void* h) { return static_cast<RefCsr*>(h)->a.num_cols; }
int64_t ref_csr_nnz(void* h) { return static_cast<RefCsr*>(h)->a.nnz(); }
int64_t ref_csr_max_row(void* h) {
  return static_cast<RefCsr*>(h)->a.max_row_nnz();
}
const char* ref_csr_name(void* h) {
  return static_cast<RefCsr*>(h)->name.c_str();
}
void ref_csr_copy(void* h, int64_t* row_ptr, int64_t* col_idx, float* val) {
  const auto& a = static_cast<RefCsr*>(h)->a;
  if (row_ptr) std::memcpy(row_ptr, a.row_ptr.data(), a.row_ptr.size() * 8);
  if (col_idx) std::memcpy(col_idx, a.col_idx.data(), a.col_idx.size() * 8);
  if (val) std::memcpy(val, a.values.data(), a.values.size() * 4);
}

// corpus.hpp:108-113 — the 27 pinned R-MAT matrices + 5 edge cases.
int64_t ref_full_corpus(uint64_t seed) {
  try {
    if (g_corpus) {
      for (auto* h : *g_corpus) delete h;
      delete g_corpus;
    }
    g_corpus = new std::vector<RefCsr*>;
    for (auto& [name, a] : full_corpus<float>(seed)) {
      auto* h = new RefCsr;
      h->a = std::move(a);
      h->name = name;
      g_corpus->push_back(h);
    }
    return static_cast<int64_t>(g_corpus->size());
  } catch (const std::exception& e) {
    return fail(e);
  }
}
void* ref_corpus_get(int64_t i) { return (*g_corpus)[i]; }

// corpus.hpp:116-122
void ref_make_dense(int64_t rows, int64_t cols, uint64_t seed, float* out) {
  auto x = make_dense<float>(rows, cols, seed);
  std::memcpy(out, x.data.data(), x.data.size() * 4);
}

// kernels.hpp:457-464 — the reference's own (multithreaded) CPU kernels.
int ref_spmm(void* h, int kernel_idx, int64_t lane_width, int64_t vdl_group,
             int64_t seq_chunk, int64_t worker_count, const float* x, int64_t n,
             float* y) {
  try {
    const auto& a = static_cast<RefCsr*>(h)->a;
    DenseMatrix<float> xm;
    xm.num_rows = a.num_cols;
    xm.num_cols = n;
    xm.data.assign(x, x + a.num_cols * n);
    auto ym = spmm(id_of(kernel_idx), a, xm,
                   cfg_of(lane_width, vdl_group, seq_chunk, worker_count));
    std::memcpy(y, ym.data.data(), ym.data.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Same call, timed exactly like bench.hpp:65-98 measure_kernel (the DenseMatrix
// X is built once outside; Y allocation+zero inside the timed call).  Returns
// seconds of the median of `repeats` after `warmup`.
double ref_time_spmm(void* h, int kernel_idx, const float* x, int64_t n,
                     int64_t repeats, int64_t warmup, int64_t worker_count) {
  try {
    const auto& a = static_cast<RefCsr*>(h)->a;
    DenseMatrix<float> xm;
    xm.num_rows = a.num_cols;
    xm.num_cols = n;
    xm.data.assign(x, x + a.num_cols * n);
    KernelConfig cfg;
    cfg.worker_count = static_cast<std::size_t>(worker_count);
    using Clock = std::chrono::steady_clock;
    for (int64_t i = 0; i < warmup; ++i) (void)spmm(id_of(kernel_idx), a, xm, cfg);
    std::vector<double> t;
    for (int64_t i = 0; i < repeats; ++i) {
      auto t0 = Clock::now();
      auto y = spmm(id_of(kernel_idx), a, xm, cfg);
      auto t1 = Clock::now();
      t.push_back(std::chrono::duration<double>(t1 - t0).count());
    }
    return detail::median(t);
  } catch (const std::exception& e) {
    fail(e);
    return -1.0;
  }
}

// csr.hpp:185-205 (fp64 ground truth, single thread).
int ref_oracle_spmm(void* h, const float* x, int64_t n, double* y) {
  try {
    const auto& a = static_cast<RefCsr*>(h)->a;
    DenseMatrix<float> xm;
    xm.num_rows = a.num_cols;
    xm.num_cols = n;
    xm.data.assign(x, x + a.num_cols * n);
    auto ym = oracle_spmm(a, xm);
    std::memcpy(y, ym.data.data(), ym.data.size() * 8);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// csr.hpp:166-181.  out = {avg_row, stdv_row, cv}
int ref_extract_features(void* h, double* out3) {
  try {
    auto f = extract_features(static_cast<RefCsr*>(h)->a);
    out3[0] = f.avg_row;
    out3[1] = f.stdv_row;
    out3[2] = f.cv;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// selector.hpp:28-34 -> kernel_index
int ref_select_kernel(double avg, double stdv, double cv, int64_t num_rows,
                      int64_t nnz, uint64_t n, uint64_t n_parallel_max,
                      double t_parallel_avg, double t_cv) {
  MatrixFeatures f;
  f.avg_row = avg;
  f.stdv_row = stdv;
  f.cv = cv;
  f.num_rows = num_rows;
  f.nnz = nnz;
  SelectorThresholds t{static_cast<std::size_t>(n_parallel_max),
                       t_parallel_avg, t_cv};
  return static_cast<int>(kernel_index(select_kernel(f, n, t)));
}

// kernels.hpp:133-149.  elem_row may be null (only num_chunks returned).
int64_t ref_plan_balanced(void* h, int64_t chunk, int64_t* elem_row) {
  try {
    auto p = plan_balanced(static_cast<RefCsr*>(h)->a, chunk);
    if (elem_row) std::memcpy(elem_row, p.elem_row.data(), p.elem_row.size() * 8);
    return p.num_chunks;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// kernels.hpp:124-129
void ref_partition(int64_t items, int64_t parts, int64_t w, int64_t* lo,
                   int64_t* hi) {
  auto [a, b] = detail::partition(items, static_cast<std::size_t>(parts),
                                  static_cast<std::size_t>(w));
  *lo = a;
  *hi = b;
}

// reduction.hpp:75-86 on float lanes (kPadRow = INT64_MAX).
int ref_conditional_scan(int64_t width, int64_t comps, const int64_t* rows,
                         float* vals) {
  try {
    LaneChunk<float> c;
    c.width = static_cast<std::size_t>(width);
    c.comps = static_cast<std::size_t>(comps);
    c.row_idx.assign(rows, rows + width);
    c.values.assign(vals, vals + width * comps);
    auto out = conditional_scan(c);
    std::memcpy(vals, out.values.data(), out.values.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// kernels.hpp:67-79 counters: run the reference kernel with stats attached.
int ref_kernel_stats(void* h, int kernel_idx, int64_t lane_width,
                     int64_t vdl_group, const float* x, int64_t n,
                     uint64_t* lane_multiplies, uint64_t* scan_ops) {
  try {
    const auto& a = static_cast<RefCsr*>(h)->a;
    DenseMatrix<float> xm;
    xm.num_rows = a.num_cols;
    xm.num_cols = n;
    xm.data.assign(x, x + a.num_cols * n);
    KernelStats st;
    KernelConfig cfg = cfg_of(lane_width, vdl_group, 256, 1);
    cfg.stats = &st;
    (void)spmm(id_of(kernel_idx), a, xm, cfg);
    *lane_multiplies = st.lane_multiplies.load();
    *scan_ops = st.scan_ops.load();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

double ref_kernel_tolerance(int64_t max_row_nnz) {
  return kernel_tolerance<float>(max_row_nnz);
}

int64_t ref_hardware_concurrency() {
  return static_cast<int64_t>(ThreadPool::default_workers());
}

}  // extern "C"
