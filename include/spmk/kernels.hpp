// spmk/kernels.hpp — drop-in for /root/reference/proj/include/spmk/kernels.hpp.
//
// Same names, types and signatures as the reference (kernels.hpp:17-472) so
// callers recompile unchanged; the four spmm_* entry points run the sm_100a
// kernels of libspmk_b200.so through the C ABI (include/spmk_capi.h):
//   host CSR + host X  --spmk_spmm_csr_host-->  upload, narrow to int32,
//   device kernel of the same KernelId, download Y.
// Results are bit-identical to the reference's fp32 kernel of the same
// KernelId at the same lane_width / seq_chunk.
//
// T = float only.  T = double throws spmk::Error ("unsupported"): there is no
// CPU fallback on this path.  KernelConfig::worker_count is accepted and
// ignored (the CUDA grid replaces the ThreadPool); KernelConfig::stats is
// filled analytically with the reference's lockstep formulas.
#pragma once

#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "spmk/csr.hpp"
#include "spmk/error.hpp"

namespace spmk {

enum class Reduction { Parallel, Sequential };
enum class Balancing { RowSplit, NonzeroSplit };

struct KernelId {
  Reduction reduction;
  Balancing balancing;
  bool operator==(const KernelId&) const = default;
};

inline constexpr KernelId kParRowSplit{Reduction::Parallel, Balancing::RowSplit};
inline constexpr KernelId kParBalanced{Reduction::Parallel, Balancing::NonzeroSplit};
inline constexpr KernelId kSeqRowSplit{Reduction::Sequential, Balancing::RowSplit};
inline constexpr KernelId kSeqBalanced{Reduction::Sequential, Balancing::NonzeroSplit};
inline constexpr std::array<KernelId, 4> kAllKernels{kParRowSplit, kParBalanced, kSeqRowSplit,
                                                     kSeqBalanced};

// kernels.hpp:47-50 numbering == spmk_kernel_id
inline std::size_t kernel_index(KernelId id) {
  return (id.reduction == Reduction::Sequential ? 2u : 0u) +
         (id.balancing == Balancing::NonzeroSplit ? 1u : 0u);
}
inline KernelId kernel_from_index(std::size_t i) { return kAllKernels.at(i); }
inline std::string kernel_name(KernelId id) {
  return spmk_kernel_name(static_cast<spmk_kernel_id>(kernel_index(id)));
}
inline KernelId parse_kernel(const std::string& name) {
  spmk_kernel_id out;
  if (spmk_parse_kernel(name.c_str(), &out) != SPMK_OK) throw Error("unknown kernel name: " + name);
  return kernel_from_index(static_cast<std::size_t>(out));
}

struct BalancedPlan {
  std::vector<Index> elem_row;
  Index chunk_size = 0;
  Index num_chunks = 0;
};

struct KernelStats {
  std::atomic<std::uint64_t> lane_multiplies{0};
  std::atomic<std::uint64_t> scan_ops{0};
  void reset() {
    lane_multiplies = 0;
    scan_ops = 0;
  }
};

// kernels.hpp:81-87: same fields, same order (designated initializers such as
// {.seq_chunk = 16} keep compiling).
struct KernelConfig {
  std::size_t lane_width = 32;
  std::size_t vdl_group = 0;
  std::size_t seq_chunk = 256;
  std::size_t worker_count = 0;
  KernelStats* stats = nullptr;
};

// Device the host-operand entry points run on (default: $SPMK_DEVICE or 0).
inline int& current_device() {
  static int dev = [] {
    const char* v = std::getenv("SPMK_DEVICE");
    return v ? std::atoi(v) : 0;
  }();
  return dev;
}
inline void set_device(int dev) { current_device() = dev; }

namespace detail {

inline bool is_pow2(std::size_t v) { return v != 0 && (v & (v - 1)) == 0; }

inline spmk_kernel_config to_c(const KernelConfig& cfg) {
  return spmk_kernel_config{cfg.lane_width, cfg.vdl_group, cfg.seq_chunk, cfg.worker_count};
}

// kernels.hpp:91-100
inline void check_config(const KernelConfig& cfg) {
  const spmk_kernel_config c = to_c(cfg);
  if (spmk_check_config(&c) != SPMK_OK) throw Error(spmk_last_error());
}

// kernels.hpp:103-109
template <typename T>
void check_dims(const CsrMatrix<T>& a, const DenseMatrix<T>& x) {
  if (a.num_cols != x.num_rows)
    throw Error("dimension mismatch: A is " + std::to_string(a.num_rows) + "x" +
                std::to_string(a.num_cols) + ", X has " + std::to_string(x.num_rows) + " rows");
}

// kernels.hpp:116-121
inline Index effective_group(const KernelConfig& cfg, Index n) {
  if (cfg.vdl_group != 0) return static_cast<Index>(cfg.vdl_group);
  return n >= 4 ? 4 : n >= 2 ? 2 : 1;
}

// kernels.hpp:124-129
inline std::pair<Index, Index> partition(Index items, std::size_t parts, std::size_t w) {
  int64_t lo = 0, hi = 0;
  spmk_partition(items, static_cast<int64_t>(parts), static_cast<int64_t>(w), &lo, &hi);
  return {lo, hi};
}

template <typename T>
DenseMatrix<T> run(KernelId id, const CsrMatrix<T>& a, const DenseMatrix<T>& x,
                   const KernelConfig& cfg) {
  check_config(cfg);
  check_dims(a, x);
  if constexpr (!std::is_same_v<T, float>) {
    throw Error("spmm: only T=float runs on the B200 device path (no CPU fallback)");
  } else {
    DenseMatrix<float> y = DenseMatrix<float>::zero(a.num_rows, x.num_cols);
    if (x.num_cols == 0 || a.num_rows == 0) return y;
    const spmk_kernel_config c = to_c(cfg);
    const auto kid = static_cast<spmk_kernel_id>(kernel_index(id));
    if (cfg.stats) {
      spmk_csr_t h = nullptr;
      check_status(spmk_csr_create(a.num_rows, a.num_cols, a.nnz(), a.row_ptr.data(), a.col_idx.data(),
                                   a.values.data(), current_device(), &h),
                   "spmm");
      std::uint64_t lm = 0, so = 0;
      spmk_status st = spmk_kernel_stats(h, kid, &c, x.num_cols, &lm, &so);
      if (st == SPMK_OK) st = spmk_spmm_host(h, kid, &c, x.data.data(), x.num_cols, y.data.data(), nullptr);
      spmk_csr_destroy(h);
      check_status(st, "spmm");
      cfg.stats->lane_multiplies += lm;
      cfg.stats->scan_ops += so;
      return y;
    }
    check_status(spmk_spmm_csr_host(a.num_rows, a.num_cols, a.nnz(), a.row_ptr.data(), a.col_idx.data(),
                                    a.values.data(), kid, &c, x.data.data(), x.num_cols, y.data.data(),
                                    current_device()),
                 "spmm");
    return y;
  }
}

}  // namespace detail

// kernels.hpp:133-149 — the COO expansion the reference's balanced kernels
// consume.  The device kernels never materialise it (they binary-search
// rowPtr per tile, spmk_plan); this host form keeps the reference API.
inline BalancedPlan plan_balanced(Index nnz, const std::vector<Index>& row_ptr, Index num_rows,
                                  Index chunk_size) {
  if (chunk_size < 1) throw Error("chunk_size must be >= 1");
  BalancedPlan p;
  p.chunk_size = chunk_size;
  p.elem_row.resize(static_cast<std::size_t>(nnz));
  for (Index r = 0; r < num_rows; ++r)
    std::fill(p.elem_row.begin() + row_ptr[r], p.elem_row.begin() + row_ptr[r + 1], r);
  p.num_chunks = (nnz + chunk_size - 1) / chunk_size;
  return p;
}
template <typename T>
BalancedPlan plan_balanced(const CsrMatrix<T>& a, Index chunk_size) {
  return plan_balanced(a.nnz(), a.row_ptr, a.num_rows, chunk_size);
}

// The four variants (kernels.hpp:157, :232, :339, :384) and the dispatcher
// (kernels.hpp:457-464).
template <typename T>
DenseMatrix<T> spmm_par_rowsplit(const CsrMatrix<T>& a, const DenseMatrix<T>& x,
                                 const KernelConfig& cfg = {}) {
  return detail::run(kParRowSplit, a, x, cfg);
}
template <typename T>
DenseMatrix<T> spmm_par_balanced(const CsrMatrix<T>& a, const DenseMatrix<T>& x,
                                 const KernelConfig& cfg = {}) {
  return detail::run(kParBalanced, a, x, cfg);
}
template <typename T>
DenseMatrix<T> spmm_seq_rowsplit(const CsrMatrix<T>& a, const DenseMatrix<T>& x,
                                 const KernelConfig& cfg = {}) {
  return detail::run(kSeqRowSplit, a, x, cfg);
}
template <typename T>
DenseMatrix<T> spmm_seq_balanced(const CsrMatrix<T>& a, const DenseMatrix<T>& x,
                                 const KernelConfig& cfg = {}) {
  return detail::run(kSeqBalanced, a, x, cfg);
}
template <typename T>
DenseMatrix<T> spmm(KernelId id, const CsrMatrix<T>& a, const DenseMatrix<T>& x,
                    const KernelConfig& cfg = {}) {
  return detail::run(id, a, x, cfg);
}

// kernels.hpp:468-472
template <typename T>
double kernel_tolerance(Index max_row_nnz) {
  const double eps = sizeof(T) == 4 ? 1e-5 : 1e-12;
  return eps * std::log2(static_cast<double>(max_row_nnz) + 2.0);
}

}  // namespace spmk
