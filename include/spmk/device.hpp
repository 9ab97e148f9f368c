// spmk/device.hpp — resident-operand API (new; no reference counterpart).
//
// The reference's spmm() takes host operands and returns Y by value
// (kernels.hpp:457-464); the drop-in keeps that shape, paying an upload per
// call.  DeviceCsr is the handle form for repeated calls: A stays resident in
// HBM (int32 indices), X and Y are caller-owned device buffers, and every
// call is asynchronous on the caller's stream.
#pragma once

#include <cstdint>
#include <utility>

#include "spmk/kernels.hpp"
#include "spmk/selector.hpp"

namespace spmk {

class DeviceCsr {
 public:
  DeviceCsr() = default;
  explicit DeviceCsr(const CsrMatrix<float>& a, int device = current_device()) {
    detail::check_status(spmk_csr_create(a.num_rows, a.num_cols, a.nnz(), a.row_ptr.data(),
                                         a.col_idx.data(), a.values.data(), device, &h_),
                         "DeviceCsr");
  }
  DeviceCsr(const DeviceCsr&) = delete;
  DeviceCsr& operator=(const DeviceCsr&) = delete;
  DeviceCsr(DeviceCsr&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  DeviceCsr& operator=(DeviceCsr&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  ~DeviceCsr() { reset(); }

  // generate_rmat<float> on the device, bit-identical to rmat.hpp:61-88.
  static DeviceCsr rmat(std::uint32_t scale, std::uint64_t edge_factor, double a, double b, double c,
                        double d, std::uint64_t seed, int device = current_device()) {
    DeviceCsr out;
    detail::check_status(spmk_generate_rmat(scale, edge_factor, a, b, c, d, seed, device, &out.h_),
                         "DeviceCsr::rmat");
    return out;
  }

  spmk_csr_t handle() const { return h_; }
  // Back to the reference's host layout (int64 indices).
  CsrMatrix<float> download() const {
    const Info i = info();
    CsrMatrix<float> a;
    a.num_rows = i.num_rows;
    a.num_cols = i.num_cols;
    a.row_ptr.assign(static_cast<std::size_t>(i.num_rows) + 1, 0);
    a.col_idx.assign(static_cast<std::size_t>(i.nnz), 0);
    a.values.assign(static_cast<std::size_t>(i.nnz), 0.f);
    detail::check_status(spmk_csr_download(h_, a.row_ptr.data(), a.col_idx.data(), a.values.data()), "download");
    return a;
  }
  Index num_rows() const { return info().num_rows; }
  Index num_cols() const { return info().num_cols; }
  Index nnz() const { return info().nnz; }

  MatrixFeatures features() const {
    spmk_features f;
    detail::check_status(spmk_features_compute(h_, &f), "features");
    return MatrixFeatures{f.avg_row, f.stdv_row, f.cv, f.num_rows, f.nnz};
  }
  KernelId select(std::size_t n, const SelectorThresholds& t = {}) const {
    const spmk_thresholds ct{t.n_parallel_max, t.t_parallel_avg, t.t_cv};
    spmk_kernel_id id;
    detail::check_status(spmk_select_for(h_, n, &ct, &id), "select");
    return kernel_from_index(static_cast<std::size_t>(id));
  }
  // Y (device, num_rows x n) = A * X (device, num_cols x n), async on stream.
  void spmm(KernelId id, const float* d_x, Index n, float* d_y, void* stream = nullptr,
            const KernelConfig& cfg = {}) const {
    const spmk_kernel_config c = detail::to_c(cfg);
    detail::check_status(
        spmk_spmm(h_, static_cast<spmk_kernel_id>(kernel_index(id)), &c, d_x, n, d_y, stream), "spmm");
  }
  // Host X in, host Y out (synchronous).
  DenseMatrix<float> spmm(KernelId id, const DenseMatrix<float>& x, const KernelConfig& cfg = {}) const {
    if (x.num_rows != num_cols()) throw Error("dimension mismatch");
    DenseMatrix<float> y = DenseMatrix<float>::zero(num_rows(), x.num_cols);
    const spmk_kernel_config c = detail::to_c(cfg);
    detail::check_status(spmk_spmm_host(h_, static_cast<spmk_kernel_id>(kernel_index(id)), &c,
                                        x.data.data(), x.num_cols, y.data.data(), nullptr),
                         "spmm");
    return y;
  }

 private:
  struct Info {
    int64_t num_rows = 0, num_cols = 0, nnz = 0, max_row = 0, empty = 0;
  };
  Info info() const {
    Info i;
    detail::check_status(spmk_csr_info(h_, &i.num_rows, &i.num_cols, &i.nnz, &i.max_row, &i.empty), "info");
    return i;
  }
  void reset() {
    if (h_) spmk_csr_destroy(h_);
    h_ = nullptr;
  }
  spmk_csr_t h_ = nullptr;
};

}  // namespace spmk
