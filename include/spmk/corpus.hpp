// spmk/corpus.hpp — drop-in for the parts of
// /root/reference/proj/include/spmk/corpus.hpp the selection harness uses:
// NamedMatrix (corpus.hpp:12-13) and make_dense<float> (corpus.hpp:116-122),
// generated on the device (spmk_make_dense_host: the same SplitMix64 stream,
// bit-identical values in [-1, 1]).  The reference's pinned acceptance corpus
// (pinned_rmat_corpus / edge_case_corpus / full_corpus) is test input and is
// not part of this header; build R-MAT corpora with generate_rmat.
#pragma once

#include <cstdint>
#include <string>
#include <type_traits>
#include <utility>

#include "spmk/csr.hpp"
#include "spmk/kernels.hpp"

namespace spmk {

template <typename T>
using NamedMatrix = std::pair<std::string, CsrMatrix<T>>;

template <typename T>
DenseMatrix<T> make_dense(Index rows, Index cols, std::uint64_t seed) {
  static_assert(std::is_same_v<T, float>, "spmk (B200): make_dense is fp32 only");
  if (rows < 0 || cols < 0) throw Error("negative dimension");
  DenseMatrix<T> x = DenseMatrix<T>::zero(rows, cols);
  detail::check_status(spmk_make_dense_host(rows, cols, seed, x.data.data(), current_device()),
                       "make_dense");
  return x;
}

}  // namespace spmk
