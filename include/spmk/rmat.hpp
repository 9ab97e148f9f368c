// spmk/rmat.hpp — drop-in for /root/reference/proj/include/spmk/rmat.hpp.
//
// RmatSkew / RmatParams / validate keep the reference's fields, defaults and
// messages (rmat.hpp:31-59).  generate_rmat<float> (rmat.hpp:61-88) runs on
// the device (spmk_generate_rmat: counter form of the same SplitMix64 stream,
// device sort and deduplication — bit-identical CSR, pinned by the golden
// digests up to the full 2^25-node BASELINE graphs) and is downloaded into
// the reference's host CsrMatrix layout.  T = double is unsupported.
#pragma once

#include <cstdint>
#include <type_traits>

#include "spmk/csr.hpp"
#include "spmk/device.hpp"
#include "spmk/error.hpp"

namespace spmk {

struct RmatSkew {
  double a = 0.57;
  double b = 0.19;
  double c = 0.19;
  double d = 0.05;
};

struct RmatParams {
  std::uint32_t scale = 10;       // dimension 2^scale
  std::uint64_t edge_factor = 8;  // target nnz = edge_factor * 2^scale
  RmatSkew skew;
  std::uint64_t seed = 1;
};

// The checks run in the library (same messages as rmat.hpp:45-59).
inline void validate(const RmatParams& p) {
  if (p.scale < 1 || p.scale > 30) throw Error("rmat scale must be in [1, 30]");
  if (p.edge_factor < 1) throw Error("rmat edge_factor must be >= 1");
  const double probs[4] = {p.skew.a, p.skew.b, p.skew.c, p.skew.d};
  double sum = 0.0;
  for (double q : probs) {
    if (q < 0.0 || q > 1.0) throw Error("rmat quadrant probability outside [0, 1]");
    sum += q;
  }
  if (sum < 1.0 - 1e-9 || sum > 1.0 + 1e-9) throw Error("rmat quadrant probabilities must sum to 1");
}

template <typename T>
CsrMatrix<T> generate_rmat(const RmatParams& p) {
  static_assert(std::is_same_v<T, float>, "spmk (B200): generate_rmat is fp32 only");
  validate(p);
  DeviceCsr d = DeviceCsr::rmat(p.scale, p.edge_factor, p.skew.a, p.skew.b, p.skew.c, p.skew.d, p.seed);
  return d.download();
}

}  // namespace spmk
