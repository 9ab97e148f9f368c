// Drop-in C++ API tests: the reference's own KATs (proj/tests/test_kernels.cpp,
// test_selector.cpp, test_core.cpp) recompiled against include/spmk/*.hpp and
// run on the device path (T=float — the reference instantiates most of them
// with T=double, which this path rejects by design).
//
//   ./test_dropin          every case (needs a GPU)
//   ./test_dropin --host   host-only cases (selector, config, names, plan)
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "spmk/spmk.hpp"

using namespace spmk;

namespace {

int g_fail = 0, g_checks = 0;
struct Case {
  const char* name;
  bool gpu;
  std::function<void()> fn;
};
std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Reg {
  Reg(const char* n, bool g, std::function<void()> f) { cases().push_back({n, g, std::move(f)}); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name, gpu) \
  static void CAT(tc_, __LINE__)(); \
  static Reg CAT(reg_, __LINE__)(name, gpu, CAT(tc_, __LINE__)); \
  static void CAT(tc_, __LINE__)()
#define CHECK(x)                                                         \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(x)) {                                                          \
      ++g_fail;                                                          \
      std::fprintf(stderr, "  FAIL %s:%d: %s\n", __FILE__, __LINE__, #x); \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, T) \
  do {                           \
    bool thrown = false;         \
    try {                        \
      (void)(expr);              \
    } catch (const T&) {         \
      thrown = true;             \
    }                            \
    CHECK(thrown);               \
  } while (0)

// make_dense (corpus.hpp:116-122): element i = float(2u-1), u the (i+1)-th
// SplitMix64 unit draw of `seed`.
DenseMatrix<float> make_dense(Index rows, Index cols, std::uint64_t seed) {
  DenseMatrix<float> d = DenseMatrix<float>::zero(rows, cols);
  for (std::size_t i = 0; i < d.data.size(); ++i) {
    std::uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    d.data[i] = static_cast<float>(2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0);
  }
  return d;
}

CsrMatrix<float> two_by_two() { return csr_from_coo<float>({{0, 0, 1.f}, {1, 0, 2.f}, {1, 1, 3.f}}, 2, 2); }

DenseMatrix<float> column(std::vector<float> v) {
  DenseMatrix<float> x = DenseMatrix<float>::zero(Index(v.size()), 1);
  x.data = std::move(v);
  return x;
}

MatrixFeatures feats(double avg, double cv, Index rows = 1000) {
  MatrixFeatures f;
  f.avg_row = avg;
  f.cv = cv;
  f.stdv_row = avg * cv;
  f.num_rows = rows;
  f.nnz = Index(avg * double(rows));
  return f;
}

}  // namespace

// ------------------------------------------------------------- host-only
TEST_CASE("kernel names, indices and parse round trip (kernels.hpp:40-57)", false) {
  const char* names[] = {"par-rs", "par-ws", "seq-rs", "seq-ws"};
  for (std::size_t i = 0; i < 4; ++i) {
    CHECK(kernel_index(kAllKernels[i]) == i);
    CHECK(kernel_name(kAllKernels[i]) == names[i]);
    CHECK(parse_kernel(names[i]) == kAllKernels[i]);
  }
  CHECK_THROWS_AS(parse_kernel("bogus"), Error);
}

TEST_CASE("decision-tree examples with default thresholds (test_selector.cpp:28-33)", false) {
  CHECK(select_kernel(feats(5, 2.0), 1) == kParBalanced);
  CHECK(select_kernel(feats(100, 0.1), 128) == kSeqRowSplit);
  CHECK(select_kernel(feats(10, 3.0), 32) == kSeqBalanced);
  CHECK(select_kernel(feats(64, 0.5), 2) == kParRowSplit);
}

TEST_CASE("threshold ties favor row-split (test_selector.cpp:35-38)", false) {
  CHECK(select_kernel(feats(32.0, 0.5), 1) == kParRowSplit);
  CHECK(select_kernel(feats(10.0, 1.0), 32) == kSeqRowSplit);
}

TEST_CASE("calibrate_thresholds picks the loss-minimising grid point", false) {
  // Two cells where seq-ws wins only above cv=3: the default t_cv=1 sends the
  // cv=2 matrix to seq-ws (loss), t_cv=2 or 4 fixes it; 2 is closer to 1.
  std::vector<CalibrationRecord> recs;
  auto add = [&](MatrixFeatures f, KernelId k, double g) { recs.push_back({f, 64, k, g}); };
  add(feats(10, 2.0, 100), kSeqRowSplit, 10.0);
  add(feats(10, 2.0, 100), kSeqBalanced, 5.0);
  add(feats(10, 8.0, 200), kSeqRowSplit, 5.0);
  add(feats(10, 8.0, 200), kSeqBalanced, 10.0);
  const SelectorThresholds t = calibrate_thresholds(recs);
  CHECK(t.t_cv == 2.0);
  CHECK(t.t_parallel_avg == 32.0);
  CHECK(t.n_parallel_max == 4u);
  CHECK_THROWS_AS(calibrate_thresholds({}), Error);
}

TEST_CASE("features KATs (test_core.cpp:59-93)", false) {
  auto a = csr_from_coo<float>({{0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {1, 2, 1}, {3, 0, 1}, {3, 1, 1},
                                {3, 2, 1}, {3, 3, 1}}, 4, 4);  // lengths [1,3,0,4]
  auto f = extract_features(a);
  CHECK(f.avg_row == 2.0);
  CHECK(f.stdv_row == 1.5811388300841898);
  CHECK(f.cv == 0.7905694150420949);
  auto e = csr_from_coo<float>({}, 3, 3);
  CHECK(extract_features(e).cv == 0.0);
  CsrMatrix<float> z;
  z.row_ptr = {0};
  CHECK_THROWS_AS(extract_features(z), Error);
}

TEST_CASE("plan_balanced KATs (test_kernels.cpp:37-58)", false) {
  auto a = csr_from_coo<float>({{0, 0, 1}, {1, 0, 1}, {1, 1, 1}}, 2, 2);
  auto p = plan_balanced(a, 2);
  CHECK(p.elem_row == (std::vector<Index>{0, 1, 1}));
  CHECK(p.num_chunks == 2);
  auto e = csr_from_coo<float>({}, 3, 3);
  CHECK(plan_balanced(e, 4).num_chunks == 0);
  CHECK_THROWS_AS(plan_balanced(a, 0), Error);
  CHECK(detail::partition(10, 3, 1) == std::make_pair(Index(3), Index(6)));
}

TEST_CASE("validate rejects malformed CSR (test_core.cpp:177-191)", false) {
  auto a = two_by_two();
  a.col_idx[2] = 0;  // row 1: 0, 0 -> not strictly increasing
  CHECK_THROWS_AS(validate(a), Error);
  auto b = two_by_two();
  b.row_ptr.back() = 5;
  CHECK_THROWS_AS(validate(b), Error);
}

TEST_CASE("matrix market: general, symmetric, pattern, integer (test_io.cpp:11-103)", false) {
  std::istringstream g("%%MatrixMarket matrix coordinate real general\n% a comment\n\n2 2 2\n1 1 1.0\n2 2 4.0\n");
  auto a = read_matrix_market<float>(g);
  CHECK(a.num_rows == 2 && a.num_cols == 2);
  CHECK(a.row_ptr == (std::vector<Index>{0, 1, 2}));
  CHECK(a.col_idx == (std::vector<Index>{0, 1}));
  CHECK(a.values == (std::vector<float>{1.f, 4.f}));
  std::istringstream sy("%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n2 1 5.0\n3 3 1.0\n3 1 2.0\n");
  auto coo = read_matrix_market<float>(sy).to_coo();
  CHECK(coo.size() == 5u);
  CHECK(coo[0].row == 0 && coo[0].col == 1 && coo[0].value == 5.f);
  CHECK(coo[1].col == 2 && coo[1].value == 2.f);
  CHECK(coo[2].row == 1 && coo[2].col == 0);
  std::istringstream pat("%%MatrixMarket matrix coordinate pattern general\n2 3 2\n1 3\n2 1\n");
  auto p = read_matrix_market<float>(pat);
  CHECK(p.values == (std::vector<float>{1.f, 1.f}));
  std::istringstream in("%%MatrixMarket matrix coordinate integer general\n1 1 1\n1 1 7\n");
  CHECK(read_matrix_market<float>(in).values == (std::vector<float>{7.f}));
}

TEST_CASE("matrix market: rejected headers and located errors (test_io.cpp:104-150)", false) {
  for (const char* h : {"%%MatrixMarket matrix coordinate complex general",
                        "%%MatrixMarket matrix coordinate real skew-symmetric",
                        "%%MatrixMarket matrix coordinate real hermitian", "%%MatrixMarket matrix array real general",
                        "%%MatrixMarket vector coordinate real general", "MatrixMarket matrix coordinate real general"}) {
    std::istringstream in(std::string(h) + "\n1 1 0\n");
    CHECK_THROWS_AS(read_matrix_market<float>(in), Error);
  }
  auto message_of = [](const std::string& text) {
    std::istringstream in(text);
    try {
      read_matrix_market<float>(in);
    } catch (const Error& e) {
      return std::string(e.what());
    }
    return std::string();
  };
  const std::string m1 = message_of("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n");
  CHECK(m1.find("line 3") != std::string::npos && m1.find("bounds") != std::string::npos);
  CHECK(message_of("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n").find("truncated") !=
        std::string::npos);
  CHECK(!message_of("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 oops 1.0\n").empty());
}

TEST_CASE("matrix market: writer format and round trip (test_io.cpp:152-198)", false) {
  auto a = csr_from_coo<float>({{0, 0, 1.f}, {1, 1, 4.f}}, 2, 2);
  std::ostringstream out;
  write_matrix_market(a, out);
  CHECK(out.str() == "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 2 4\n");
  std::ostringstream e;
  write_matrix_market(csr_from_coo<float>({}, 3, 3), e);
  CHECK(e.str() == "%%MatrixMarket matrix coordinate real general\n3 3 0\n");
  std::vector<Triple<float>> t;
  for (Index i = 0; i < 50; ++i)
    for (Index j = 0; j < 50; j += 1 + (i % 7)) t.push_back({i, j, 1.0f / float(1 + i + j)});
  auto b = csr_from_coo(std::move(t), 50, 50);
  std::stringstream buf;
  write_matrix_market(b, buf);
  CHECK(read_matrix_market<float>(buf) == b);
}

// ------------------------------------------------------------- device path
TEST_CASE("all four kernels on the 2x2 hand example (test_kernels.cpp:60-69)", true) {
  auto a = two_by_two();
  auto x = column({10.f, 20.f});
  for (KernelId id : kAllKernels) {
    auto y = spmm(id, a, x);
    CHECK(y(0, 0) == 10.f);
    CHECK(y(1, 0) == 80.f);
  }
}

TEST_CASE("seq_rowsplit hand arithmetic with N=2 (test_kernels.cpp:71-87)", true) {
  auto a = two_by_two();
  DenseMatrix<float> x = DenseMatrix<float>::zero(2, 2);
  x(0, 0) = 10.f;
  x(0, 1) = 1.f;
  x(1, 0) = 20.f;
  x(1, 1) = 2.f;
  auto y = spmm_seq_rowsplit(a, x);
  CHECK(y(0, 0) == 10.f);
  CHECK(y(0, 1) == 1.f);
  CHECK(y(1, 0) == 80.f);
  CHECK(y(1, 1) == 8.f);
}

TEST_CASE("identity passes X through bit-exactly (test_kernels.cpp:89-99)", true) {
  std::vector<Triple<float>> t;
  for (Index i = 0; i < 4; ++i) t.push_back({i, i, 1.f});
  auto a = csr_from_coo(std::move(t), 4, 4);
  auto x = make_dense(4, 8, 17);
  for (KernelId id : kAllKernels) CHECK(spmm(id, a, x).data == x.data);
}

TEST_CASE("single 100-nonzero row across chunks (test_kernels.cpp:101-111)", true) {
  std::vector<Triple<float>> t;
  for (Index j = 0; j < 100; ++j) t.push_back({0, j, 1.f});
  auto a = csr_from_coo(std::move(t), 1, 100);
  DenseMatrix<float> x = DenseMatrix<float>::zero(100, 1);
  x.data.assign(100, 1.f);
  CHECK(spmm_par_balanced(a, x)(0, 0) == 100.f);
  CHECK(spmm_seq_balanced(a, x, {.seq_chunk = 16})(0, 0) == 100.f);
}

TEST_CASE("seq_balanced splits a row across chunks (test_kernels.cpp:132-138)", true) {
  auto a = two_by_two();
  auto x = column({10.f, 20.f});
  auto y = spmm_seq_balanced(a, x, {.seq_chunk = 2});
  CHECK(y(0, 0) == 10.f);
  CHECK(y(1, 0) == 80.f);
}

TEST_CASE("dimension mismatch and invalid configs throw (test_kernels.cpp:231-246)", true) {
  auto a = two_by_two();
  auto bad = DenseMatrix<float>::zero(3, 1);
  for (KernelId id : kAllKernels) CHECK_THROWS_AS(spmm(id, a, bad), Error);
  auto x = column({1.f, 1.f});
  CHECK_THROWS_AS(spmm_par_rowsplit(a, x, {.lane_width = 3}), Error);
  CHECK_THROWS_AS(spmm_par_rowsplit(a, x, {.lane_width = 128}), Error);
  CHECK_THROWS_AS(spmm_par_rowsplit(a, x, {.vdl_group = 3}), Error);
  CHECK_THROWS_AS(spmm_seq_balanced(a, x, {.seq_chunk = 0}), Error);
}

TEST_CASE("T=double is rejected (no CPU fallback)", true) {
  auto a = csr_from_coo<double>({{0, 0, 1.0}}, 1, 1);
  DenseMatrix<double> x = DenseMatrix<double>::zero(1, 1);
  CHECK_THROWS_AS(spmm(kSeqBalanced, a, x), Error);
}

TEST_CASE("lane-multiply counters (test_kernels.cpp:248-272)", true) {
  std::vector<Triple<float>> t;
  std::uint64_t s = 55;
  for (Index i = 0; i < 200; ++i) {
    s += 0x9e3779b97f4a7c15ULL;
    const Index len = 1 + Index((s >> 33) % 7);
    for (Index j = 0; j < len; ++j) t.push_back({i, (i + 13 * j) % 200, 1.f});
  }
  auto a = csr_from_coo(std::move(t), 200, 200);
  auto x = make_dense(200, 1, 77);
  KernelStats bal, rs;
  KernelConfig cfg;
  cfg.stats = &bal;
  (void)spmm_par_balanced(a, x, cfg);
  cfg.stats = &rs;
  (void)spmm_par_rowsplit(a, x, cfg);
  CHECK(bal.lane_multiplies.load() <= std::uint64_t(a.nnz()) + cfg.lane_width);
  CHECK(bal.lane_multiplies.load() <= rs.lane_multiplies.load());
}

TEST_CASE("resident handle: device R-MAT, features, rule, both call shapes agree", true) {
  DeviceCsr d = DeviceCsr::rmat(10, 8, 0.57, 0.19, 0.19, 0.05, 7);
  CHECK(d.num_rows() == 1024);
  const KernelId k = d.select(32);
  const MatrixFeatures f = d.features();
  CHECK(select_kernel(f, 32) == k);
  auto x = make_dense(d.num_cols(), 32, 0x00D5EED + 32);
  auto y1 = d.spmm(k, x);
  auto y2 = d.spmm(k, x);
  CHECK(y1.data == y2.data);
}

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::strcmp(argv[1], "--host") == 0;
  int ran = 0;
  for (auto& c : cases()) {
    if (host_only && c.gpu) continue;
    const int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "  FAIL %s: unexpected exception: %s\n", c.name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", c.name);
    ++ran;
  }
  std::printf("%d cases, %d checks, %d failures\n", ran, g_checks, g_fail);
  return g_fail ? 1 : 0;
}
