// Drop-in C++ API tests: the reference's own KATs (proj/tests/test_kernels.cpp,
// test_selector.cpp, test_core.cpp) recompiled against include/spmk/*.hpp and
// run on the device path (T=float — the reference instantiates most of them
// with T=double, which this path rejects by design).
//
//   ./test_dropin          every case (needs a GPU)
//   ./test_dropin --host   host-only cases (selector, config, names, plan)
#include <array>
#include <cmath>
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
DenseMatrix<float> host_make_dense(Index rows, Index cols, std::uint64_t seed) {
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

// test_bench.cpp helpers: a 32x32 random corpus (SplitMix64 rmat.hpp:15-29)
struct Mix {
  std::uint64_t s;
  std::uint64_t next() {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};
std::vector<NamedMatrix<float>> tiny_corpus() {
  std::vector<Triple<float>> t;
  Mix rng{1};
  for (int i = 0; i < 200; ++i) {
    const Index r = Index(rng.next() % 32), c = Index(rng.next() % 32);
    t.push_back({r, c, static_cast<float>(2.0 * rng.unit() - 1.0)});
  }
  std::vector<NamedMatrix<float>> corpus;
  corpus.emplace_back("tiny", csr_from_coo(std::move(t), 32, 32));
  return corpus;
}
BenchRecord make_record(const std::string& m, std::size_t n, KernelId k, double g, bool a) {
  BenchRecord r;
  r.matrix_name = m;
  r.nnz = 100;
  r.n = n;
  r.kernel = kernel_name(k);
  r.gflops = g;
  r.time_seconds = 2.0 * 100 * double(n) / g / 1e9;
  r.selected_by_rule = a;
  return r;
}
void add_cell(std::vector<BenchRecord>& rec, const std::string& m, std::size_t n, std::array<double, 4> g,
              KernelId chosen) {
  for (std::size_t k = 0; k < 4; ++k) rec.push_back(make_record(m, n, kAllKernels[k], g[k], false));
  rec.push_back(make_record(m, n, chosen, g[kernel_index(chosen)], true));
}
bool near(double a, double b, double eps = 1e-9) { return std::fabs(a - b) <= eps * std::max(1.0, std::fabs(b)); }

}  // namespace

// ------------------------------------------------------------- host-only
TEST_CASE("summarize: auto matching best gives zero loss (test_bench.cpp:87-95)", false) {
  std::vector<BenchRecord> r;
  add_cell(r, "m1", 1, {1, 2, 3, 4}, kSeqBalanced);
  add_cell(r, "m1", 8, {5, 2, 3, 4}, kParRowSplit);
  auto s = summarize_selection_loss(r);
  CHECK(near(s.per_n_loss.at(1), 0.0) && near(s.per_n_loss.at(8), 0.0));
  CHECK(near(s.single_kernel_loss.at("seq-ws"), 0.1));
}

TEST_CASE("summarize: half the best, shifting landscape, fixed-kernel loss (test_bench.cpp:97-135)", false) {
  std::vector<BenchRecord> r;
  add_cell(r, "m1", 4, {2, 4, 1, 1}, kParRowSplit);
  add_cell(r, "m2", 4, {3, 6, 1, 1}, kParRowSplit);
  CHECK(near(summarize_selection_loss(r).per_n_loss.at(4), 0.5));
  r.clear();
  for (int m = 0; m < 4; ++m) {
    const std::string name = "m" + std::to_string(m);
    add_cell(r, name, 1, {10, 9, 2, 2}, kParRowSplit);
    add_cell(r, name, 4, {9, 10, 2, 2}, kParBalanced);
    add_cell(r, name, 32, {2, 2, 10, 9}, kSeqRowSplit);
    add_cell(r, name, 128, {2, 2, 9, 10}, kSeqBalanced);
  }
  auto s = summarize_selection_loss(r);
  for (const auto& [k, l] : s.single_kernel_loss) CHECK(mean_per_n_loss(s) < l);
  CHECK(min_single_kernel_loss(s) > 0.0);
  r.clear();
  add_cell(r, "m1", 2, {5, 1, 1, 1}, kParRowSplit);
  add_cell(r, "m1", 16, {5, 1, 1, 1}, kSeqRowSplit);
  s = summarize_selection_loss(r);
  CHECK(s.single_kernel_loss.at("par-rs") == 0.0 && s.single_kernel_loss.at("par-ws") > 0.0);
}

TEST_CASE("summarize rejects incomplete record sets; emit_csv shapes (test_bench.cpp:137-175)", false) {
  std::vector<BenchRecord> r;
  add_cell(r, "m1", 1, {1, 2, 3, 4}, kSeqBalanced);
  r.pop_back();
  CHECK_THROWS_AS(summarize_selection_loss(r), Error);
  r.clear();
  add_cell(r, "m1", 1, {1, 2, 3, 4}, kSeqBalanced);
  r.erase(r.begin());
  CHECK_THROWS_AS(summarize_selection_loss(r), Error);
  std::ostringstream out;
  emit_csv({}, SelectionLossSummary{}, out);
  CHECK(out.str() == "matrix_name,num_rows,num_cols,nnz,n,kernel,time_seconds,gflops,correct,selected_by_rule\n");
  r.clear();
  add_cell(r, "m1", 1, {1, 2, 3, 4}, kSeqBalanced);
  std::ostringstream out2;
  emit_csv(r, summarize_selection_loss(r), out2);
  std::istringstream lines(out2.str());
  std::string line;
  int data = 0, comments = 0;
  std::getline(lines, line);
  while (std::getline(lines, line)) (line[0] == '#' ? comments : data) += 1;
  CHECK(data == 5 && comments == 5);
}

TEST_CASE("rmat params validation (test_rmat.cpp)", false) {
  RmatParams p;
  p.scale = 0;
  CHECK_THROWS_AS(validate(p), Error);
  p.scale = 8;
  p.edge_factor = 0;
  CHECK_THROWS_AS(validate(p), Error);
  p.edge_factor = 8;
  p.skew = RmatSkew{0.5, 0.5, 0.5, 0.0};
  CHECK_THROWS_AS(validate(p), Error);
}
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
  auto x = host_make_dense(4, 8, 17);
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
  auto x = host_make_dense(200, 1, 77);
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
  auto x = host_make_dense(d.num_cols(), 32, 0x00D5EED + 32);
  auto y1 = d.spmm(k, x);
  auto y2 = d.spmm(k, x);
  CHECK(y1.data == y2.data);
}

TEST_CASE("generate_rmat<float> and make_dense<float> on the device (rmat.hpp:61-88, corpus.hpp:116-122)", true) {
  RmatParams p;
  p.scale = 10;
  p.edge_factor = 8;
  p.seed = 7;
  const CsrMatrix<float> a = generate_rmat<float>(p);
  validate(a);
  CHECK(a.num_rows == 1024 && a.nnz() > 0);
  const CsrMatrix<float> b = DeviceCsr::rmat(10, 8, 0.57, 0.19, 0.19, 0.05, 7).download();
  CHECK(a.row_ptr == b.row_ptr && a.col_idx == b.col_idx && a.values == b.values);
  for (float v : a.values) CHECK(v == 1.0f);
  const auto x = make_dense<float>(1000, 7, 17);
  const auto h = host_make_dense(1000, 7, 17);
  CHECK(x.num_rows == 1000 && x.num_cols == 7 && x.data == h.data);
}

TEST_CASE("run_benchmark: records, correctness, gflops, the auto record (test_bench.cpp:56-85)", true) {
  auto records = run_benchmark(tiny_corpus(), {1}, {}, {}, 3, 0);
  CHECK(records.size() == 5);
  int autos = 0;
  for (const auto& r : records) {
    CHECK(r.correct && r.time_seconds > 0.0);
    CHECK(near(r.gflops, 2.0 * double(r.nnz) * double(r.n) / r.time_seconds / 1e9));
    autos += r.selected_by_rule;
  }
  CHECK(autos == 1);
  auto corpus = tiny_corpus();
  records = run_benchmark(corpus, {1, 8}, {}, {}, 2, 0);
  const auto f = extract_features(corpus[0].second);
  for (const auto& r : records)
    if (r.selected_by_rule) CHECK(r.kernel == kernel_name(select_kernel(f, r.n)));
  auto s = summarize_selection_loss(records);
  CHECK(s.per_n_loss.size() == 2);
  CHECK_THROWS_AS(run_benchmark<float>({}, {1}, {}, {}, 1, 0), Error);
  CHECK_THROWS_AS(run_benchmark(tiny_corpus(), {1}, {}, {}, 0, 0), Error);
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
