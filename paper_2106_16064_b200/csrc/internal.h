// internal.h — host-side state shared by the translation units of
// libspmk_b200.so (the C ABI in include/spmk_capi.h).
//
//   capi_handle.cu  handles, row metadata, plans, features, partition,
//                   validation, fix-up / zero-fill launches (aux_kernels.cuh)
//   capi_spmm.cu    the spmm dispatcher (run_spmm) and its C entry points
//   launch_seq.cu   sequential-reduction sweeps (seq_kernels.cuh)
//   launch_par.cu   par-rs / par-ws / hub-row kernels (par_*.cuh, hub_kernels.cuh)
//   capi_gen.cu     device generators (gen_kernels.cuh)
//   capi_iter.cu    iterative SpMV / PageRank support + CUDA IPC (iter_kernels.cuh)
//   capi_bench.cu   selection-harness measurement (spmk_measure_kernel) + host make_dense
//   capi_mg.cu      multi-GPU layer over NCCL (spmk_mg_*)
//
// Every kernel header is included by exactly one translation unit (they define
// non-template __global__ functions).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/spmk_capi.h"

namespace spmk_host {

// Last error on this thread (spmk_last_error).
spmk_status fail(spmk_status st, const std::string& msg);

struct CudaError {
  spmk_status st;
  std::string msg;
};

#define CK(expr)                                                                     \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      throw ::spmk_host::CudaError{                                                  \
          _e == cudaErrorMemoryAllocation ? SPMK_ENOMEM : SPMK_ECUDA,                \
          std::string(#expr) + ": " + cudaGetErrorString(_e)};                       \
  } while (0)

inline int grid_for(long long n, int threads = 256, int cap = 148 * 16) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

template <typename T>
T* dev_alloc(size_t count) {
  T* p = nullptr;
  CK(cudaMalloc(&p, sizeof(T) * (count ? count : 1)));
  return p;
}

extern std::atomic<uint64_t> g_launches;
#define LAUNCHED(n) ::spmk_host::g_launches.fetch_add((n), std::memory_order_relaxed)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

inline bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }
inline int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Plan for a nonzero-split kernel (tiles of TS nonzeros made of CH-chunks),
// a row-split tile list, or a hub-row list (cached per handle and shape).
struct Plan {
  int4* desc = nullptr;    // ntiles per-tile start descriptors
  int* rlo = nullptr;      // ntiles + 1
  long long ntiles = 0;
  long long TS = 0, CH = 0, EXT = 0;
  int* longrows = nullptr;
  int4* longinfo = nullptr;  // ws plans: fix-up descriptors (long_info_kernel), big rows first
  int nlong = 0;
  int nbig = 0;              // ws plans: long rows with > kFixupLaneMax partials
  std::vector<int> hrows;    // hub plans: hub rows in ascending order (host copy)
  std::vector<int> hlen;     // hub plans: hub row lengths in launch order
};

// Lane-per-job seq-ws layout (sell_kernels.cuh), per seq_chunk.
constexpr long long kSellMaxChunk = 512;
struct SellPlan {
  long long CH = 0;
  int shape = 0;            // sweep shape (launch_sell.cu kSellShapes)
  int cw = 32;              // column width (8 / 16 / 32: 4 / 2 / 1 jobs per lane)
  int* steps = nullptr;     // nsteps x 64 ints
  long long nsteps = 0;
  int* cstep = nullptr;     // nchunks + 1 work-queue chunk starts (step indices)
  int nchunks = 0;
  int* sched = nullptr;     // per column tile {claim counter, warps done}
  int nwarps = 0, blocks = 0;
  int4* fold = nullptr;     // {row, first slot, slots} of the rows of >= 3 segments
  int nfold = 0;
  int nbig = 0;             // leading fold rows with > kFoldWarpMax slots (one CTA each)
  int n4 = 0, n2 = 0;       // first fold rows with <= 4 / <= 2 slots (short-row tiers)
  int sms = 0;              // SMs of the device the plan was built for
  long long nslots = 0;     // H slots (x N floats)
};

// Products-buffer layout of the hub rows for one N (par-rs two-pass path).
struct HubLayout {
  long long* po = nullptr;  // per hub: offset in floats (multiple of 4)
  int2* segs = nullptr;     // per products block: {hub, first position}
  int nsegs = 0;
  long long floats = 0;     // buffer size (+ 16-byte slack)
};

// Performance knobs of one handle.  None of them changes a result bit (they
// pick tile shapes and kernel paths, never a summation order).  Initialised
// once at handle creation from the environment (SPMK_<NAME>, see DESIGN.md
// §4), then owned by the handle: spmk_csr_set_tuning / spmk_csr_get_tuning.
struct Tuning {
  long long seq_tile_nnz = 0;    // 0 = automatic (256; seq-rs at N <= 2 on small matrices: smaller)
  long long seq_ext = 32;        // owner-extension limit of seq-ws tiles
  long long parws_ext = 32;      // owner-extension limit of par-ws tiles
  long long parws_t = 4;         // par-ws chunks per tile (4 or 8)
  long long parrs_vl = 0;        // par-rs virtual lanes per lane (0 = automatic)
  long long hub_nnz = -1;        // row-split hub threshold (-1 = automatic: 2048 par-rs, 1024 seq-rs; 0 = off)
  long long hub_two_pass = -1;   // -1 automatic (par-rs on, seq-rs off)
  long long hub_smem = 0;        // shared-memory pad of the seq-rs hub CTA
  long long l2_persist = 0;      // 1 = access-policy window over X on every spmm
  long long parws_impl = 2;      // par-ws at lane_width 32, N <= 2: 2 = streaming head-flag kernel (par_ws2.cuh), 1 = tile kernel
  long long parws_cpt = 0;       // par_ws2 chunks per tile (0 = automatic)
  long long parws3 = 2;          // par-ws at W 32, N = 1 … 4: par_ws3.cuh (2 = every plan, 1 = plans without long rows), 0 = par_ws2 / tile kernel
  long long sell_cfg = 0;        // lane-per-job sweep shape (launch_sell.cu)
  long long seq_impl = 2;        // seq-ws, seq_chunk <= kSellMaxChunk: 2 = lane-per-job sweep (sell_kernels.cuh) at N = 32, 3 = also at N % 32 == 0, 1 = tile sweep only
  void from_env();
  bool set(const std::string& key, long long v);
  bool get(const std::string& key, long long* v) const;
};

// Scratch buffers superseded by a larger request stay allocated until the
// handle is destroyed: a CUDA graph captured earlier may still point at them.
struct GrowBuffer {
  float* ptr = nullptr;
  size_t floats = 0;
  std::vector<float*> retired;
  float* get(size_t n);
  void release();
};

}  // namespace spmk_host

struct spmk_csr_s {
  int device = 0;
  long long m = 0, k = 0, nnz = 0;
  int* rp = nullptr;
  int* col = nullptr;
  float* val = nullptr;
  bool own_rp = true, own_col = true, own_val = true;
  bool canonical = true;  // columns strictly increasing in every row (csr.hpp:95-119)
  // resident row metadata
  int mne = 0;            // non-empty rows
  int* crp = nullptr;     // mne+1
  int* rid = nullptr;     // mne
  int nempty = 0;
  int* erow = nullptr;    // nempty
  unsigned* hflag32 = nullptr;  // segment heads of the 32-nonzero chunks (par_ws2), lazily built
  long long max_row = 0;
  unsigned long long sum_len2 = 0;
  spmk_host::Tuning tune;
  // caches
  std::map<std::tuple<int, long long, long long, long long>, spmk_host::Plan> plans;
  spmk_host::GrowBuffer scratch;   // long-row partial slots (H, T)
  std::map<std::tuple<long long, int, int>, spmk_host::SellPlan> sell_plans;  // (seq_chunk, shape, row cap)
  std::map<std::pair<int, int>, spmk_host::HubLayout> hub_layouts;  // (L, N)
  spmk_host::GrowBuffer hub_prod;  // par-rs two-pass hub products
  // host-operand staging: kStageSlots rotating (X, Y) device buffer pairs;
  // slot_done[i] marks the end of the last call that used slot i
  static constexpr int kStageSlots = 2;
  float* stage_x[kStageSlots] = {nullptr, nullptr};
  float* stage_y[kStageSlots] = {nullptr, nullptr};
  size_t stage_x_n[kStageSlots] = {0, 0}, stage_y_n[kStageSlots] = {0, 0};
  cudaEvent_t slot_done[kStageSlots] = {nullptr, nullptr};
  int next_slot = 0;
  // side stream for work that overlaps the variant kernels (empty-row fill)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // calls on different streams share the handle's scratch (long-row partial
  // slots) and side stream: a call waits for the previous call's kernels when
  // it comes on another stream (copies around the call still overlap)
  cudaEvent_t ev_last = nullptr;
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  std::mutex mu;
};

namespace spmk_host {

// ---- capi_handle.cu
spmk_status create_from_device32(long long m, long long k, long long nnz, int* rp, int* col, float* val,
                                 bool own, int device, spmk_csr_t* out, cudaStream_t s);
Plan& get_plan(spmk_csr_s* h, int kind, long long TS, long long CH, long long EXT, cudaStream_t s);
Plan& get_hub_plan(spmk_csr_s* h, int L, cudaStream_t s);
const unsigned* get_head_flags32(spmk_csr_s* h, cudaStream_t s);
Plan& get_rs_desc(spmk_csr_s* h, long long TS, int L, const Plan* hub, cudaStream_t s);
void launch_zero_all(float* y, long long total, cudaStream_t s);
void launch_zero_rows(const spmk_csr_s* h, int N, float* y, bool vec4, cudaStream_t s);
void launch_fixup(const Plan& p, const float* H, const float* Tsl, float* y, int N, cudaStream_t s);
int fixup_lane_max();

// ---- launch_seq.cu
struct SeqLaunch {
  const int* crp;
  const int* rid;
  const int* col;
  const float* val;
  const float* X;
  float* Y;
  float* H;
  float* Tsl;
  const int* rlo;
  const int4* desc;
  int mne, nnz, N, nunits;
  long long TS, CH, EXT;
};
void launch_seq(const SeqLaunch& a, bool ws, bool aligned, cudaStream_t s);

// ---- launch_sell.cu
// column width of the lane-per-job sweep for (seq_chunk, N), 0 = not eligible
int sell_width(const spmk_csr_s* h, long long CH, int N, bool aligned);
// CH = kSellNoChunk: seq-rs (one job per row); rows of >= lmax nonzeros excluded (hub rows)
constexpr long long kSellNoChunk = 1LL << 40;
SellPlan& get_sell_plan(spmk_csr_s* h, long long CH, int lmax, int cw, cudaStream_t s);
void free_sell_plan(SellPlan& p);
// side_busy: a side-stream kernel (seq-rs hub rows) runs concurrently
void launch_sell(spmk_csr_s* h, SellPlan& p, const float* X, int N, float* Y, float* H, bool side_busy,
                 cudaStream_t s);

// ---- launch_par.cu
struct ParLaunch {
  const int* crp;
  const int* rid;
  const int* col;
  const float* val;
  const float* X;
  float* Y;
  float* H;
  float* Tsl;
  const int* rlo;
  const int4* desc;
  int mne, nnz, N, nunits, hub;
  long long TS;
};
void launch_par_rs(const ParLaunch& a, int W, int vl, bool aligned, cudaStream_t s);
void launch_par_ws(const ParLaunch& a, int W, int T, bool aligned, cudaStream_t s);
void launch_par_ws64(const ParLaunch& a, float* slots, cudaStream_t s);  // lane_width 64
void launch_par_ws2(const ParLaunch& a, const unsigned* hflag, bool aligned, cudaStream_t s);
// W 32, N = 1 … 4; rid_ident: no empty rows; long_rows: the plan has long rows (H / T partials)
void launch_par_ws3(const ParLaunch& a, const unsigned* hflag, bool rid_ident, bool aligned, bool long_rows,
                    cudaStream_t s);  // W 32, N <= 2
void launch_hubs(spmk_csr_s* h, const Plan& hub, spmk_kernel_id id, int W, int L, const float* d_x, int N,
                 float* d_y, cudaStream_t s);
void launch_hub_rows(const int* crp, int mne, int L, int2* list, int* cnt, cudaStream_t s);

}  // namespace spmk_host
