// spmk_capi.cu — C ABI of the B200-native adaptive SpMV/SpMM engine.
// See include/spmk_capi.h for the contract (reference interface per entry).
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/spmk_capi.h"
#include "aux_kernels.cuh"
#include "gen_kernels.cuh"
#include "hub_kernels.cuh"
#include "iter_kernels.cuh"
#include "par_kernels.cuh"
#include "seq_kernels.cuh"

using namespace spmk_dev;

namespace {

thread_local std::string g_err;

spmk_status fail(spmk_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

struct CudaError {
  spmk_status st;
  std::string msg;
};

#define CK(expr)                                                                     \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      throw CudaError{_e == cudaErrorMemoryAllocation ? SPMK_ENOMEM : SPMK_ECUDA,    \
                      std::string(#expr) + ": " + cudaGetErrorString(_e)};           \
  } while (0)

int grid_for(long long n, int threads = 256, int cap = 148 * 16) {
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

struct Plan {
  int4* desc = nullptr;    // ntiles per-tile start descriptors
  int* rlo = nullptr;      // ntiles + 1
  long long ntiles = 0;
  long long TS = 0, CH = 0, EXT = 0;
  int* longrows = nullptr;
  int4* longinfo = nullptr;  // ws plans: fixup descriptors (long_info_kernel), big rows first
  int nlong = 0;
  int nbig = 0;              // ws plans: long rows with > kFixupLaneMax partials
  std::vector<int> hrows;  // hub plans: hub rows in ascending order (host copy)
  std::vector<int> hlen;   // hub plans: hub row lengths in launch order
};

// Products-buffer layout of the hub rows for one N (par-rs two-pass path).
struct HubLayout {
  long long* po = nullptr;  // per hub: offset in floats (multiple of 4)
  int2* segs = nullptr;     // per products block: {hub, first position}
  int nsegs = 0;
  long long floats = 0;     // buffer size (+ 16-byte slack)
};

std::atomic<uint64_t> g_launches{0};
#define LAUNCHED(n) g_launches.fetch_add((n), std::memory_order_relaxed)

struct Timing {
  bool on = false;
  int device = -1;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // call0, main0, main1, call1
};
thread_local Timing g_timing;

void timing_record(int which, cudaStream_t s) {
  if (!g_timing.on) return;
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_timing.device != dev) {
    for (auto& e : g_timing.ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : g_timing.ev) cudaEventCreate(&e);
    g_timing.device = dev;
  }
  cudaEventRecord(g_timing.ev[which], s);
}

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

}  // namespace

struct spmk_csr_s {
  int device = 0;
  long long m = 0, k = 0, nnz = 0;
  int* rp = nullptr;
  int* col = nullptr;
  float* val = nullptr;
  bool own_rp = true, own_col = true, own_val = true;
  // resident row metadata
  int mne = 0;            // non-empty rows
  int* crp = nullptr;     // mne+1
  int* rid = nullptr;     // mne
  int nempty = 0;
  int* erow = nullptr;    // nempty
  long long max_row = 0;
  unsigned long long sum_len2 = 0;
  // caches
  std::map<std::tuple<int, long long, long long, long long>, Plan> plans;
  float* scratch = nullptr;
  size_t scratch_floats = 0;
  std::map<std::pair<int, int>, HubLayout> hub_layouts;  // (L, N)
  float* hub_prod = nullptr;
  size_t hub_prod_floats = 0;
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

namespace {

void free_handle(spmk_csr_s* h) {
  DeviceGuard g(h->device);
  if (h->own_rp) cudaFree(h->rp);
  if (h->own_col) cudaFree(h->col);
  if (h->own_val) cudaFree(h->val);
  cudaFree(h->crp);
  cudaFree(h->rid);
  cudaFree(h->erow);
  for (auto& kv : h->plans) {
    cudaFree(kv.second.rlo);
    cudaFree(kv.second.desc);
    cudaFree(kv.second.longrows);
    cudaFree(kv.second.longinfo);
  }
  cudaFree(h->scratch);
  for (auto& kv : h->hub_layouts) {
    cudaFree(kv.second.po);
    cudaFree(kv.second.segs);
  }
  cudaFree(h->hub_prod);
  if (h->side) {
    cudaStreamSynchronize(h->side);
    cudaStreamDestroy(h->side);
    cudaEventDestroy(h->ev_fork);
    cudaEventDestroy(h->ev_join);
  }
  if (h->ev_last) cudaEventDestroy(h->ev_last);
  for (int i = 0; i < spmk_csr_s::kStageSlots; ++i) {
    cudaFree(h->stage_x[i]);
    cudaFree(h->stage_y[i]);
    if (h->slot_done[i]) cudaEventDestroy(h->slot_done[i]);
  }
  delete h;
}

// Row metadata: non-empty compaction + moments (one-time, at create).
void build_meta(spmk_csr_s* h, cudaStream_t s) {
  const int m = (int)h->m;
  h->crp = dev_alloc<int>((size_t)m + 1);
  h->rid = dev_alloc<int>((size_t)m);
  h->erow = dev_alloc<int>((size_t)m);
  int* flag = dev_alloc<int>((size_t)m + 1);
  int* pos = dev_alloc<int>((size_t)m + 1);
  unsigned long long* mom = dev_alloc<unsigned long long>(4);
  CK(cudaMemsetAsync(mom, 0, 4 * sizeof(unsigned long long), s));
  if (m > 0) {
    nonempty_flag_kernel<<<grid_for(m), 256, 0, s>>>(h->rp, m, flag); LAUNCHED(1);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flag, pos, m + 1, s);
    void* tmp = dev_alloc<char>(tmp_bytes);
    CK(cudaMemsetAsync(flag + m, 0, sizeof(int), s));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, pos, m + 1, s);
    compact_scatter_kernel<<<grid_for(m), 256, 0, s>>>(h->rp, m, pos, h->crp, h->rid, h->erow); LAUNCHED(1);
    row_moments_kernel<<<grid_for(m), 256, 0, s>>>(h->rp, m, mom); LAUNCHED(1);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&h->mne, pos + m, sizeof(int), cudaMemcpyDeviceToHost, s));
    unsigned long long hm[4];
    CK(cudaMemcpyAsync(hm, mom, sizeof(hm), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(tmp);
    h->sum_len2 = hm[1];
    h->max_row = (long long)hm[2];
    h->nempty = m - h->mne;
  }
  // crp[mne] = nnz
  const int nnz32 = (int)h->nnz;
  CK(cudaMemcpyAsync(h->crp + h->mne, &nnz32, sizeof(int), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  cudaFree(flag);
  cudaFree(pos);
  cudaFree(mom);
}

// Plan for a nonzero-split kernel: tiles of TS nonzeros made of CH-chunks.
Plan& get_plan(spmk_csr_s* h, int kind, long long TS, long long CH, long long EXT, cudaStream_t s) {
  EXT = std::max(1LL, std::min(EXT, TS));
  auto key = std::make_tuple(kind, TS, CH, EXT);
  auto it = h->plans.find(key);
  if (it != h->plans.end()) return it->second;
  Plan p;
  p.TS = TS;
  p.CH = CH;
  p.EXT = EXT;
  p.ntiles = (h->nnz + TS - 1) / TS;
  p.rlo = dev_alloc<int>((size_t)p.ntiles + 1);
  tile_plan_kernel<<<grid_for(p.ntiles + 1), 256, 0, s>>>(h->crp, h->mne, p.ntiles, TS, p.rlo); LAUNCHED(1);
  p.desc = dev_alloc<int4>((size_t)p.ntiles);
  ws_tile_desc_kernel<<<grid_for(p.ntiles), 256, 0, s>>>(h->crp, p.rlo, p.ntiles, TS, EXT, h->nnz, p.desc); LAUNCHED(1);
  int* cnt = dev_alloc<int>(1);
  CK(cudaMemsetAsync(cnt, 0, sizeof(int), s));
  // upper bound on long rows: every long row crosses a tile boundary
  const long long cap = p.ntiles + 1;
  p.longrows = dev_alloc<int>((size_t)cap);
  if (h->mne > 0)
    long_rows_kernel<<<grid_for(h->mne), 256, 0, s>>>(h->crp, h->mne, TS, EXT, p.longrows, cnt); LAUNCHED(1);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&p.nlong, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  cudaFree(cnt);
  if (p.nlong > 0) {
    p.longinfo = dev_alloc<int4>((size_t)p.nlong);
    long_info_kernel<<<grid_for(p.nlong), 256, 0, s>>>(p.longrows, p.nlong, h->crp, h->rid, TS, CH, p.longinfo); LAUNCHED(1);
    CK(cudaGetLastError());
    // big rows first (stable partition on the host, once per plan)
    std::vector<int4> info((size_t)p.nlong);
    CK(cudaMemcpyAsync(info.data(), p.longinfo, sizeof(int4) * info.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    auto it = std::stable_partition(info.begin(), info.end(),
                                    [](const int4& d) { return d.w - d.z >= kFixupLaneMax; });
    p.nbig = (int)(it - info.begin());
    CK(cudaMemcpyAsync(p.longinfo, info.data(), sizeof(int4) * info.size(), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  return h->plans.emplace(key, p).first->second;
}

// Hub rows of the row-split variants (rows with >= L nonzeros, hub_kernels.cuh):
// device list longest first (launch order), host copy ascending.
Plan& get_hub_plan(spmk_csr_s* h, int L, cudaStream_t s) {
  auto key = std::make_tuple(4, (long long)L, 0LL, 0LL);
  auto it = h->plans.find(key);
  if (it != h->plans.end()) return it->second;
  Plan p;
  const long long cap = h->nnz / L + 1;
  int2* list = dev_alloc<int2>((size_t)cap);
  int* cnt = dev_alloc<int>(1);
  CK(cudaMemsetAsync(cnt, 0, sizeof(int), s));
  hub_rows_kernel<<<grid_for(h->mne), 256, 0, s>>>(h->crp, h->mne, L, list, cnt); LAUNCHED(1);
  CK(cudaGetLastError());
  int n = 0;
  CK(cudaMemcpyAsync(&n, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (n > 0) {
    std::vector<int2> hl((size_t)n);
    CK(cudaMemcpyAsync(hl.data(), list, sizeof(int2) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::sort(hl.begin(), hl.end(), [](int2 x, int2 y) { return x.y != y.y ? x.y > y.y : x.x < y.x; });
    std::vector<int> rows((size_t)n);
    for (int i = 0; i < n; ++i) rows[i] = hl[i].x;
    p.hlen.resize((size_t)n);
    for (int i = 0; i < n; ++i) p.hlen[i] = hl[i].y;
    p.longrows = dev_alloc<int>((size_t)n);
    CK(cudaMemcpyAsync(p.longrows, rows.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    std::sort(rows.begin(), rows.end());
    p.hrows = std::move(rows);
    CK(cudaStreamSynchronize(s));
  }
  p.nlong = n;
  cudaFree(list);
  cudaFree(cnt);
  return h->plans.emplace(key, p).first->second;
}

// Row-split tile descriptors, cached like a plan: tile t holds the whole rows
// that start in [t*TS, (t+1)*TS) (rlo of tile_plan_kernel), so tiles are
// nnz-balanced without ever splitting a row (the row-split contract).  With
// hub rows (hub plan `hub`), a tile holding hubs is cut into the runs of
// non-hub rows between them: the first run keeps the tile's slot, the others
// are appended; hub rows belong to no tile.
Plan& get_rs_desc(spmk_csr_s* h, long long TS, int L, const Plan* hub, cudaStream_t s) {
  auto key = std::make_tuple(3, TS, (long long)L, 0LL);
  auto it = h->plans.find(key);
  if (it != h->plans.end()) return it->second;
  Plan p;
  p.TS = TS;
  p.ntiles = (h->nnz + TS - 1) / TS;
  p.rlo = dev_alloc<int>((size_t)p.ntiles + 1);
  tile_plan_kernel<<<grid_for(p.ntiles + 1), 256, 0, s>>>(h->crp, h->mne, p.ntiles, TS, p.rlo); LAUNCHED(1);
  p.desc = dev_alloc<int4>((size_t)p.ntiles);
  rs_tile_desc_kernel<<<grid_for(p.ntiles), 256, 0, s>>>(h->crp, p.rlo, p.ntiles, p.desc); LAUNCHED(1);
  CK(cudaGetLastError());
  if (hub && !hub->hrows.empty()) {
    // one round trip: row metadata and descriptors down, edited, back up
    const std::vector<int>& hr = hub->hrows;
    std::vector<int> rlo((size_t)p.ntiles + 1), rp((size_t)h->mne + 1);
    std::vector<int4> desc((size_t)p.ntiles);
    CK(cudaMemcpyAsync(rlo.data(), p.rlo, sizeof(int) * rlo.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(rp.data(), h->crp, sizeof(int) * rp.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(desc.data(), p.desc, sizeof(int4) * desc.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (size_t i = 0; i < hr.size();) {
      // the tile whose rows [rlo[t], rlo[t+1]) contain hub row hr[i]
      const long long t = (long long)(std::upper_bound(rlo.begin(), rlo.end(), hr[i]) - rlo.begin()) - 1;
      const int r0 = rlo[t], r1 = rlo[t + 1];
      std::vector<int4> pieces;
      int a0 = r0;
      for (; i < hr.size() && hr[i] < r1; ++i) {
        if (hr[i] > a0) pieces.push_back(make_int4(a0, rp[a0], rp[hr[i]], MODE_NORMAL));
        a0 = hr[i] + 1;
      }
      if (a0 < r1) pieces.push_back(make_int4(a0, rp[a0], rp[r1], MODE_NORMAL));
      // an empty first run keeps the slot as an idle tile (start == end)
      desc[t] = pieces.empty() ? make_int4(r0, 0, 0, MODE_NORMAL) : pieces[0];
      for (size_t k = 1; k < pieces.size(); ++k) desc.push_back(pieces[k]);
    }
    if ((long long)desc.size() != p.ntiles) {
      cudaFree(p.desc);
      p.desc = nullptr;
      p.desc = dev_alloc<int4>(desc.size());
      p.ntiles = (long long)desc.size();
    }
    CK(cudaMemcpyAsync(p.desc, desc.data(), sizeof(int4) * desc.size(), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  return h->plans.emplace(key, p).first->second;
}

float* get_scratch(spmk_csr_s* h, size_t floats) {
  if (floats > h->scratch_floats) {
    cudaFree(h->scratch);
    h->scratch = nullptr;
    h->scratch_floats = 0;
    h->scratch = dev_alloc<float>(floats);
    h->scratch_floats = floats;
  }
  return h->scratch;
}

spmk_kernel_config cfg_or_default(const spmk_kernel_config* cfg) {
  spmk_kernel_config c;
  spmk_default_config(&c);
  return cfg ? *cfg : c;
}

bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

long long env_ll(const char* name, long long dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoll(v) : dflt;
}

// The dynamic-shared-memory opt-in is per (kernel, device): remember which
// pairs have it so multi-device processes set it on every device.
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, bool> g_attr_done;
bool need_smem_attr(const void* fn) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  return !std::exchange(g_attr_done[{fn, dev}], true);
}

// Hub threshold of the row-split variants (0 disables the hub path).
// Measured on B200 (R-MAT s20..s25 heavy): par-rs 2048 (s25 N=1: 3.91 ms at
// 1024, 3.37 ms at 2048, 3.50 ms at 4096), seq-rs 1024 (s20 N=32: 0.77 ms,
// 0.88 ms at 4096).
int hub_threshold(spmk_kernel_id id) {
  const long long dflt = id == SPMK_PAR_ROWSPLIT ? 2048 : 1024;
  return (int)std::max(0LL, std::min<long long>(env_ll("SPMK_HUB_NNZ", dflt), INT32_MAX));
}

template <int CW>
void launch_seq_hub(const HubArgs& g, int nhub, int N, cudaStream_t s) {
  // SPMK_HUB_SMEM pads the shared-memory request (e.g. 120 KB: one hub CTA
  // per SM); measured neutral at N = 32 and slower at N = 128, so off.
  const int smem = (int)std::max<long long>(hub_smem_bytes<CW>(), env_ll("SPMK_HUB_SMEM", 0));
  if (need_smem_attr(reinterpret_cast<const void*>(seq_rs_hub_kernel<CW>)))
    CK(cudaFuncSetAttribute(seq_rs_hub_kernel<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  seq_rs_hub_kernel<CW><<<dim3((unsigned)nhub, (unsigned)((N + CW - 1) / CW)), kHubThreads, smem, s>>>(g); LAUNCHED(1);
}

const HubLayout& get_hub_layout(spmk_csr_s* h, const Plan& hub, int L, int N, cudaStream_t s) {
  auto key = std::make_pair(L, N);
  auto it = h->hub_layouts.find(key);
  if (it != h->hub_layouts.end()) return it->second;
  HubLayout lay;
  std::vector<long long> po(hub.hlen.size());
  std::vector<int2> segs;
  long long off = 0;
  for (size_t i = 0; i < hub.hlen.size(); ++i) {
    po[i] = off;
    off += ((long long)hub.hlen[i] * N + 3) / 4 * 4;
    for (int q = 0; q < hub.hlen[i]; q += kHubSeg) segs.push_back(make_int2((int)i, q));
  }
  lay.floats = off + 4;
  lay.nsegs = (int)segs.size();
  lay.po = dev_alloc<long long>(po.size());
  lay.segs = dev_alloc<int2>(segs.size());
  CK(cudaMemcpyAsync(lay.po, po.data(), sizeof(long long) * po.size(), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(lay.segs, segs.data(), sizeof(int2) * segs.size(), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  return h->hub_layouts.emplace(key, lay).first->second;
}

void launch_hubs(spmk_csr_s* h, const Plan& hub, spmk_kernel_id id, int W, const float* d_x, int N, float* d_y,
                 cudaStream_t s) {
  HubArgs g{hub.longrows, h->crp, h->rid, h->col, h->val, d_x, d_y, N};
  // seq-rs is the fold with one chain per column (W = 1: every position in
  // order, no tree) — kernels.hpp:366-370
  const bool seq = id == SPMK_SEQ_ROWSPLIT;
  const int FW = seq ? 1 : W;
  const long long two_pass = env_ll("SPMK_HUB_TWO_PASS", seq ? 0 : 1);
  if (two_pass && FW * N <= kHubThreads) {
    const HubLayout& lay = get_hub_layout(h, hub, hub_threshold(id), N, s);
    if ((size_t)lay.floats > h->hub_prod_floats) {
      cudaFree(h->hub_prod);
      h->hub_prod = nullptr;
      h->hub_prod_floats = 0;
      h->hub_prod = dev_alloc<float>((size_t)lay.floats);
      h->hub_prod_floats = (size_t)lay.floats;
    }
    HubProdArgs pa{hub.longrows, lay.segs, lay.po, h->crp, h->col, h->val, d_x, h->hub_prod, N};
    hub_products_kernel<<<lay.nsegs, 256, 0, s>>>(pa); LAUNCHED(1);
    constexpr int smem = 128 + kFoldStages * kFoldStageBytes;
    if (need_smem_attr(reinterpret_cast<const void*>(par_rs_hub_fold_kernel)))
      CK(cudaFuncSetAttribute(par_rs_hub_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    par_rs_hub_fold_kernel<<<hub.nlong, FW * N, smem, s>>>(pa, h->rid, d_y, FW); LAUNCHED(1);
    CK(cudaGetLastError());
    return;
  }
  int cw = 1;
  while (cw < N && cw < 32) cw *= 2;  // columns per CTA
  if (id == SPMK_SEQ_ROWSPLIT) {
    switch (cw) {
      case 1: launch_seq_hub<1>(g, hub.nlong, N, s); break;
      case 2: launch_seq_hub<2>(g, hub.nlong, N, s); break;
      case 4: launch_seq_hub<4>(g, hub.nlong, N, s); break;
      case 8: launch_seq_hub<8>(g, hub.nlong, N, s); break;
      case 16: launch_seq_hub<16>(g, hub.nlong, N, s); break;
      default: launch_seq_hub<32>(g, hub.nlong, N, s); break;
    }
  } else {
    cw = std::min(cw, kHubThreads / W);
    const dim3 grid((unsigned)hub.nlong, (unsigned)((N + cw - 1) / cw));
    par_rs_hub_kernel<<<grid, W * cw, 0, s>>>(g, W, cw); LAUNCHED(1);
  }
  CK(cudaGetLastError());
}

// ------------------------------------------------------------ seq launch
template <int LPU, int CPL, bool VEC, int B, bool WS>
void launch_seq_t(const SeqArgs& a, int ncol_tiles, cudaStream_t s) {
  const int upb = 256 / LPU;
  dim3 grid((a.nunits + upb - 1) / upb, ncol_tiles);
  seq_kernel<LPU, CPL, VEC, B, WS><<<grid, 256, 0, s>>>(a); LAUNCHED(1);
}

// Column mapping of the sequential sweep: a group of LPU lanes covers one
// column tile; each lane owns CPL columns (float4/float2 when aligned), so
// one warp instruction serves 32/LPU work units at once.
template <bool WS, int CPL, bool VEC, int B>
void launch_seq_lpu(const SeqArgs& a, int lpu, int tiles, cudaStream_t s) {
  switch (lpu) {
    case 1: launch_seq_t<1, CPL, VEC, B, WS>(a, tiles, s); break;
    case 2: launch_seq_t<2, CPL, VEC, B, WS>(a, tiles, s); break;
    case 4: launch_seq_t<4, CPL, VEC, B, WS>(a, tiles, s); break;
    case 8: launch_seq_t<8, CPL, VEC, B, WS>(a, tiles, s); break;
    case 16: launch_seq_t<16, CPL, VEC, B, WS>(a, tiles, s); break;
    default: launch_seq_t<32, CPL, VEC, B, WS>(a, tiles, s); break;
  }
}

template <int LPU, int B, int S, bool WS, int NT>
void launch_seq_async_t(const SeqArgs& a, int ncol_tiles, cudaStream_t s) {
  constexpr int smem = seq_async_smem_bytes<LPU, B, S, NT>();
  if (need_smem_attr(reinterpret_cast<const void*>(seq_kernel_async<LPU, B, S, WS, NT>)))
    CK(cudaFuncSetAttribute(seq_kernel_async<LPU, B, S, WS, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int upb = NT / LPU;
  dim3 grid((a.nunits + upb - 1) / upb, ncol_tiles);
  seq_kernel_async<LPU, B, S, WS, NT><<<grid, NT, smem, s>>>(a); LAUNCHED(1);
}

// N = 4..28 (1, 2 or 4 lanes per unit): the 3-stage ring, 128 threads
template <bool WS, int B, int S, int NT>
void launch_seq_async(const SeqArgs& a, int lpu, int tiles, cudaStream_t s) {
  switch (lpu) {
    case 1: launch_seq_async_t<1, B, S, WS, NT>(a, tiles, s); break;
    case 2: launch_seq_async_t<2, B, S, WS, NT>(a, tiles, s); break;
    default: launch_seq_async_t<4, B, S, WS, NT>(a, tiles, s); break;
  }
}

template <int LPU, int B, int S, bool WS, int NT, bool EXACT>
void launch_seq_a2_t(const SeqArgs& a, int ncol_tiles, cudaStream_t s) {
  constexpr int smem = seq_async2_smem_bytes<LPU, B, S, NT>();
  if (need_smem_attr(reinterpret_cast<const void*>(seq_async2_kernel<LPU, B, S, WS, NT, EXACT>)))
    CK(cudaFuncSetAttribute(seq_async2_kernel<LPU, B, S, WS, NT, EXACT>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int upb = NT / LPU;
  dim3 grid((a.nunits + upb - 1) / upb, ncol_tiles);
  seq_async2_kernel<LPU, B, S, WS, NT, EXACT><<<grid, NT, smem, s>>>(a); LAUNCHED(1);
}

// N >= 32 (8, 16 or 32 lanes per unit): the 2-stage lean sweep
template <bool WS, int B, int S, int NT, bool EXACT>
void launch_seq_a2(const SeqArgs& a, int lpu, int tiles, cudaStream_t s) {
  switch (lpu) {
    case 8: launch_seq_a2_t<8, B, S, WS, NT, EXACT>(a, tiles, s); break;
    case 16: launch_seq_a2_t<16, B, S, WS, NT, EXACT>(a, tiles, s); break;
    default: launch_seq_a2_t<32, B, S, WS, NT, EXACT>(a, tiles, s); break;
  }
}

template <bool WS>
void launch_seq(SeqArgs a, bool aligned, cudaStream_t s) {
  const int N = a.N;
  if (aligned && N % 4 == 0) {
    const int lpu = std::min(32, next_pow2(N / 4));
    a.ncol_tile = 4 * lpu;
    const int tiles = (N + a.ncol_tile - 1) / a.ncol_tile;
    // Measured on B200 (R-MAT s20 heavy/uniform, tools/probe_perf.py): the
    // lean 2-stage ring wins from 8 lanes per unit up (N >= 32), the 3-stage
    // ring below (a register-pipelined sweep and a 6-stage ring were slower).
    if (lpu >= 8) launch_seq_a2<WS, 8, 2, 128, true>(a, lpu, tiles, s);
    else launch_seq_async<WS, 8, 3, 128>(a, lpu, tiles, s);
  } else if (aligned && N % 2 == 0 && N <= 64) {
    const int lpu = next_pow2(N / 2);
    a.ncol_tile = 2 * lpu;
    launch_seq_lpu<WS, 2, true, 16>(a, lpu, 1, s);
  } else if (N <= 32) {
    const int lpu = next_pow2(N);
    a.ncol_tile = lpu;
    launch_seq_lpu<WS, 1, false, 16>(a, lpu, 1, s);
  } else if (N <= 64) {
    a.ncol_tile = 64;
    launch_seq_t<32, 2, false, 16, WS>(a, 1, s);
  } else {
    a.ncol_tile = 128;
    launch_seq_t<32, 4, false, 8, WS>(a, (N + 127) / 128, s);
  }
}

// ------------------------------------------------------------ par launch
template <int W, int VL, int CT, bool V4>
void launch_par_rs_t(const ParArgs& a, int ncol_tiles, cudaStream_t s) {
  constexpr int G = W / VL;
  const long long groups_needed = a.mne;
  const long long threads = groups_needed * G;
  long long blocks = (threads + 255) / 256;
  blocks = std::max(1LL, std::min(blocks, 148LL * 32));
  par_rs_kernel<W, VL, CT, V4><<<dim3((unsigned)blocks, ncol_tiles), 256, 0, s>>>(a); LAUNCHED(1);
}

template <int W, int VL>
void launch_par_rs_w(ParArgs a, bool aligned, cudaStream_t s) {
  const int N = a.N;
  int ct = N <= 1 ? 1 : N <= 2 ? 2 : N <= 4 ? 4 : N <= 8 ? 8 : N <= 16 ? 16 : 32;
  a.ncol_tile = ct;
  const int tiles = (N + ct - 1) / ct;
  const bool v4 = aligned && (N % 4 == 0) && ct >= 4;
  switch (ct) {
    case 1: launch_par_rs_t<W, VL, 1, false>(a, tiles, s); break;
    case 2: launch_par_rs_t<W, VL, 2, false>(a, tiles, s); break;
    case 4: v4 ? launch_par_rs_t<W, VL, 4, true>(a, tiles, s) : launch_par_rs_t<W, VL, 4, false>(a, tiles, s); break;
    case 8: v4 ? launch_par_rs_t<W, VL, 8, true>(a, tiles, s) : launch_par_rs_t<W, VL, 8, false>(a, tiles, s); break;
    case 16: v4 ? launch_par_rs_t<W, VL, 16, true>(a, tiles, s) : launch_par_rs_t<W, VL, 16, false>(a, tiles, s); break;
    default: v4 ? launch_par_rs_t<W, VL, 32, true>(a, tiles, s) : launch_par_rs_t<W, VL, 32, false>(a, tiles, s); break;
  }
}

// Narrow dense rows (N <= 4): VL virtual lanes per physical lane, so a row
// group is W/VL threads and several short rows share a warp; the tree levels
// inside a physical lane run in registers (same order, kernels.hpp:193-199).
template <int W, int VL>
void launch_par_rs_narrow(ParArgs a, bool aligned, cudaStream_t s) {
  const int N = a.N;
  const int ct = N <= 1 ? 1 : N <= 2 ? 2 : 4;
  a.ncol_tile = ct;
  const bool v4 = aligned && (N % 4 == 0) && ct == 4;
  switch (ct) {
    case 1: launch_par_rs_t<W, VL, 1, false>(a, 1, s); break;
    case 2: launch_par_rs_t<W, VL, 2, false>(a, 1, s); break;
    default: v4 ? launch_par_rs_t<W, VL, 4, true>(a, 1, s) : launch_par_rs_t<W, VL, 4, false>(a, 1, s); break;
  }
}

// Virtual lanes per physical lane for par-rs at lane_width 32, N <= 4 (the
// results do not depend on it).  Measured on B200: rows averaging >= 24
// nonzeros fill a 32-lane group (cfg5 8-way slices 0-3, avg 27..443: VL=1
// 0.36-0.41 ms vs VL=4 0.41-0.45 ms); shorter rows want narrow groups (tail
// slice, avg 4.5: 0.75 -> 0.60 ms at VL=4), 8 on low-cv graphs at N=1
// (s20 uniform: 159 us at 1, 128 at 4, 112 at 8).
int par_rs_vl(const spmk_csr_s* h, int W, int N) {
  const long long env = env_ll("SPMK_PARRS_VL", 0);
  if (env > 0) return (int)env;
  if (W != 32 || N > 4) return 1;
  const double M = (double)h->m, avg = (double)h->nnz / M;
  const double var = std::max(0.0, (double)h->sum_len2 / M - avg * avg);
  const double cv = avg > 0.0 ? std::sqrt(var) / avg : 0.0;
  if (avg >= 24.0) return 1;
  if (N == 2 && cv > 1.0) return 1;  // s22 heavy N=2: 543 us at 1, 577 at 4
  return (N == 1 && cv <= 1.0) ? 8 : 4;
}

void launch_par_rs(const ParArgs& a, int W, int vl, bool aligned, cudaStream_t s) {
  if (a.N <= 4 && vl > 1) {
    if (W == 32 && vl == 4) return launch_par_rs_narrow<32, 4>(a, aligned, s);
    if (W == 32 && vl == 8) return launch_par_rs_narrow<32, 8>(a, aligned, s);
    if (W == 64 && vl == 8) return launch_par_rs_narrow<64, 8>(a, aligned, s);
    if (W == 16 && vl == 4) return launch_par_rs_narrow<16, 4>(a, aligned, s);
  }
  switch (W) {
    case 2: launch_par_rs_w<2, 1>(a, aligned, s); break;
    case 4: launch_par_rs_w<4, 1>(a, aligned, s); break;
    case 8: launch_par_rs_w<8, 1>(a, aligned, s); break;
    case 16: launch_par_rs_w<16, 1>(a, aligned, s); break;
    case 32: launch_par_rs_w<32, 1>(a, aligned, s); break;
    default: launch_par_rs_w<64, 2>(a, aligned, s); break;
  }
}

template <int W, int CT, int T, int MINB, bool BT>
void launch_par_ws_t(const ParArgs& a, int ncol_tiles, cudaStream_t s) {
  const int upb = 256 / W;
  dim3 grid((a.nunits + upb - 1) / upb, ncol_tiles);
  par_ws_kernel<W, CT, T, MINB, BT><<<grid, 256, 0, s>>>(a); LAUNCHED(1);
}

template <int W, int T, int MINB, bool BT>
void launch_par_ws_w(ParArgs a, bool aligned, cudaStream_t s) {
  const int N = a.N;
  int ct = N <= 1 ? 1 : N <= 2 ? 2 : N <= 4 ? 4 : 8;
  a.xvec = aligned && ((ct % 4 == 0 && N % 4 == 0) || (ct == 2 && N % 2 == 0));
  a.ncol_tile = ct;
  const int tiles = (N + ct - 1) / ct;
  switch (ct) {
    case 1: launch_par_ws_t<W, 1, T, MINB, BT>(a, tiles, s); break;
    case 2: launch_par_ws_t<W, 2, T, MINB, BT>(a, tiles, s); break;
    case 4: launch_par_ws_t<W, 4, T, MINB, BT>(a, tiles, s); break;
    default: launch_par_ws_t<W, 8, T, MINB, BT>(a, tiles, s); break;
  }
}

// Tile shape of par-ws: T chunks of W nonzeros per group (a pure performance
// knob: any T keeps the results bit-exact).
int par_ws_chunks_per_tile() { return env_ll("SPMK_PARWS_T", 4) == 8 ? 8 : 4; }  // the two compiled shapes

template <int T, int MINB, bool BT = true>
void launch_par_ws_tt(const ParArgs& a, int W, bool aligned, cudaStream_t s) {
  switch (W) {
    case 2: launch_par_ws_w<2, T, MINB, BT>(a, aligned, s); break;
    case 4: launch_par_ws_w<4, T, MINB, BT>(a, aligned, s); break;
    case 8: launch_par_ws_w<8, T, MINB, BT>(a, aligned, s); break;
    case 16: launch_par_ws_w<16, T, MINB, BT>(a, aligned, s); break;
    default: launch_par_ws_w<32, T, MINB, BT>(a, aligned, s); break;
  }
}

void launch_par_ws(const ParArgs& a, int W, bool aligned, cudaStream_t s) {
  const int T = par_ws_chunks_per_tile();
  // T = 4 chunks per tile, 5 blocks per SM: measured best on B200 (R-MAT
  // s20 heavy/uniform, N = 1 and 4; T = 6 / 8 and 4 / 6 blocks were slower)
  if (T == 8) launch_par_ws_tt<8, 4>(a, W, aligned, s);
  else launch_par_ws_tt<4, 5>(a, W, aligned, s);
}

// seq-rs tile (nonzeros whose rows start in one span): 256; at N <= 2 (one
// lane per unit) shrunk on small matrices so there are >= 256 tiles per SM
// (measured: R-MAT s16 N=1 87 -> 23.5 us, s18 heavy N=1 281 -> 133 us; at
// N >= 4 smaller tiles lost 5-40 %, sweep r01n vs r01o).  Tiles hold whole
// rows, so the size never changes the results.
long long rs_tile_nnz(long long nnz, int N) {
  if (N > 2) return 256;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  long long ts = 256;
  while (ts > 32 && nnz / ts < (long long)sms * 256) ts >>= 1;
  return ts;
}

// Tile sizes (nonzeros per work unit).  Any multiple of the chunk keeps the
// results bit-exact; these are pure performance knobs (env overridable).
long long tile_chunks(long long chunk, long long target) {
  long long t = target / chunk;
  return t < 1 ? 1 : t;
}

spmk_status run_spmm(spmk_csr_s* h, spmk_kernel_id id, const spmk_kernel_config& cfg,
                     const float* d_x, int64_t n, float* d_y, cudaStream_t s) {
  const long long M = h->m;
  if (n == 0 || M == 0) return SPMK_OK;
  if (h->nnz == 0 || h->mne == 0) {
    zero_all_kernel<<<grid_for(M * n), 256, 0, s>>>(d_y, M * n); LAUNCHED(1);
    CK(cudaGetLastError());
    return SPMK_OK;
  }
  if (n > INT32_MAX / 2) return fail(SPMK_EUNSUPPORTED, "n too large");
  if (id == SPMK_PAR_BALANCED && cfg.lane_width > 32)
    return fail(SPMK_EUNSUPPORTED, "par-ws with lane_width 64 is not supported on the device");
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(s, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (!capturing && h->has_last && h->last_stream != s) CK(cudaStreamWaitEvent(s, h->ev_last, 0));
  timing_record(0, s);
  const int N = (int)n;
  const bool aligned = ((uintptr_t)d_x % 16 == 0) && ((uintptr_t)d_y % 16 == 0);
  // Empty rows -> 0 (the reference's zero-initialised Y).  The variant
  // kernels never touch empty rows, so the zero fill runs on the handle's
  // side stream concurrently with them (fork/join through events: HBM writes
  // overlap the gather-bound sweep; capturable into CUDA graphs).
  // Row-split variants: hub rows (>= L nonzeros) run in hub_kernels.cuh on
  // the side stream, concurrently with the main kernel (disjoint rows of Y).
  const bool rs = id == SPMK_PAR_ROWSPLIT || id == SPMK_SEQ_ROWSPLIT;
  const int L = rs ? hub_threshold(id) : 0;
  const Plan* hub = L > 0 ? &get_hub_plan(h, L, s) : nullptr;
  const bool hubs = hub && hub->nlong > 0;
  const bool fork = h->nempty > 0 || hubs;
  if (fork) {
    if (!h->side) {
      CK(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(h->ev_fork, s));
    CK(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    if (hubs) launch_hubs(h, *hub, id, (int)cfg.lane_width, d_x, N, d_y, h->side);
    if (h->nempty == 0) {
    } else if (aligned && N % 4 == 0) {
      zero_rows_kernel<4><<<grid_for((long long)h->nempty * N / 4), 256, 0, h->side>>>(h->erow, h->nempty, N, d_y); LAUNCHED(1);
    } else {
      zero_rows_kernel<1><<<grid_for((long long)h->nempty * N), 256, 0, h->side>>>(h->erow, h->nempty, N, d_y); LAUNCHED(1);
    }
    CK(cudaEventRecord(h->ev_join, h->side));
  }

  if (id == SPMK_SEQ_ROWSPLIT || id == SPMK_SEQ_BALANCED) {
    SeqArgs a{};
    a.crp = h->crp;
    a.rid = h->rid;
    a.col = h->col;
    a.val = h->val;
    a.X = d_x;
    a.Y = d_y;
    a.mne = h->mne;
    a.nnz = (int)h->nnz;
    a.N = N;
    a.cvvec = ((uintptr_t)h->col % 16 == 0) && ((uintptr_t)h->val % 16 == 0);
    if (id == SPMK_SEQ_ROWSPLIT) {
      const long long TS = std::max(1LL, env_ll("SPMK_SEQ_TILE_NNZ", rs_tile_nnz(h->nnz, N)));
      Plan& p = get_rs_desc(h, TS, L, hubs ? hub : nullptr, s);
      a.nunits = (int)p.ntiles;
      a.desc = p.desc;
      timing_record(1, s);
      launch_seq<false>(a, aligned, s);
      timing_record(2, s);
    } else {
      const long long CH = (long long)cfg.seq_chunk;
      const long long TS = CH * tile_chunks(CH, env_ll("SPMK_SEQ_TILE_NNZ", 256));
      Plan& p = get_plan(h, 1, TS, CH, env_ll("SPMK_SEQ_EXT", 32), s);  // EXT: measured (cfg2 -7 %)
      a.rlo = p.rlo;
      a.desc = p.desc;
      a.TS = TS;
      a.CH = CH;
      a.EXT = p.EXT;
      a.nunits = (int)p.ntiles;
      if (p.nlong > 0) {
        const long long nch = (h->nnz + CH - 1) / CH;
        float* sc = get_scratch(h, (size_t)(nch + p.ntiles) * N);
        a.H = sc;
        a.Tsl = sc + (size_t)nch * N;
      }
      timing_record(1, s);
      launch_seq<true>(a, aligned, s);
      timing_record(2, s);
      if (p.nlong > 0)
        fixup_kernel<<<fixup_blocks(p.nlong, p.nbig, N), kFixupWarps * 32, 0, s>>>(
            p.longinfo, p.nlong, p.nbig, a.H, a.Tsl, d_y, N); LAUNCHED(1);
    }
  } else {
    ParArgs a{};
    a.crp = h->crp;
    a.rid = h->rid;
    a.col = h->col;
    a.val = h->val;
    a.X = d_x;
    a.Y = d_y;
    a.mne = h->mne;
    a.nnz = (int)h->nnz;
    a.N = N;
    const int W = (int)cfg.lane_width;
    if (id == SPMK_PAR_ROWSPLIT) {
      a.hub = hubs ? L : INT32_MAX;
      timing_record(1, s);
      launch_par_rs(a, W, par_rs_vl(h, W, N), aligned, s);
      timing_record(2, s);
    } else {
      const long long CH = W;
      const long long TS = CH * par_ws_chunks_per_tile();  // par_ws_kernel tile shape
      Plan& p = get_plan(h, 2, TS, CH, env_ll("SPMK_PARWS_EXT", 32), s);
      a.rlo = p.rlo;
      a.desc = p.desc;
      a.TS = TS;
      a.nunits = (int)p.ntiles;
      if (p.nlong > 0) {
        const long long nch = (h->nnz + CH - 1) / CH;
        float* sc = get_scratch(h, (size_t)(nch + p.ntiles) * N);
        a.H = sc;
        a.Tsl = sc + (size_t)nch * N;
      }
      timing_record(1, s);
      launch_par_ws(a, W, aligned, s);
      timing_record(2, s);
      if (p.nlong > 0)
        fixup_kernel<<<fixup_blocks(p.nlong, p.nbig, N), kFixupWarps * 32, 0, s>>>(
            p.longinfo, p.nlong, p.nbig, a.H, a.Tsl, d_y, N); LAUNCHED(1);
    }
  }
  if (fork) CK(cudaStreamWaitEvent(s, h->ev_join, 0));
  CK(cudaGetLastError());
  timing_record(3, s);
  if (!capturing) {
    if (!h->ev_last) CK(cudaEventCreateWithFlags(&h->ev_last, cudaEventDisableTiming));
    CK(cudaEventRecord(h->ev_last, s));
    h->last_stream = s;
    h->has_last = true;
  }
  return SPMK_OK;
}

spmk_status create_from_device32(long long m, long long k, long long nnz, int* rp, int* col,
                                 float* val, bool own, int device, spmk_csr_t* out,
                                 cudaStream_t s) {
  auto* h = new spmk_csr_s;
  h->device = device;
  h->m = m;
  h->k = k;
  h->nnz = nnz;
  h->rp = rp;
  h->col = col;
  h->val = val;
  h->own_rp = h->own_col = h->own_val = own;
  try {
    int* err = dev_alloc<int>(1);
    CK(cudaMemsetAsync(err, 0, sizeof(int), s));
    validate_kernel<<<grid_for(std::max(m, 1LL)), 256, 0, s>>>(rp, col, (int)m, (int)k, nnz, err); LAUNCHED(1);
    CK(cudaGetLastError());
    int herr = 0;
    CK(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(err);
    if (herr) {
      free_handle(h);
      return fail(SPMK_EINVAL, (herr & 1) ? "row_ptr malformed (csr.hpp:95-119)"
                               : (herr & 2) ? "column index out of range"
                                            : "columns not strictly increasing within a row");
    }
    build_meta(h, s);
  } catch (const CudaError& e) {
    free_handle(h);
    return fail(e.st, e.msg);
  }
  *out = h;
  return SPMK_OK;
}

}  // namespace

// =============================================================== C ABI
extern "C" {

const char* spmk_last_error(void) { return g_err.c_str(); }
int spmk_version(void) { return SPMK_CAPI_VERSION; }

void spmk_default_config(spmk_kernel_config* cfg) {
  cfg->lane_width = 32;
  cfg->vdl_group = 0;
  cfg->seq_chunk = 256;
  cfg->worker_count = 0;
}
void spmk_default_thresholds(spmk_thresholds* t) {
  t->n_parallel_max = 4;
  t->t_parallel_avg = 32.0;
  t->t_cv = 1.0;
}

spmk_status spmk_check_config(const spmk_kernel_config* cfg) {
  if (!cfg) return SPMK_OK;
  if (!is_pow2(cfg->lane_width) || cfg->lane_width < 2 || cfg->lane_width > 64)
    return fail(SPMK_EINVAL, "lane_width must be a power of two in [2, 64]");
  if (cfg->vdl_group != 0 && cfg->vdl_group != 1 && cfg->vdl_group != 2 && cfg->vdl_group != 4)
    return fail(SPMK_EINVAL, "vdl_group must be 0 (auto), 1, 2 or 4");
  if (cfg->seq_chunk < 1) return fail(SPMK_EINVAL, "seq_chunk must be >= 1");
  if (cfg->seq_chunk > (1ull << 30)) return fail(SPMK_EUNSUPPORTED, "seq_chunk too large for the device path");
  return SPMK_OK;
}

const char* spmk_kernel_name(spmk_kernel_id id) {
  switch (id) {
    case SPMK_PAR_ROWSPLIT: return "par-rs";
    case SPMK_PAR_BALANCED: return "par-ws";
    case SPMK_SEQ_ROWSPLIT: return "seq-rs";
    default: return "seq-ws";
  }
}

spmk_status spmk_parse_kernel(const char* name, spmk_kernel_id* out) {
  for (int i = 0; i < 4; ++i) {
    if (std::strcmp(name, spmk_kernel_name((spmk_kernel_id)i)) == 0) {
      *out = (spmk_kernel_id)i;
      return SPMK_OK;
    }
  }
  return fail(SPMK_EINVAL, std::string("unknown kernel name: ") + name);
}

spmk_status spmk_csr_create(int64_t num_rows, int64_t num_cols, int64_t nnz,
                            const int64_t* row_ptr, const int64_t* col_idx,
                            const float* values, int device, spmk_csr_t* out) {
  if (!out || !row_ptr || (nnz > 0 && (!col_idx || !values)))
    return fail(SPMK_EINVAL, "null argument");
  if (num_rows < 0 || num_cols < 0 || nnz < 0) return fail(SPMK_EINVAL, "negative dimension");
  if (num_rows >= INT32_MAX || num_cols >= INT32_MAX || nnz >= INT32_MAX)
    return fail(SPMK_EUNSUPPORTED, "device path narrows indices to int32 (need < 2^31)");
  if (row_ptr[0] != 0 || row_ptr[num_rows] != nnz)
    return fail(SPMK_EINVAL, "row_ptr[0] must be 0 and row_ptr[M] must equal nnz");
  DeviceGuard g(device);
  cudaStream_t s = nullptr;
  int *rp = nullptr, *col = nullptr;
  float* val = nullptr;
  long long* tmp = nullptr;
  int* bad = nullptr;
  try {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    rp = dev_alloc<int>((size_t)num_rows + 1);
    col = dev_alloc<int>((size_t)nnz);
    val = dev_alloc<float>((size_t)nnz);
    const long long chunk = 1LL << 24;
    tmp = dev_alloc<long long>((size_t)std::min<long long>(chunk, std::max<long long>(nnz, num_rows + 1)));
    bad = dev_alloc<int>(1);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
    auto narrow = [&](const int64_t* src, int* dst, long long n) {
      for (long long o = 0; o < n; o += chunk) {
        const long long c = std::min(chunk, n - o);
        CK(cudaMemcpyAsync(tmp, src + o, c * 8, cudaMemcpyHostToDevice, s));
        narrow_kernel<<<grid_for(c), 256, 0, s>>>(tmp, dst + o, c, bad); LAUNCHED(1);
        CK(cudaGetLastError());
      }
    };
    narrow(row_ptr, rp, num_rows + 1);
    narrow(col_idx, col, nnz);
    if (nnz) CK(cudaMemcpyAsync(val, values, nnz * 4, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    int hbad = 0;
    CK(cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(tmp);
    cudaFree(bad);
    tmp = nullptr;
    bad = nullptr;
    if (hbad) {
      cudaFree(rp);
      cudaFree(col);
      cudaFree(val);
      cudaStreamDestroy(s);
      return fail(SPMK_EINVAL, "index out of int32 range");
    }
    spmk_status st = create_from_device32(num_rows, num_cols, nnz, rp, col, val, true, device, out, s);
    cudaStreamDestroy(s);
    return st;
  } catch (const CudaError& e) {
    cudaFree(rp);
    cudaFree(col);
    cudaFree(val);
    cudaFree(tmp);
    cudaFree(bad);
    if (s) cudaStreamDestroy(s);
    return fail(e.st, e.msg);
  }
}

spmk_status spmk_csr_create_device(int64_t num_rows, int64_t num_cols, int64_t nnz,
                                   const int32_t* d_row_ptr, const int32_t* d_col_idx,
                                   const float* d_values, int copy, spmk_csr_t* out) {
  if (!out || !d_row_ptr) return fail(SPMK_EINVAL, "null argument");
  if (num_rows < 0 || num_cols < 0 || nnz < 0) return fail(SPMK_EINVAL, "negative dimension");
  if (num_rows >= INT32_MAX || num_cols >= INT32_MAX || nnz >= INT32_MAX)
    return fail(SPMK_EUNSUPPORTED, "device path needs indices < 2^31");
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, d_row_ptr) != cudaSuccess || attr.type != cudaMemoryTypeDevice)
    return fail(SPMK_EINVAL, "d_row_ptr is not device memory");
  const int device = attr.device;
  DeviceGuard g(device);
  cudaStream_t s = nullptr;
  try {
    // the arrays may still be in flight on any of the caller's streams
    CK(cudaDeviceSynchronize());
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int* rp = const_cast<int*>(d_row_ptr);
    int* col = const_cast<int*>(d_col_idx);
    float* val = const_cast<float*>(d_values);
    if (copy) {
      rp = dev_alloc<int>((size_t)num_rows + 1);
      col = dev_alloc<int>((size_t)nnz);
      val = dev_alloc<float>((size_t)nnz);
      CK(cudaMemcpyAsync(rp, d_row_ptr, (num_rows + 1) * 4, cudaMemcpyDeviceToDevice, s));
      if (nnz) {
        CK(cudaMemcpyAsync(col, d_col_idx, nnz * 4, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(val, d_values, nnz * 4, cudaMemcpyDeviceToDevice, s));
      }
    }
    spmk_status st = create_from_device32(num_rows, num_cols, nnz, rp, col, val, copy != 0,
                                          device, out, s);
    cudaStreamDestroy(s);
    return st;
  } catch (const CudaError& e) {
    if (s) cudaStreamDestroy(s);
    return fail(e.st, e.msg);
  }
}

spmk_status spmk_csr_slice(spmk_csr_t a, int64_t row_begin, int64_t row_end, int device,
                           spmk_csr_t* out) {
  if (!a || !out || row_begin < 0 || row_end < row_begin || row_end > a->m)
    return fail(SPMK_EINVAL, "bad slice");
  try {
    int rp_b = 0, rp_e = 0;
    {
      DeviceGuard g(a->device);
      CK(cudaMemcpy(&rp_b, a->rp + row_begin, 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&rp_e, a->rp + row_end, 4, cudaMemcpyDeviceToHost));
    }
    const long long rows = row_end - row_begin, nnz = rp_e - rp_b;
    DeviceGuard g(device);
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int* rp = dev_alloc<int>((size_t)rows + 1);
    int* col = dev_alloc<int>((size_t)nnz);
    float* val = dev_alloc<float>((size_t)nnz);
    int* rpsrc = a->rp;
    int* tmp = nullptr;
    if (device != a->device) {
      tmp = dev_alloc<int>((size_t)rows + 1);
      CK(cudaMemcpyPeerAsync(tmp, device, a->rp + row_begin, a->device, (rows + 1) * 4, s));
      CK(cudaMemcpyPeerAsync(col, device, a->col + rp_b, a->device, nnz * 4, s));
      CK(cudaMemcpyPeerAsync(val, device, a->val + rp_b, a->device, nnz * 4, s));
      rebase_kernel<<<grid_for(rows + 1), 256, 0, s>>>(tmp, 0, rows, rp); LAUNCHED(1);
    } else {
      CK(cudaMemcpyAsync(col, a->col + rp_b, nnz * 4, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(val, a->val + rp_b, nnz * 4, cudaMemcpyDeviceToDevice, s));
      rebase_kernel<<<grid_for(rows + 1), 256, 0, s>>>(rpsrc, row_begin, rows, rp); LAUNCHED(1);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    if (tmp) cudaFree(tmp);
    spmk_status st = create_from_device32(rows, a->k, nnz, rp, col, val, true, device, out, s);
    cudaStreamDestroy(s);
    return st;
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
}

spmk_status spmk_csr_abs_copy(spmk_csr_t a, spmk_csr_t* out) {
  if (!a || !out) return fail(SPMK_EINVAL, "null argument");
  DeviceGuard g(a->device);
  cudaStream_t s = nullptr;
  try {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int* rp = dev_alloc<int>((size_t)a->m + 1);
    int* col = dev_alloc<int>((size_t)a->nnz);
    float* val = dev_alloc<float>((size_t)a->nnz);
    CK(cudaMemcpyAsync(rp, a->rp, (a->m + 1) * 4, cudaMemcpyDeviceToDevice, s));
    if (a->nnz) {
      CK(cudaMemcpyAsync(col, a->col, a->nnz * 4, cudaMemcpyDeviceToDevice, s));
      abs_copy_kernel<<<grid_for(a->nnz), 256, 0, s>>>(a->val, val, a->nnz); LAUNCHED(1);
      CK(cudaGetLastError());
    }
    spmk_status st = create_from_device32(a->m, a->k, a->nnz, rp, col, val, true, a->device, out, s);
    cudaStreamDestroy(s);
    return st;
  } catch (const CudaError& e) {
    if (s) cudaStreamDestroy(s);
    return fail(e.st, e.msg);
  }
}

spmk_status spmk_csr_destroy(spmk_csr_t a) {
  if (a) free_handle(a);
  return SPMK_OK;
}

spmk_status spmk_csr_info(spmk_csr_t a, int64_t* num_rows, int64_t* num_cols, int64_t* nnz,
                          int64_t* max_row_nnz, int64_t* empty_rows) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  if (num_rows) *num_rows = a->m;
  if (num_cols) *num_cols = a->k;
  if (nnz) *nnz = a->nnz;
  if (max_row_nnz) *max_row_nnz = a->max_row;
  if (empty_rows) *empty_rows = a->nempty;
  return SPMK_OK;
}

spmk_status spmk_csr_device_arrays(spmk_csr_t a, const int32_t** d_row_ptr,
                                   const int32_t** d_col_idx, const float** d_values) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  if (d_row_ptr) *d_row_ptr = a->rp;
  if (d_col_idx) *d_col_idx = a->col;
  if (d_values) *d_values = a->val;
  return SPMK_OK;
}

spmk_status spmk_csr_download(spmk_csr_t a, int64_t* row_ptr, int64_t* col_idx, float* values) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  DeviceGuard g(a->device);
  try {
    auto widen = [&](const int* src, int64_t* dst, long long n) {
      if (!dst || n == 0) return;
      long long* tmp = dev_alloc<long long>((size_t)n);
      widen_kernel<<<grid_for(n), 256>>>(src, tmp, n); LAUNCHED(1);
      CK(cudaGetLastError());
      CK(cudaMemcpy(dst, tmp, n * 8, cudaMemcpyDeviceToHost));
      cudaFree(tmp);
    };
    widen(a->rp, row_ptr, a->m + 1);
    widen(a->col, col_idx, a->nnz);
    if (values && a->nnz) CK(cudaMemcpy(values, a->val, a->nnz * 4, cudaMemcpyDeviceToHost));
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

// csr.hpp:166-181, sequential double sum (the reference order).
spmk_status spmk_features_host(int64_t num_rows, const int64_t* row_ptr, spmk_features* out) {
  if (num_rows < 1) return fail(SPMK_EINVAL, "extract_features requires num_rows >= 1");
  const long long nnz = row_ptr[num_rows];
  out->num_rows = num_rows;
  out->nnz = nnz;
  out->avg_row = (double)nnz / (double)num_rows;
  double ss = 0.0;
  for (long long i = 0; i < num_rows; ++i) {
    const double d = (double)(row_ptr[i + 1] - row_ptr[i]) - out->avg_row;
    ss += d * d;
  }
  out->stdv_row = std::sqrt(ss / (double)num_rows);
  out->cv = out->avg_row == 0.0 ? 0.0 : out->stdv_row / out->avg_row;
  return SPMK_OK;
}

spmk_status spmk_features_compute(spmk_csr_t a, spmk_features* out) {
  if (!a || !out) return fail(SPMK_EINVAL, "null argument");
  if (a->m < 1) return fail(SPMK_EINVAL, "extract_features requires num_rows >= 1");
  // exact integer moments (computed at create); host finalize
  const long double m = (long double)a->m, nnz = (long double)a->nnz;
  out->num_rows = a->m;
  out->nnz = a->nnz;
  out->avg_row = (double)a->nnz / (double)a->m;  // bit-identical to csr.hpp:170
  long double ss = (long double)a->sum_len2 - nnz * nnz / m;
  if (ss < 0) ss = 0;
  out->stdv_row = (double)std::sqrt(ss / m);
  out->cv = out->avg_row == 0.0 ? 0.0 : out->stdv_row / out->avg_row;
  return SPMK_OK;
}

spmk_kernel_id spmk_select(const spmk_features* f, uint64_t n, const spmk_thresholds* t) {
  spmk_thresholds d;
  spmk_default_thresholds(&d);
  const spmk_thresholds& th = t ? *t : d;
  if (n <= th.n_parallel_max) return f->avg_row < th.t_parallel_avg ? SPMK_PAR_BALANCED : SPMK_PAR_ROWSPLIT;
  return f->cv > th.t_cv ? SPMK_SEQ_BALANCED : SPMK_SEQ_ROWSPLIT;
}

spmk_status spmk_select_for(spmk_csr_t a, uint64_t n, const spmk_thresholds* t,
                            spmk_kernel_id* out) {
  spmk_features f;
  spmk_status st = spmk_features_compute(a, &f);
  if (st != SPMK_OK) return st;
  spmk_thresholds d;
  spmk_default_thresholds(&d);
  const spmk_thresholds& th = t ? *t : d;
  // tie-guard: near a threshold recompute in the reference's exact order
  if (std::fabs(f.cv - th.t_cv) <= 1e-9 * std::fabs(th.t_cv)) {
    std::vector<int64_t> rp((size_t)a->m + 1);
    st = spmk_csr_download(a, rp.data(), nullptr, nullptr);
    if (st != SPMK_OK) return st;
    spmk_features_host(a->m, rp.data(), &f);
  }
  *out = spmk_select(&f, n, &th);
  return SPMK_OK;
}

spmk_status spmk_plan(spmk_csr_t a, int64_t chunk, int64_t* chunk_first_row, int64_t* num_chunks) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  if (chunk < 1) return fail(SPMK_EINVAL, "chunk_size must be >= 1");
  const long long nch = (a->nnz + chunk - 1) / chunk;
  if (num_chunks) *num_chunks = nch;
  if (!chunk_first_row || nch == 0) return SPMK_OK;
  DeviceGuard g(a->device);
  try {
    long long* d = dev_alloc<long long>((size_t)nch);
    chunk_first_row_kernel<<<grid_for(nch), 256>>>(a->rp, (int)a->m, nch, chunk, d); LAUNCHED(1);
    CK(cudaGetLastError());
    CK(cudaMemcpy(chunk_first_row, d, nch * 8, cudaMemcpyDeviceToHost));
    cudaFree(d);
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_plan_elem_row(spmk_csr_t a, int64_t* elem_row) {
  if (!a || !elem_row) return fail(SPMK_EINVAL, "null argument");
  if (a->nnz == 0) return SPMK_OK;
  DeviceGuard g(a->device);
  try {
    long long* d = dev_alloc<long long>((size_t)a->nnz);
    elem_row_kernel<<<grid_for(a->nnz), 256>>>(a->rp, (int)a->m, a->nnz, d); LAUNCHED(1);
    CK(cudaGetLastError());
    CK(cudaMemcpy(elem_row, d, a->nnz * 8, cudaMemcpyDeviceToHost));
    cudaFree(d);
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

void spmk_partition(int64_t items, int64_t parts, int64_t w, int64_t* lo, int64_t* hi) {
  *lo = items * w / parts;
  *hi = items * (w + 1) / parts;
}

spmk_status spmk_row_slices(spmk_csr_t a, int64_t parts, int64_t* bounds) {
  if (!a || !bounds || parts < 1) return fail(SPMK_EINVAL, "bad argument");
  DeviceGuard g(a->device);
  try {
    long long* d = dev_alloc<long long>((size_t)parts + 1);
    row_slices_kernel<<<grid_for(parts + 1), 256>>>(a->rp, (int)a->m, a->nnz, parts, d); LAUNCHED(1);
    CK(cudaGetLastError());
    CK(cudaMemcpy(bounds, d, (parts + 1) * 8, cudaMemcpyDeviceToHost));
    cudaFree(d);
    for (int64_t g2 = 1; g2 <= parts; ++g2)
      if (bounds[g2] < bounds[g2 - 1]) bounds[g2] = bounds[g2 - 1];
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_spmm(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg,
                      const float* d_x, int64_t n, float* d_y, void* stream) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  if ((int)id < 0 || (int)id > 3) return fail(SPMK_EINVAL, "bad kernel id");
  spmk_status st = spmk_check_config(cfg);
  if (st != SPMK_OK) return st;
  if (n < 0) return fail(SPMK_EDIM, "negative n");
  if (n > 0 && a->m > 0 && !d_y) return fail(SPMK_EINVAL, "null Y");
  if (n > 0 && a->k > 0 && !d_x) return fail(SPMK_EINVAL, "null X");
  const spmk_kernel_config c = cfg_or_default(cfg);
  std::lock_guard<std::mutex> lk(a->mu);
  DeviceGuard g(a->device);
  try {
    return run_spmm(a, id, c, d_x, n, d_y, (cudaStream_t)stream);
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
}

spmk_status spmk_spmm_auto(spmk_csr_t a, const spmk_thresholds* t, const spmk_kernel_config* cfg,
                           const float* d_x, int64_t n, float* d_y, void* stream,
                           spmk_kernel_id* chosen) {
  spmk_kernel_id id;
  spmk_status st = spmk_select_for(a, (uint64_t)n, t, &id);
  if (st != SPMK_OK) return st;
  if (chosen) *chosen = id;
  return spmk_spmm(a, id, cfg, d_x, n, d_y, stream);
}

namespace {
// H2D(x) -> spmm -> D2H(y) on `s` through one of the handle's staging slots;
// the slot's previous user is awaited on the device (event), not the host.
spmk_status spmm_host_enqueue(spmk_csr_s* a, spmk_kernel_id id, const spmk_kernel_config& c,
                              const float* x, int64_t n, float* y, cudaStream_t s) {
  const size_t nx = (size_t)a->k * n, ny = (size_t)a->m * n;
  const int slot = a->next_slot;
  a->next_slot = (slot + 1) % spmk_csr_s::kStageSlots;
  if (!a->slot_done[slot]) CK(cudaEventCreateWithFlags(&a->slot_done[slot], cudaEventDisableTiming));
  if (nx > a->stage_x_n[slot] || ny > a->stage_y_n[slot]) {
    CK(cudaEventSynchronize(a->slot_done[slot]));  // previous user done before freeing
    if (nx > a->stage_x_n[slot]) {
      cudaFree(a->stage_x[slot]);
      a->stage_x[slot] = nullptr;
      a->stage_x_n[slot] = 0;
      a->stage_x[slot] = dev_alloc<float>(nx);
      a->stage_x_n[slot] = nx;
    }
    if (ny > a->stage_y_n[slot]) {
      cudaFree(a->stage_y[slot]);
      a->stage_y[slot] = nullptr;
      a->stage_y_n[slot] = 0;
      a->stage_y[slot] = dev_alloc<float>(ny);
      a->stage_y_n[slot] = ny;
    }
  }
  CK(cudaStreamWaitEvent(s, a->slot_done[slot], 0));
  if (nx) CK(cudaMemcpyAsync(a->stage_x[slot], x, nx * 4, cudaMemcpyHostToDevice, s));
  spmk_status st = run_spmm(a, id, c, a->stage_x[slot], n, a->stage_y[slot], s);
  if (st != SPMK_OK) return st;
  CK(cudaMemcpyAsync(y, a->stage_y[slot], ny * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaEventRecord(a->slot_done[slot], s));
  return SPMK_OK;
}
}  // namespace

spmk_status spmk_spmm_host(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg,
                           const float* x, int64_t n, float* y, void* stream) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  spmk_status st = spmk_check_config(cfg);
  if (st != SPMK_OK) return st;
  if (n < 0) return fail(SPMK_EDIM, "negative n");
  if (n == 0 || a->m == 0) return SPMK_OK;
  const spmk_kernel_config c = cfg_or_default(cfg);
  std::lock_guard<std::mutex> lk(a->mu);
  DeviceGuard g(a->device);
  cudaStream_t s = (cudaStream_t)stream;
  try {
    st = spmm_host_enqueue(a, id, c, x, n, y, s);
    if (st != SPMK_OK) return st;
    CK(cudaStreamSynchronize(s));
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_spmm_host_async(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg,
                                 const float* x, int64_t n, float* y, void* stream) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  spmk_status st = spmk_check_config(cfg);
  if (st != SPMK_OK) return st;
  if (n < 0) return fail(SPMK_EDIM, "negative n");
  if (n == 0 || a->m == 0) return SPMK_OK;
  const spmk_kernel_config c = cfg_or_default(cfg);
  std::lock_guard<std::mutex> lk(a->mu);
  DeviceGuard g(a->device);
  try {
    return spmm_host_enqueue(a, id, c, x, n, y, (cudaStream_t)stream);
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
}

spmk_status spmk_spmm_csr_host(int64_t num_rows, int64_t num_cols, int64_t nnz,
                               const int64_t* row_ptr, const int64_t* col_idx,
                               const float* values, spmk_kernel_id id,
                               const spmk_kernel_config* cfg, const float* x, int64_t n,
                               float* y, int device) {
  spmk_status st = spmk_check_config(cfg);
  if (st != SPMK_OK) return st;
  spmk_csr_t h = nullptr;
  st = spmk_csr_create(num_rows, num_cols, nnz, row_ptr, col_idx, values, device, &h);
  if (st != SPMK_OK) return st;
  st = spmk_spmm_host(h, id, cfg, x, n, y, nullptr);
  spmk_csr_destroy(h);
  return st;
}

spmk_status spmk_kernel_stats(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg,
                              int64_t n, uint64_t* lane_multiplies, uint64_t* scan_ops) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  spmk_status st = spmk_check_config(cfg);
  if (st != SPMK_OK) return st;
  const spmk_kernel_config c = cfg_or_default(cfg);
  *lane_multiplies = 0;
  *scan_ops = 0;
  if (n == 0 || id == SPMK_SEQ_ROWSPLIT || id == SPMK_SEQ_BALANCED) return SPMK_OK;
  const uint64_t w = c.lane_width;
  uint64_t levels = 0;
  for (uint64_t off = 1; off < w; off <<= 1) ++levels;
  int64_t group = c.vdl_group ? (int64_t)c.vdl_group : (n >= 4 ? 4 : n >= 2 ? 2 : 1);
  if (group > n) group = n;
  const uint64_t wc_sum = (uint64_t)((n / group) * group + (n % group));
  if (id == SPMK_PAR_ROWSPLIT) {
    // sum over non-empty rows of ceil(len/W) * W (kernels.hpp:187)
    std::vector<int64_t> rp((size_t)a->m + 1);
    st = spmk_csr_download(a, rp.data(), nullptr, nullptr);
    if (st != SPMK_OK) return st;
    uint64_t lm = 0, rows = 0;
    for (int64_t i = 0; i < a->m; ++i) {
      const uint64_t len = (uint64_t)(rp[i + 1] - rp[i]);
      if (!len) continue;
      lm += (len + w - 1) / w * w;
      ++rows;
    }
    *lane_multiplies = lm * wc_sum;
    *scan_ops = rows * levels * w * wc_sum;
  } else {
    if (a->nnz == 0) return SPMK_OK;
    const uint64_t chunks = ((uint64_t)a->nnz + w - 1) / w;
    *lane_multiplies = chunks * w * wc_sum;
    *scan_ops = chunks * levels * w * wc_sum;
  }
  return SPMK_OK;
}

double spmk_kernel_tolerance(int64_t max_row_nnz) {
  return 1e-5 * std::log2((double)max_row_nnz + 2.0);
}

spmk_status spmk_l2_persist_x(void* stream, const float* d_x, size_t bytes) {
  cudaStream_t s = (cudaStream_t)stream;
  try {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaStreamAttrValue attr;
    std::memset(&attr, 0, sizeof(attr));
    if (bytes == 0 || d_x == nullptr) {
      attr.accessPolicyWindow.num_bytes = 0;
      CK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &attr));
      CK(cudaCtxResetPersistingL2Cache());
      return SPMK_OK;
    }
    int max_win = 0, max_persist = 0;
    CK(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
    if (max_win <= 0 || max_persist <= 0) return fail(SPMK_EUNSUPPORTED, "no L2 persistence");
    const size_t persist = std::min<size_t>(bytes, (size_t)max_persist);
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist));
    const size_t win = std::min<size_t>(bytes, (size_t)max_win);
    attr.accessPolicyWindow.base_ptr = const_cast<float*>(d_x);
    attr.accessPolicyWindow.num_bytes = win;
    attr.accessPolicyWindow.hitRatio = std::min(1.0f, (float)persist / (float)win);
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &attr));
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_make_dense(int64_t rows, int64_t cols, uint64_t seed, float* d_out, void* stream) {
  const long long total = rows * cols;
  if (total <= 0) return SPMK_OK;
  make_dense_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(d_out, total, seed); LAUNCHED(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SPMK_ECUDA, cudaGetErrorString(e));
  return SPMK_OK;
}

spmk_status spmk_generate_rmat(uint32_t scale, uint64_t edge_factor, double a, double b, double c,
                               double d, uint64_t seed, int device, spmk_csr_t* out) {
  // rmat.hpp:46-59 validate
  if (scale < 1 || scale > 30) return fail(SPMK_EINVAL, "rmat scale must be in [1, 30]");
  if (edge_factor < 1) return fail(SPMK_EINVAL, "rmat edge_factor must be >= 1");
  const double pr[4] = {a, b, c, d};
  double sum = 0.0;
  for (double q : pr) {
    if (q < 0.0 || q > 1.0) return fail(SPMK_EINVAL, "rmat quadrant probability outside [0, 1]");
    sum += q;
  }
  if (std::abs(sum - 1.0) > 1e-9) return fail(SPMK_EINVAL, "rmat quadrant probabilities must sum to 1");
  if (scale > 30 || (edge_factor << scale) >= (1ull << 31))
    return fail(SPMK_EUNSUPPORTED, "edge count must be < 2^31 on the device path");
  DeviceGuard g(device);
  const long long m = 1LL << scale;
  const long long edges = (long long)(edge_factor << scale);
  const double t_a = a, t_ab = a + b, t_abc = a + b + c;  // rmat.hpp:66-68
  cudaStream_t s = nullptr;
  try {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    unsigned long long* keys = dev_alloc<unsigned long long>((size_t)edges);
    unsigned long long* sorted = dev_alloc<unsigned long long>((size_t)edges);
    rmat_edges_kernel<<<grid_for(edges, 256, 148 * 64), 256, 0, s>>>(keys, edges, (int)scale, seed,
                                                                     t_a, t_ab, t_abc); LAUNCHED(1);
    CK(cudaGetLastError());
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, edges, 0, 2 * (int)scale, s);
    void* tmp = dev_alloc<char>(tb);
    cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, edges, 0, 2 * (int)scale, s);
    cudaFree(tmp);
    int* flag = reinterpret_cast<int*>(keys);  // reuse: edges*8 bytes >= 2*edges ints
    int* pos = flag + edges;
    unique_flag_kernel<<<grid_for(edges), 256, 0, s>>>(sorted, edges, flag); LAUNCHED(1);
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, flag, pos, edges, s);
    tmp = dev_alloc<char>(sb);
    cub::DeviceScan::ExclusiveSum(tmp, sb, flag, pos, edges, s);
    int last_flag = 0, last_pos = 0;
    CK(cudaMemcpyAsync(&last_flag, flag + edges - 1, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&last_pos, pos + edges - 1, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(tmp);
    const long long nnz = (long long)last_pos + last_flag;
    int* col = dev_alloc<int>((size_t)nnz);
    float* val = dev_alloc<float>((size_t)nnz);
    unsigned long long* rows = dev_alloc<unsigned long long>((size_t)nnz);
    unique_scatter_kernel<<<grid_for(edges), 256, 0, s>>>(sorted, edges, flag, pos, (int)scale, col,
                                                           val, rows); LAUNCHED(1);
    cudaFree(keys);
    cudaFree(sorted);
    int* rp = dev_alloc<int>((size_t)m + 1);
    rowptr_from_rows_kernel<<<grid_for(m + 1), 256, 0, s>>>(rows, nnz, m, rp); LAUNCHED(1);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    cudaFree(rows);
    spmk_status st = create_from_device32(m, m, nnz, rp, col, val, true, device, out, s);
    cudaStreamDestroy(s);
    return st;
  } catch (const CudaError& e) {
    if (s) cudaStreamDestroy(s);
    return fail(e.st, e.msg);
  }
}

// ------------------------------------------------------------ iterative SpMV
spmk_status spmk_column_counts(spmk_csr_t a, int32_t* d_counts, void* stream) {
  if (!a || !d_counts) return fail(SPMK_EINVAL, "null argument");
  DeviceGuard g(a->device);
  cudaStream_t s = (cudaStream_t)stream;
  try {
    CK(cudaMemsetAsync(d_counts, 0, (size_t)a->k * 4, s));
    if (a->nnz) {
      column_counts_kernel<<<grid_for(a->nnz), 256, 0, s>>>(a->col, a->nnz, d_counts); LAUNCHED(1);
    }
    CK(cudaGetLastError());
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_csr_values_inv_column_counts(spmk_csr_t a, const int32_t* d_counts, void* stream) {
  if (!a || !d_counts) return fail(SPMK_EINVAL, "null argument");
  if (!a->own_val) return fail(SPMK_EINVAL, "handle borrows its values; create it with copy=1");
  DeviceGuard g(a->device);
  try {
    if (a->nnz) {
      inv_count_values_kernel<<<grid_for(a->nnz), 256, 0, (cudaStream_t)stream>>>(a->col, a->nnz, d_counts, a->val);
      LAUNCHED(1);
    }
    CK(cudaGetLastError());
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

static const int kIterBlocks = 148 * 8;

int64_t spmk_pagerank_scratch_doubles(void) { return 2 * kIterBlocks; }

spmk_status spmk_pagerank_init(const float* d_r, const int32_t* d_counts, int64_t m, int64_t m_total,
                               double alpha, double* d_state, double* d_scratch, void* stream) {
  if (!d_r || !d_counts || !d_state || !d_scratch || m < 0 || m_total < 1) return fail(SPMK_EINVAL, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  dangling_mass_kernel<<<kIterBlocks, kIterThreads, 0, s>>>(d_r, d_counts, m, d_scratch); LAUNCHED(1);
  pagerank_finalize_kernel<<<1, 32, 0, s>>>(d_scratch, kIterBlocks, m_total, alpha, d_state, nullptr, 0); LAUNCHED(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPMK_OK : fail(SPMK_ECUDA, cudaGetErrorString(e));
}

spmk_status spmk_pagerank_step(const float* d_y, float* d_r, const int32_t* d_counts, int64_t m,
                               int64_t m_total, double alpha, double* d_state, double* d_scratch,
                               double* d_hist, int32_t t, void* stream) {
  if (!d_y || !d_r || !d_counts || !d_state || !d_scratch || m < 0 || m_total < 1)
    return fail(SPMK_EINVAL, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  pagerank_update_kernel<<<kIterBlocks, kIterThreads, 0, s>>>(d_y, d_r, d_counts, m, (float)alpha, d_state,
                                                              d_scratch); LAUNCHED(1);
  pagerank_finalize_kernel<<<1, 32, 0, s>>>(d_scratch, kIterBlocks, m_total, alpha, d_state, d_hist, t); LAUNCHED(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPMK_OK : fail(SPMK_ECUDA, cudaGetErrorString(e));
}

spmk_status spmk_pagerank_step_p2p(const float* d_y, const float* d_x_cur, float* const* peer_x_next,
                                   int32_t npeers, const int32_t* d_counts, int64_t row0, int64_t m,
                                   int64_t m_total, double alpha, double* d_state, double* d_scratch,
                                   void* stream) {
  if (!d_y || !d_x_cur || !peer_x_next || !d_counts || !d_state || !d_scratch || m < 0 || m_total < 1 ||
      row0 < 0 || npeers < 1 || npeers > kMaxPeers)
    return fail(SPMK_EINVAL, "bad argument");
  PeerPtrs pp{};
  for (int q = 0; q < npeers; ++q) {
    if (!peer_x_next[q]) return fail(SPMK_EINVAL, "null peer buffer");
    pp.p[q] = peer_x_next[q];
  }
  cudaStream_t s = (cudaStream_t)stream;
  pagerank_update_p2p_kernel<<<kIterBlocks, kIterThreads, 0, s>>>(d_y, d_x_cur, d_counts, row0, m, (float)alpha,
                                                                  d_state, pp, npeers, d_scratch); LAUNCHED(1);
  pagerank_finalize_kernel<<<1, 32, 0, s>>>(d_scratch, kIterBlocks, m_total, alpha, d_state, nullptr, 0); LAUNCHED(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPMK_OK : fail(SPMK_ECUDA, cudaGetErrorString(e));
}

spmk_status spmk_ipc_handle(const void* d_ptr, void* handle64) {
  if (!d_ptr || !handle64) return fail(SPMK_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr));
  if (e != cudaSuccess) return fail(SPMK_ECUDA, cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  std::memcpy(handle64, &h, 64);
  return SPMK_OK;
}

spmk_status spmk_ipc_open(const void* handle64, void** d_ptr) {
  if (!handle64 || !d_ptr) return fail(SPMK_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(SPMK_ECUDA, cudaGetErrorString(e));
  return SPMK_OK;
}

spmk_status spmk_ipc_close(void* d_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  return e == cudaSuccess ? SPMK_OK : fail(SPMK_ECUDA, cudaGetErrorString(e));
}

uint64_t spmk_launch_count(void) { return g_launches.load(); }

spmk_status spmk_timing_enable(int on) {
  g_timing.on = on != 0;
  return SPMK_OK;
}

spmk_status spmk_timing_last(float* main_kernel_ms, float* whole_call_ms) {
  if (!g_timing.on || !g_timing.ev[0]) return fail(SPMK_EINVAL, "timing not enabled / no call recorded");
  if (cudaEventSynchronize(g_timing.ev[3]) != cudaSuccess) return fail(SPMK_ECUDA, "event sync");
  if (main_kernel_ms) cudaEventElapsedTime(main_kernel_ms, g_timing.ev[1], g_timing.ev[2]);
  if (whole_call_ms) cudaEventElapsedTime(whole_call_ms, g_timing.ev[0], g_timing.ev[3]);
  return SPMK_OK;
}

}  // extern "C"
