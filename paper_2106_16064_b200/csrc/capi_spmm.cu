// capi_spmm.cu — the spmm dispatcher (kernels.hpp:457-464) and its C entry
// points: device operands (spmk_spmm), rule-selected (spmk_spmm_auto), host
// operands through the handle's staging slots (spmk_spmm_host[_async]) and the
// reference's one-shot value-returning call shape (spmk_spmm_csr_host).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace spmk_host {
namespace {

// Event sets of the last kRing calls (one per call, reused cyclically), so a
// caller can time many calls without synchronizing between them.
struct Timing {
  static constexpr int kRing = 256;
  bool on = false;
  int device = -1;
  long long calls = 0;  // calls recorded since enable
  cudaEvent_t ev[kRing][4] = {};  // call0, main0, main1, call1
};
thread_local Timing g_timing;

void timing_record(int which, cudaStream_t s) {
  if (!g_timing.on) return;
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_timing.device != dev) {
    for (auto& q : g_timing.ev)
      for (auto& e : q) {
        if (e) cudaEventDestroy(e);
        cudaEventCreate(&e);
      }
    g_timing.device = dev;
  }
  if (which == 0) ++g_timing.calls;
  cudaEventRecord(g_timing.ev[(g_timing.calls - 1) % Timing::kRing][which], s);
}

spmk_kernel_config cfg_or_default(const spmk_kernel_config* cfg) {
  spmk_kernel_config c;
  spmk_default_config(&c);
  return cfg ? *cfg : c;
}

// Hub threshold of the row-split variants (0 disables the hub path).
// Measured on B200 (R-MAT s20..s25 heavy): par-rs 2048 (s25 N=1: 3.91 ms at
// 1024, 3.37 ms at 2048, 3.50 ms at 4096), seq-rs 1024 (s20 N=32: 0.77 ms,
// 0.88 ms at 4096).
int hub_threshold(const spmk_csr_s* h, spmk_kernel_id id) {
  const long long dflt = id == SPMK_PAR_ROWSPLIT ? 2048 : 1024;
  const long long v = h->tune.hub_nnz < 0 ? dflt : h->tune.hub_nnz;
  return (int)std::max(0LL, std::min<long long>(v, INT32_MAX));
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
// results bit-exact; these are pure performance knobs.
long long tile_chunks(long long chunk, long long target) {
  long long t = target / chunk;
  return t < 1 ? 1 : t;
}

// Virtual lanes per physical lane for par-rs at lane_width 32, N <= 4 (the
// results do not depend on it).  Measured on B200: rows averaging >= 24
// nonzeros fill a 32-lane group (cfg5 8-way slices 0-3, avg 27..443: VL=1
// 0.36-0.41 ms vs VL=4 0.41-0.45 ms); shorter rows want narrow groups (tail
// slice, avg 4.5: 0.75 -> 0.60 ms at VL=4), 8 on low-cv graphs at N=1
// (s20 uniform: 159 us at 1, 128 at 4, 112 at 8).
int par_rs_vl(const spmk_csr_s* h, int W, int N) {
  if (h->tune.parrs_vl > 0) return (int)h->tune.parrs_vl;
  if (W != 32 || N > 4) return 1;
  const double M = (double)h->m, avg = (double)h->nnz / M;
  const double var = std::max(0.0, (double)h->sum_len2 / M - avg * avg);
  const double cv = avg > 0.0 ? std::sqrt(var) / avg : 0.0;
  if (avg >= 24.0) return 1;
  if (N == 2 && cv > 1.0) return 1;  // s22 heavy N=2: 543 us at 1, 577 at 4
  return (N == 1 && cv <= 1.0) ? 8 : 4;
}

// Access-policy window over X on `s` (persisting hits, streaming misses),
// clamped to the device limits; bytes == 0 clears it.
void set_l2_window(cudaStream_t s, const void* d_x, size_t bytes) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  cudaStreamAttrValue attr;
  std::memset(&attr, 0, sizeof(attr));
  if (bytes == 0 || d_x == nullptr) {
    attr.accessPolicyWindow.num_bytes = 0;
    CK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &attr));
    CK(cudaCtxResetPersistingL2Cache());
    return;
  }
  int max_win = 0, max_persist = 0;
  CK(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev));
  CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
  if (max_win <= 0 || max_persist <= 0) throw CudaError{SPMK_EUNSUPPORTED, "no L2 persistence on this device"};
  const size_t persist = std::min<size_t>(bytes, (size_t)max_persist);
  size_t cur = 0;
  CK(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
  if (cur != persist) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist));
  const size_t win = std::min<size_t>(bytes, (size_t)max_win);
  attr.accessPolicyWindow.base_ptr = const_cast<void*>(d_x);
  attr.accessPolicyWindow.num_bytes = win;
  attr.accessPolicyWindow.hitRatio = std::min(1.0f, (float)persist / (float)win);
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  CK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &attr));
}

spmk_status run_spmm(spmk_csr_s* h, spmk_kernel_id id, const spmk_kernel_config& cfg, const float* d_x,
                     int64_t n, float* d_y, cudaStream_t s) {
  const long long M = h->m;
  if (n == 0 || M == 0) return SPMK_OK;
  if (h->nnz == 0 || h->mne == 0) {
    launch_zero_all(d_y, M * n, s);
    CK(cudaGetLastError());
    return SPMK_OK;
  }
  if (n > INT32_MAX / 2) return fail(SPMK_EUNSUPPORTED, "n too large");
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(s, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (!capturing && h->has_last && h->last_stream != s) CK(cudaStreamWaitEvent(s, h->ev_last, 0));
  if (h->tune.l2_persist) set_l2_window(s, d_x, (size_t)h->k * (size_t)n * 4);
  timing_record(0, s);
  const int N = (int)n;
  const bool aligned = ((uintptr_t)d_x % 16 == 0) && ((uintptr_t)d_y % 16 == 0);
  // Empty rows -> 0 (the reference's zero-initialised Y).  The variant
  // kernels never touch empty rows, so the zero fill runs on the handle's
  // side stream concurrently with them (fork/join through events: HBM writes
  // overlap the gather-bound sweep; capturable into CUDA graphs).
  // Row-split variants: hub rows (>= L nonzeros) run in hub_kernels.cuh on
  // the side stream, concurrently with the main kernel (disjoint rows of Y).
  // seq-ws / seq-rs at N = 32: the lane-per-job sweep (it writes the empty
  // rows itself); seq-rs rows of >= L nonzeros go to the hub kernels
  const int cw_ws = id == SPMK_SEQ_BALANCED ? sell_width(h, (long long)cfg.seq_chunk, N, aligned) : 0;
  const int cw_rs = id == SPMK_SEQ_ROWSPLIT ? sell_width(h, kSellNoChunk, N, aligned) : 0;
  const bool sell_ws = cw_ws > 0, sell_rs = cw_rs > 0;
  const bool sell = sell_ws || sell_rs;
  const bool rs = id == SPMK_PAR_ROWSPLIT || id == SPMK_SEQ_ROWSPLIT;
  // seq-rs hub threshold under the sweep (measured on B200, R-MAT heavy):
  // N = 32 1024 (s22: 1343 us vs 1443 at 512, 1843 at 256; s20 equal);
  // N = 8 / 16 (4 / 2 jobs per lane: longer slices) 512 (N=8 s20 282 vs 402
  // us at 1024, s22 equal; N=16 s20 309 vs 367, s22 1107 vs 974)
  const int L = rs ? ((cw_rs > 0 && cw_rs < 32 && h->tune.hub_nnz < 0) ? 512 : hub_threshold(h, id)) : 0;
  const Plan* hub = L > 0 ? &get_hub_plan(h, L, s) : nullptr;
  const bool hubs = hub && hub->nlong > 0;
  const bool zero_side = h->nempty > 0 && !sell;
  const bool fork = zero_side || hubs;
  if (fork) {
    if (!h->side) {
      CK(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(h->ev_fork, s));
    CK(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    if (hubs) launch_hubs(h, *hub, id, (int)cfg.lane_width, L, d_x, N, d_y, h->side);
    if (zero_side) launch_zero_rows(h, N, d_y, aligned && N % 4 == 0, h->side);
    CK(cudaEventRecord(h->ev_join, h->side));
  }

  if (id == SPMK_SEQ_ROWSPLIT || id == SPMK_SEQ_BALANCED) {
    SeqLaunch a{};
    a.crp = h->crp;
    a.rid = h->rid;
    a.col = h->col;
    a.val = h->val;
    a.X = d_x;
    a.Y = d_y;
    a.mne = h->mne;
    a.nnz = (int)h->nnz;
    a.N = N;
    if (sell_rs) {
      SellPlan& sp = get_sell_plan(h, kSellNoChunk, L > 0 ? L : INT32_MAX, cw_rs, s);
      timing_record(1, s);
      launch_sell(h, sp, d_x, N, d_y, nullptr, hubs, s);
      timing_record(2, s);
    } else if (id == SPMK_SEQ_ROWSPLIT) {
      const long long TS = h->tune.seq_tile_nnz > 0 ? h->tune.seq_tile_nnz : rs_tile_nnz(h->nnz, N);
      Plan& p = get_rs_desc(h, TS, L, hubs ? hub : nullptr, s);
      a.nunits = (int)p.ntiles;
      a.desc = p.desc;
      timing_record(1, s);
      launch_seq(a, false, aligned, s);
      timing_record(2, s);
    } else if (sell_ws) {
      SellPlan& sp = get_sell_plan(h, (long long)cfg.seq_chunk, INT32_MAX, cw_ws, s);
      float* H = sp.nslots > 0 ? h->scratch.get((size_t)sp.nslots * N) : nullptr;
      timing_record(1, s);
      launch_sell(h, sp, d_x, N, d_y, H, false, s);
      timing_record(2, s);
    } else {
      const long long CH = (long long)cfg.seq_chunk;
      const long long TS = CH * tile_chunks(CH, h->tune.seq_tile_nnz > 0 ? h->tune.seq_tile_nnz : 256);
      Plan& p = get_plan(h, 1, TS, CH, h->tune.seq_ext, s);  // EXT: measured (cfg2 -7 %)
      a.rlo = p.rlo;
      a.desc = p.desc;
      a.TS = TS;
      a.CH = CH;
      a.EXT = p.EXT;
      a.nunits = (int)p.ntiles;
      if (p.nlong > 0) {
        const long long nch = (h->nnz + CH - 1) / CH;
        float* sc = h->scratch.get((size_t)(nch + p.ntiles) * N);
        a.H = sc;
        a.Tsl = sc + (size_t)nch * N;
      }
      timing_record(1, s);
      launch_seq(a, true, aligned, s);
      timing_record(2, s);
      if (p.nlong > 0) launch_fixup(p, a.H, a.Tsl, d_y, N, s);
    }
  } else {
    ParLaunch a{};
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
    } else if (W == 64) {
      const long long nch = (h->nnz + 63) / 64;
      float* slots = h->scratch.get((size_t)(2 * nch) * N);
      timing_record(1, s);
      launch_par_ws64(a, slots, s);
      timing_record(2, s);
    } else {
      // W = 32, N <= 4: par_ws3 (below); with parws3 = 0, N <= 2 the streaming
      // head-flag kernel par_ws2, otherwise T chunks of W nonzeros per tile (4
      // or 8: the two compiled shapes of the tile kernel)
      const bool ws2 = W == 32 && N <= 2 && h->tune.parws_impl == 2;
      const int T = h->tune.parws_t == 8 ? 8 : 4;
      const long long CH = W;
      const long long chunks = (h->nnz + 31) / 32;
      // N = 1 … 4: par_ws3 (long rows too unless parws3 = 1) on ~16K tiles
      // (measured best on R-MAT uniform s16..s22 and banded s20: 4 .. 64; 8K or
      // 32K tiles up to 1.3x slower); with long
      // rows, par_ws2 (N <= 2) on its own tiles (the largest power of two <= 64
      // that still gives >= 8 waves of 32 resident warps per SM) or the tile kernel
      bool ws3 = W == 32 && N <= 4 && h->tune.parws_impl == 2 && h->tune.parws3 != 0;
      auto ws_cpt = [&](bool three) {
        long long c = h->tune.parws_cpt;
        if (c > 0) return c;
        c = 4;
        if (three) {  // tiles closest to 16K (log scale): double while > 16K * sqrt(2)
          if (chunks < 65536) c = 8;  // small (cfg1): 8.5 -> 7.9 us per call from a graph, 15.2 -> 15.1 flushed
          while (c < 64 && chunks > 23170LL * c) c *= 2;
        } else {
          while (c < 64 && chunks / (c * 2) >= 8LL * 148 * 32) c *= 2;
        }
        return c;
      };
      long long TS = ws3 ? CH * ws_cpt(true) : (ws2 ? CH * ws_cpt(false) : CH * T);
      Plan* pp = &get_plan(h, 2, TS, CH, h->tune.parws_ext, s);
      if (ws3 && pp->nlong > 0 && h->tune.parws3 < 2) {
        ws3 = false;
        TS = ws2 ? CH * ws_cpt(false) : CH * T;
        pp = &get_plan(h, 2, TS, CH, h->tune.parws_ext, s);
      }
      Plan& p = *pp;
      a.rlo = p.rlo;
      a.desc = p.desc;
      a.TS = TS;
      a.nunits = (int)p.ntiles;
      if (p.nlong > 0) {
        const long long nch = (h->nnz + CH - 1) / CH;
        float* sc = h->scratch.get((size_t)(nch + p.ntiles) * N);
        a.H = sc;
        a.Tsl = sc + (size_t)nch * N;
      }
      const unsigned* hf = ws2 || ws3 ? get_head_flags32(h, s) : nullptr;
      timing_record(1, s);
      if (ws3) launch_par_ws3(a, hf, h->mne == h->m, aligned, p.nlong > 0, s);
      else if (ws2) launch_par_ws2(a, hf, aligned, s);
      else launch_par_ws(a, W, T, aligned, s);
      timing_record(2, s);
      if (p.nlong > 0) launch_fixup(p, a.H, a.Tsl, d_y, N, s);
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

// H2D(x) -> spmm -> D2H(y) on `s` through one of the handle's staging slots;
// the slot's previous user is awaited on the device (event), not the host.
spmk_status spmm_host_enqueue(spmk_csr_s* a, spmk_kernel_id id, const spmk_kernel_config& c, const float* x,
                              int64_t n, float* y, cudaStream_t s) {
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

spmk_status check_call(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg, int64_t n) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  if ((int)id < 0 || (int)id > 3) return fail(SPMK_EINVAL, "bad kernel id");
  spmk_status st = spmk_check_config(cfg);
  if (st != SPMK_OK) return st;
  if (n < 0) return fail(SPMK_EDIM, "negative n");
  return SPMK_OK;
}

}  // namespace
}  // namespace spmk_host

using namespace spmk_host;

extern "C" {

spmk_status spmk_spmm(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg,
                      const float* d_x, int64_t n, float* d_y, void* stream) {
  spmk_status st = check_call(a, id, cfg, n);
  if (st != SPMK_OK) return st;
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

spmk_status spmk_spmm_host(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg,
                           const float* x, int64_t n, float* y, void* stream) {
  spmk_status st = check_call(a, id, cfg, n);
  if (st != SPMK_OK) return st;
  if (n == 0 || a->m == 0) return SPMK_OK;
  if (!y || (a->k > 0 && !x)) return fail(SPMK_EINVAL, "null operand");
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
  spmk_status st = check_call(a, id, cfg, n);
  if (st != SPMK_OK) return st;
  if (n == 0 || a->m == 0) return SPMK_OK;
  if (!y || (a->k > 0 && !x)) return fail(SPMK_EINVAL, "null operand");
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
  // One call per handle: the lane-per-job layout (a sorted copy of A) could
  // not be amortised, so the tile sweeps run unless SPMK_SEQ_IMPL asks.
  if (!std::getenv("SPMK_SEQ_IMPL")) h->tune.seq_impl = 1;
  st = spmk_spmm_host(h, id, cfg, x, n, y, nullptr);
  spmk_csr_destroy(h);
  return st;
}

spmk_status spmk_l2_persist_x(void* stream, const float* d_x, size_t bytes) {
  try {
    set_l2_window((cudaStream_t)stream, d_x, bytes);
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_timing_enable(int on) {
  g_timing.on = on != 0;
  g_timing.calls = 0;
  return SPMK_OK;
}

spmk_status spmk_timing_last(float* main_kernel_ms, float* whole_call_ms) {
  if (!g_timing.on || g_timing.calls == 0) return fail(SPMK_EINVAL, "timing not enabled / no call recorded");
  cudaEvent_t* q = g_timing.ev[(g_timing.calls - 1) % Timing::kRing];
  if (cudaEventSynchronize(q[3]) != cudaSuccess) return fail(SPMK_ECUDA, "event sync");
  if (main_kernel_ms) cudaEventElapsedTime(main_kernel_ms, q[1], q[2]);
  if (whole_call_ms) cudaEventElapsedTime(whole_call_ms, q[0], q[3]);
  return SPMK_OK;
}

spmk_status spmk_timing_summary(float* main_kernel_ms, float* whole_call_ms, int* calls) {
  if (!g_timing.on || g_timing.calls == 0) return fail(SPMK_EINVAL, "timing not enabled / no call recorded");
  const long long n = std::min<long long>(g_timing.calls, Timing::kRing);
  if (cudaEventSynchronize(g_timing.ev[(g_timing.calls - 1) % Timing::kRing][3]) != cudaSuccess)
    return fail(SPMK_ECUDA, "event sync");
  double m = 0, w = 0;
  for (long long i = g_timing.calls - n; i < g_timing.calls; ++i) {
    cudaEvent_t* q = g_timing.ev[i % Timing::kRing];
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, q[1], q[2]);
    cudaEventElapsedTime(&b, q[0], q[3]);
    m += a;
    w += b;
  }
  if (main_kernel_ms) *main_kernel_ms = (float)m;
  if (whole_call_ms) *whole_call_ms = (float)w;
  if (calls) *calls = (int)n;
  return SPMK_OK;
}

spmk_status spmk_spmm_path(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg, int64_t n,
                           int* path) {
  if (!a || !path) return fail(SPMK_EINVAL, "null argument");
  const spmk_kernel_config c = cfg_or_default(cfg);
  const bool ok = n > 0 && n <= INT32_MAX;
  *path = ok && ((id == SPMK_SEQ_BALANCED && spmk_host::sell_width(a, (long long)c.seq_chunk, (int)n, true) > 0) ||
                 (id == SPMK_SEQ_ROWSPLIT && spmk_host::sell_width(a, spmk_host::kSellNoChunk, (int)n, true) > 0))
              ? 1
              : 0;
  return SPMK_OK;
}

}  // extern "C"
