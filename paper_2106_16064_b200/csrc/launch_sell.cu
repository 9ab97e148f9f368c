// launch_sell.cu — plan and launch of the lane-per-job seq-ws sweep
// (sell_kernels.cuh; spmm_seq_balanced kernels.hpp:384-455).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cub/cub.cuh>
#include <map>
#include <mutex>
#include <vector>

#include "internal.h"
#include "sell_kernels.cuh"

using namespace spmk_dev;

namespace spmk_host {
namespace {

// Work-queue chunk sizes in steps: >= every shape's S + C - 1 (the rings run
// at most one chunk ahead, and the sweep resolves the next chunk once per S
// steps); the smallest allowed measured best at cfg2 (finer tail).
constexpr int kSellChunkMin = 12, kSellChunkMax = 512;
constexpr int kSellGuide = 4;  // target chunk = remaining steps / (kSellGuide x warps)
constexpr int kSellMaxTiles = 64;                        // column tiles (N <= 2048)
constexpr unsigned long long kSellMaxXBytes = 768ull << 20;  // seq-ws default: X up to 768 MB
// Sweep shapes (ring depths S / C, warps per CTA, CTAs per SM); tuning knob
// sell_cfg picks one (measured on B200).
struct SellShape {
  const void* fn;
  void (*launch)(dim3, const SellArgs&, cudaStream_t);
  int wpc, smem;
};
template <int CW, int S, int C, int WPC, int MINB>
void sell_launch_t(dim3 grid, const SellArgs& a, cudaStream_t s) {
  seq_sell_kernel<CW, S, C, WPC, MINB><<<grid, WPC * 32, sell_smem_bytes<CW, S, C, WPC>(), s>>>(a);
}
template <int CW, int S, int C, int WPC, int MINB>
constexpr SellShape sell_shape() {
  return SellShape{reinterpret_cast<const void*>(seq_sell_kernel<CW, S, C, WPC, MINB>),
                   sell_launch_t<CW, S, C, WPC, MINB>, WPC, sell_smem_bytes<CW, S, C, WPC>()};
}
// [column width 32 / 16 / 8][sell_cfg]; a step's rows are 4 KB at every width,
// its A part 256 B x (32 / CW)
constexpr int kSellShapeCount = 4;
const SellShape kSellShapes[3][kSellShapeCount] = {
    {
        sell_shape<32, 4, 8, 4, 3>(),   // 0: 12 warps / SM, 3 steps of rows in flight per warp
        sell_shape<32, 2, 4, 8, 2>(),   // 1: 16 warps, 1 in flight
        sell_shape<32, 4, 8, 12, 1>(),  // 2: 12 warps in one CTA
        sell_shape<32, 3, 6, 4, 4>(),   // 3: 16 warps, 2 in flight
    },
    {
        sell_shape<16, 4, 8, 5, 2>(),   // 0: 10 warps / SM
        sell_shape<16, 3, 6, 4, 3>(),   // 1: 12 warps, 2 in flight
        sell_shape<16, 2, 4, 8, 2>(),   // 2: 16 warps, 1 in flight
        sell_shape<16, 3, 6, 5, 2>(),   // 3: 10 warps, 2 in flight
    },
    {
        sell_shape<8, 4, 8, 3, 3>(),    // 0: 9 warps / SM
        sell_shape<8, 3, 6, 4, 3>(),    // 1: 12 warps, 2 in flight
        sell_shape<8, 2, 4, 8, 2>(),    // 2: 16 warps, 1 in flight
        sell_shape<8, 3, 6, 5, 2>(),    // 3: 10 warps, 2 in flight
    },
};
int cw_index(int cw) { return cw == 32 ? 0 : (cw == 16 ? 1 : 2); }

template <typename T>
struct DevTmp {
  T* p = nullptr;
  explicit DevTmp(size_t n) { p = dev_alloc<T>(n); }
  ~DevTmp() { cudaFree(p); }
  DevTmp(const DevTmp&) = delete;
  DevTmp& operator=(const DevTmp&) = delete;
};

template <typename In, typename Out>
void exclusive_scan(const In* in, Out* out, int n, cudaStream_t s) {
  size_t bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
  DevTmp<unsigned char> tmp(bytes);
  CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, s));
}

__global__ void fold_keys_kernel(const int4* f, int n, int* key, int* idx) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    key[i] = f[i].z;
    idx[i] = i;
  }
}
__global__ void gather_int4_kernel(const int4* in, const int* idx, int n, int4* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[idx[i]];
}
__global__ void iota_kernel(int* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}

// Resident CTAs per SM of a sweep shape (and its shared-memory opt-in), per device.
int sell_blocks_per_sm(int cw, int shape) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, int> cache;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, cw, shape});
  if (it != cache.end()) return it->second;
  const SellShape& sh = kSellShapes[cw_index(cw)][shape];
  int bps = 1;
  CK(cudaFuncSetAttribute(sh.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, sh.smem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, sh.fn, sh.wpc * 32, sh.smem));
  if (bps < 1) bps = 1;
  cache[{dev, cw, shape}] = bps;
  return bps;
}

int sell_shape_of(const spmk_csr_s* h) {
  const long long v = h->tune.sell_cfg;
  return v >= 0 && v < kSellShapeCount ? (int)v : 0;
}

// Dev tracing (SPMK_SELL_TRACE=1): per-warp start / end times of the last
// sweep, read back with spmk_sell_trace (not part of the drop-in surface).
unsigned long long* g_trace = nullptr;
int g_trace_n = 0;
unsigned long long* sell_trace_buffer(int nwarps) {
  static const bool on = [] {
    const char* v = std::getenv("SPMK_SELL_TRACE");
    return v && *v == '1';
  }();
  if (!on) return nullptr;
  if (g_trace_n < nwarps) {
    cudaFree(g_trace);
    g_trace = dev_alloc<unsigned long long>((size_t)4 * nwarps);
    g_trace_n = nwarps;
  }
  return g_trace;
}

}  // namespace

extern "C" int spmk_sell_trace(unsigned long long* out, int cap) {
  const int n = std::min(cap, g_trace_n);
  if (n > 0 && cudaMemcpy(out, g_trace, sizeof(unsigned long long) * 4 * n, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return n;
}

int sell_width(const spmk_csr_s* h, long long CH, int N, bool aligned) {
  // N = 8 / 16 / 32 (one tile of 8 / 16 / 32 columns, 4 / 2 / 1 jobs per
  // lane); at N = 64 / 128 the tile sweep (16 / 32 lanes per unit, 256 /
  // 512-byte rows per gather) measured 7 % / 34 % faster on B200, so 32-column
  // tiles of wider X only with seq_impl 3
  if (h->tune.seq_impl < 2) return 0;
  int cw = 0;
  // seq-ws with an X far beyond L2 (DRAM-bound gathers): the tile sweep's
  // row-order locality wins (R-MAT s24 e32: N = 16 / 32 tile 4.9 / 7.0 ms vs
  // 5.8 / 8.0; X 1.07 / 2.1 GB), below it the sweep (s22 N = 32, X 537 MB:
  // 830 vs 934 us; s24 N = 8, X 537 MB: 3.6 vs 4.3 ms); seq-rs always
  const bool big_x = CH != kSellNoChunk && (unsigned long long)h->k * N * 4 > kSellMaxXBytes;
  if (h->tune.seq_impl == 2 && big_x) return 0;
  if (N == 32 || N == 16 || N == 8) cw = N;
  else if (h->tune.seq_impl == 3 && N % 32 == 0 && N / 32 <= kSellMaxTiles) cw = 32;
  const bool ok = cw > 0 && aligned && (CH <= kSellMaxChunk || CH == kSellNoChunk) && h->k < INT32_MAX &&
                  (unsigned long long)h->k * (unsigned long long)(N / 4) < (1ull << 32) && h->nnz < INT32_MAX &&
                  h->m < INT32_MAX;
  return ok ? cw : 0;
}

SellPlan& get_sell_plan(spmk_csr_s* h, long long CH, int lmax, int cw, cudaStream_t s) {
  const int shape = sell_shape_of(h);
  const auto key = std::make_tuple(CH, shape * 64 + cw, lmax);
  const int jps = 32 * (32 / cw);  // jobs per slice
  auto it = h->sell_plans.find(key);
  if (it != h->sell_plans.end()) return it->second;
  const int mne = h->mne;
  SellPlan p;
  p.CH = CH;
  p.shape = shape;
  p.cw = cw;
  // jobs per compact row, H slots, fold rows
  DevTmp<int> njob(mne + 1), nslot(mne + 1), nmulti(mne + 1);
  DevTmp<int> joff(mne + 1), soff(mne + 1), moff(mne + 1);
  CK(cudaMemsetAsync(njob.p + mne, 0, sizeof(int), s));
  CK(cudaMemsetAsync(nslot.p + mne, 0, sizeof(int), s));
  CK(cudaMemsetAsync(nmulti.p + mne, 0, sizeof(int), s));
  sell_count_kernel<<<grid_for(mne), 256, 0, s>>>(h->crp, mne, CH, lmax, njob.p, nslot.p, nmulti.p); LAUNCHED(1);
  exclusive_scan(njob.p, joff.p, mne + 1, s);
  exclusive_scan(nslot.p, soff.p, mne + 1, s);
  exclusive_scan(nmulti.p, moff.p, mne + 1, s);
  int tot[3];
  CK(cudaMemcpyAsync(&tot[0], joff.p + mne, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&tot[1], soff.p + mne, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&tot[2], moff.p + mne, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int Jr = tot[0];
  const int J = Jr + h->nempty;
  p.nslots = tot[1];
  p.nfold = tot[2];
  DevTmp<int> jstart(J), jlen(J), jout(J);
  if (p.nfold > 0) p.fold = dev_alloc<int4>(p.nfold);
  sell_jobs_kernel<<<grid_for(mne), 256, 0, s>>>(h->crp, h->rid, mne, CH, lmax, joff.p, soff.p, moff.p, jstart.p,
                                                 jlen.p, jout.p, p.fold); LAUNCHED(1);
  if (p.nfold > 1) {  // fold rows with the most slots first (the jobs address H slots, not fold rows)
    DevTmp<int> key(p.nfold), key_s(p.nfold), fidx(p.nfold), fidx_s(p.nfold);
    DevTmp<int4> tmpf(p.nfold);
    fold_keys_kernel<<<grid_for(p.nfold), 256, 0, s>>>(p.fold, p.nfold, key.p, fidx.p); LAUNCHED(1);
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, key.p, key_s.p, fidx.p, fidx_s.p, p.nfold, 0, 32, s));
    DevTmp<unsigned char> tmp(bytes);
    CK(cub::DeviceRadixSort::SortPairsDescending(tmp.p, bytes, key.p, key_s.p, fidx.p, fidx_s.p, p.nfold, 0, 32, s));
    gather_int4_kernel<<<grid_for(p.nfold), 256, 0, s>>>(p.fold, fidx_s.p, p.nfold, tmpf.p); LAUNCHED(1);
    CK(cudaMemcpyAsync(p.fold, tmpf.p, sizeof(int4) * p.nfold, cudaMemcpyDeviceToDevice, s));
    std::vector<int> ks((size_t)p.nfold);
    CK(cudaMemcpyAsync(ks.data(), key_s.p, sizeof(int) * p.nfold, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    while (p.nbig < p.nfold && ks[(size_t)p.nbig] > kFoldWarpMax) ++p.nbig;
    p.n4 = p.nbig;
    while (p.n4 < p.nfold && ks[(size_t)p.n4] > 4) ++p.n4;
    p.n2 = p.n4;
    while (p.n2 < p.nfold && ks[(size_t)p.n2] > 2) ++p.n2;
  } else if (p.nfold == 1) {
    int4 f1;
    CK(cudaMemcpyAsync(&f1, p.fold, sizeof(int4), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    p.nbig = f1.z > kFoldWarpMax ? 1 : 0;
    p.n4 = f1.z > 4 ? 1 : 0;
    p.n2 = f1.z > 2 ? 1 : 0;
  }
  if (h->nempty > 0) {
    sell_empty_jobs_kernel<<<grid_for(h->nempty), 256, 0, s>>>(h->erow, h->nempty, Jr, jstart.p, jlen.p, jout.p); LAUNCHED(1);
  }
  // jobs by length, descending (stable: equal lengths keep row order)
  DevTmp<int> idx(J), sidx(J), slen(J);
  iota_kernel<<<grid_for(J), 256, 0, s>>>(idx.p, J); LAUNCHED(1);
  {
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, jlen.p, slen.p, idx.p, sidx.p, J, 0, 16, s));
    DevTmp<unsigned char> tmp(bytes);
    CK(cub::DeviceRadixSort::SortPairsDescending(tmp.p, bytes, jlen.p, slen.p, idx.p, sidx.p, J, 0, 16, s));
  }
  const int nsl = (int)(((long long)J + jps - 1) / jps);
  DevTmp<long long> lsteps(nsl + 1), lcost(nsl + 1), step_ex(nsl + 1);
  CK(cudaMemsetAsync(lsteps.p + nsl, 0, sizeof(long long), s));
  sell_slice_kernel<<<grid_for(nsl), 256, 0, s>>>(slen.p, nsl, jps, lsteps.p, lcost.p); LAUNCHED(1);
  exclusive_scan(lsteps.p, step_ex.p, nsl + 1, s);
  std::vector<long long> sx((size_t)nsl + 1);
  CK(cudaMemcpyAsync(sx.data(), step_ex.p, sizeof(long long) * sx.size(), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const long long T = sx[(size_t)nsl];
  if (T >= INT32_MAX) throw CudaError{SPMK_EUNSUPPORTED, "sell layout: too many steps"};
  p.nsteps = T;
  p.steps = dev_alloc<int>((size_t)T * 2 * jps);
  int dev = 0, sms = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  p.sms = sms;
  p.blocks = sms * sell_blocks_per_sm(cw, shape);
  p.nwarps = p.blocks * kSellShapes[cw_index(cw)][shape].wpc;
  // Chunks of whole slices for the warps' work queue, guided sizes: about
  // remaining / (4 W) steps, clamped to [kSellChunkMin, kSellChunkMax] (a
  // slice longer than that is one chunk); the first W are the warps' first
  // chunks, the rest are claimed in order.
  std::vector<int> cs;
  cs.reserve(4 * (size_t)p.nwarps + 16);
  int si = 0;
  while (si < nsl) {
    cs.push_back((int)sx[(size_t)si]);
    const long long rem = T - sx[(size_t)si];
    const long long target = std::max<long long>(kSellChunkMin, std::min<long long>(kSellChunkMax, rem / ((long long)kSellGuide * p.nwarps)));
    const long long start = sx[(size_t)si];
    while (si < nsl && sx[(size_t)si] - start < target) ++si;
  }
  cs.push_back((int)T);
  p.nchunks = (int)cs.size() - 1;
  p.cstep = dev_alloc<int>(cs.size());
  CK(cudaMemcpyAsync(p.cstep, cs.data(), sizeof(int) * cs.size(), cudaMemcpyHostToDevice, s));
  p.sched = dev_alloc<int>(2 * kSellMaxTiles);
  CK(cudaMemsetAsync(p.sched, 0, sizeof(int) * 2 * kSellMaxTiles, s));
  sell_fill_kernel<<<grid_for((long long)nsl * 32), 256, 0, s>>>(sidx.p, slen.p, J, nsl, jps, cw == 32 ? 0 : 512 / (4 * cw), step_ex.p, jstart.p, jout.p,
                                                                 h->col, h->val, p.steps); LAUNCHED(1);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));  // temporaries (and cs) are freed on return
  return h->sell_plans.emplace(key, p).first->second;
}

void free_sell_plan(SellPlan& p) {
  cudaFree(p.steps);
  cudaFree(p.cstep);
  cudaFree(p.sched);
  cudaFree(p.fold);
  p = SellPlan{};
}

void launch_sell(spmk_csr_s* h, SellPlan& p, const float* X, int N, float* Y, float* H, bool side_busy,
                 cudaStream_t s) {
  const int tiles = N / p.cw;
  SellArgs a{};
  a.steps = p.steps;
  a.cstep = p.cstep;
  a.sched = p.sched;
  a.nchunks = p.nchunks;
  a.X = X;
  a.Y = Y;
  a.H = H;
  a.N = N;
  a.K = (int)std::min<long long>(h->k, 1 << 30);
  a.claim_first = side_busy ? 1 : 0;
  a.one2 = kOnePair;
  a.trace = sell_trace_buffer(p.nwarps);
  sell_blocks_per_sm(p.cw, p.shape);  // shared-memory opt-in on this device
  kSellShapes[cw_index(p.cw)][p.shape].launch(dim3(p.blocks, tiles), a, s); LAUNCHED(1);
  if (p.nfold > 0) {
    // programmatic dependent launch: scheduled while the sweep drains
    cudaLaunchConfig_t lc = {};
    FoldTiers ft;
    ft.n4 = p.n4;
    ft.n2 = p.n2;
    ft.w8 = (int)(((long long)(p.n4 - p.nbig) * tiles + 3) / 4);
    ft.w4 = (int)(((long long)(p.n2 - p.n4) * tiles + 3) / 4);
    const long long small_warps = (long long)ft.w8 + ft.w4 + ((long long)(p.nfold - p.n2) * tiles + 7) / 8;
    constexpr int wpb = kFoldThreads / 32;
    lc.gridDim = dim3((unsigned)((long long)p.nbig * tiles + (small_warps + wpb - 1) / wpb));
    lc.blockDim = dim3(kFoldThreads);
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, sell_fold_kernel, (const int4*)p.fold, p.nfold, p.nbig, ft, (const float*)H, Y, N)); LAUNCHED(1);
  }
}

}  // namespace spmk_host
