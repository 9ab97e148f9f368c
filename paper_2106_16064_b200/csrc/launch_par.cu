// launch_par.cu — launches of the parallel-reduction kernels (north_star b
// par-rs kernels.hpp:157-224 in par_kernels.cuh; north_star d par-ws
// kernels.hpp:232-330 in par_ws.cuh) and of the row-split hub-row kernels
// (hub_kernels.cuh) that both row-split variants use for rows >= L nonzeros.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "hub_kernels.cuh"
#include "internal.h"
#include "par_kernels.cuh"
#include "par_ws.cuh"
#include "par_ws64.cuh"
#include "par_ws2.cuh"
#include "par_ws3.cuh"

using namespace spmk_dev;

namespace spmk_host {
namespace {

std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, bool> g_attr_done;
bool need_smem_attr(const void* fn) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  return !std::exchange(g_attr_done[{fn, dev}], true);
}

ParArgs to_args(const ParLaunch& l) {
  ParArgs a{};
  a.crp = l.crp;
  a.rid = l.rid;
  a.col = l.col;
  a.val = l.val;
  a.X = l.X;
  a.Y = l.Y;
  a.H = l.H;
  a.Tsl = l.Tsl;
  a.rlo = l.rlo;
  a.desc = l.desc;
  a.mne = l.mne;
  a.nnz = l.nnz;
  a.N = l.N;
  a.TS = l.TS;
  a.nunits = l.nunits;
  a.hub = l.hub;
  return a;
}

// ------------------------------------------------------------ par-rs
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

// ------------------------------------------------------------ par-ws
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

// ------------------------------------------------------------ hub rows
template <int CW>
void launch_seq_hub(const HubArgs& g, int nhub, int N, long long pad, cudaStream_t s) {
  // hub_smem pads the shared-memory request (e.g. 120 KB: one hub CTA per
  // SM); measured neutral at N = 32 and slower at N = 128, so off.
  const int smem = (int)std::max<long long>(hub_smem_bytes<CW>(), pad);
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

}  // namespace

void launch_par_rs(const ParLaunch& l, int W, int vl, bool aligned, cudaStream_t s) {
  const ParArgs a = to_args(l);
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

// T = 4 chunks per tile, 5 blocks per SM: measured best on B200 (R-MAT s20
// heavy/uniform, N = 1 and 4; T = 6 / 8 and 4 / 6 blocks were slower).
void launch_par_ws(const ParLaunch& l, int W, int T, bool aligned, cudaStream_t s) {
  const ParArgs a = to_args(l);
  if (T == 8) launch_par_ws_tt<8, 4>(a, W, aligned, s);
  else launch_par_ws_tt<4, 5>(a, W, aligned, s);
}

void launch_par_ws2(const ParLaunch& l, const unsigned* hflag, bool aligned, cudaStream_t s) {
  ParWs2Args A{to_args(l), hflag};
  const int N = A.p.N;
  const int ct = N <= 1 ? 1 : 2;
  A.p.xvec = aligned && ct == 2 && N % 2 == 0;
  A.p.ncol_tile = ct;
  const dim3 grid((unsigned)((A.p.nunits + 7) / 8), (unsigned)((N + ct - 1) / ct));
  // groups of 2 chunks (measured: 4-chunk groups need 79 registers and run
  // slower, cfg5 2.72 vs 2.88 ms)
  if (ct == 1) par_ws2_kernel<1, 2><<<grid, 256, 0, s>>>(A);
  else par_ws2_kernel<2, 2><<<grid, 256, 0, s>>>(A);
  LAUNCHED(1);
}

template <bool LONG>
void launch_par_ws3_t(const ParWs2Args& A, cudaStream_t s) {
  const unsigned grid = (unsigned)((A.p.nunits + 7) / 8);
  if (A.p.N == 1) par_ws3_kernel<1, LONG><<<grid, 256, 0, s>>>(A);
  else if (A.p.N == 2) par_ws3_kernel<2, LONG><<<grid, 256, 0, s>>>(A);
  else if (A.p.N == 3) par_ws3_kernel<3, LONG><<<grid, 256, 0, s>>>(A);
  else par_ws3_kernel<4, LONG><<<grid, 256, 0, s>>>(A);
  LAUNCHED(1);
}
void launch_par_ws3(const ParLaunch& l, const unsigned* hflag, bool rid_ident, bool aligned, bool long_rows,
                    cudaStream_t s) {
  ParWs2Args A{to_args(l), hflag};
  if (rid_ident) A.p.rid = nullptr;  // no empty rows: compact row r is row r
  A.p.xvec = aligned ? 1 : 0;
  if (long_rows) launch_par_ws3_t<true>(A, s);
  else launch_par_ws3_t<false>(A, s);
}

void launch_par_ws64(const ParLaunch& l, float* slots, cudaStream_t s) {
  ParWs64Args a{l.crp, l.rid, l.col, l.val, l.X, l.Y, slots, l.mne, l.nnz, l.N, ((long long)l.nnz + 63) / 64};
  par_ws64_chunk_kernel<<<grid_for(a.chunks * 32, 256, 148 * 64), 256, 0, s>>>(a); LAUNCHED(1);
  par_ws64_merge_kernel<<<grid_for((long long)a.mne * a.N), 256, 0, s>>>(a); LAUNCHED(1);
  CK(cudaGetLastError());
}

void launch_hubs(spmk_csr_s* h, const Plan& hub, spmk_kernel_id id, int W, int L, const float* d_x, int N,
                 float* d_y, cudaStream_t s) {
  HubArgs g{hub.longrows, h->crp, h->rid, h->col, h->val, d_x, d_y, N};
  // seq-rs is the fold with one chain per column (W = 1: every position in
  // order, no tree) — kernels.hpp:366-370
  const bool seq = id == SPMK_SEQ_ROWSPLIT;
  const int FW = seq ? 1 : W;
  const long long two_pass = h->tune.hub_two_pass < 0 ? (seq ? 0 : 1) : h->tune.hub_two_pass;
  if (two_pass && FW * N <= kHubThreads) {
    const HubLayout& lay = get_hub_layout(h, hub, L, N, s);
    float* prod = h->hub_prod.get((size_t)lay.floats);
    HubProdArgs pa{hub.longrows, lay.segs, lay.po, h->crp, h->col, h->val, d_x, prod, N};
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
  if (seq) {
    const long long pad = h->tune.hub_smem;
    switch (cw) {
      case 1: launch_seq_hub<1>(g, hub.nlong, N, pad, s); break;
      case 2: launch_seq_hub<2>(g, hub.nlong, N, pad, s); break;
      case 4: launch_seq_hub<4>(g, hub.nlong, N, pad, s); break;
      case 8: launch_seq_hub<8>(g, hub.nlong, N, pad, s); break;
      case 16: launch_seq_hub<16>(g, hub.nlong, N, pad, s); break;
      default: launch_seq_hub<32>(g, hub.nlong, N, pad, s); break;
    }
  } else {
    cw = std::min(cw, kHubThreads / W);
    const dim3 grid((unsigned)hub.nlong, (unsigned)((N + cw - 1) / cw));
    par_rs_hub_kernel<<<grid, W * cw, 0, s>>>(g, W, cw); LAUNCHED(1);
  }
  CK(cudaGetLastError());
}

}  // namespace spmk_host
