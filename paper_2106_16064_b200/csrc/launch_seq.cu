// launch_seq.cu — launches of the sequential-reduction sweeps (north_star a
// and c: seq-rs kernels.hpp:339-376, seq-ws kernels.hpp:384-455); the kernels
// are in seq_kernels.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "internal.h"
#include "seq_kernels.cuh"

using namespace spmk_dev;

namespace spmk_host {
namespace {

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
void launch_seq_ws(SeqArgs a, bool aligned, cudaStream_t s) {
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

}  // namespace

void launch_seq(const SeqLaunch& l, bool ws, bool aligned, cudaStream_t s) {
  SeqArgs a{};
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
  a.CH = l.CH;
  a.EXT = l.EXT;
  a.nunits = l.nunits;
  a.cvvec = ((uintptr_t)l.col % 16 == 0) && ((uintptr_t)l.val % 16 == 0);
  a.one2 = kOnePair;
  if (ws) launch_seq_ws<true>(a, aligned, s);
  else launch_seq_ws<false>(a, aligned, s);
}

}  // namespace spmk_host
