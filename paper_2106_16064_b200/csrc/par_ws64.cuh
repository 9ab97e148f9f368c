// par_ws64.cuh — par-ws at lane_width 64 (kernels.hpp:92-94 accepts W = 64;
// chunk W at :244).  A chunk of 64 nonzeros is swept by one warp with two
// virtual lanes per physical lane (lane gl holds virtual lanes 2gl, 2gl+1),
// in the reference's order:
//   * rounded products v = val*X[col, j]                    (kernels.hpp:277)
//   * the lockstep conditional Hillis-Steele scan over the 64 virtual lanes
//     (reduction.hpp:75-86): level `off` adds lane i-off's pre-level value iff
//     both hold the same row (i - off >= run start); off = 1 pairs the two
//     virtual lanes of a thread and crosses one lane, off = 2k moves both
//     virtual lanes k physical lanes (shfl_up);
//   * the last lane of each run emits (:296-309): complete rows store to Y,
//     rows crossing a chunk edge write the reference's boundary slot
//     (2q + [row starts in chunk q]);
// then par_ws64_merge_kernel forms Y = ((+0 + slot) + slot) ... in ascending
// slot order for every row crossing a chunk edge (:316-323).
// Rows are the handle's compacted non-empty rows (empty rows are zero-filled
// separately), so at most 64 rows start inside a chunk.  A plain, exact path
// for the one lane width the tuned kernel (par_ws.cuh, W <= 32) leaves out.
#pragma once
#include "common.cuh"

namespace spmk_dev {

struct ParWs64Args {
  const int* __restrict__ crp;   // compact rowPtr (mne+1)
  const int* __restrict__ rid;   // compact -> original row
  const int* __restrict__ col;
  const float* __restrict__ val;
  const float* __restrict__ X;
  float* __restrict__ Y;
  float* __restrict__ slots;     // (2 * chunks) x N
  int mne, nnz, N;
  long long chunks;
};

__global__ void __launch_bounds__(256) par_ws64_chunk_kernel(const ParWs64Args a) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * 8;
  for (long long q = blockIdx.x * 8LL + threadIdx.x / 32; q < a.chunks; q += nwarps) {
    const int e0 = (int)(q * 64);
    const int e1 = min(e0 + 64, a.nnz);
    // compact row containing e0: upper_bound(crp, e0) - 1
    int c = 0;
    if (lane == 0) {
      int lo = 0, hi = a.mne;  // crp[lo] <= e0 < crp[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (a.crp[mid] <= e0) lo = mid; else hi = mid;
      }
      c = lo;
    }
    c = __shfl_sync(FULL, c, 0);
    // in-chunk row starts: bit (end - e0) for the row ends inside (e0, e0+64)
    unsigned long long M = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = c + 1 + lane + 32 * h;
      const int end = k <= a.mne ? a.crp[k] : 0x7fffffff;
      const bool in = end > e0 && end < e0 + 64;
      const unsigned b = __ballot_sync(FULL, in);
      // ends are increasing in k: OR the bit of every in-range end
      unsigned long long mine = in ? (1ull << (end - e0)) : 0ull;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) mine |= __shfl_xor_sync(FULL, mine, o);
      M |= mine;
      (void)b;
    }
    const int i0 = 2 * lane, i1 = 2 * lane + 1;
    const bool live0 = e0 + i0 < e1, live1 = e0 + i1 < e1;
    auto below = [&](int i) { return M & ((i == 63) ? ~0ull : ((2ull << i) - 1ull)); };
    auto runstart = [&](int i) {
      const unsigned long long m = below(i);
      return m ? 63 - __clzll(m) : 0;
    };
    const int s0 = runstart(i0), s1 = runstart(i1);
    const int k0 = __popcll(below(i0)), k1 = __popcll(below(i1));
    const bool last0 = live0 && (!live1 || ((M >> i1) & 1ull));
    const bool last1 = live1 && (i1 == 63 || e0 + i1 + 1 == e1 || ((M >> (i1 + 1)) & 1ull));
    const int c0i = live0 ? a.col[e0 + i0] : 0, c1i = live1 ? a.col[e0 + i1] : 0;
    const float w0 = live0 ? a.val[e0 + i0] : 0.f, w1 = live1 ? a.val[e0 + i1] : 0.f;
    // emission targets (per virtual lane that ends a run)
    auto target = [&](bool last, int k, int j) -> float* {
      if (!last) return nullptr;
      const int r = c + k;
      const int rs = a.crp[r], re = a.crp[r + 1];
      if (rs >= e0 && re <= e1) return a.Y + (size_t)a.rid[r] * a.N + j;  // complete (:300-302)
      const long long slot = 2 * q + (rs < e0 ? 0 : 1);                   // boundary slot (:303-307)
      return a.slots + (size_t)slot * a.N + j;
    };
    for (int j = 0; j < a.N; ++j) {
      float v0 = live0 ? __fmul_rn(w0, a.X[(size_t)c0i * a.N + j]) : 0.f;
      float v1 = live1 ? __fmul_rn(w1, a.X[(size_t)c1i * a.N + j]) : 0.f;
      {  // off = 1
        const float up = __shfl_up_sync(FULL, v1, 1);
        const float n0 = (lane > 0 && i0 - 1 >= s0) ? __fadd_rn(v0, up) : v0;
        const float n1 = (i1 - 1 >= s1) ? __fadd_rn(v1, v0) : v1;
        v0 = n0;
        v1 = n1;
      }
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {  // off = 2k
        const float u0 = __shfl_up_sync(FULL, v0, k), u1 = __shfl_up_sync(FULL, v1, k);
        if (lane >= k && i0 - 2 * k >= s0) v0 = __fadd_rn(v0, u0);
        if (lane >= k && i1 - 2 * k >= s1) v1 = __fadd_rn(v1, u1);
      }
      if (float* t = target(last0, k0, j)) *t = v0;
      if (float* t = target(last1, k1, j)) *t = v1;
    }
  }
}

// Rows crossing a chunk edge: Y = +0, then + slot 2q0+1, + slot 2q+0 for the
// later chunks it touches, ascending (kernels.hpp:316-323).
__global__ void par_ws64_merge_kernel(const ParWs64Args a) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)a.mne * a.N;
       t += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(t / a.N), j = (int)(t % a.N);
    const int rs = a.crp[r], re = a.crp[r + 1];
    const long long q0 = rs / 64, q1 = (re - 1) / 64;
    if (q0 == q1) continue;
    float y = 0.f;
    y = __fadd_rn(y, a.slots[(size_t)(2 * q0 + 1) * a.N + j]);
    for (long long q = q0 + 1; q <= q1; ++q) y = __fadd_rn(y, a.slots[(size_t)(2 * q) * a.N + j]);
    a.Y[(size_t)a.rid[r] * a.N + j] = y;
  }
}

}  // namespace spmk_dev
