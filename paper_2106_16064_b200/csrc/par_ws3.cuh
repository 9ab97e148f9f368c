// par_ws3.cuh — par-ws (north_star d) at lane_width 32 for SpMV (N = 1) on
// matrices without long rows: the par_ws2 sweep with one chunk per
// iteration and only the arithmetic that case needs.
//
// Same arithmetic as spmm_par_balanced (kernels.hpp:232-330) for W = 32 and
// as par_ws2_kernel: per 32-nonzero chunk q lane l takes position 32q + l,
// forms the rounded product (:277), runs the lockstep conditional
// Hillis-Steele scan (reduction.hpp:75-86), and the last lane of each run
// emits (:296-309); a row crossing chunk edges gets
// Y = ((+0 + P_first) + P_next) + ... in ascending chunk order (:316-323)
// through the running carry.  Tiles are the ws plan's (owner-extends, so a
// row never crosses into another warp's tile when the plan has no long rows:
// no H / T partials, no fix-up).
//
// Why a separate kernel: on regular matrices (uniform / banded, ~16 nonzeros
// per row) par_ws2 is issue-bound at ~110 warp instructions per chunk (two
// interleaved chunks, the long-row modes, 48 registers for 5 blocks / SM so
// nvcc rematerialises); here ~70, the compact-row lookup of the next chunk's
// row ends is issued a chunk ahead (the store no longer waits on it), and the
// next-head flags come from one funnel shift of two head words.
#pragma once
#include "common.cuh"
#include "par_kernels.cuh"
#include "par_ws2.cuh"

namespace spmk_dev {

__global__ void __launch_bounds__(256)
par_ws3_kernel(const ParWs2Args A) {
  constexpr unsigned FULL = 0xffffffffu;
  const ParArgs& a = A.p;
  const int lane = threadIdx.x & 31;
  const int unit = blockIdx.x * 8 + threadIdx.x / 32;
  if (unit >= a.nunits) return;  // whole warps only
  const uint64_t pol = evict_first_policy();
  const unsigned le = (lane == 31) ? FULL : ((2u << lane) - 1u);
  const int4 dsc = a.desc[unit];
  const int lo = dsc.y;        // first live position (a row head)
  const int hard_end = dsc.z;  // end of the last row this tile owns
  if (lo >= hard_end) return;
  // compact row containing the first swept chunk's first position
  int cur = dsc.x;
  if ((lo & 31) != 0) cur = dsc.x - 1;  // lanes before lo: row r-1 (dead)
  const int q_beg = lo >> 5;
  const int q_end = (hard_end + 31) >> 5;  // exclusive
  const int* const rid = a.rid;
  const int rmax = a.mne - 1;

  // chunk q's colIdx / val / head word, zero outside [lo, hard_end)
  auto load_cv = [&](int q, int& c, float& v, unsigned& m) {
    const int p = (q << 5) + lane;
    const bool live = q < q_end && p >= lo && p < hard_end;
    c = live ? ld_stream(a.col + p, pol) : 0;
    v = live ? ld_stream(a.val + p, pol) : 0.f;
    m = q <= q_end ? __ldg(A.hflag + q) : 0u;  // q_end <= ceil(nnz/32): in range
  };
  // compact row of lane l's run end in a chunk with head word M, first row cr
  auto row_of = [&](int cr, unsigned M) { return cr + __popc(M & le & ~1u); };

  // pipeline: chunk q computing, q + 1 gathered, q + 2 loading
  int c1, c2;
  float v0, v1, v2, x0;
  unsigned m0, m1, m2;
  int c0;
  load_cv(q_beg, c0, v0, m0);
  load_cv(q_beg + 1, c1, v1, m1);
  load_cv(q_beg + 2, c2, v2, m2);
  x0 = ld_x(a.X + (size_t)(unsigned)c0);
  // row-end row ids of chunk q (prefetched a chunk ahead)
  int rid0 = 0;
  if (rid) rid0 = rid[min(row_of(cur, m0), rmax)];
  float carry = 0.f;
  bool has_carry = false;

#pragma unroll 1
  for (int q = q_beg; q < q_end; ++q) {
    // gather chunk q + 1, look up its row ids, load chunk q + 3
    const float x1 = ld_x(a.X + (size_t)(unsigned)c1);
    const int cur1 = cur + __popc(m0 & ~1u) + (int)(m1 & 1u);  // compact row containing 32(q+1)
    int rid1 = 0;
    if (rid) rid1 = rid[min(row_of(cur1, m1), rmax)];
    int c3;
    float v3;
    unsigned m3;
    load_cv(q + 3, c3, v3, m3);

    // chunk q
    const int cq = q << 5;
    const int p = cq + lane;
    const bool live = p >= lo && p < hard_end;
    float v = __fmul_rn(v0, x0);  // kernels.hpp:277 (dead lanes: val 0, never read by live runs)
    const unsigned mle = m0 & le;
    const int sst = max(31 - __clz(mle), 0);  // first lane of this lane's run in the chunk
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {  // reduction.hpp:77-85, lockstep
      const float up = __shfl_up_sync(FULL, v, off);
      if (lane - off >= sst) v = __fadd_rn(v, up);
    }
    const unsigned nh = __funnelshift_r(m0, m1, 1);  // bit l: position 32q + l + 1 starts a row
    const bool first_run = mle == 0;                 // run open since before this chunk
    const float t = (first_run && has_carry) ? __fadd_rn(carry, v) : v;
    if (live && ((nh >> lane) & 1u)) {
      const int row = rid ? rid0 : row_of(cur, m0);
      st_y(a.Y + (size_t)(unsigned)row, t);
    }
    // the run crossing the chunk's last live lane (if any) becomes the carry
    const int ll = min(hard_end - cq, 32) - 1;
    const float tl = __shfl_sync(FULL, t, ll);
    if (!((nh >> ll) & 1u)) {
      const unsigned le_ll = (ll == 31) ? FULL : ((2u << ll) - 1u);
      if ((m0 & le_ll) != 0) {  // a run starting in this chunk
        carry = __fadd_rn(0.f, tl);  // Y starts at +0
        has_carry = true;
      } else {
        carry = tl;
      }
    } else {
      has_carry = false;
    }
    cur = cur1;
    // rotate
    c0 = c1; v0 = v1; m0 = m1; x0 = x1; rid0 = rid1;
    c1 = c2; v1 = v2; m1 = m2;
    c2 = c3; v2 = v3; m2 = m3;
  }
}

}  // namespace spmk_dev
