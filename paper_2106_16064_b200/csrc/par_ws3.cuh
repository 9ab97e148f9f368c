// par_ws3.cuh — par-ws (north_star d) at lane_width 32 for N = 1 … 4: the par_ws2 sweep with one chunk per
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

// dense row of CT columns at column index c (CT = 2 / 4: one 8- / 16-byte
// load when X is 16-byte aligned)
template <int CT>
__device__ __forceinline__ void ws3_gather(const float* X, int c, bool vec, float (&x)[CT]) {
  const float* r = X + (size_t)(unsigned)c * CT;
  if constexpr (CT == 1) {
    x[0] = ld_x(r);
  } else if constexpr (CT == 2) {
    if (vec) {
      const float2 t = ld_x2(r);
      x[0] = t.x;
      x[1] = t.y;
    } else {
      x[0] = ld_x(r);
      x[1] = ld_x(r + 1);
    }
  } else if constexpr (CT == 3) {
#pragma unroll
    for (int j = 0; j < CT; ++j) x[j] = ld_x(r + j);
  } else {
    if (vec) {
      const float4 t = ld_x4(r);
      x[0] = t.x;
      x[1] = t.y;
      x[2] = t.z;
      x[3] = t.w;
    } else {
#pragma unroll
      for (int j = 0; j < CT; ++j) x[j] = ld_x(r + j);
    }
  }
}

template <int CT, bool LONG>
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
  const int lo = dsc.y;        // first live position (a row head, or the tile start inside a long row)
  const int hard_end = dsc.z;  // end of the last row this tile owns
  if (lo >= hard_end) return;
  // LONG (plans with long rows): the row entering the tile may be long; its
  // per-chunk partials go to H, an owner's prefix of a long row crossing the
  // tile end to T (fixup_kernel merges them), as in par_ws2
  int mode = LONG ? dsc.w : MODE_NORMAL;
  // compact row containing the first swept chunk's first position
  int cur = dsc.x;
  if (mode == MODE_NORMAL && (lo & 31) != 0) cur = dsc.x - 1;  // lanes before lo: row r-1 (dead)
  const int q_beg = lo >> 5;
  const int q_end = (hard_end + 31) >> 5;  // exclusive
  const int* const rid = a.rid;
  const int rmax = a.mne - 1;
  const bool vec = a.xvec != 0;

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
  int c0, c1, c2;
  float v0, v1, v2, x0[CT];
  unsigned m0, m1, m2;
  load_cv(q_beg, c0, v0, m0);
  load_cv(q_beg + 1, c1, v1, m1);
  load_cv(q_beg + 2, c2, v2, m2);
  ws3_gather<CT>(a.X, c0, vec, x0);
  // row-end row ids of chunk q (looked up a chunk ahead)
  int rid0 = 0;
  if (rid) rid0 = rid[min(row_of(cur, m0), rmax)];
  float carry[CT];
#pragma unroll
  for (int j = 0; j < CT; ++j) carry[j] = 0.f;
  bool has_carry = LONG && mode == MODE_ENTER_LONG;

#pragma unroll 1
  for (int q = q_beg; q < q_end; ++q) {
    // gather chunk q + 1, look up its row ids, load chunk q + 3
    float x1[CT];
    ws3_gather<CT>(a.X, c1, vec, x1);
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
    float v[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) v[j] = __fmul_rn(v0, x0[j]);  // kernels.hpp:277 (dead lanes: never read by live runs)
    const unsigned mle = m0 & le;
    const int sst = max(31 - __clz(mle), 0);  // first lane of this lane's run in the chunk
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {  // reduction.hpp:77-85, lockstep
      const bool same = lane - off >= sst;
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        const float up = __shfl_up_sync(FULL, v[j], off);
        if (same) v[j] = __fadd_rn(v[j], up);
      }
    }
    const unsigned nh = __funnelshift_r(m0, m1, 1);  // bit l: position 32q + l + 1 starts a row
    const bool first_run = mle == 0;                 // run open since before this chunk
    const bool add_carry = first_run && has_carry && (!LONG || mode == MODE_NORMAL);
    float t[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) t[j] = add_carry ? __fadd_rn(carry[j], v[j]) : v[j];
    if (LONG && first_run && mode == MODE_ENTER_LONG) {
      // long row: this chunk's partial from its last lane in the chunk
      if (live && (((nh >> lane) & 1u) || p + 1 == min(cq + 32, hard_end))) {
        float* h = a.H + (size_t)q * CT;
#pragma unroll
        for (int j = 0; j < CT; ++j) h[j] = t[j];
      }
    } else if (live && ((nh >> lane) & 1u)) {
      const int row = rid ? rid0 : row_of(cur, m0);
      float* y = a.Y + (size_t)(unsigned)row * CT;
      if constexpr (CT == 1) {
        st_y(y, t[0]);
      } else if (CT != 3 && vec) {  // X and Y 16-byte aligned: rows of CT floats are 4 CT-byte aligned
        if constexpr (CT == 2) st_y2(y, t[0], t[1]);
        else if constexpr (CT == 4) st_y4(y, t[0], t[1], t[2], t[3]);
      } else {
#pragma unroll
        for (int j = 0; j < CT; ++j) st_y(y + j, t[j]);
      }
    }
    // the run crossing the chunk's last live lane (if any) becomes the carry
    const int ll = min(hard_end - cq, 32) - 1;
    float tl[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) tl[j] = __shfl_sync(FULL, t[j], ll);
    if (!((nh >> ll) & 1u)) {
      const unsigned le_ll = (ll == 31) ? FULL : ((2u << ll) - 1u);
      if ((m0 & le_ll) != 0) {  // a run starting in this chunk
#pragma unroll
        for (int j = 0; j < CT; ++j) carry[j] = __fadd_rn(0.f, tl[j]);  // Y starts at +0
        has_carry = true;
        mode = MODE_NORMAL;
      } else if (!LONG || mode == MODE_NORMAL) {
#pragma unroll
        for (int j = 0; j < CT; ++j) carry[j] = tl[j];
      }
    } else {
      has_carry = false;
      mode = MODE_NORMAL;
    }
    cur = cur1;
    // rotate
    c0 = c1; v0 = v1; m0 = m1; rid0 = rid1;
#pragma unroll
    for (int j = 0; j < CT; ++j) x0[j] = x1[j];
    c1 = c2; v1 = v2; m1 = m2;
    c2 = c3; v2 = v3; m2 = m3;
  }
  if constexpr (LONG) {
    // long row crossing the tile end (its owner does not extend): prefix -> T slot
    const int te = min(unit * (int)a.TS + (int)a.TS, a.nnz);
    if (hard_end == te && te < a.nnz && has_carry && mode == MODE_NORMAL && lane == 0) {
#pragma unroll
      for (int j = 0; j < CT; ++j) a.Tsl[(size_t)unit * CT + j] = carry[j];
    }
  }
}

}  // namespace spmk_dev
