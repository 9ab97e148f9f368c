// par_ws2.cuh — par-ws (north_star d) at lane_width 32, the reference's
// default, for N <= 2 (SpMV: cfg1, cfg5, PageRank): a
// streaming form of the paper's vectorized segment reduction built on
// precomputed segment-head flags instead of per-tile row windows.
//
// Same arithmetic as spmm_par_balanced (kernels.hpp:232-330) for W = 32:
// per 32-nonzero chunk q (plan_balanced chunks, kernels.hpp:244), lane l
// takes position 32q + l, forms the rounded product (:277), runs the lockstep
// conditional Hillis-Steele scan (reduction.hpp:75-86: at offset off lane l
// adds lane l-off's pre-level value iff both hold the same row), and the
// last lane of each run emits (:296-309).  A row crossing chunk edges gets
// Y = ((+0 + P_first) + P_next) + ... in ascending chunk order (:316-323):
// the running carry below, a fixed left-to-right chain.
//
// Layout (built once per handle, aux_kernels.cuh head_flags_kernel):
//   hflag[q]  bit l set iff position 32q + l starts a (non-empty) row; a
//             phantom head at position nnz closes the last row.
// One warp sweeps one tile of TS = 32*C consecutive chunks (the ws plan:
// tile descriptors {first row, first live position, last position, mode},
// owner-extends for rows ending in the next tile, per-chunk H partials +
// owner prefix T for long rows, merged by fixup_kernel).  The row of lane l
// is cur + popc(heads <= l, excluding bit 0) and advances by the chunk's head
// count, so no row window, no bitmap construction and no per-tile setup
// beyond one 16-byte descriptor; colIdx/val/hflag stream two groups ahead,
// the X gathers of the next group are in flight while the current group's
// scans (independent, interleaved) run.
#pragma once
#include "common.cuh"
#include "par_kernels.cuh"

namespace spmk_dev {

struct ParWs2Args {
  ParArgs p;
  const unsigned* __restrict__ hflag;  // ceil(nnz/32)+1 words
};

template <int CT, int D>
__global__ void __launch_bounds__(256)
par_ws2_kernel(const ParWs2Args A) {
  constexpr unsigned FULL = 0xffffffffu;
  const ParArgs& a = A.p;
  const int lane = threadIdx.x & 31;
  const int unit = blockIdx.x * 8 + threadIdx.x / 32;
  if (unit >= a.nunits) return;  // whole warps only
  const int col0 = blockIdx.y * CT;
  const int nt = min(CT, a.N - col0);
  const int N = a.N;
  const bool vec = a.xvec != 0;
  const uint64_t pol = evict_first_policy();
  const unsigned le = (lane == 31) ? FULL : ((2u << lane) - 1u);
  const char* const xb = reinterpret_cast<const char*>(a.X + col0);
  const unsigned xs = (unsigned)N * 4u;
  char* const ybase = reinterpret_cast<char*>(a.Y + col0);

  const int TS = (int)a.TS;
  const int tb = unit * TS;
  const int te = min(tb + TS, a.nnz);
  const int4 dsc = a.desc[unit];
  const int lo = dsc.y;          // first live position
  const int hard_end = dsc.z;    // te, or the end of the owned row crossing te
  int mode = dsc.w;              // mode of the row entering the first chunk
  if (lo >= hard_end) return;
  // compact row containing the first swept chunk's first position
  int cur = dsc.x;
  if (mode == MODE_NORMAL && (lo & 31) != 0) cur = dsc.x - 1;  // lanes before lo: row r-1 (dead)
  bool has_carry = mode == MODE_ENTER_LONG;
  const int q_beg = lo >> 5;
  const int q_end = (hard_end + 31) >> 5;  // exclusive

  float carry[CT];
#pragma unroll
  for (int j = 0; j < CT; ++j) carry[j] = 0.f;

  // Software pipeline over groups of G chunks: colIdx/val/head words of
  // group g+2 load while group g is processed (2G slots), the X rows of
  // group g+1 are gathered right after group g's products are formed (G
  // slots); within a group the G conditional scans are independent
  // straight-line code (interleaved level by level), only the emission /
  // carry pass is sequential over the chunks.
  constexpr int G = D;
  constexpr int S = 2 * G;
  int cr[S];
  float vr[S];
  unsigned hr[S];
  float xr[G][CT];
  auto load_cv = [&](int q, int i) {
    const int p = (q << 5) + lane;
    const bool live = q < q_end && p >= lo && p < hard_end;
    cr[i] = live ? ld_stream(a.col + p, pol) : 0;
    vr[i] = live ? ld_stream(a.val + p, pol) : 0.f;
    hr[i] = q <= q_end ? __ldg(A.hflag + q) : 0u;  // q_end <= ceil(nnz/32): in range
  };
  auto load_x = [&](int q, int ci, int xi) {
    const int p = (q << 5) + lane;
    const bool live = q < q_end && p >= lo && p < hard_end;
    load_dense_cols<CT>(reinterpret_cast<const float*>(xb + (size_t)(unsigned)cr[ci] * xs), nt, vec, live, xr[xi]);
  };

#pragma unroll
  for (int i = 0; i < S; ++i) load_cv(q_beg + i, i);
#pragma unroll
  for (int i = 0; i < G; ++i) load_x(q_beg + i, i, i);

#pragma unroll 1
  for (int qg = q_beg; qg < q_end; qg += S) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // two groups per iteration: slots h*G .. h*G+G-1
      const int q0 = qg + h * G;
      if (q0 >= q_end) break;  // warp-uniform
      float v[G][CT];
      int sst[G];
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const unsigned mle = hr[h * G + i] & le;
        sst[i] = mle ? 31 - __clz(mle) : 0;
#pragma unroll
        for (int j = 0; j < CT; ++j) v[i][j] = __fmul_rn(vr[h * G + i], xr[i][j]);  // kernels.hpp:277
      }
      // X rows of the next group into the freed slots (its colIdx landed a group ago)
#pragma unroll
      for (int i = 0; i < G; ++i) load_x(q0 + G + i, ((h + 1) % 2) * G + i, i);
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {  // reduction.hpp:77-85, lockstep; G chunks interleaved
#pragma unroll
        for (int i = 0; i < G; ++i) {
          const bool same = lane - off >= sst[i];
#pragma unroll
          for (int j = 0; j < CT; ++j) {
            const float up = __shfl_up_sync(FULL, v[i][j], off);
            if (same) v[i][j] = __fadd_rn(v[i][j], up);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int q = q0 + i;
        if (q >= q_end) break;  // warp-uniform
        const int c0 = q << 5;
        const int p = c0 + lane;
        const int hi = min(c0 + 32, hard_end);
        const bool live = p >= lo && p < hi;
        const unsigned M = hr[h * G + i];
        const unsigned Mn = hr[(h * G + i + 1) % S];  // chunk q+1's heads (loaded earlier)
        const unsigned mle = M & le;
        // lane l closes its run iff position l+1 starts a row (head bit, or
        // bit 0 of the next chunk's word, or the phantom head at nnz) or the
        // unit's range ends there
        const bool next_head = (lane < 31) ? ((M >> (lane + 1)) & 1u) : (Mn & 1u);
        const bool last = live && (next_head || p + 1 == hi);
        const bool first_run = (mle & ~1u) == 0 && !(M & 1u);  // run open since before c0
        float t[CT];
#pragma unroll
        for (int j = 0; j < CT; ++j)
          t[j] = (first_run && has_carry && mode == MODE_NORMAL) ? __fadd_rn(carry[j], v[i][j]) : v[i][j];
        if (last) {
          if (first_run && mode == MODE_ENTER_LONG) {
            store_cols<CT>(a.H + (size_t)q * N + col0, nt, t, false);  // long row: per-chunk partial
          } else if (next_head) {
            const int r = cur + __popc(mle & ~1u);
            store_cols<CT>(reinterpret_cast<float*>(ybase + (size_t)(unsigned)a.rid[r] * xs), nt, t, true);
          }
        }
        // the run crossing c0+32 (if any) becomes the carried row
        // (warp-uniform: computed from the chunk's head word, no shuffle)
        const int ll = min(hi - c0, 32) - 1;  // last live lane of the chunk
        const bool cont = !((ll < 31) ? ((M >> (ll + 1)) & 1u) : (Mn & 1u));
        const unsigned le_ll = (ll == 31) ? FULL : ((2u << ll) - 1u);
        const bool lfirst = (M & le_ll & ~1u) == 0 && !(M & 1u);
        float tl[CT];
#pragma unroll
        for (int j = 0; j < CT; ++j) tl[j] = __shfl_sync(FULL, t[j], ll);
        if (cont) {
          if (!lfirst) {
#pragma unroll
            for (int j = 0; j < CT; ++j) carry[j] = __fadd_rn(0.f, tl[j]);  // Y starts at +0
            has_carry = true;
            mode = MODE_NORMAL;
          } else if (mode == MODE_NORMAL) {
#pragma unroll
            for (int j = 0; j < CT; ++j) carry[j] = tl[j];
          }
        } else {
          has_carry = false;
          mode = MODE_NORMAL;
        }
        cur += __popc(M & ~1u) + (int)(Mn & 1u);  // compact row containing c0 + 32
      }
      // colIdx/val/heads of group g+2 into this group's slots
#pragma unroll
      for (int i = 0; i < G; ++i) load_cv(q0 + S + i, h * G + i);
    }
  }
  // long row crossing te (its owner does not extend): prefix -> T slot
  if (hard_end == te && te < a.nnz && has_carry && mode == MODE_NORMAL && lane == 0)
    store_cols<CT>(a.Tsl + (size_t)unit * N + col0, nt, carry, false);
}

}  // namespace spmk_dev
