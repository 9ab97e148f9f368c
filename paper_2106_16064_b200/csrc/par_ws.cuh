// par_ws.cuh — par-ws (north_star d): nonzero-split + parallel reduction, the
// paper's vectorized segment reduction (VSR), restating
// spmm_par_balanced (kernels.hpp:232-330) and the lane-model scan
// conditional_scan_inplace (reduction.hpp:75-86) as warp code.
//
// A group of W lanes (W = lane_width) owns a tile of T consecutive W-nonzero
// chunks (the reference's plan_balanced(a, W) chunks, kernels.hpp:244).  Per
// chunk, lane l takes nonzero c0+l:
//   * rounded product v = val*X[col, cols]            (kernels.hpp:277)
//   * segment heads: the row ends of the next W rows (a shared-memory window
//     of the compact rowPtr) mark the in-chunk row starts in a bit mask M
//     (one REDUX.OR); a lane's row is cur + popc(M & lanes<=l) and its segment
//     starts at the highest head <= l;
//   * conditional Hillis-Steele scan: at offset off, lane l adds lane l-off's
//     pre-level value iff both hold the same row, i.e. l-off >= segstart(l)
//     (shfl_up, lockstep) — the reference scan, add for add;
//   * the last lane of each run stores its total: complete rows go to Y; the
//     run entering from the previous chunk folds into the carried row
//     (carry + P, the reference's ascending boundary merge, kernels.hpp:
//     316-323); a row entering the tile from >= 2 tiles back (long) emits one
//     partial per chunk (H slots, the reference's head[q]) for fixup_kernel.
// A row crossing the tile end is finished by the tile that owns its start
// when it ends within the next tile ("owner extends"); otherwise the owner
// writes its prefix to the T slot.  The per-tile decisions come precomputed
// in the plan's descriptors (ws_tile_desc_kernel).
//
// Positions are 32-bit (nnz < 2^31 on the device path).  All T chunks of
// colIdx/val and the dense-row gathers are issued before the first scan.
#pragma once
#include "common.cuh"

namespace spmk_dev {

constexpr int kParWsChunksPerTile = 8;  // tile = 8 chunks of W nonzeros

// OR over the W-lane group (W | 32), all 32 lanes converged.
template <int W>
__device__ __forceinline__ unsigned group_or(unsigned v) {
  if constexpr (W == 32) {
    return __reduce_or_sync(0xffffffffu, v);
  } else {
#pragma unroll
    for (int o = 1; o < W; o <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, o, W);
    return v;
  }
}

// CT columns of one dense row (cols [col0, col0+nt) of X), zero when !live.
// vec: 16-byte (CT % 4 == 0) or 8-byte (CT == 2) aligned vector loads.
template <int CT>
__device__ __forceinline__ void load_dense_cols(const float* __restrict__ xr, int nt, bool vec,
                                                bool live, float (&x)[CT]) {
  if constexpr (CT % 4 == 0) {
    if (vec) {
#pragma unroll
      for (int j = 0; j < CT; j += 4) {
        if (live && j < nt) {
          const float4 t = ld_x4(xr + j);
          x[j] = t.x; x[j + 1] = t.y; x[j + 2] = t.z; x[j + 3] = t.w;
        } else {
          x[j] = x[j + 1] = x[j + 2] = x[j + 3] = 0.f;
        }
      }
      return;
    }
  } else if constexpr (CT == 2) {
    if (vec) {  // N even => nt == 2
      if (live) {
        const float2 t = ld_x2(xr);
        x[0] = t.x; x[1] = t.y;
      } else {
        x[0] = x[1] = 0.f;
      }
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < CT; ++j) x[j] = (live && j < nt) ? ld_x(xr + j) : 0.f;
}

template <int CT>
__device__ __forceinline__ void store_cols(float* __restrict__ p, int nt, const float (&v)[CT], bool stream) {
#pragma unroll
  for (int j = 0; j < CT; ++j)
    if (j < nt) {
      if (stream) st_y(p + j, v[j]); else p[j] = v[j];
    }
}

template <int W, int CT, int T = kParWsChunksPerTile, int MINB = 1, bool BATCHED = true>
__global__ void __launch_bounds__(256, MINB)
par_ws_kernel(const ParArgs a) {
  static_assert(W >= 2 && W <= 32, "W");
  constexpr int NG = 256 / W;      // groups per block
  constexpr int WINP = T * W + 2;  // rows touching a tile <= T*W + 1
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int BIG = 0x7fffffff;
  __shared__ int s_crp[NG * WINP];  // wcrp[i] = crp[rbase + 1 + i] (row ends)
  __shared__ int s_rid[NG * WINP];  // wrid[i] = rid[rbase + i]

  const int lane = threadIdx.x & 31;
  const int gl = lane & (W - 1);
  const int gidx = threadIdx.x / W;
  int unit = blockIdx.x * NG + gidx;
  const bool active = unit < a.nunits;
  if (!active) unit = 0;
  int* wcrp = s_crp + gidx * WINP;
  int* wrid = s_rid + gidx * WINP;
  const int col0 = blockIdx.y * a.ncol_tile;
  const int nt = min(a.ncol_tile, a.N - col0);
  const int N = a.N;
  const bool vec = a.xvec != 0;
  const uint64_t pol = evict_first_policy();
  const unsigned le = (gl == 31) ? FULL : ((2u << gl) - 1u);  // lanes <= gl
  // dense-row address = xb + col * xs: one IMAD.WIDE.U32 per gather
  const char* const xb = reinterpret_cast<const char*>(a.X + col0);
  const unsigned xs = (unsigned)N * 4u;
  auto xrow = [&](int c) { return reinterpret_cast<const float*>(xb + (size_t)(unsigned)c * xs); };

  // ---- tile setup from the precomputed descriptor {cur, start, hard_end, mode}
  const int TS = (int)a.TS;
  const int tb = unit * TS;
  const int te = min(tb + TS, a.nnz);
  const int4 d = a.desc[unit];
  const int r2 = a.rlo[unit + 1];  // first compact row starting >= te
  int lo = d.y;                     // first live position
  int hard_end = d.z;               // te, or the end of the owned row crossing te
  int mode = d.w;                   // mode of the carried row
  const bool work = active && lo < hard_end;
  if (!work) lo = hard_end = tb;
  int cur = d.x;
  if (mode == MODE_NORMAL && lo > tb && ((lo - tb) % W) != 0) cur = d.x - 1;  // dead lanes of row r-1
  bool has_carry = work && mode == MODE_ENTER_LONG;
  const int rbase = cur;
  const int cnt = work ? r2 - rbase : 0;  // rows [cur, r2) touch the tile

  // ---- issue every load of the tile: colIdx/val, then the row window, then X
  int cidx[T];
  float wv[T];
  const int* const colp = a.col + (tb + gl);  // chunk k at immediate offset k*W
  const float* const valp = a.val + (tb + gl);
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const int p = tb + k * W + gl;
    const bool live = work && p >= lo && p < te;
    cidx[k] = live ? ld_stream(colp + k * W, pol) : 0;
    wv[k] = live ? ld_stream(valp + k * W, pol) : 0.f;
  }
  {
    const int* const wsrc_crp = a.crp + (rbase + 1);
    const int* const wsrc_rid = a.rid + rbase;
#pragma unroll 1
    for (int i = gl; i < cnt; i += W) {
      wcrp[i] = wsrc_crp[(unsigned)i];
      wrid[i] = wsrc_rid[(unsigned)i];
    }
  }
  float xv[T][CT];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const int p = tb + k * W + gl;
    const bool live = work && p >= lo && p < te;
    load_dense_cols<CT>(xrow(cidx[k]), nt, vec, live, xv[k]);
  }
  __syncwarp();

  float carry[CT];
#pragma unroll
  for (int j = 0; j < CT; ++j) carry[j] = 0.f;

  // One chunk [c0, c0+W), executed by the whole warp (shuffles full-mask).
  // Row ends beyond the last window entry read as BIG.  Dead lanes need no
  // run boundaries of their own: lanes before `lo` belong to row cur, whose
  // end (= lo) is already a head bit of M; lanes at or past `hi` only follow
  // live lanes (they never feed a live lane's scan), and the last live lane
  // is flagged explicitly.  Dead lanes carry w = x = 0.
  char* const ybase = reinterpret_cast<char*>(a.Y + col0);
  const unsigned ystride = (unsigned)N * 4u;
  auto chunk = [&](bool en, int c0, float w, const float (&x)[CT]) {
    const int p = c0 + gl;
    const int hi = min(c0 + W, hard_end);
    const bool live = en && p >= lo && p < hi;
    const int wbase = cur - rbase;
    const int wi = wbase + gl;
    const int wend = (en && wi < cnt) ? wcrp[wi] : BIG;
    const unsigned b = (unsigned)(wend - c0);
    const unsigned M = group_or<W>((b - 1u < (unsigned)(W - 1)) ? (1u << b) : 0u);  // in-chunk row starts
    const unsigned mle = M & le;
    const int sst = mle ? 31 - __clz(mle) : 0;  // first lane of this lane's run
    const int kidx = __popc(mle);               // row(l) - cur
    float v[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) v[j] = __fmul_rn(w, x[j]);  // kernels.hpp:277
#pragma unroll
    for (int off = 1; off < W; off <<= 1) {  // reduction.hpp:77-85, lockstep
      const bool same = gl - off >= sst;
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        const float up = __shfl_up_sync(FULL, v[j], off, W);
        if (same) v[j] = __fadd_rn(v[j], up);
      }
    }
    // emission by the last lane of each run
    const bool last = live && (gl == W - 1 || p + 1 == hi || ((M >> (gl + 1)) & 1u));
    const bool first_run = has_carry && kidx == 0;  // run continuing from before c0
    float t[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j)
      t[j] = (first_run && mode == MODE_NORMAL) ? __fadd_rn(carry[j], v[j]) : v[j];
    const int ri = wbase + kidx;
    const int rend = (last && ri < cnt) ? wcrp[ri] : BIG;
    if (last) {
      if (first_run && mode == MODE_ENTER_LONG) {
        store_cols<CT>(a.H + (size_t)(c0 / W) * N + col0, nt, t, false);
      } else if (rend <= c0 + W) {
        store_cols<CT>(reinterpret_cast<float*>(ybase + (size_t)(unsigned)wrid[ri] * ystride), nt, t, true);
      }
    }
    // the last live run continuing past the chunk becomes the carried row
    const int ll = max(min(hi - c0, W), 1) - 1;
    const int flags = __shfl_sync(FULL, (rend != BIG && rend > c0 + W ? 1 : 0) | (first_run ? 2 : 0), ll, W);
    float tl[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) tl[j] = __shfl_sync(FULL, t[j], ll, W);
    const int nb = __popc(M);
    const int wn_i = wbase + nb;
    const int wn = (en && wn_i < cnt) ? wcrp[wn_i] : BIG;
    if (en) {
      if (flags & 1) {
        if (!(flags & 2)) {
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
      cur += nb + (wn == c0 + W ? 1 : 0);  // row containing c0 + W
    }
  };

  if constexpr (!BATCHED) {
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const int c0 = tb + k * W;
      chunk(work && c0 < te && c0 + W > lo, c0, wv[k], xv[k]);
    }
  } else {
    // Batched form: the segment heads of the whole tile are known up front
    // (one bitmap word per chunk: bit e-tb for every row end e inside the
    // tile), so the T conditional scans are independent straight-line code
    // the scheduler interleaves; only the (cheap) emission/carry pass below
    // is sequential over the chunks.
    unsigned hw[T];
#pragma unroll
    for (int k = 0; k < T; ++k) hw[k] = 0u;
#pragma unroll 1
    for (int i = gl; i < cnt; i += W) {
      const int off = wcrp[i] - tb;
      if (off > 0 && off < T * W) {
#pragma unroll
        for (int k = 0; k < T; ++k)
          if ((off / W) == k) hw[k] |= 1u << (off % W);
      }
    }
    unsigned M[T];
    int base[T + 1];
    base[0] = 0;
#pragma unroll
    for (int k = 0; k < T; ++k) {
      M[k] = group_or<W>(hw[k]);
      base[k + 1] = base[k] + __popc(M[k]);
    }
    float v[T][CT];
#pragma unroll
    for (int k = 0; k < T; ++k)
#pragma unroll
      for (int j = 0; j < CT; ++j) v[k][j] = __fmul_rn(wv[k], xv[k][j]);  // kernels.hpp:277
    int sst[T];
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const unsigned mle = M[k] & le;
      sst[k] = mle ? 31 - __clz(mle) : 0;
    }
#pragma unroll
    for (int off = 1; off < W; off <<= 1) {  // reduction.hpp:77-85, lockstep, T chunks interleaved
#pragma unroll
      for (int k = 0; k < T; ++k) {
        const bool same = gl - off >= sst[k];
#pragma unroll
        for (int j = 0; j < CT; ++j) {
          const float up = __shfl_up_sync(FULL, v[k][j], off, W);
          if (same) v[k][j] = __fadd_rn(v[k][j], up);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const int c0 = tb + k * W;
      const bool en = work && c0 < te && c0 + W > lo;
      const int p = c0 + gl;
      const int hi = min(c0 + W, hard_end);
      const bool live = en && p >= lo && p < hi;
      const int kl = __popc(M[k] & le);
      const bool last = live && (gl == W - 1 || p + 1 == hi || ((M[k] >> (gl + 1)) & 1u));
      const bool first_run = has_carry && kl == 0;  // run continuing from before c0
      float t[CT];
#pragma unroll
      for (int j = 0; j < CT; ++j)
        t[j] = (first_run && mode == MODE_NORMAL) ? __fadd_rn(carry[j], v[k][j]) : v[k][j];
      const int ri = base[k] + kl;  // window index of this lane's row
      const int rend = (last && ri < cnt) ? wcrp[ri] : BIG;
      if (last) {
        if (first_run && mode == MODE_ENTER_LONG) {
          store_cols<CT>(a.H + (size_t)(c0 / W) * N + col0, nt, t, false);
        } else if (rend <= c0 + W) {
          store_cols<CT>(reinterpret_cast<float*>(ybase + (size_t)(unsigned)wrid[ri] * ystride), nt, t, true);
        }
      }
      const int ll = max(min(hi - c0, W), 1) - 1;
      const int flags = __shfl_sync(FULL, (rend != BIG && rend > c0 + W ? 1 : 0) | (first_run ? 2 : 0), ll, W);
      float tl[CT];
#pragma unroll
      for (int j = 0; j < CT; ++j) tl[j] = __shfl_sync(FULL, t[j], ll, W);
      if (en) {
        if (flags & 1) {
          if (!(flags & 2)) {
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
      }
    }
    cur = rbase + base[T];  // row containing te (the extension row, if any)
  }
  // long row crossing te (its owner does not extend): prefix -> T slot
  if (work && hard_end == te && has_carry && mode == MODE_NORMAL && gl == 0)
    store_cols<CT>(a.Tsl + (size_t)unit * N + col0, nt, carry, false);
  // owner extends: finish the row crossing te (it ends within the next tile)
#pragma unroll 1
  for (int c0 = te; __any_sync(FULL, c0 < hard_end); c0 += W) {
    const bool en = c0 < hard_end;
    const int p = c0 + gl;
    const bool live = en && p < hard_end;
    const int ci = live ? ld_stream(a.col + p, pol) : 0;
    const float w = live ? ld_stream(a.val + p, pol) : 0.f;
    float x[CT];
    load_dense_cols<CT>(xrow(ci), nt, vec, live, x);
    chunk(en, c0, w, x);
  }
}

}  // namespace spmk_dev
