// par_kernels.cuh — parallel-reduction kernels (north_star b and d):
//   par-rs  spmm_par_rowsplit  kernels.hpp:157-224  (VDL + merge tree)
//   par-ws  spmm_par_balanced  kernels.hpp:232-330  (VSR segmented scan)
#pragma once
#include "common.cuh"

namespace spmk_dev {

// ============================================================================
// par-rs.  A group of W lanes (W = lane_width) per non-empty row.  Lane l
// accumulates nonzeros base+l, base+W, ... (kernels.hpp:179-188) for a column
// tile of CT columns, loading the dense row with 128-bit vectors (VDL,
// PAPER.md:60-66).  The cross-lane merge reproduces the reference's pairwise
// tree acc[l] = acc[2l+1] + acc[2l] (kernels.hpp:193-199) exactly:
//   * while a lane still holds >1 column: butterfly reduce-scatter with
//     shfl_xor offsets 1,2,4,... — pairs adjacent lane groups exactly like the
//     tree, but each level halves the columns a lane carries (W-1 shuffles per
//     row instead of CT*log2 W);
//   * remaining levels: shfl_down with the next offsets.
// VL = 2 emulates lane_width 64: each physical lane holds virtual lanes 2l and
// 2l+1 and performs the tree's first level in registers.
// ============================================================================
struct ParArgs {
  const int* __restrict__ crp;
  const int* __restrict__ rid;
  const int* __restrict__ col;
  const float* __restrict__ val;
  const float* __restrict__ X;
  float* __restrict__ Y;
  float* __restrict__ H;
  float* __restrict__ Tsl;
  const int* __restrict__ rlo;
  int mne, nnz, N;
  int ncol_tile;      // columns per blockIdx.y pass
  long long TS;       // par-ws tile (T chunks of W)
  int nunits;
};

template <int W, int VL, int CT, bool VEC4>
__global__ void __launch_bounds__(256)
par_rs_kernel(const ParArgs a) {
  constexpr int G = W / VL;  // physical lanes per row group (<= 32)
  static_assert(G >= 1 && G <= 32, "group");
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const unsigned gmask = group_mask<G>();
  const int groups_total = (gridDim.x * blockDim.x) / G;
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int col0 = blockIdx.y * a.ncol_tile;
  const int nt = min(a.ncol_tile, a.N - col0);  // columns this pass (<= CT)
  const int N = a.N;
  const uint64_t pol = evict_first_policy();

  // number of butterfly (reduce-scatter) levels: halve while CT allows
  constexpr int LOGG = (G >= 32) ? 5 : (G >= 16) ? 4 : (G >= 8) ? 3 : (G >= 4) ? 2 : (G >= 2) ? 1 : 0;
  constexpr int V2CT = (CT % 32 == 0) ? 5 : (CT % 16 == 0) ? 4 : (CT % 8 == 0) ? 3 : (CT % 4 == 0) ? 2 : (CT % 2 == 0) ? 1 : 0;
  constexpr int HL = LOGG < V2CT ? LOGG : V2CT;

  // software pipeline over this group's rows: bounds two rows ahead, the
  // first W-batch of colIdx/val one row ahead, dense rows for the current one
  auto bounds = [&](int row, int& s, int& f) {
    if (row < a.mne) {
      s = a.crp[row];
      f = a.crp[row + 1];
    } else {
      s = f = 0;
    }
  };
  auto first_batch = [&](int s, int f, int (&c)[VL], float (&w)[VL]) {
#pragma unroll
    for (int v = 0; v < VL; ++v) {
      const int p = s + gl * VL + v;
      const bool live = p < f && p < s + W;
      c[v] = live ? ld_stream(a.col + p, pol) : -1;
      w[v] = live ? ld_stream(a.val + p, pol) : 0.f;
    }
  };
  auto accumulate = [&](const int (&c)[VL], const float (&w)[VL], float (&acc)[CT], float (&acc2)[VL == 2 ? CT : 1]) {
#pragma unroll
    for (int v = 0; v < VL; ++v) {
      if (c[v] >= 0) {
        const float* xr = a.X + (size_t)c[v] * N + col0;
        float xv[CT];
        if constexpr (VEC4 && CT % 4 == 0) {
#pragma unroll
          for (int k = 0; k < CT; k += 4) {
            if (k < nt) {
              const float4 t = ld_x4(xr + k);
              xv[k] = t.x; xv[k + 1] = t.y; xv[k + 2] = t.z; xv[k + 3] = t.w;
            } else {
              xv[k] = xv[k + 1] = xv[k + 2] = xv[k + 3] = 0.f;
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < CT; ++k) xv[k] = (k < nt) ? ld_x(xr + k) : 0.f;
        }
        if constexpr (VL == 2) {
          if (v == 1) {
#pragma unroll
            for (int k = 0; k < CT; ++k) acc2[k] = mul_add_rn(acc2[k], w[v], xv[k]);
          } else {
#pragma unroll
            for (int k = 0; k < CT; ++k) acc[k] = mul_add_rn(acc[k], w[v], xv[k]);
          }
        } else {
#pragma unroll
          for (int k = 0; k < CT; ++k) acc[k] = mul_add_rn(acc[k], w[v], xv[k]);
        }
      }
    }
  };

  int s0, f0, s1, f1;
  bounds(gid, s0, f0);
  bounds(gid + groups_total, s1, f1);
  int c0[VL];
  float w0[VL];
  first_batch(s0, f0, c0, w0);
  for (int r = gid; r < a.mne; r += groups_total) {
    int s2, f2;
    bounds(r + 2 * groups_total, s2, f2);
    int c1[VL];
    float w1[VL];
    first_batch(s1, f1, c1, w1);
    const int s = s0, f = f0;
    float acc[CT];
#pragma unroll
    for (int k = 0; k < CT; ++k) acc[k] = 0.f;
    float acc2[VL == 2 ? CT : 1];
#pragma unroll
    for (int k = 0; k < (VL == 2 ? CT : 1); ++k) acc2[k] = 0.f;
    accumulate(c0, w0, acc, acc2);
    for (int base = s + W; base < f; base += W) {  // rows longer than W
      int c[VL];
      float w[VL];
#pragma unroll
      for (int v = 0; v < VL; ++v) {
        const int p = base + gl * VL + v;
        c[v] = p < f ? ld_stream(a.col + p, pol) : -1;
        w[v] = p < f ? ld_stream(a.val + p, pol) : 0.f;
      }
      accumulate(c, w, acc, acc2);
    }
    if constexpr (VL == 2) {
      // tree level 1 of the 64-lane model: acc[l] = acc[2l+1] + acc[2l]
#pragma unroll
      for (int k = 0; k < CT; ++k) acc[k] = __fadd_rn(acc2[k], acc[k]);
    }
    // butterfly reduce-scatter levels (offsets 1..2^(HL-1))
    int cbase = 0;  // first column of the contiguous run this lane holds
#pragma unroll
    for (int h = 0; h < HL; ++h) {
      const int off = 1 << h;
      const int half = CT >> (h + 1);
      const bool upper = (gl & off) != 0;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const float send = upper ? acc[i] : acc[i + half];
        const float keep = upper ? acc[i + half] : acc[i];
        const float recv = __shfl_xor_sync(gmask, send, off, G);
        acc[i] = __fadd_rn(keep, recv);
      }
      if (upper) cbase += half;
    }
    constexpr int REM = CT >> HL;  // columns still held per lane
    // remaining tree levels on the held columns
#pragma unroll
    for (int h = HL; h < LOGG; ++h) {
      const int off = 1 << h;
#pragma unroll
      for (int i = 0; i < REM; ++i) {
        const float o = __shfl_down_sync(gmask, acc[i], off, G);
        acc[i] = __fadd_rn(acc[i], o);
      }
    }
    // lanes gl < 2^HL hold the final values of columns [cbase, cbase+REM)
    if (gl < (1 << HL)) {
      float* yr = a.Y + (size_t)a.rid[r] * N + col0;
#pragma unroll
      for (int i = 0; i < REM; ++i)
        if (cbase + i < nt) st_y(yr + cbase + i, acc[i]);
    }
    s0 = s1; f0 = f1; s1 = s2; f1 = f2;
#pragma unroll
    for (int v = 0; v < VL; ++v) {
      c0[v] = c1[v];
      w0[v] = w1[v];
    }
  }
}

// ============================================================================
// par-ws (VSR; kernels.hpp:232-330 + reduction.hpp:75-86).
// A group of W lanes processes a tile of T consecutive W-nonzero chunks.  Per
// chunk: lane l takes nonzero c0+l, forms the rounded product v*x
// (kernels.hpp:277), and the conditional Hillis-Steele scan adds lane l-off
// iff both lanes hold the same row (shfl_up offsets 1..W/2, lockstep) — the
// reference scan exactly.  Row ids come from segment-head flags: a window of
// the next W row ends (coalesced crp load) marks the in-chunk row starts in
// a bit mask M (redux.or); a lane's row is cur + popc(M & lanes<=l), so the
// equality test of two lanes is bit arithmetic, not a shuffle.
// The last lane of each run emits: runs complete in the chunk store Y; the
// run entering from the previous chunk is folded into the carried row
// (carry = carry + P, the reference's ascending merge); a long entering row
// (>= 2 tiles back) emits one partial per chunk (H) for fixup_kernel.
// ============================================================================
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

template <int W, int CT>
__global__ void __launch_bounds__(256)
par_ws_kernel(const ParArgs a) {
  static_assert(W >= 2 && W <= 32, "W");
  constexpr int T = kParWsChunksPerTile;
  constexpr int NG = 256 / W;         // groups per block
  constexpr int WINP = T * W + 2;     // rows touching a tile <= T*W + 1
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ int s_crp[NG * WINP];    // s_crp[i] = crp[rbase + 1 + i]
  __shared__ int s_rid[NG * WINP];    // s_rid[i] = rid[rbase + i]

  const int lane = threadIdx.x & 31;
  const int gl = lane & (W - 1);
  const int gidx = threadIdx.x / W;
  int unit = blockIdx.x * NG + gidx;
  // All 32 lanes run every loop below (warp-uniform trip counts); an idle or
  // finished group just has no live lanes.  Shuffles are full-mask.
  bool active = unit < a.nunits;
  if (!active) unit = 0;
  int* wcrp = s_crp + gidx * WINP;
  int* wrid = s_rid + gidx * WINP;
  const int col0 = blockIdx.y * a.ncol_tile;
  const int nt = min(a.ncol_tile, a.N - col0);
  const int N = a.N;
  const uint64_t pol = evict_first_policy();
  const bool vec4 = (CT % 4 == 0) && (N % 4 == 0);
  const unsigned le = (gl == 31) ? 0xffffffffu : ((2u << gl) - 1u);  // lanes <= gl

  const long long tb = (long long)unit * a.TS;
  long long te = min(tb + a.TS, (long long)a.nnz);
  const int r = a.rlo[unit];
  const int r2 = a.rlo[unit + 1];
  long long lo = tb;        // first live position of this tile
  long long hard_end = te;  // te, or the end of an owned row crossing te
  int kstart = 0;           // first chunk of the tile with live lanes
  int cur;                  // compact row containing the current chunk start
  int mode = MODE_NORMAL;   // mode of the carried row
  bool has_carry = false;   // a row continues into the chunk from before it
  float carry[CT];
#pragma unroll
  for (int k = 0; k < CT; ++k) carry[k] = 0.f;

  if (te < a.nnz) {
    const int c2 = a.crp[r2];
    if (c2 > te) {
      const int cs = a.crp[r2 - 1];
      if (cs >= tb && (c2 - 1) / a.TS < unit + 2) hard_end = c2;
    }
  }
  const int cr = a.crp[r];
  if (cr > tb) {  // row r-1 enters from the left
    const int rs = a.crp[r - 1];
    if ((cr - 1) / a.TS - rs / a.TS >= 2) {
      cur = r - 1;
      mode = MODE_ENTER_LONG;
      has_carry = true;
    } else {
      lo = cr;  // finished by its owner tile
      if (lo >= te) active = false;
      kstart = (int)((min(lo, te) - tb) / W);
      cur = (lo > tb + (long long)kstart * W) ? r - 1 : r;
    }
  } else {
    cur = r;
  }
  if (!active) {
    lo = hard_end = te = tb;  // no live lanes anywhere
    has_carry = false;
  }

  // row window for the rows touching the tile: [cur, r2)
  const int rbase = cur;
  const int cnt = active ? r2 - rbase : 0;  // <= T*W + 1
  for (int i = gl; i < WINP; i += W) {
    wcrp[i] = (i < cnt) ? a.crp[rbase + 1 + i] : 0x7fffffff;
    wrid[i] = (i < cnt) ? a.rid[rbase + i] : 0;
  }

  // issue every load of the tile up front: colIdx/val, then the dense rows
  int cidx[T];
  float wv[T];
  float xv[T][CT];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const long long p = tb + (long long)k * W + gl;
    const bool live = k >= kstart && p >= lo && p < te;
    cidx[k] = live ? ld_stream(a.col + p, pol) : 0;
    wv[k] = live ? ld_stream(a.val + p, pol) : 0.f;
  }
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const long long p = tb + (long long)k * W + gl;
    const bool live = k >= kstart && p >= lo && p < te;
    const float* xr = a.X + (size_t)cidx[k] * N + col0;
    if (vec4) {
#pragma unroll
      for (int j = 0; j < CT; j += 4) {
        if (live && j < nt) {
          const float4 t = ld_x4(xr + j);
          xv[k][j] = t.x; xv[k][j + 1] = t.y; xv[k][j + 2] = t.z; xv[k][j + 3] = t.w;
        } else {
          xv[k][j] = xv[k][j + 1] = xv[k][j + 2] = xv[k][j + 3] = 0.f;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < CT; ++j) xv[k][j] = (live && j < nt) ? ld_x(xr + j) : 0.f;
    }
  }
  __syncwarp();

  // One chunk (executed by the whole warp; `en` says whether this group has
  // a chunk here): rounded products, conditional scan, emission, carry.
  auto chunk = [&](bool en, long long c0, float w, const float (&x)[CT], int wrow_end, int wrow_id) {
    const long long p = c0 + gl;
    const long long hi = min(c0 + W, hard_end);
    const bool live = en && p >= lo && p < hi;
    const int llo = (int)max(0LL, min(lo - c0, (long long)W));
    const int lhi = (int)max(1LL, min(hi - c0, (long long)W));
    const long long b = (long long)wrow_end - c0;
    const unsigned M = group_or<W>((b > 0 && b < W) ? (1u << (int)b) : 0u);
    unsigned Mrun = M;  // dead lanes form their own runs
    if (llo > 0 && llo < W) Mrun |= 1u << llo;
    if (lhi < W) Mrun |= 1u << lhi;
    const int kidx = __popc(M & le);  // row(l) - cur
    const int runid = __popc(Mrun & le);
    float v[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) v[j] = live ? __fmul_rn(w, x[j]) : 0.f;  // kernels.hpp:277
#pragma unroll
    for (int off = 1; off < W; off <<= 1) {  // reduction.hpp:77-85, lockstep
      const int src = gl - off;
      const bool same =
          src >= 0 && __popc(Mrun & ((src == 31) ? 0xffffffffu : ((2u << src) - 1u))) == runid;
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        const float up = __shfl_up_sync(FULL, v[j], off, W);
        if (same) v[j] = __fadd_rn(v[j], up);
      }
    }
    const bool last_of_run = live && (gl == W - 1 || ((Mrun >> (gl + 1)) & 1u));
    const int rend = __shfl_sync(FULL, wrow_end, kidx, W);  // crp[row+1]
    const int orow = __shfl_sync(FULL, wrow_id, kidx, W);   // rid[row]
    const bool starts_here = kidx > 0 || !has_carry;
    const bool ends_here = rend <= c0 + W;
    if (last_of_run && starts_here && ends_here) {  // complete run: Y = P
      float* yr = a.Y + (size_t)orow * N + col0;
#pragma unroll
      for (int j = 0; j < CT; ++j)
        if (j < nt) st_y(yr + j, v[j]);
    }
    // run entering from the previous chunk (lanes [0, first boundary))
    const bool carried_in = en && has_carry;
    const unsigned rest = Mrun & ~1u;
    const int first_last = rest ? (__ffs(rest) - 2) : (W - 1);
    const bool fin = __shfl_sync(FULL, wrow_end, 0, W) <= c0 + W;
    float pf[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) pf[j] = __shfl_sync(FULL, v[j], first_last, W);
    if (carried_in) {
      if (mode == MODE_ENTER_LONG) {
        if (gl == 0) {
          float* hr = a.H + (size_t)(c0 / W) * N + col0;
#pragma unroll
          for (int j = 0; j < CT; ++j)
            if (j < nt) hr[j] = pf[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < CT; ++j) carry[j] = __fadd_rn(carry[j], pf[j]);
        if (fin && gl == 0) {
          float* yr = a.Y + (size_t)wrow_id * N + col0;  // lane 0 holds rid[cur]
#pragma unroll
          for (int j = 0; j < CT; ++j)
            if (j < nt) st_y(yr + j, carry[j]);
        }
      }
      if (fin) {
        has_carry = false;
        mode = MODE_NORMAL;
      }
    }
    // last live run continuing past the chunk becomes the carried row
    const int last_live = lhi - 1;
    const int klast = __shfl_sync(FULL, kidx, last_live, W);
    const int rend_last = __shfl_sync(FULL, rend, last_live, W);
    float pl[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) pl[j] = __shfl_sync(FULL, v[j], last_live, W);
    if (en && rend_last > c0 + W && !(carried_in && klast == 0)) {
#pragma unroll
      for (int j = 0; j < CT; ++j) carry[j] = pl[j];
      has_carry = true;
      mode = MODE_NORMAL;
    }
    const int nb = __popc(M);  // advance to the row containing c0 + W
    const int wnext = __shfl_sync(FULL, wrow_end, nb, W);
    if (en) cur = cur + nb + (wnext == c0 + W ? 1 : 0);
  };

  // rolled chunk loop (keeps the kernel inside the instruction cache); the
  // preloaded operands rotate down one slot per chunk
#pragma unroll 1
  for (int k = 0; k < T; ++k) {
    const long long c0 = tb + (long long)k * W;
    const bool en = k >= kstart && c0 < te;
    const int wi = cur - rbase + gl;
    const int wre = (wi >= 0 && wi < WINP) ? wcrp[wi] : 0x7fffffff;
    const int wid = (wi >= 0 && wi < WINP) ? wrid[wi] : 0;
    chunk(en, c0, wv[0], xv[0], wre, wid);
#pragma unroll
    for (int kk = 0; kk + 1 < T; ++kk) {
      wv[kk] = wv[kk + 1];
#pragma unroll
      for (int j = 0; j < CT; ++j) xv[kk][j] = xv[kk + 1][j];
    }
  }
  if (hard_end == te) {
    // a carried NORMAL row here crosses te and is long: owner prefix -> T
    if (has_carry && mode == MODE_NORMAL && gl == 0) {
      float* tr = a.Tsl + (size_t)unit * N + col0;
#pragma unroll
      for (int j = 0; j < CT; ++j)
        if (j < nt) tr[j] = carry[j];
    }
  }
  // owner extends: finish the crossing row (it ends in the next tile)
  const int wi0 = min(max(cur - rbase, 0), WINP - 1);
  const int wre = (gl == 0) ? wcrp[wi0] : 0x7fffffff;
  const int wid = (gl == 0) ? wrid[wi0] : 0;
#pragma unroll 1
  for (long long c0 = te; __any_sync(FULL, c0 < hard_end); c0 += W) {
    const bool en = c0 < hard_end;
    const long long p = c0 + gl;
    const bool live = en && p < hard_end;
    const int ci = live ? ld_stream(a.col + p, pol) : 0;
    const float w = live ? ld_stream(a.val + p, pol) : 0.f;
    float x[CT];
    const float* xr = a.X + (size_t)ci * N + col0;
#pragma unroll
    for (int j = 0; j < CT; ++j) x[j] = (live && j < nt) ? ld_x(xr + j) : 0.f;
    chunk(en, c0, w, x, wre, wid);
  }
}

}  // namespace spmk_dev
