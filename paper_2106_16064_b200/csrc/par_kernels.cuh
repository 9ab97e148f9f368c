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

  for (int r = gid; r < a.mne; r += groups_total) {
    const int s = a.crp[r], f = a.crp[r + 1];
    float acc[CT];
#pragma unroll
    for (int k = 0; k < CT; ++k) acc[k] = 0.f;
    float acc2[VL == 2 ? CT : 1];
#pragma unroll
    for (int k = 0; k < (VL == 2 ? CT : 1); ++k) acc2[k] = 0.f;

    for (int base = s; base < f; base += W) {
#pragma unroll
      for (int v = 0; v < VL; ++v) {
        const int p = base + gl * VL + v;  // virtual lane gl*VL+v
        if (p < f) {
          const int c = ld_stream(a.col + p, pol);
          const float w = ld_stream(a.val + p, pol);
          const float* xr = a.X + (size_t)c * N + col0;
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
              for (int k = 0; k < CT; ++k) acc2[k] = mul_add_rn(acc2[k], w, xv[k]);
            } else {
#pragma unroll
              for (int k = 0; k < CT; ++k) acc[k] = mul_add_rn(acc[k], w, xv[k]);
            }
          } else {
#pragma unroll
            for (int k = 0; k < CT; ++k) acc[k] = mul_add_rn(acc[k], w, xv[k]);
          }
        }
      }
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
template <int W, int CT>
__global__ void __launch_bounds__(256)
par_ws_kernel(const ParArgs a) {
  static_assert(W >= 2 && W <= 32, "W");
  const int lane = threadIdx.x & 31;
  const int gl = lane & (W - 1);
  const unsigned gmask = group_mask<W>();
  const int upb = blockDim.x / W;
  const int unit = blockIdx.x * upb + threadIdx.x / W;
  if (unit >= a.nunits) return;  // group-uniform
  const int col0 = blockIdx.y * a.ncol_tile;
  const int nt = min(a.ncol_tile, a.N - col0);
  const int N = a.N;
  const uint64_t pol = evict_first_policy();
  const bool vec4 = (CT % 4 == 0) && (N % 4 == 0);
  const unsigned le = (gl == 31) ? 0xffffffffu : ((2u << gl) - 1u);  // lanes <= gl

  const long long tb = (long long)unit * a.TS;
  const long long te = min(tb + a.TS, (long long)a.nnz);
  const int r = a.rlo[unit];
  long long lo = tb;        // first live position of this tile
  long long hard_end = te;  // te, or the end of an owned row crossing te
  long long c0 = tb;
  int cur;                  // compact row containing c0
  int mode = MODE_NORMAL;   // mode of the carried row
  bool has_carry = false;   // a row continues into chunk c0 from before it
  float carry[CT];
#pragma unroll
  for (int k = 0; k < CT; ++k) carry[k] = 0.f;

  if (te < a.nnz) {
    const int r2 = a.rlo[unit + 1];
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
      if (lo >= te) return;
      c0 = tb + ((lo - tb) / W) * W;
      cur = (lo > c0) ? r - 1 : r;
    }
  } else {
    cur = r;
  }

  for (; c0 < hard_end; c0 += W) {
    const long long p = c0 + gl;
    const long long hi = min(c0 + W, hard_end);
    const bool live = p >= lo && p < hi;
    const int llo = (int)max(0LL, lo - c0);
    const int lhi = (int)(hi - c0);
    // segment heads: window of the next W row ends crp[cur+1 .. cur+W]
    const int wi = cur + 1 + gl;
    const int wv = wi <= a.mne ? a.crp[wi] : 0x7fffffff;
    const int ridw = (cur + gl < a.mne) ? a.rid[cur + gl] : 0;
    const long long b = (long long)wv - c0;
    const unsigned M = __reduce_or_sync(gmask, (b > 0 && b < W) ? (1u << (int)b) : 0u);
    unsigned Mrun = M;  // dead lanes form their own runs
    if (llo > 0) Mrun |= 1u << llo;
    if (lhi < W) Mrun |= 1u << lhi;
    const int kidx = __popc(M & le);     // row(l) - cur
    const int runid = __popc(Mrun & le);

    // rounded products v*x (kernels.hpp:277)
    int cidx = 0;
    float w = 0.f;
    if (live) {
      cidx = ld_stream(a.col + p, pol);
      w = ld_stream(a.val + p, pol);
    }
    float v[CT];
    const float* xr = a.X + (size_t)cidx * N + col0;
    if (vec4) {
#pragma unroll
      for (int k = 0; k < CT; k += 4) {
        if (live && k < nt) {
          const float4 t = ld_x4(xr + k);
          v[k] = __fmul_rn(w, t.x);
          v[k + 1] = __fmul_rn(w, t.y);
          v[k + 2] = __fmul_rn(w, t.z);
          v[k + 3] = __fmul_rn(w, t.w);
        } else {
          v[k] = v[k + 1] = v[k + 2] = v[k + 3] = 0.f;
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < CT; ++k) v[k] = (live && k < nt) ? __fmul_rn(w, ld_x(xr + k)) : 0.f;
    }
    // conditional Hillis-Steele scan (reduction.hpp:77-85), lockstep
#pragma unroll
    for (int off = 1; off < W; off <<= 1) {
      const int src = gl - off;
      const bool same =
          src >= 0 && __popc(Mrun & ((src == 31) ? 0xffffffffu : ((2u << src) - 1u))) == runid;
#pragma unroll
      for (int k = 0; k < CT; ++k) {
        const float up = __shfl_up_sync(gmask, v[k], off, W);
        if (same) v[k] = __fadd_rn(v[k], up);
      }
    }
    const bool last_of_run = live && (gl == W - 1 || ((Mrun >> (gl + 1)) & 1u));
    const int rend = __shfl_sync(gmask, wv, kidx, W);   // crp[row+1]
    const int orow = __shfl_sync(gmask, ridw, kidx, W); // rid[row]
    const bool starts_here = kidx > 0 || !has_carry;
    const bool ends_here = rend <= c0 + W;
    // runs complete in this chunk: Y = P (kernels.hpp:299-301)
    if (last_of_run && starts_here && ends_here) {
      float* yr = a.Y + (size_t)orow * N + col0;
#pragma unroll
      for (int k = 0; k < CT; ++k)
        if (k < nt) st_y(yr + k, v[k]);
    }
    const bool carried_in = has_carry;
    // run entering from the previous chunk (lanes [0, first boundary))
    if (carried_in) {
      const unsigned rest = Mrun & ~1u;
      const int first_last = rest ? (__ffs(rest) - 2) : (W - 1);
      const bool fin = __shfl_sync(gmask, wv, 0, W) <= c0 + W;
      float pf[CT];
#pragma unroll
      for (int k = 0; k < CT; ++k) pf[k] = __shfl_sync(gmask, v[k], first_last, W);
      if (mode == MODE_ENTER_LONG) {
        if (gl == 0) {
          float* hr = a.H + (size_t)(c0 / W) * N + col0;
#pragma unroll
          for (int k = 0; k < CT; ++k)
            if (k < nt) hr[k] = pf[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < CT; ++k) carry[k] = __fadd_rn(carry[k], pf[k]);
        if (fin && gl == 0) {
          float* yr = a.Y + (size_t)ridw * N + col0;  // lane 0 holds rid[cur]
#pragma unroll
          for (int k = 0; k < CT; ++k)
            if (k < nt) st_y(yr + k, carry[k]);
        }
      }
      if (fin) {
        has_carry = false;
        mode = MODE_NORMAL;
      }
    }
    // last live run continuing past the chunk becomes the carried row
    const int last_live = lhi - 1;
    const int klast = __shfl_sync(gmask, kidx, last_live, W);
    const int rend_last = __shfl_sync(gmask, rend, last_live, W);
    if (rend_last > c0 + W && !(carried_in && klast == 0)) {
#pragma unroll
      for (int k = 0; k < CT; ++k) carry[k] = __shfl_sync(gmask, v[k], last_live, W);
      has_carry = true;
      mode = MODE_NORMAL;
    }
    // advance to the row containing c0 + W
    const int nb = __popc(M);
    const int wnext = __shfl_sync(gmask, wv, nb, W);
    cur = cur + nb + (wnext == c0 + W ? 1 : 0);
    if (c0 + W >= te && hard_end == te) {
      // a carried NORMAL row here crosses te and is long: owner prefix -> T
      if (has_carry && mode == MODE_NORMAL && gl == 0) {
        float* tr = a.Tsl + (size_t)unit * N + col0;
#pragma unroll
        for (int k = 0; k < CT; ++k)
          if (k < nt) tr[k] = carry[k];
      }
      break;
    }
  }
}

}  // namespace spmk_dev
