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
  const int4* __restrict__ desc;  // par-ws per-tile start descriptors (ws_tile_desc_kernel)
  int mne, nnz, N;
  int xvec;           // dense rows loadable as aligned float2/float4
  int ncol_tile;      // columns per blockIdx.y pass
  long long TS;       // par-ws tile (T chunks of W)
  int nunits;
  int hub;            // par-rs: rows with >= hub nonzeros belong to par_rs_hub_kernel
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
  const char* const xb = reinterpret_cast<const char*>(a.X + col0);
  const unsigned xs = (unsigned)N * 4u;
  // dense-row loads of one batch (issued before any of the batch's FMAs)
  auto load_x = [&](const int (&c)[VL], float (&xv)[VL][CT]) {
#pragma unroll
    for (int v = 0; v < VL; ++v) {
      const float* xr = reinterpret_cast<const float*>(xb + (size_t)(unsigned)max(c[v], 0) * xs);
      const bool ok = c[v] >= 0;
      if constexpr (VEC4 && CT % 4 == 0) {
#pragma unroll
        for (int k = 0; k < CT; k += 4) {
          if (ok && k < nt) {
            const float4 t = ld_x4(xr + k);
            xv[v][k] = t.x; xv[v][k + 1] = t.y; xv[v][k + 2] = t.z; xv[v][k + 3] = t.w;
          } else {
            xv[v][k] = xv[v][k + 1] = xv[v][k + 2] = xv[v][k + 3] = 0.f;
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < CT; ++k) xv[v][k] = (ok && k < nt) ? ld_x(xr + k) : 0.f;
      }
    }
  };
  // lane-sequential FMA chain (kernels.hpp:181-186); dead lanes add nothing.
  // Virtual lane gl*VL+v keeps its own chain acc[v].
  auto fma_batch = [&](const int (&c)[VL], const float (&w)[VL], const float (&xall)[VL][CT],
                       float (&acc)[VL][CT]) {
#pragma unroll
    for (int v = 0; v < VL; ++v) {
      if (c[v] >= 0) {
#pragma unroll
        for (int k = 0; k < CT; ++k) acc[v][k] = mul_add_rn(acc[v][k], w[v], xall[v][k]);
      }
    }
  };

  // Software pipeline over this group's rows: bounds two rows ahead, the
  // first W-batch of colIdx/val one row ahead.  Refills happen after the
  // rotation, so the register moves only read values loaded an iteration
  // earlier.
  int s0, f0, s1, f1, s2, f2;
  bounds(gid, s0, f0);
  bounds(gid + groups_total, s1, f1);
  bounds(gid + 2 * groups_total, s2, f2);
  int c0[VL], c1[VL];
  float w0[VL], w1[VL];
  first_batch(s0, f0, c0, w0);
  first_batch(s1, f1, c1, w1);
  for (int r = gid; r < a.mne; r += groups_total) {
    const int s = s0, f = f0;
    if (f - s < a.hub) {
    float accv[VL][CT];
#pragma unroll
    for (int v = 0; v < VL; ++v)
#pragma unroll
      for (int k = 0; k < CT; ++k) accv[v][k] = 0.f;
    {
      float x0[VL][CT];
      load_x(c0, x0);
      fma_batch(c0, w0, x0, accv);
    }
    // rows longer than W: U batches of colIdx/val, then their dense rows, are
    // in flight before the (in-order) FMAs of the first one
    // (wider virtual-lane groups already hold VL loads per lane)
    constexpr int U0 = CT <= 1 ? 4 : (CT <= 4 ? 2 : 1);
    constexpr int U = VL <= 2 ? U0 : (U0 * 2 / VL > 0 ? U0 * 2 / VL : 1);
    for (int base = s + W; base < f; base += U * W) {
      int c[U][VL];
      float w[U][VL];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < VL; ++v) {
          const int p = base + u * W + gl * VL + v;
          c[u][v] = p < f ? ld_stream(a.col + p, pol) : -1;
          w[u][v] = p < f ? ld_stream(a.val + p, pol) : 0.f;
        }
      float xv[U][VL][CT];
#pragma unroll
      for (int u = 0; u < U; ++u) load_x(c[u], xv[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) fma_batch(c[u], w[u], xv[u], accv);
    }
    // the tree levels inside one physical lane (virtual lanes gl*VL .. +VL-1):
    // acc[l] = acc[2l+1] + acc[2l] (kernels.hpp:193-199)
#pragma unroll
    for (int wv = VL; wv > 1; wv >>= 1)
#pragma unroll
      for (int v = 0; v < wv / 2; ++v)
#pragma unroll
        for (int k = 0; k < CT; ++k) accv[v][k] = __fadd_rn(accv[2 * v + 1][k], accv[2 * v][k]);
    float acc[CT];
#pragma unroll
    for (int k = 0; k < CT; ++k) acc[k] = accv[0][k];
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
    s0 = s1; f0 = f1; s1 = s2; f1 = f2;
#pragma unroll
    for (int v = 0; v < VL; ++v) {
      c0[v] = c1[v];
      w0[v] = w1[v];
    }
    bounds(r + 3 * groups_total, s2, f2);
    first_batch(s1, f1, c1, w1);
  }
}

}  // namespace spmk_dev

#include "par_ws.cuh"
