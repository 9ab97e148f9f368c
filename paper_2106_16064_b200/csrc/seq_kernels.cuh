// seq_kernels.cuh — sequential-reduction kernels (north_star a and c):
//   seq-rs  spmm_seq_rowsplit  kernels.hpp:339-376  (row blocks, CSC staging)
//   seq-ws  spmm_seq_balanced  kernels.hpp:384-455  (nnz chunks of seq_chunk)
//
// One work unit = one group of LPU lanes (LPU | 32).  The group sweeps its
// nonzero range in ascending order; every lane owns CPL output columns and
// keeps one fp32 accumulator per column, so each column's sum is the
// reference's strictly sequential `acc += v*x` chain (bit-identical).
//
// CSC (coalesced sparse-row caching): each batch of B
// nonzeros' colIdx/val is loaded coalesced across the group (lane gl loads
// entries gl, gl+LPU, ...) and broadcast with shuffles, so all dense-row
// gathers of the batch are issued before the sequential adds consume them.
//
// Rows come from the handle's compacted row list (non-empty rows only;
// empty rows are zero-filled by zero_rows_kernel), so a row change is
// "position == crp[cur+1]" with no empty-row skipping.
//
// seq-ws chunk semantics (kernels.hpp:410-453): the reference's per-chunk
// partials for rows crossing chunk boundaries are merged as
// Y = ((0 + P_q1) + P_q1+1) + ... in ascending chunk order.  A unit here is a
// tile of T chunks; at every chunk boundary inside a row the running
// `carry = carry + acc; acc = 0` reproduces exactly that order.  A row that
// crosses the tile end is finished by the tile that owns its start when it
// ends in the next tile ("owner extends", no partial traffic); rows spanning
// >= 2 more tiles emit per-chunk partials (H) plus the owner prefix (T) and
// are merged by fixup_kernel in ascending order.
#pragma once
#include "common.cuh"

namespace spmk_dev {

struct SeqArgs {
  const int* __restrict__ crp;   // compact rowPtr (mne+1)
  const int* __restrict__ rid;   // compact -> original row (mne)
  const int* __restrict__ col;   // nnz
  const float* __restrict__ val; // nnz
  const float* __restrict__ X;   // K x N
  float* __restrict__ Y;         // M x N
  float* __restrict__ H;         // chunk partial slots (nchunks x N)
  float* __restrict__ Tsl;       // tile prefix slots (ntiles x N)
  const int* __restrict__ rlo;   // ws: first compact row starting >= tile start
  int mne;                       // non-empty rows
  int nnz;
  int N;                         // columns of X / Y
  int ncol_tile;                 // columns handled per blockIdx.y
  long long TS;                  // ws: tile size in nnz (= T * CH)
  long long CH;                  // ws: chunk size (seq_chunk)
  int RB;                        // rs: rows per tile
  int nunits;                    // tiles
};

template <int LPU, int CPL, bool VEC, int B, bool WS>
__global__ void __launch_bounds__(256)
seq_kernel(const SeqArgs a) {
  static_assert(B % LPU == 0 || LPU > B, "batch");
  constexpr int SLOTS = (B + LPU - 1) / LPU;  // entries loaded per lane per batch
  const int lane = threadIdx.x & 31;
  const int gl = lane & (LPU - 1);
  const int upb = blockDim.x / LPU;
  const int unit = blockIdx.x * upb + threadIdx.x / LPU;
  if (unit >= a.nunits) return;  // group-uniform

  const int col0 = blockIdx.y * a.ncol_tile;
  ColMap<LPU, CPL, VEC> cm{gl, min(a.ncol_tile, a.N - col0)};
  const int N = a.N;
  const uint64_t pol = evict_first_policy();

  // ---- tile setup -------------------------------------------------------
  long long e, te, hard_end;
  int cur, cur_end, orow = 0, mode = MODE_NORMAL;
  float carry[CPL], acc[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) carry[k] = acc[k] = 0.f;
  long long next_cb;

  if constexpr (WS) {
    const long long tb = (long long)unit * a.TS;
    te = min(tb + a.TS, (long long)a.nnz);
    const int r = a.rlo[unit];
    // crossing row at te: the row containing position te started before te.
    hard_end = te;
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
        cur_end = cr;
        mode = MODE_ENTER_LONG;
        e = tb;
      } else {
        e = cr;  // skipped: finished by the owner tile
        if (e >= te) return;
        cur = r;
        cur_end = a.crp[cur + 1];
        orow = a.rid[cur];
      }
    } else {
      e = tb;
      cur = r;
      cur_end = a.crp[cur + 1];
      orow = a.rid[cur];
    }
    if (mode == MODE_NORMAL && cur_end > te && (cur_end - 1) / a.TS >= unit + 2)
      mode = MODE_OWNER_LONG;
    next_cb = (e / a.CH + 1) * a.CH;
  } else {
    const int r0 = unit * a.RB;
    const int r1 = min(r0 + a.RB, a.mne);
    e = a.crp[r0];
    te = a.crp[r1];
    hard_end = te;
    cur = r0;
    cur_end = a.crp[cur + 1];
    orow = a.rid[cur];
    next_cb = 0x7fffffffffffffffLL;
  }
  long long nev = min((long long)cur_end, next_cb);

  // ---- sweep ---------------------------------------------------------------
  bool live = true;
  for (long long eb = e; live; eb += B) {
    int cr_[SLOTS];
    float vr_[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const long long p = eb + (long long)s * LPU + gl;
      if (p < hard_end) {
        cr_[s] = ld_stream(a.col + p, pol);
        vr_[s] = ld_stream(a.val + p, pol);
      } else {
        cr_[s] = 0;
        vr_[s] = 0.f;
      }
    }
    float xv[B][CPL];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int c = gshfl<LPU>(cr_[j / LPU], j % LPU);
      if (eb + j < hard_end) {
        cm.load(a.X + (size_t)c * N + col0, xv[j]);
      } else {
#pragma unroll
        for (int k = 0; k < CPL; ++k) xv[j][k] = 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const long long p = eb + j;
      if (p == nev) {
        if (p == cur_end) {
          if (mode == MODE_ENTER_LONG) {
            cm.store_slot(a.H + (size_t)((p - 1) / a.CH) * N + col0, acc);
          } else {
            float o[CPL];
#pragma unroll
            for (int k = 0; k < CPL; ++k) o[k] = __fadd_rn(carry[k], acc[k]);
            cm.store(a.Y + (size_t)orow * N + col0, o);
          }
          if (p >= te) {
            live = false;
          } else {
            ++cur;
            cur_end = a.crp[cur + 1];
            orow = a.rid[cur];
            mode = MODE_NORMAL;
            if constexpr (WS) {
              if (cur_end > te && (cur_end - 1) / a.TS >= unit + 2) mode = MODE_OWNER_LONG;
            }
#pragma unroll
            for (int k = 0; k < CPL; ++k) carry[k] = acc[k] = 0.f;
          }
        }
        if constexpr (WS) {
          if (live && p == next_cb) {
            if (mode == MODE_ENTER_LONG) {
              cm.store_slot(a.H + (size_t)(p / a.CH - 1) * N + col0, acc);
#pragma unroll
              for (int k = 0; k < CPL; ++k) acc[k] = 0.f;
              if (p >= te) live = false;
            } else if (mode == MODE_OWNER_LONG && p >= te) {
              float o[CPL];
#pragma unroll
              for (int k = 0; k < CPL; ++k) o[k] = __fadd_rn(carry[k], acc[k]);
              cm.store_slot(a.Tsl + (size_t)unit * N + col0, o);
              live = false;
            } else {
#pragma unroll
              for (int k = 0; k < CPL; ++k) {
                carry[k] = __fadd_rn(carry[k], acc[k]);
                acc[k] = 0.f;
              }
            }
            next_cb += a.CH;
          }
        }
        nev = min((long long)cur_end, next_cb);
      }
      if (!live) break;
      const float v = gshfl<LPU>(vr_[j / LPU], j % LPU);
#pragma unroll
      for (int k = 0; k < CPL; ++k) acc[k] = mul_add_rn(acc[k], v, xv[j][k]);
    }
  }
}

}  // namespace spmk_dev
