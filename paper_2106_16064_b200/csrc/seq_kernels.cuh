// seq_kernels.cuh — sequential-reduction kernels (north_star a and c):
//   seq-rs  spmm_seq_rowsplit  kernels.hpp:339-376  (row blocks, CSC staging)
//   seq-ws  spmm_seq_balanced  kernels.hpp:384-455  (nnz chunks of seq_chunk)
//
// One work unit = one group of LPU lanes (LPU | 32) sweeping a tile of
// nonzeros in ascending order; every lane owns CPL output columns with one
// fp32 accumulator each, so a column's sum is the reference's strictly
// sequential `acc += v*x` chain (bit-identical, two roundings).
//
// Latency hiding (the sweep is a gather-multiply-reduce, HBM/L2 bound):
//   * 3-stage software pipeline over batches of B nonzeros: colIdx/val of
//     batch b+2 and the dense-row gathers of batch b+1 are in flight while
//     batch b is consumed — no load sits on the critical path of the adds.
//   * CSC: each batch's colIdx/val is loaded coalesced across
//     the group (lane gl takes entries gl, gl+LPU, ...) and broadcast with
//     shuffles.
//   * Row metadata (row ends, output row ids) of the next WIN rows sit in a
//     per-group shared-memory window, so a row change is a shared-memory
//     broadcast, not a dependent global load.
//
// Rows come from the handle's compacted row list (non-empty rows only;
// empty rows are zero-filled by zero_rows_kernel).
//
// seq-ws chunk semantics (kernels.hpp:410-453): the reference merges the
// per-chunk partials of a row that crosses chunk boundaries as
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
  const int* __restrict__ order; // rs: tile processing order (heavy first) or null
  int mne;                       // non-empty rows
  int nnz;
  int N;                         // columns of X / Y
  int ncol_tile;                 // columns handled per blockIdx.y
  long long TS;                  // ws: tile size in nnz (= T * CH)
  long long CH;                  // ws: chunk size (seq_chunk)
  int RB;                        // rs: rows per tile
  int nunits;                    // tiles
};

constexpr int kSeqThreads = 256;

template <int LPU>
struct SeqWin {
  static constexpr int WIN = LPU >= 8 ? 64 : (LPU >= 2 ? 32 : 16);
};

template <int LPU, int CPL, bool VEC, int B, bool WS>
__global__ void __launch_bounds__(kSeqThreads, 2)
seq_kernel(const SeqArgs a) {
  constexpr int SLOTS = (B + LPU - 1) / LPU;  // entries loaded per lane per batch
  constexpr int WIN = SeqWin<LPU>::WIN;
  constexpr int NGROUPS = kSeqThreads / LPU;
  constexpr int BIG = 0x7fffffff;
  __shared__ int s_win[NGROUPS * 2 * WIN];

  const int lane = threadIdx.x & 31;
  const int gl = lane & (LPU - 1);
  const int gidx = threadIdx.x / LPU;
  const unsigned gmask = group_mask<LPU>();
  int unit = blockIdx.x * NGROUPS + gidx;
  // Every lane of the warp stays in the sweep loop until all groups are done
  // (warp-uniform trip count), so all shuffles run converged on a full mask.
  bool live = unit < a.nunits;
  if (!live) unit = 0;
  if constexpr (!WS) {
    if (a.order && live) unit = a.order[unit];
  }
  int* wcrp = s_win + gidx * 2 * WIN;  // wcrp[i] = crp[wb + 1 + i]
  int* wrid = wcrp + WIN;              // wrid[i] = rid[wb + i]

  const int col0 = blockIdx.y * a.ncol_tile;
  const ColMap<LPU, CPL, VEC> cm{gl, min(a.ncol_tile, a.N - col0)};
  const int N = a.N;
  const uint64_t pol = evict_first_policy();

  // ---- tile setup (all divisions happen here, none in the sweep) ----------
  int e, te, hard_end, cur;
  int mode = MODE_NORMAL;
  int q = 0, next_cb = BIG, long_thresh = BIG, CH = BIG;
  if constexpr (WS) {
    CH = (int)a.CH;
    const long long tb = (long long)unit * a.TS;
    te = (int)min(tb + a.TS, (long long)a.nnz);
    long_thresh = (int)min((long long)(unit + 2) * a.TS, (long long)BIG);  // row end > this => long
    const int r = a.rlo[unit];
    hard_end = te;
    if (te < a.nnz) {  // row crossing te, finished here if it ends in the next tile
      const int r2 = a.rlo[unit + 1];
      const int c2 = a.crp[r2];
      if (c2 > te && a.crp[r2 - 1] >= tb && c2 <= long_thresh) hard_end = c2;
    }
    const int cr = a.crp[r];
    if (cr > tb) {  // row r-1 enters from the left
      const int rs = a.crp[r - 1];
      if ((cr - 1) / a.TS - rs / a.TS >= 2) {
        cur = r - 1;
        mode = MODE_ENTER_LONG;
        e = (int)tb;
      } else {
        e = cr;  // skipped: finished by its owner tile
        if (e >= te) live = false;
        cur = r;
      }
    } else {
      e = (int)tb;
      cur = r;
    }
    q = e / CH;
    next_cb = (int)min((long long)(q + 1) * CH, (long long)BIG);
  } else {
    const int r0 = unit * a.RB;
    const int r1 = min(r0 + a.RB, a.mne);
    e = a.crp[r0];
    te = a.crp[r1];
    hard_end = te;
    cur = r0;
  }

  int wb = cur;
  auto refill = [&](int base) {
    __syncwarp(gmask);
#pragma unroll 1
    for (int i = gl; i < WIN; i += LPU) {
      const int ci = base + 1 + i;
      wcrp[i] = ci <= a.mne ? a.crp[ci] : BIG;
      wrid[i] = (base + i < a.mne) ? a.rid[base + i] : 0;
    }
    __syncwarp(gmask);
    wb = base;
  };
  refill(cur);
  int cur_end = wcrp[0];
  int orow = wrid[0];
  if (WS && mode == MODE_NORMAL && cur_end > long_thresh) mode = MODE_OWNER_LONG;
  float carry[CPL], acc[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) carry[k] = acc[k] = 0.f;
  int nev = min(cur_end, next_cb);

  // ---- pipelined sweep -----------------------------------------------------
  auto load_cv = [&](int eb, int (&cr)[SLOTS], float (&vr)[SLOTS]) {
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int o = s * LPU + gl;
      const int p = eb + o;
      if (o < B && p < hard_end) {
        if constexpr (LPU >= 8) {
          cr[s] = ld_stream(a.col + p, pol);
          vr[s] = ld_stream(a.val + p, pol);
        } else {
          cr[s] = __ldg(a.col + p);
          vr[s] = __ldg(a.val + p);
        }
      } else {
        cr[s] = 0;
        vr[s] = 0.f;
      }
    }
  };
  auto load_x = [&](int eb, const int (&cr)[SLOTS], float (&xv)[B][CPL]) {
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int c = gshfl<LPU>(cr[j / LPU], j % LPU);
      if (eb + j < hard_end) {
        cm.load(a.X + (size_t)c * N + col0, xv[j]);
      } else {
#pragma unroll
        for (int k = 0; k < CPL; ++k) xv[j][k] = 0.f;
      }
    }
  };

  int c_c[SLOTS], c_n[SLOTS], c_nn[SLOTS];
  float v_c[SLOTS], v_n[SLOTS], v_nn[SLOTS];
  float x_c[B][CPL], x_n[B][CPL];
  load_cv(e, c_c, v_c);
  load_cv(e + B, c_n, v_n);
  load_x(e, c_c, x_c);

  if (!live) hard_end = 0;  // no loads for idle groups
#pragma unroll 1
  for (int eb = e; __any_sync(0xffffffffu, live); eb += B) {
    load_cv(eb + 2 * B, c_nn, v_nn);
    load_x(eb + B, c_n, x_n);
    float vv[B];
#pragma unroll
    for (int j = 0; j < B; ++j) vv[j] = gshfl<LPU>(v_c[j / LPU], j % LPU);
    // Segments between events: one predicated, event-free pass over the
    // batch per segment, and a single copy of the (rare) event handler, so
    // the hot loop stays small in the instruction cache.  No shuffles below:
    // groups may diverge here.
    int js = 0;
#pragma unroll 1
    while (live) {
      const int je = (nev < eb + B) ? nev - eb : B;
#pragma unroll
      for (int j = 0; j < B; ++j) {
        if (j >= js && j < je) {
#pragma unroll
          for (int k = 0; k < CPL; ++k) acc[k] = mul_add_rn(acc[k], vv[j], x_c[j][k]);
        }
      }
      if (je >= B) break;
      const int p = eb + je;  // event before consuming position p
      if (p == cur_end) {
        if (WS && mode == MODE_ENTER_LONG) {
          cm.store_slot(a.H + (size_t)q * N + col0, acc);
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
          if (cur - wb >= WIN) refill(cur);
          cur_end = wcrp[cur - wb];
          orow = wrid[cur - wb];
          mode = (WS && cur_end > long_thresh) ? MODE_OWNER_LONG : MODE_NORMAL;
#pragma unroll
          for (int k = 0; k < CPL; ++k) carry[k] = acc[k] = 0.f;
        }
      }
      if (WS && live && p == next_cb) {
        if (mode == MODE_ENTER_LONG) {
          cm.store_slot(a.H + (size_t)q * N + col0, acc);
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
        ++q;
        next_cb = (next_cb > BIG - CH) ? BIG : next_cb + CH;
      }
      nev = min(cur_end, next_cb);
      js = je;
    }
    // rotate the pipeline
#pragma unroll
    for (int j = 0; j < B; ++j)
#pragma unroll
      for (int k = 0; k < CPL; ++k) x_c[j][k] = x_n[j][k];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      v_c[s] = v_n[s];
      c_n[s] = c_nn[s];
      v_n[s] = v_nn[s];
    }
  }
}

}  // namespace spmk_dev
