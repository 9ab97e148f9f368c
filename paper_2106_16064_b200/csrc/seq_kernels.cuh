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
  const int4* __restrict__ desc; // per-tile start descriptors (ws_/rs_tile_desc_kernel)
  int mne;                       // non-empty rows
  int nnz;
  int N;                         // columns of X / Y
  int ncol_tile;                 // columns handled per blockIdx.y
  long long TS;                  // ws: tile size in nnz (= T * CH)
  long long CH;                  // ws: chunk size (seq_chunk)
  long long EXT;                 // ws: owner-extension limit (row_is_long)
  int nunits;                    // tiles
  int cvvec;                     // colIdx/val 16-byte aligned (vector batch loads)
  f32x2 one2;                    // {1.0f, 1.0f} (kOnePair), opaque to ptxas: see f2_add
};

constexpr int kSeqThreads = 256;

template <int LPU>
struct SeqWin {
  static constexpr int WIN = LPU >= 8 ? 64 : (LPU >= 2 ? 32 : 16);
};

// Per-group sweep state: tile setup, the row window and the (rare) event
// handler.  Every member function is force-inlined, so the state lives in
// registers; the two kernels below differ only in how dense rows arrive.
template <int LPU, int CPL, bool VEC, bool WS, int NT = kSeqThreads>
struct SeqSweep {
  static constexpr int WIN = SeqWin<LPU>::WIN;
  static constexpr int BIG = 0x7fffffff;
  int e, te, hard_end, cur, cur_end, orow, mode, q, next_cb, long_thresh, CH, wb, unit, nev;
  bool live;
  float carry[CPL], acc[CPL];
  int* wcrp;  // wcrp[i] = crp[wb + 1 + i]
  int* wrid;  // wrid[i] = rid[wb + i]
  int gl, col0, N;
  char* ybase;         // Y + col0: row address = ybase + row * ystride (32-bit math)
  unsigned ystride;
  unsigned gmask;
  ColMap<LPU, CPL, VEC> cm;

  __device__ __forceinline__ void refill(const SeqArgs& a, int base) {
    __syncwarp(gmask);
#pragma unroll 1
    for (int i = gl; i < WIN; i += LPU) {
      const int ci = base + 1 + i;
      wcrp[i] = ci <= a.mne ? a.crp[ci] : BIG;
      wrid[i] = (base + i < a.mne) ? a.rid[base + i] : 0;
    }
    __syncwarp(gmask);
    wb = base;
  }

  // Tile setup, part 1: one 16-byte descriptor load (the plan precomputed the
  // entering/crossing-row decisions), so the colIdx/val prefetch can be issued
  // right after it without further dependent round trips.
  __device__ __forceinline__ void setup_begin(const SeqArgs& a, int* swin) {
    const int lane = threadIdx.x & 31;
    gl = lane & (LPU - 1);
    const int gidx = threadIdx.x / LPU;
    gmask = group_mask<LPU>();
    constexpr int NGROUPS = NT / LPU;
    unit = blockIdx.x * NGROUPS + gidx;
    // Every lane of the warp stays in the sweep loop until all groups are done
    // (warp-uniform trip count), so all shuffles run converged on a full mask.
    live = unit < a.nunits;
    if (!live) unit = 0;
    if constexpr (!WS) {
      if (a.order && live) unit = a.order[unit];
    }
    wcrp = swin + gidx * 2 * WIN;
    wrid = wcrp + WIN;
    col0 = blockIdx.y * a.ncol_tile;
    cm = ColMap<LPU, CPL, VEC>{gl, min(a.ncol_tile, a.N - col0)};
    N = a.N;
    ybase = reinterpret_cast<char*>(a.Y + col0);
    ystride = (unsigned)a.N * 4u;
    const int4 d = a.desc[unit];
    cur = d.x;
    e = d.y;
    hard_end = d.z;
    mode = d.w;
    q = 0;
    next_cb = BIG;
    long_thresh = BIG;
    CH = BIG;
    if constexpr (WS) {
      CH = (int)a.CH;
      const long long tb = (long long)unit * a.TS;
      te = (int)min(tb + a.TS, (long long)a.nnz);
      long_thresh = (int)min(tb + a.TS + a.EXT, (long long)BIG);  // row end > this => long (row_is_long)
      q = e / CH;
      next_cb = (int)min((long long)(q + 1) * CH, (long long)BIG);
    } else {
      te = hard_end;
    }
    if (e >= hard_end) live = false;
    if (!live) hard_end = 0;  // no loads for idle groups
  }
  // Tile setup, part 2 (after the prefetch is in flight): the row window.
  __device__ __forceinline__ void setup_end(const SeqArgs& a) {
    refill(a, cur);
    cur_end = wcrp[0];
    orow = wrid[0];
    if (WS && mode == MODE_NORMAL && cur_end > long_thresh) mode = MODE_OWNER_LONG;
#pragma unroll
    for (int k = 0; k < CPL; ++k) carry[k] = acc[k] = 0.f;
    nev = min(cur_end, next_cb);
  }

  // Events at position p (before consuming it): row end and/or chunk boundary.
  __device__ __forceinline__ void event(const SeqArgs& a, int p) {
    if (p == cur_end) {
      if (WS && mode == MODE_ENTER_LONG) {
        cm.store_slot(a.H + (size_t)q * N + col0, acc);
      } else {
        float o[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) o[k] = __fadd_rn(carry[k], acc[k]);
        cm.store(reinterpret_cast<float*>(ybase + (size_t)(unsigned)orow * ystride), o);
      }
      if (p >= te) {
        live = false;
      } else {
        ++cur;
        if (cur - wb >= WIN) refill(a, cur);
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
  }
};

// --------------------------------------------------------------------------
// Register-pipelined sweep (any column mapping).
// --------------------------------------------------------------------------
template <int LPU, int CPL, bool VEC, int B, bool WS>
__global__ void __launch_bounds__(kSeqThreads, 2)
seq_kernel(const SeqArgs a) {
  constexpr int SLOTS = (B + LPU - 1) / LPU;  // entries loaded per lane per batch
  using SW = SeqSweep<LPU, CPL, VEC, WS>;
  __shared__ int s_win[(kSeqThreads / LPU) * 2 * SW::WIN];
  SW st;
  st.setup_begin(a, s_win);
  const uint64_t pol = evict_first_policy();

  auto load_cv = [&](int eb, int (&cr)[SLOTS], float (&vr)[SLOTS]) {
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int o = s * LPU + st.gl;
      const int p = eb + o;
      if (o < B && p < st.hard_end) {
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
      if (eb + j < st.hard_end) {
        st.cm.load(reinterpret_cast<const float*>(reinterpret_cast<const char*>(a.X + st.col0) +
                                                  (size_t)(unsigned)c * ((unsigned)st.N * 4u)),
                   xv[j]);
      } else {
#pragma unroll
        for (int k = 0; k < CPL; ++k) xv[j][k] = 0.f;
      }
    }
  };

  // colIdx/val two batches ahead (refilled after the rotation, so the moves
  // read registers loaded an iteration earlier); dense rows one batch ahead in
  // two register sets whose roles swap between the two unrolled halves.
  int c_c[SLOTS], c_n[SLOTS], c_nn[SLOTS];
  float v_c[SLOTS], v_n[SLOTS], v_nn[SLOTS];
  float x_a[B][CPL], x_b[B][CPL];
  load_cv(st.e, c_c, v_c);
  load_cv(st.e + B, c_n, v_n);
  load_cv(st.e + 2 * B, c_nn, v_nn);
  st.setup_end(a);
  load_x(st.e, c_c, x_a);

  auto step = [&](int eb, float (&xc)[B][CPL], float (&xn)[B][CPL]) {
    load_x(eb + B, c_n, xn);
    float vv[B];
#pragma unroll
    for (int j = 0; j < B; ++j) vv[j] = gshfl<LPU>(v_c[j / LPU], j % LPU);
    // Segments between events: one predicated, event-free pass over the
    // batch per segment, and a single copy of the (rare) event handler, so
    // the hot loop stays small in the instruction cache.  No shuffles below:
    // groups may diverge here.
    int js = 0;
#pragma unroll 1
    while (st.live) {
      const int je = (st.nev < eb + B) ? st.nev - eb : B;
#pragma unroll
      for (int j = 0; j < B; ++j) {
        if (j >= js && j < je) {
#pragma unroll
          for (int k = 0; k < CPL; ++k) st.acc[k] = mul_add_rn(st.acc[k], vv[j], xc[j][k]);
        }
      }
      if (je >= B) break;
      st.event(a, eb + je);
      js = je;
    }
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      v_c[s] = v_n[s];
      c_n[s] = c_nn[s];
      v_n[s] = v_nn[s];
    }
    load_cv(eb + 3 * B, c_nn, v_nn);
  };

#pragma unroll 1
  for (int eb = st.e; __any_sync(0xffffffffu, st.live); eb += 2 * B) {
    step(eb, x_a, x_b);
    if (!__any_sync(0xffffffffu, st.live)) break;
    step(eb + B, x_b, x_a);
  }
}

// --------------------------------------------------------------------------
// Shared-memory-staged sweep for 4-aligned widths (float4 per lane): the
// dense-row gathers are cp.async (LDGSTS) 16-byte copies into an S-stage ring,
// so the bytes in flight live in shared memory, not registers.  Each lane
// reads back exactly the 16 bytes it copied, so completion is the per-thread
// cp.async.wait_group — no cross-lane barrier.
// --------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(unsigned smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(g));
}
__device__ __forceinline__ void cp_async16_hint(unsigned smem, const void* g, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem), "l"(g), "l"(pol));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(NPEND));
}

template <int LPU, int B, int S, int NT>
constexpr int seq_async_smem_bytes() {
  return NT * S * B * 16 + (NT / LPU) * 2 * SeqWin<LPU>::WIN * 4;
}

template <int LPU, int B, int S, bool WS, int NT>
__global__ void __launch_bounds__(NT, 512 / NT)
seq_kernel_async(const SeqArgs a) {
  constexpr int SLOTS = (B + LPU - 1) / LPU;
  using SW = SeqSweep<LPU, 4, true, WS, NT>;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  float4* ring = reinterpret_cast<float4*>(s_dyn);  // [S][B][NT threads]
  int* s_win = reinterpret_cast<int*>(s_dyn + NT * S * B * 16);
  SW st;
  st.setup_begin(a, s_win);
  const uint64_t pol = evict_first_policy();
  const bool colok = 4 * st.gl < st.cm.nt;
  const unsigned ring_base = (unsigned)__cvta_generic_to_shared(ring) + threadIdx.x * 16;
  const float* xg = a.X + st.col0 + 4 * st.gl;

  auto load_cv = [&](int eb, int (&cr)[SLOTS], float (&vr)[SLOTS]) {
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int o = s * LPU + st.gl;
      const int p = eb + o;
      if (o < B && p < st.hard_end) {
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
  // issue the gathers of batch `eb` into ring stage `stg`
  auto issue = [&](int eb, int stg, const int (&cr)[SLOTS]) {
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int c = gshfl<LPU>(cr[j / LPU], j % LPU);
      if (colok && eb + j < st.hard_end)
        cp_async16(ring_base + (unsigned)((stg * B + j) * NT * 16), xg + (size_t)c * st.N);
    }
    cp_async_commit();
  };

  // Pipeline depths: colIdx/val are loaded R-1 batches ahead of consumption
  // (they stream from HBM), dense rows are gathered S-1 batches ahead.
  constexpr int R = S + 4;
  int cring[R][SLOTS];
  float vring[R][SLOTS];
#pragma unroll
  for (int r = 0; r < R - 1; ++r) load_cv(st.e + r * B, cring[r], vring[r]);
#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(st.e + s * B, s, cring[s]);
  st.setup_end(a);

  int stage = 0;
#pragma unroll 1
  for (int eb = st.e; __any_sync(0xffffffffu, st.live); eb += B) {
    load_cv(eb + (R - 1) * B, cring[R - 1], vring[R - 1]);
    issue(eb + (S - 1) * B, (stage + S - 1) % S, cring[S - 1]);
    cp_async_wait<S - 1>();  // this thread's copies of batch eb have landed
    // products of the whole batch up front (smem latency off the add chain);
    // positions that end up unconsumed are simply never added
    const float4* xs = ring + stage * B * NT + threadIdx.x;
    float pr[B][4];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const float v = gshfl<LPU>(vring[0][j / LPU], j % LPU);
      const float4 x = xs[j * NT];
      pr[j][0] = __fmul_rn(v, x.x);
      pr[j][1] = __fmul_rn(v, x.y);
      pr[j][2] = __fmul_rn(v, x.z);
      pr[j][3] = __fmul_rn(v, x.w);
    }
    // Consume in rounds: every group adds its products up to its next event
    // (predicated adds, no branches), then all groups that reached an event
    // handle it together (converged), until the batch is done.  (With 16
    // groups per warp nearly every position holds some group's event, so the
    // per-position dispatch of seq_async2 measured slower here: uniform N=8
    // 150 -> 222 us.)
    int js = st.live ? 0 : B;
#pragma unroll 1
    while (true) {
      const int je = st.live ? min(B, st.nev - eb) : B;
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const bool m = j >= js && j < je;
#pragma unroll
        for (int k = 0; k < 4; ++k) st.acc[k] = m ? __fadd_rn(st.acc[k], pr[j][k]) : st.acc[k];
      }
      const bool ev = st.live && je < B;
      if (!__any_sync(0xffffffffu, ev)) break;
      if (ev) st.event(a, eb + je);
      js = ev ? je : B;
    }
    stage = (stage + 1 == S) ? 0 : stage + 1;
    // (Refilling the top slot after the rotation instead, so the moves never
    // wait on this iteration's loads, measured 15 % slower on B200.)
#pragma unroll
    for (int r = 0; r + 1 < R; ++r)
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        cring[r][s] = cring[r + 1][s];
        vring[r][s] = vring[r + 1][s];
      }
  }
  cp_async_wait<0>();
}

}  // namespace spmk_dev

namespace spmk_dev {

// --------------------------------------------------------------------------
// seq_async2: the production sequential sweep for 4-aligned column tiles.
// Dense rows are gathered with cp.async (LDGSTS, 16 B per lane) into an
// S-stage shared-memory ring (S a power of two), S-1 batches of B nonzeros
// ahead of consumption; colIdx/val stream through registers S batches ahead
// (lane gl holds entries gl, gl+LPU, ... of a batch, broadcast by shuffles).
// The hot loop carries no per-element predicates: positions outside the
// unit's range read clamped, in-bounds addresses and are never added (values
// before the unit start are zeroed while acc is +0; the unit stops at its
// final event).  Events are located per batch with REDUX.OR over the units'
// next-event bits; the adds run in rounds between event positions, so a
// batch without events costs one predicated pass.
// --------------------------------------------------------------------------
template <int LPU, int B, int S, int NT>
constexpr int seq_async2_smem_bytes() {
  return NT * S * B * 16 + (NT / LPU) * 2 * SeqWin<LPU>::WIN * 4;
}

template <int LPU, int B, int S, bool WS, int NT, bool EXACT>
__global__ void __launch_bounds__(NT, NT <= 64 ? 10 : NT <= 128 ? 5 : 1)
seq_async2_kernel(const SeqArgs a) {
  static_assert((S & (S - 1)) == 0 && S >= 2, "S must be a power of two");
  static_assert(B <= 16, "B");
  constexpr int SLOTS = (B + LPU - 1) / LPU;
  constexpr unsigned FULL = 0xffffffffu;
  using SW = SeqSweep<LPU, 4, true, WS, NT>;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  float4* ring = reinterpret_cast<float4*>(s_dyn);  // [S][B][NT]
  int* s_win = reinterpret_cast<int*>(s_dyn + NT * S * B * 16);
  SW st;
  st.setup_begin(a, s_win);
  const uint64_t pol = evict_first_policy();
  const int last = a.nnz - 1;
  const int xoff = (4 * st.gl < st.cm.nt) ? 4 * st.gl : 0;  // idle lanes re-read column 0
  const char* xg = reinterpret_cast<const char*>(a.X + st.col0 + xoff);
  const unsigned xstride = (unsigned)a.N * 4u;
  const unsigned ring0 = (unsigned)__cvta_generic_to_shared(ring) + threadIdx.x * 16u;
  const int ea = st.e & ~(B - 1);

  auto load_cv = [&](int eb, int (&c)[SLOTS], float (&v)[SLOTS]) {
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int o = s * LPU + st.gl;
      const int p = min(eb + o, last);
      if (SLOTS * LPU == B || o < B) {
        c[s] = ld_stream(a.col + p, pol);
        v[s] = ld_stream(a.val + p, pol);
      } else {
        c[s] = 0;
        v[s] = 0.f;
      }
    }
  };
  auto issue = [&](int stg, const int (&c)[SLOTS]) {
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const unsigned cj = (unsigned)gshfl<LPU>(c[j / LPU], j % LPU);
      cp_async16(ring0 + (unsigned)((stg * B + j) * NT * 16), xg + (size_t)cj * xstride);
    }
    cp_async_commit();
  };

  int cring[S + 1][SLOTS];
  float vring[S + 1][SLOTS];
#pragma unroll
  for (int i = 0; i < S; ++i) load_cv(ea + i * B, cring[i], vring[i]);
#pragma unroll
  for (int s = 0; s < SLOTS; ++s)
    if (ea + s * LPU + st.gl < st.e) vring[0][s] = 0.f;  // other rows before the unit start
  // first gathers before the row window: its loads then overlap them
#pragma unroll
  for (int i = 0; i < S - 1; ++i) issue(i, cring[i]);
  st.setup_end(a);

  int stage = 0;
#pragma unroll 1
  for (int eb = ea; __any_sync(FULL, st.live); eb += B) {
    load_cv(eb + S * B, cring[S], vring[S]);  // refilled before the rotation (a refill after it: +15 %)
    issue((stage + S - 1) & (S - 1), cring[S - 1]);
    cp_async_wait<S - 1>();  // this thread's copies of batch eb have landed
    const float4* xs = ring + stage * B * NT + threadIdx.x;
    // products off the add chain (EXACT: rounded product, kernels.hpp:439-441,
    // as FMUL2 pairs); fast mode keeps (v, x) and fuses them into the add
    float pv[B], px[B][4];
    f32x2 pp[B][2];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const float v = gshfl<LPU>(vring[0][j / LPU], j % LPU);
      const float4 x = xs[j * NT];
      if constexpr (EXACT) {
        pp[j][0] = f2_mul(v, f2_pack(x.x, x.y));
        pp[j][1] = f2_mul(v, f2_pack(x.z, x.w));
      } else {
        px[j][0] = x.x; px[j][1] = x.y; px[j][2] = x.z; px[j][3] = x.w;
      }
      pv[j] = v;
    }
    // positions holding some unit's next event: with B <= LPU lane gl of a
    // unit votes for position gl and the units' bytes are folded, else REDUX
    auto next_bits = [&](int from) -> unsigned {
      const int d = st.nev - eb;
      if constexpr (B <= LPU) {
        unsigned m = __ballot_sync(FULL, st.live && d == st.gl && d >= from);
        if constexpr (LPU < 32) m |= m >> 16;
        if constexpr (LPU < 16) m |= m >> 8;
        return m & ((1u << B) - 1u);
      } else {
        return __reduce_or_sync(FULL, (st.live && d >= from && d < B) ? (1u << d) : 0u);
      }
    };
    unsigned wm = next_bits(0);
    // unrolled positions; a warp-uniform branch into the event handler only
    // where some unit has an event (measured 9 % faster than add rounds
    // between events: cfg2 320 -> 290 us)
#pragma unroll
    for (int j = 0; j < B; ++j) {
      if (wm & (1u << j)) {
        if (st.live && st.nev == eb + j) st.event(a, eb + j);
        wm = next_bits(j + 1);
      }
      if constexpr (EXACT) {
        // acc += product, FFMA2 by one (two roundings in all: FMUL2 above, this)
        f32x2 a01 = f2_add(f2_pack(st.acc[0], st.acc[1]), pp[j][0], a.one2);
        f32x2 a23 = f2_add(f2_pack(st.acc[2], st.acc[3]), pp[j][1], a.one2);
        f2_unpack(a01, st.acc[0], st.acc[1]);
        f2_unpack(a23, st.acc[2], st.acc[3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) st.acc[k] = fmaf(pv[j], px[j][k], st.acc[k]);
      }
    }
    stage = (stage + 1) & (S - 1);
#pragma unroll
    for (int i = 0; i < S; ++i)
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        cring[i][s] = cring[i + 1][s];
        vring[i][s] = vring[i + 1][s];
      }
  }
  cp_async_wait<0>();
}

}  // namespace spmk_dev
