// sell_kernels.cuh — seq-ws (spmm_seq_balanced, kernels.hpp:384-455) as a
// lane-per-job sweep over a segment-sliced layout of A.
//
// Decomposition (exact in the reference's order).  Cut every non-empty row at
// the seq_chunk boundaries (multiples of CH): a piece of a row inside one chunk
// is a *segment*.  The reference computes every segment as one sequential
// chain acc = ((0 + v0 x0) + v1 x1) + ... (kernels.hpp:426-443), writes it
// straight into Y when the row is complete in the chunk, into a boundary slot
// otherwise, and folds the slots into the zero-initialised Y in ascending
// chunk order: Y[r] = ((0 + P_first) + P_next) + ... (:448-453).  A *job* is
//   * a row of one segment: one lane runs it and writes acc into Y (acc is
//     never -0, so the reference's Y = acc and 0 + acc have the same bits);
//   * one segment of a row that crosses a chunk boundary: its chain goes to
//     an H slot (slots of a row are consecutive) and sell_fold_kernel folds
//     the row's slots in ascending order after the sweep.  (Running rows of
//     two segments in one lane with a carry measured 5 % slower: 32 more
//     registers and a per-step boundary test, for a smaller fold);
//   * an empty row (length 0): writes the zeros of Y.
// Any assignment of jobs to lanes gives the same bits, so jobs are sorted by
// length (descending, stable) and cut into slices of 32 (SELL-32): the lanes of
// a warp run jobs of nearly equal length in lockstep (R-MAT s20: 0.5 % of the
// data positions are padding).
//
// Layout in HBM (built once per handle and seq_chunk, sell_*_kernel below):
// one *step* = 64 ints = 256 bytes = the 32 lanes' (column, value) at one
// position.  A slice is a header step followed by L data steps:
//   header: [lane] = output code (Y row, 0x80000000 | H slot, or -1 = none),
//           [32 + lane] = the lane's job length (lane 0: the slice's L)
//   data:   [lane] = column (0 for padding), [32 + lane] = value bits (0 for padding)
// Padding positions (t >= the lane's job length) gather row 0 and are not added.
//
// Sweep (seq_sell_kernel): persistent warps pulling chunks of whole slices
// (heaviest first, sizes shrinking toward the end) from an atomic counter —
// static per-warp ranges left the slowest warp at 1.6x the median (the
// per-step time varies with the rows' L2 hit rates).  Per warp, in shared memory, filled with
// cp.async (LDGSTS, 16 B per lane, one commit group per iteration):
//   * a C-stage ring of steps, C - 1 steps ahead of the consumer;
//   * an S-stage ring of dense rows, S - 1 steps ahead: 8 LDGSTS per step,
//     each copying 4 whole 128-B rows X[col, col0 .. col0 + 31] (lanes 8g..8g+7
//     take rows 8g + i, one 16-B chunk each: every instruction coalesced).
// Lane j reads its own row with 8 LDS.128 in rotated chunk order (chunk
// (c + j) & 7 at step c: the 8 lanes of a quarter warp hit 8 different bank
// groups; accumulator slot c holds columns 4((c + j) & 7) .. +3).  Measured:
// an XOR-swizzled ring (chunk k of row r at k ^ (r & 7), static slots) was 24 %
// slower on B200, a 144-byte padded row pitch cost 12.5 % of the ring's
// in-flight bytes and was slower too.  The exact products / adds run as
// FMUL2 / FFMA2-by-one pairs.  No shuffles and no per-nonzero row events (the
// tile sweep of seq_kernels.cuh spends ~7.5 warp instructions per nonzero on
// them).
#pragma once
#include <type_traits>

#include "common.cuh"

namespace spmk_dev {

// One step of a slice of 32 G jobs (G = 32 / CW jobs per lane, CW = the
// sweep's column width): 32 G columns + 32 G values.
__host__ __device__ constexpr int sell_step_ints(int cw) { return 2 * 32 * (32 / cw); }

// ---------------------------------------------------------------- plan
// Per compact row: jobs (= segments), H slots and fold flag (rows of >= 2
// segments).  seq-rs (spmm_seq_rowsplit, kernels.hpp:339-376) is the same
// sweep with no chunk cuts (CH beyond any row): one job per row, rows of
// >= lmax nonzeros left to the hub kernels.
__global__ void sell_count_kernel(const int* __restrict__ crp, int mne, long long CH, int lmax,
                                  int* __restrict__ njob, int* __restrict__ nslot, int* __restrict__ nmulti) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < mne; i += gridDim.x * blockDim.x) {
    const long long s = crp[i], e = crp[i + 1];
    if (e - s >= lmax) {  // seq-rs hub row: computed by the hub kernel
      njob[i] = nslot[i] = nmulti[i] = 0;
      continue;
    }
    const int nseg = (int)((e - 1) / CH - s / CH + 1);
    const bool split = nseg > 1;
    njob[i] = split ? nseg : 1;
    nslot[i] = split ? nseg : 0;
    nmulti[i] = split ? 1 : 0;
  }
}

// Jobs of every compact row (offsets from exclusive scans of the counts) and
// the fold list {row, first slot, slots, 0} of the split rows.
__global__ void sell_jobs_kernel(const int* __restrict__ crp, const int* __restrict__ rid, int mne, long long CH,
                                 int lmax, const int* __restrict__ joff, const int* __restrict__ soff,
                                 const int* __restrict__ moff, int* __restrict__ jstart, int* __restrict__ jlen,
                                 int* __restrict__ jout, int4* __restrict__ fold) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < mne; i += gridDim.x * blockDim.x) {
    const long long s = crp[i], e = crp[i + 1];
    if (e - s >= lmax) continue;
    const long long q0 = s / CH;
    const long long nseg = (e - 1) / CH - q0 + 1;
    const int j = joff[i];
    if (nseg == 1) {
      jstart[j] = (int)s;
      jlen[j] = (int)(e - s);
      jout[j] = rid[i];
    } else {
      const int s0 = soff[i];
      for (long long k = 0; k < nseg; ++k) {
        const long long a = k == 0 ? s : (q0 + k) * CH;
        const long long b = k == nseg - 1 ? e : (q0 + k + 1) * CH;
        jstart[j + k] = (int)a;
        jlen[j + k] = (int)(b - a);
        jout[j + k] = (int)(0x80000000u | (unsigned)(s0 + k));
      }
      fold[moff[i]] = make_int4(rid[i], s0, (int)nseg, 0);
    }
  }
}

// Empty rows: jobs of length 0 (their slice writes the zeros).
__global__ void sell_empty_jobs_kernel(const int* __restrict__ erow, int nempty, int j0, int* __restrict__ jstart,
                                       int* __restrict__ jlen, int* __restrict__ jout) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nempty; i += gridDim.x * blockDim.x) {
    jstart[j0 + i] = 0;
    jlen[j0 + i] = 0;
    jout[j0 + i] = erow[i];
  }
}

// Slice lengths (jobs sorted by length, descending: the slice's first job is
// its longest) -> steps (1 + L) and balancing cost (steps + 1: the header and
// the epilogue cost about one more step).
__global__ void sell_slice_kernel(const int* __restrict__ slen_sorted, int nsl, int jps,
                                  long long* __restrict__ steps, long long* __restrict__ cost) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsl; s += gridDim.x * blockDim.x) {
    const int L = slen_sorted[(long long)jps * s];
    steps[s] = 1 + L;
    cost[s] = 2 + L;
  }
}

// One warp per slice (jps = 32 G jobs: position g * 32 + lane): header + data
// steps of 2 jps ints.
__global__ void sell_fill_kernel(const int* __restrict__ sidx, const int* __restrict__ slen, int J, int nsl, int jps,
                                 int rpi,
                                 const long long* __restrict__ step_ex, const int* __restrict__ jstart,
                                 const int* __restrict__ jout,
                                 const int* __restrict__ col, const float* __restrict__ val, int* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (long long s = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; s < nsl;
       s += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int L = slen[(long long)jps * s];
    int* p = out + step_ex[s] * 2 * jps;
    // column of position pos at its producer index (see seq_sell_kernel: at
    // CW < 32 an LDGSTS copies rpi consecutive ring rows, lane group g needs
    // rows g, rpi + g, ...: stored contiguously)
    auto cidx = [&](int pos) { return rpi ? (pos % rpi) * 8 + pos / rpi : pos; };
    for (int pos = lane; pos < jps; pos += 32) {
      const long long j = (long long)jps * s + pos;
      const bool ok = j < J;
      const int idx = ok ? sidx[j] : 0;
      const int len = ok ? slen[j] : 0;
      const int st = ok ? jstart[idx] : 0;
      p[pos] = ok ? jout[idx] : -1;
      p[jps + pos] = len;
      for (int t = 0; t < L; ++t) {
        int* q = p + (long long)(t + 1) * 2 * jps;
        const bool in = t < len;
        q[cidx(pos)] = in ? col[st + t] : 0;
        q[jps + pos] = in ? __float_as_int(val[st + t]) : 0;
      }
    }
  }
}

// ---------------------------------------------------------------- sweep
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// predicated forms: a predicate instead of a branch around the copy
__device__ __forceinline__ void cp16_if(unsigned dst, const void* src, bool on) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.cg.shared.global [%0], [%1], 16;\n}" ::"r"(dst),
               "l"(src), "r"((int)on)
               : "memory");
}
__device__ __forceinline__ void cp8_if(unsigned dst, const void* src, bool on) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.ca.shared.global [%0], [%1], 8;\n}" ::"r"(dst),
               "l"(src), "r"((int)on)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// U = 0 .. N-1 in order as compile-time constants, stopping at the first false
template <int U, int N>
struct SellUnroll {
  template <class F, class P>
  __device__ __forceinline__ static bool run(F& f, P p) {
    return f(std::integral_constant<int, U>{}, p) && SellUnroll<U + 1, N>::run(f, p);
  }
};
template <int N>
struct SellUnroll<N, N> {
  template <class F, class P>
  __device__ __forceinline__ static bool run(F&, P) {
    return true;
  }
};
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// (a0, a1) += v * (x0, x1), each element rounded twice like the reference's
// `acc += v * x` (kernels.hpp:439-441): FMUL2, then FFMA2 by `one` (opaque to
// ptxas, see f2_add) so the product is not fused into the add.  One asm block
// over scalar operands: ptxas keeps the accumulators in place (64-bit asm
// operands cost ~16 register moves per step).
__device__ __forceinline__ void f2_mac(float& a0, float& a1, float v, float x0, float x1, f32x2 one) {
  asm("{\n .reg .b64 p, q, r;\n mov.b64 q, {%2, %2};\n mov.b64 r, {%3, %4};\n mul.rn.f32x2 p, q, r;\n"
      " mov.b64 r, {%0, %1};\n fma.rn.f32x2 r, p, %5, r;\n mov.b64 {%0, %1}, r;\n}"
      : "+f"(a0), "+f"(a1)
      : "f"(v), "f"(x0), "f"(x1), "l"(one));
}

struct SellArgs {
  const int* __restrict__ steps;  // T steps x 64 ints
  const int* __restrict__ cstep;  // nchunks + 1 chunk starts (step indices; whole slices, heaviest first)
  int* __restrict__ sched;        // per column tile {claim counter, warps done}, zero between calls
  int nchunks;
  const float* __restrict__ X;    // K x N
  float* __restrict__ Y;          // M x N
  float* __restrict__ H;          // partial slots x N
  int N;
  int K;                          // rows of X (0: no X row 0 to test)
  int claim_first;                // 1: first chunks claimed per CTA (a concurrent side-stream kernel)
  f32x2 one2;                     // {1, 1}, opaque to ptxas (see f2_add)
  unsigned long long* trace;      // dev: per-warp {start, end, steps, slices} (%globaltimer), or null
};

constexpr int kSellStage = 4096;  // one step's 32 G dense rows of CW floats in the ring
template <int CW, int S, int C>
__host__ __device__ constexpr int sell_warp_bytes() {
  // row ring + step ring + the output codes of the slice being stored
  return S * kSellStage + C * sell_step_ints(CW) * 4 + sell_step_ints(CW) * 2;
}
template <int CW, int S, int C, int WPC>
__host__ __device__ constexpr int sell_smem_bytes() {
  return WPC * sell_warp_bytes<CW, S, C>();
}

template <int CW, int S, int C, int WPC, int MINB>
__global__ void __launch_bounds__(WPC * 32, MINB)
seq_sell_kernel(const SellArgs a) {
  static_assert(CW == 8 || CW == 16 || CW == 32, "column width");
  static_assert(S >= 2 && C == 2 * S, "ring depths (the step ring is two halves of S slots)");
  constexpr int G = 32 / CW;           // jobs per lane
  constexpr int JPS = 32 * G;          // jobs per slice = dense rows per step
  constexpr int SI = 2 * JPS;          // ints per step
  constexpr int RB = 4 * CW;           // bytes per dense row
  constexpr int CPR = CW / 4;          // 16-byte chunks per row
  constexpr int LPR = CW / 4;          // LDGSTS lanes per row
  extern __shared__ __align__(128) unsigned char s_sell[];
  // the fold pass (a programmatic dependent) may be scheduled as CTAs drain;
  // it still waits for this grid's completion before reading H
  asm volatile("griddepcontrol.launch_dependents;");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * WPC + warp;
  const int W = gridDim.x * WPC;
  int* sched = a.sched + 2 * blockIdx.y;  // {chunks claimed, warps done}
  // First chunks: warp w takes chunk w (the W heaviest, no atomics) unless a
  // side-stream kernel competes for the SMs (seq-rs hub rows): then one claim
  // of WPC chunks per CTA, so a CTA that becomes resident late starts on
  // later, lighter chunks instead of a statically assigned heavy one
  // (measured: static 187 us at cfg2; claimed 200 us, but seq-rs with hubs
  // 390 -> 553 us in some runs when static).
  __shared__ int s_first;
  int first = w;
  if (a.claim_first) {
    if (threadIdx.x == 0) s_first = atomicAdd(sched, WPC);
    __syncthreads();
    first = s_first + warp;
  }
  unsigned long long t_start = 0;
  int nsteps = 0, nslices = 0;
  if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

  unsigned char* wb = s_sell + warp * sell_warp_bytes<CW, S, C>();
  const int* cr = reinterpret_cast<const int*>(wb + S * kSellStage);  // [C][SI]
  const unsigned xr0 = smem_addr(wb);
  const unsigned cr0 = xr0 + S * kSellStage;
  const int col0 = blockIdx.y * CW;
  const float x00 = a.K > 0 ? __ldg(a.X + col0 + lane % CW) : 0.f;  // X row 0 (padding rows), tested below
  const int* steps = a.steps;
  // LDGSTS lanes: group q = lane / LPR copies chunk lane % LPR of 8 rows, one
  // per instruction: rows 8 q + i at CW = 32 (4 rows 1 KB apart: 4 wavefronts,
  // the minimum), rows i RPI + q below (the instruction's RPI rows contiguous;
  // 8 q + i there put 16 / 8 rows on the same banks: 16- / 8-way conflicts)
  const int q = lane / LPR, ch = lane % LPR;
  // 32-bit row offsets in 16-byte units (the plan checks K * N / 4 < 2^32)
  const float4* xg = reinterpret_cast<const float4*>(a.X + col0);
  const unsigned n16 = (unsigned)a.N / 4;
  constexpr int RPI = 512 / RB;                       // rows per LDGSTS instruction
  constexpr int ISTRIDE = CW == 32 ? RB : 512;         // ring bytes between a lane's rows
  const unsigned xdst0 = xr0 + (unsigned)((CW == 32 ? q * 8 * RB : q * RB) + ch * 16);

  // Work: chunks of whole slices (plan: a.cstep), heaviest first.  A warp
  // claims the next chunk (atomic counter) as soon as it enters one; the claim and the chunk bounds load are consumed only
  // when the step ring reaches the chunk end (every chunk but the last has
  // >= C steps, so the rings never run more than one chunk ahead).
  int a0 = 0, alen = 0;                   // chunk the consumer is in (real start, steps)
  int b0 = 0, blen = 0, bknown = 1;       // next chunk (bknown = 0: claim in flight)
  int pc0 = 0, pc1 = 0;                   // lane 0: the claim's bounds
  auto claim = [&]() {
    if (lane == 0) {
      const int c = atomicAdd(sched, 1) + (a.claim_first ? 0 : W);
      pc0 = c < a.nchunks ? a.cstep[c] : 0;
      pc1 = c < a.nchunks ? a.cstep[c + 1] : 0;
    }
    bknown = 0;
  };
  auto resolve = [&]() {
    if (!bknown) {
      b0 = __shfl_sync(0xffffffffu, pc0, 0);
      blen = __shfl_sync(0xffffffffu, pc1, 0) - b0;
      bknown = 1;
    }
  };
  // real step at virtual position v of the consumer's chunk (-1: none)
  auto map = [&](int v) -> int {
    if (v < alen) return a0 + v;
    resolve();
    return v - alen < blen ? b0 + (v - alen) : -1;
  };
  if (first < a.nchunks) {
    a0 = a.cstep[first];
    alen = a.cstep[first + 1] - a0;
    claim();
  } else {
    blen = 0;
  }

  // step g into step-ring slot cs: every lane copies SI / 32 ints (8-byte
  // copies at CW = 32, 16-byte ones below: no lane predicate)
  auto fetch_step = [&](int g, int cs) {
    if (g < 0) return;
    if constexpr (SI / 32 == 2) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(cr0 + (cs * SI + lane * 2) * 4),
                   "l"(steps + (size_t)g * SI + lane * 2)
                   : "memory");
    } else {
#pragma unroll
      for (int o = 0; o < SI / 128; ++o)
        cp16(cr0 + (cs * SI + (o * 32 + lane) * 4) * 4, steps + (size_t)g * SI + (o * 32 + lane) * 4);
    }
  };
  int prem = 0;  // producer: data steps left in the current slice
  // dense rows of step p (step slot pcs) into row-ring slot pxs (prologue)
  auto produce = [&](int p, int pcs, int pxs) {
    if (p < 0) return;
    if (prem == 0) {  // header: no rows
      prem = cr[pcs * SI + JPS];
      return;
    }
    --prem;
    const int4 c0 = reinterpret_cast<const int4*>(cr + pcs * SI)[2 * q];
    const int4 c1 = reinterpret_cast<const int4*>(cr + pcs * SI)[2 * q + 1];
    const int cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const unsigned d = xdst0 + pxs * kSellStage;
#pragma unroll
    for (int i = 0; i < 8; ++i) cp16(d + i * ISTRIDE, xg + ((unsigned)cc[i] * n16 + ch));
  };

  // prologue: steps 0 .. C-2 (one group each), then rows of steps 0 .. S-2
#pragma unroll 1
  for (int i = 0; i < C - 1; ++i) {
    fetch_step(map(i), i);
    cp_commit();
  }
#pragma unroll 1
  for (int i = 0; i < S - 1; ++i) {
    cp_wait<C - 2>();
    __syncwarp();
    produce(map(i), i, i);
    cp_commit();
  }

  // This lane's jobs sit at positions g * 32 + lane of a slice; their rows are
  // read in rotated chunk order (chunk (c + rot) % CPR at slot c) so the 8
  // lanes of a quarter warp hit 8 different bank groups.  Offsets from s_sell
  // (this warp's ring included): every row read is one register + a constant.
  constexpr int ROT_SHIFT = CW == 32 ? 0 : (CW == 16 ? 1 : 2);
  const int rot = (lane >> ROT_SHIFT) & (CPR - 1);
  const unsigned wofs = (unsigned)(warp * sell_warp_bytes<CW, S, C>());
  unsigned roff[G][CPR];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int c = 0; c < CPR; ++c)
      roff[g][c] = wofs + (unsigned)((g * 32 + lane) * RB + (((c + rot) & (CPR - 1)) * 16));
  float acc[G][CW];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int c = 0; c < CW; ++c) acc[g][c] = 0.f;
  int out[G], len[G];
#pragma unroll
  for (int g = 0; g < G; ++g) out[g] = -1, len[g] = 0;
  int crem = 0, t = 0;  // steps left in the slice, position in it
  const size_t ystride = (size_t)a.N;
  // Epilogue of a slice: its 32 G rows go through a free ring stage (the one
  // of the header step, whose position gathers no rows) so the stores are
  // coalesced like the gathers: each STG.128 writes 4 G whole rows (storing
  // from registers, 32 rows of 16 B per instruction, cost ~35 us at cfg2).
  int* ocode = reinterpret_cast<int*>(wb + S * kSellStage + C * SI * 4);  // [JPS]
  auto epilogue = [&](int slot) {
    unsigned char* stg = s_sell + slot * kSellStage;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      ocode[g * 32 + lane] = out[g];
#pragma unroll
      for (int c = 0; c < CPR; ++c) {
        const float* o = &acc[g][4 * c];
        *reinterpret_cast<float4*>(stg + roff[g][c]) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = CW == 32 ? 8 * q + i : i * RPI + q;  // this lane's row (producer mapping)
      const int oc = ocode[r];
      if (oc == -1) continue;
      const float4 v = *reinterpret_cast<const float4*>(stg + wofs + r * RB + ch * 16);
      if (oc >= 0) {
        st_y4(a.Y + (size_t)oc * ystride + col0 + ch * 4, v.x, v.y, v.z, v.w);
      } else {
        *reinterpret_cast<float4*>(a.H + (size_t)(oc & 0x7fffffff) * ystride + col0 + ch * 4) = v;
      }
    }
    __syncwarp();
  };

  // Padding positions gather X row 0 and multiply it by 0: when this tile of
  // row 0 is finite that adds +-0 to an accumulator that is never -0 (same
  // bits), so the sweep runs without the per-job length test.
  const bool row0_finite = __all_sync(0xffffffffu, isfinite(x00));

  // Main loop, in groups of S iterations (C = 2 S).  Iteration u of a group
  // consumes position k from step slot (half h, u) and row stage u, produces
  // the rows of position k + S - 1 into stage (u - 1) % S and fetches position
  // k + C - 1 into the step slot iteration u - 1 consumed; h flips per group.
  // Every ring address is a register plus a constant, and the only per-step
  // branch is the consumer's header test: the producer's header / end cases
  // are predicates, the next chunk is resolved once per group (work chunks
  // but the last are >= S + C - 1 steps, kSellChunkMin).
  constexpr unsigned HALF = S * SI * 4;
  const unsigned cro = wofs + S * kSellStage;  // step ring, from s_sell
  unsigned hoff = 0;                           // byte offset of half h
  int k = 0;
  auto step = [&](auto uc, auto chk) -> bool {
    constexpr int u = decltype(uc)::value;
    constexpr bool CHECK = decltype(chk)::value;
    // one wait per iteration: the rows of position k (issued S - 1 iterations
    // ago) and the step of position k + S - 1 (fetched C - S iterations ago)
    cp_wait<S - 2>();
    __syncwarp();
    const unsigned oth = HALF - hoff;
    // producer, part 1: position k + S - 1 (slot u = 0: half h, S - 1; else the other half, u - 1)
    const int* ps = reinterpret_cast<const int*>(s_sell + cro + (u == 0 ? hoff + (S - 1) * SI * 4 : oth + (u - 1) * SI * 4));
    const bool pv = k + (S - 1) < alen + blen;
    const int hv = ps[JPS];
    const int4 c0 = reinterpret_cast<const int4*>(ps)[2 * q];
    const int4 c1 = reinterpret_cast<const int4*>(ps)[2 * q + 1];
    const bool issue = pv && prem != 0;
    prem = pv ? (prem == 0 ? hv : prem - 1) : prem;
    const int fv = k + (C - 1);
    const bool fok = fv < alen + blen;
    const int f = (fv < alen ? a0 : b0 - alen) + fv;  // real step (fok)
    // producer, part 2: the rows of position k + S - 1 into row stage (u - 1) % S
    auto gather = [&]() {
      const int cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      const unsigned d = xdst0 + ((u + S - 1) % S) * kSellStage;
#pragma unroll
      for (int i = 0; i < 8; ++i) cp16_if(d + i * ISTRIDE, xg + ((unsigned)cc[i] * n16 + ch), issue);
    };
    // consumer: position k
    const int* cw = reinterpret_cast<const int*>(s_sell + cro + hoff + u * SI * 4);
    if (crem == 0) {  // header: finish the previous slice, start the next
      if (k == alen) {  // the consumer leaves its chunk
        resolve();
        if (blen <= 0) {
          nsteps += u;
          return false;
        }
        a0 = b0;
        alen = blen;
        k = 0;
        claim();
        if (alen < S + C - 1) resolve();  // the last chunk may be short
      }
      ++nslices;
      epilogue(u);  // this position's row stage is free (a header gathers nothing)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        out[g] = cw[g * 32 + lane];
        len[g] = cw[JPS + g * 32 + lane];
#pragma unroll
        for (int c = 0; c < CW; ++c) acc[g][c] = 0.f;
      }
      crem = cw[JPS];  // position 0 holds the slice's longest job
      t = 0;
      gather();
    } else {
      // the row reads first, the gathers while they are in flight, then the math
      const unsigned char* xrow = s_sell + u * kSellStage;
      float4 xs[G][CPR];
      float vs[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        vs[g] = __int_as_float(cw[JPS + g * 32 + lane]);
#pragma unroll
        for (int c = 0; c < CPR; ++c) xs[g][c] = *reinterpret_cast<const float4*>(xrow + roff[g][c]);
      }
      gather();
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (!CHECK || t < len[g]) {  // padding adds nothing (also when X row 0 holds inf / NaN)
#pragma unroll
          for (int c = 0; c < CPR; ++c) {
            f2_mac(acc[g][4 * c], acc[g][4 * c + 1], vs[g], xs[g][c].x, xs[g][c].y, a.one2);
            f2_mac(acc[g][4 * c + 2], acc[g][4 * c + 3], vs[g], xs[g][c].z, xs[g][c].w, a.one2);
          }
        }
      }
      ++t;
      --crem;
    }
    // and the step of position k + C - 1 (slot u = 0: the other half, S - 1; else half h, u - 1)
    {
      const unsigned fs = smem_addr(s_sell) + cro + (u == 0 ? oth + (S - 1) * SI * 4 : hoff + (u - 1) * SI * 4);
      const int* src = steps + (size_t)(unsigned)f * SI;  // not read unless fok
      if constexpr (SI / 32 == 2) {
        cp8_if(fs + lane * 8, src + lane * 2, fok);
      } else {
#pragma unroll
        for (int o = 0; o < SI / 128; ++o) cp16_if(fs + (o * 32 + lane) * 16, src + (o * 32 + lane) * 4, fok);
      }
    }
    cp_commit();
    ++k;
    return true;
  };
  auto sweep = [&](auto chk) {
#pragma unroll 1
    for (;;) {
      if (!bknown && k + (S + C - 2) >= alen) resolve();  // positions up to k + S + C - 2 this group
      if (!SellUnroll<0, S>::run(step, chk)) return;
      nsteps += S;
      hoff = HALF - hoff;
    }
  };
  if (row0_finite)
    sweep(std::false_type{});
  else
    sweep(std::true_type{});
  cp_wait<0>();
  __syncwarp();
  epilogue(0);
  if (lane == 0) {
    // the last warp out resets the counters for the next call (every claim of
    // this warp has returned its value already: no fence needed before the count)
    if (atomicAdd(sched + 1, 1) == W - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
    if (a.trace && blockIdx.y == 0) {
      unsigned long long t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      a.trace[4 * w] = t_start;
      a.trace[4 * w + 1] = t_end;
      a.trace[4 * w + 2] = (unsigned long long)nsteps;
      a.trace[4 * w + 3] = (unsigned long long)nslices;
    }
  }
}

// Y[row] = ((0 + H[s0]) + H[s0 + 1]) + ... (kernels.hpp:448-453: ascending
// chunk order) for the rows that cross a chunk boundary, per 32-column tile.
// The fold list is sorted by slot count, longest first:
//   * rows of > kFoldWarpMax slots (few; chains up to nnz / seq_chunk long):
//     one CTA per (row, tile) stages up to kFoldStage slots in shared memory
//     with all its threads (every load in flight at once), then warp 0 adds
//     them in order, lane = column;
//   * the others (most rows: 2 slots): several (row, tile) items per warp by
//     slot-count tier (below), all their loads in flight, lane = column.
// Launched as a programmatic dependent of the sweep: the descriptor load
// overlaps the sweep's tail, griddepcontrol.wait orders the H reads after it.
constexpr int kFoldWarpMax = 8;
constexpr int kFoldStage = 96;    // slots staged per round of a long row (12.7 KB)
constexpr int kFoldThreads = 64;  // 2 warps per block (measured: 128 the same, 32 slower)
// Short rows (<= 8 slots) in three tiers of the slot-sorted fold list, each
// warp taking R consecutive (row, tile) items with every load in flight:
// 5..8 slots R = 4, 3..4 slots R = 4 (4 loads each), 2 slots R = 8 (most
// split rows cross one boundary: 2 loads per item, none predicated off).
struct FoldTiers {
  int n4, n2;        // first fold row with <= 4 / <= 2 slots
  int w8, w4;        // work units of the 5..8 and 3..4 tiers
};
// H is written by the sweep this kernel overlaps (programmatic dependent
// launch): no __restrict__ on it, or its loads count as invariant and may be
// hoisted above griddepcontrol.wait (seen: stale slots on a plan's first call).
template <int R, int Z>
__device__ __forceinline__ void fold_items(const int4* __restrict__ fold, int it0, int it_end, int tiles,
                                           const float* H, float* __restrict__ Y, int N, int lane) {
  int4 d[R];
  int c[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int it = it0 + r;
    const int f = tiles == 1 ? it : it / tiles;
    c[r] = (it - f * tiles) * 32 + lane;
    d[r] = it < it_end && c[r] < N ? fold[f] : make_int4(0, 0, 0, 0);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float v[R][Z];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const float* h = H + (size_t)d[r].y * N + c[r];
#pragma unroll
    for (int u = 0; u < Z; ++u) v[r][u] = u < d[r].z ? h[(size_t)u * N] : 0.f;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (d[r].z == 0) continue;
    float y = 0.f;
#pragma unroll
    for (int u = 0; u < Z; ++u)
      if (u < d[r].z) y = __fadd_rn(y, v[r][u]);
    st_y(Y + (size_t)d[r].x * N + c[r], y);
  }
}
__global__ void __launch_bounds__(kFoldThreads, 16)
sell_fold_kernel(const int4* __restrict__ fold, int nfold, int nbig, FoldTiers ft, const float* H,
                 float* __restrict__ Y, int N) {
  constexpr int WPB = kFoldThreads / 32;
  __shared__ float buf[kFoldStage][33];
  const int tiles = N >= 32 ? N >> 5 : 1;  // N < 32 (the 8 / 16-column sweeps): lanes >= N idle
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nbig_items = nbig * tiles;
  if ((int)blockIdx.x < nbig_items) {
    const int f = (int)blockIdx.x / tiles;
    const int c0 = ((int)blockIdx.x - f * tiles) * 32;
    const int4 d = fold[f];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const bool colok = c0 + lane < N;
    const float* h = H + (size_t)d.y * N + (colok ? c0 + lane : 0);
    float y = 0.f;
    for (int k0 = 0; k0 < d.z; k0 += kFoldStage) {
      const int n = min(kFoldStage, d.z - k0);
      // every slot of the round in flight at once, straight into shared memory
      // (4-byte cp.async: no register staging, so a round covers kFoldStage
      // slots; cfg2: the rows of > 96 slots take two)
      for (int r = warp; r < n; r += WPB)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(&buf[r][lane])),
                     "l"(h + (size_t)(k0 + r) * N)
                     : "memory");
      cp_commit();
      cp_wait<0>();
      __syncthreads();
      if (warp == 0) {
        int r = 0;
        for (; r + 8 <= n; r += 8) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = buf[r + e][lane];
#pragma unroll
          for (int e = 0; e < 8; ++e) y = __fadd_rn(y, v[e]);
        }
        for (; r < n; ++r) y = __fadd_rn(y, buf[r][lane]);
      }
      __syncthreads();
    }
    if (warp == 0 && colok) st_y(Y + (size_t)d.x * N + c0 + lane, y);
    return;
  }
  // one short-row work unit per warp (a grid-stride loop over fewer warps
  // measured slower: 13-15 vs 9-11 us at cfg2)
  const int gw = ((int)blockIdx.x - nbig_items) * WPB + warp;
  if (gw < ft.w8)
    fold_items<4, 8>(fold, nbig_items + gw * 4, ft.n4 * tiles, tiles, H, Y, N, lane);
  else if (gw < ft.w8 + ft.w4)
    fold_items<4, 4>(fold, ft.n4 * tiles + (gw - ft.w8) * 4, ft.n2 * tiles, tiles, H, Y, N, lane);
  else
    fold_items<8, 2>(fold, ft.n2 * tiles + (gw - ft.w8 - ft.w4) * 8, nfold * tiles, tiles, H, Y, N, lane);
}

}  // namespace spmk_dev
