// Hub rows of the row-split variants (par-rs, seq-rs).
//
// The row-split variants give one worker to one row (kernels.hpp:157-224 and
// :339-376): a row's sum is a single ordered chain (seq-rs) or W per-lane
// chains plus a fixed tree (par-rs).  On power-law matrices one group then
// serialises a 40K-nonzero row behind ~2 dependent memory round trips per
// step.  Rows with >= L nonzeros ("hubs", plan-time list) are skipped by the
// main row-split kernels and computed here instead, one CTA per (hub row,
// column tile), in exactly the reference's order:
//
//   * seq-rs: products v*x (rounded) are formed in parallel by 7 producer
//     warps into a double-buffered shared-memory chunk while warp 0 folds
//     the previous chunk in position order (acc += p; one chain per column).
//     The chain is then the only serial part: ~4 cycles per nonzero.
//   * par-rs: one thread per (lane chain l, column): chain l sums positions
//     s + l + j*W in j order with 16 steps of gathers in flight; the tree
//     acc[l] = acc[2l+1] + acc[2l] (kernels.hpp:193-199) runs per column
//     from shared memory.
#pragma once

#include "common.cuh"

namespace spmk_dev {

constexpr int kHubThreads = 256;
constexpr int kHubProducers = 7;                // seq-rs: warps 1..7 form products
constexpr int kHubChunk = kHubProducers * 32;   // positions per shared-memory chunk
template <int CW>
constexpr int hub_smem_bytes() { return 2 * kHubChunk * CW * 4; }  // double buffer (57,344 B at CW = 32)

struct HubArgs {
  const int* __restrict__ hubs;  // compact rows, longest first
  const int* __restrict__ crp;
  const int* __restrict__ rid;
  const int* __restrict__ col;
  const float* __restrict__ val;
  const float* __restrict__ X;
  float* __restrict__ Y;
  int N;
};

// seq-rs (kernels.hpp:339-376): acc = 0; for e in row: acc += val[e]*x[col[e]].
// CW columns per CTA (power of two <= 32); a producer lane (sg, cl) gathers
// positions sg + (32/CW)*t of its warp's 32, so small N wastes no lanes.
// Producers run two chunks ahead in registers (colIdx/val) and one chunk
// ahead in flight (the gathers), so each barrier interval costs about one
// fold of kHubChunk dependent adds.
template <int CW>
__global__ void __launch_bounds__(kHubThreads, 1) seq_rs_hub_kernel(const HubArgs a) {
  constexpr int SG = 32 / CW;
  extern __shared__ float hub_buf[];  // [2][kHubChunk][CW]
  const int r = a.hubs[blockIdx.x];
  const int s = a.crp[r], f = a.crp[r + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = lane / CW, cl = lane % CW;
  const int c = blockIdx.y * CW + cl;
  const bool cok = c < a.N;
  const int cx = min(c, a.N - 1);  // gathers are unpredicated (a dead slot is never folded)
  const unsigned xs = (unsigned)a.N;
  const int nch = (f - s + kHubChunk - 1) / kHubChunk;
  const int pw = warp - 1;
  auto ldcv = [&](int it, int& cc, float& vv) {
    const int p = s + it * kHubChunk + pw * 32 + lane;
    cc = p < f ? a.col[p] : 0;
    vv = p < f ? a.val[p] : 0.f;
  };
  // Plain loads into registers consumed one barrier interval later: no
  // select on the loaded value, so all CW gathers stay in flight.
  auto gather = [&](int cc, float (&xv)[CW]) {
#pragma unroll
    for (int t = 0; t < CW; ++t) {
      const int ci = __shfl_sync(0xffffffffu, cc, sg + SG * t);
      xv[t] = ld_x(a.X + (size_t)(unsigned)ci * xs + cx);
    }
  };
  int cc0 = 0, cc1 = 0;
  float vv0 = 0.f, vv1 = 0.f;
  float xv[CW];
  if (warp > 0) {
    ldcv(0, cc0, vv0);
    ldcv(1, cc1, vv1);
    gather(cc0, xv);
  }
  float acc = 0.f;
  for (int it = 0; it <= nch; ++it) {
    if (warp > 0) {
      if (it < nch) {
        float* b = hub_buf + (it & 1) * kHubChunk * CW + pw * 32 * CW;
#pragma unroll
        for (int t = 0; t < CW; ++t) {
          const int i = sg + SG * t;
          b[i * CW + cl] = __fmul_rn(__shfl_sync(0xffffffffu, vv0, i), xv[t]);
        }
        cc0 = cc1;
        vv0 = vv1;
        if (it + 1 < nch) gather(cc0, xv);
        ldcv(it + 2, cc1, vv1);
      }
    } else if (it > 0 && lane < CW) {
      const float* b = hub_buf + ((it - 1) & 1) * kHubChunk * CW + cl;
      const int cnt = min(kHubChunk, f - s - (it - 1) * kHubChunk);
      if (cnt == kHubChunk && CW >= 16) {
#pragma unroll 16
        for (int i = 0; i < kHubChunk; ++i) acc = __fadd_rn(acc, b[i * CW]);
      } else if (cnt == kHubChunk) {
        // 32 products per batch, the next batch's shared-memory loads issued
        // before this batch's adds: the add chain never waits on LDS latency
        float nx[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) nx[k] = b[k * CW];
#pragma unroll 1
        for (int bb = 0; bb < kHubProducers; ++bb) {
          float cur[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) cur[k] = nx[k];
          if (bb + 1 < kHubProducers) {
#pragma unroll
            for (int k = 0; k < 32; ++k) nx[k] = b[((bb + 1) * 32 + k) * CW];
          }
#pragma unroll
          for (int k = 0; k < 32; ++k) acc = __fadd_rn(acc, cur[k]);
        }
      } else {
#pragma unroll 4
        for (int i = 0; i < cnt; ++i) acc = __fadd_rn(acc, b[i * CW]);
      }
    }
    __syncthreads();
  }
  if (warp == 0 && lane < CW && cok) a.Y[(size_t)(unsigned)a.rid[r] * xs + c] = acc;
}

// par-rs (kernels.hpp:157-224) with W lanes: thread (l, cl) of a W x CW CTA
// owns lane chain l (positions s + l + j*W, in j order) of column cl; U steps
// of colIdx/val are loaded one batch ahead so a batch costs one gather round
// trip.  Then the tree acc[l] = acc[2l+1] + acc[2l] (kernels.hpp:193-199).
__global__ void __launch_bounds__(kHubThreads) par_rs_hub_kernel(const HubArgs a, int W, int CW) {
  constexpr int U = 16;
  __shared__ float sacc[kHubThreads];
  const int t = threadIdx.x;
  const int l = t / CW, cl = t % CW;
  const int r = a.hubs[blockIdx.x];
  const int s = a.crp[r], f = a.crp[r + 1];
  const int c = blockIdx.y * CW + cl;
  const bool cok = c < a.N;
  const int cx = min(c, a.N - 1);
  const unsigned xs = (unsigned)a.N;
  int cc[U];
  float vv[U];
  auto load = [&](int p) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = p + u * W;
      cc[u] = q < f ? a.col[q] : 0;
      vv[u] = q < f ? a.val[q] : 0.f;
    }
  };
  float acc = 0.f;
  int p = s + l;
  load(p);
  for (; p < f; p += U * W) {
    float xv[U], vc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vc[u] = vv[u];
      xv[u] = ld_x(a.X + (size_t)(unsigned)cc[u] * xs + cx);  // unpredicated: dead steps are not added
    }
    load(p + U * W);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (p + u * W < f) acc = mul_add_rn(acc, vc[u], xv[u]);
  }
  sacc[t] = acc;
  __syncthreads();
  if (l == 0) {
#pragma unroll 1
    for (int len = W; len > 1; len >>= 1)
#pragma unroll 1
      for (int i = 0; i < len / 2; ++i)
        sacc[i * CW + cl] = __fadd_rn(sacc[(2 * i + 1) * CW + cl], sacc[2 * i * CW + cl]);
    if (cok) a.Y[(size_t)(unsigned)a.rid[r] * xs + c] = sacc[cl];
  }
}


// ---------------------------------------------------------------- par-rs,
// two passes for the longest rows.  A 373K-nonzero hub (cfg5's 8-way slice 0)
// gives each of the W lane chains 11.7K dependent steps; gathering inside the
// chain leaves ~16 gathers in flight per chain and the row takes ~1 ms.  So:
//   1. hub_products_kernel: every rounded product v*x of every hub row, in
//      parallel over all SMs (segments of kHubSeg positions), into a
//      products buffer laid out [hub][position][column] (16-byte aligned rows);
//   2. par_rs_hub_fold_kernel: one CTA per hub row streams its products
//      through a shared-memory ring with 1-D bulk copies (cp.async.bulk, TMA
//      engine, mbarrier completion) while thread (l, c) adds chain l of column
//      c in j order — the reference's order — and then runs the tree.
// The fold is then bound by the add chains, not by gather latency.
constexpr int kHubSeg = 2048;        // positions per products block
constexpr int kFoldStages = 6;       // ring stages (48 KB)
constexpr int kFoldStageBytes = 8192;

struct HubProdArgs {
  const int* __restrict__ hubs;       // compact rows, launch order
  const int2* __restrict__ segs;      // {hub index, first position} per block
  const long long* __restrict__ po;   // products offset (floats) per hub
  const int* __restrict__ crp;
  const int* __restrict__ col;
  const float* __restrict__ val;
  const float* __restrict__ X;
  float* __restrict__ prod;
  int N;
};

__global__ void __launch_bounds__(256) hub_products_kernel(const HubProdArgs a) {
  const int2 sg = a.segs[blockIdx.x];
  const int r = a.hubs[sg.x];
  const int s = a.crp[r], len = a.crp[r + 1] - s;
  const int q1 = min(sg.y + kHubSeg, len);
  const unsigned N = (unsigned)a.N;
  float* const out = a.prod + a.po[sg.x];
  const long long i0 = (long long)sg.y * N, i1 = (long long)q1 * N;
  if (N == 1) {
    const uint64_t pol = evict_first_policy();
#pragma unroll 4
    for (long long i = i0 + threadIdx.x; i < i1; i += 256) {
      const int e = s + (int)i;
      out[i] = __fmul_rn(ld_stream(a.val + e, pol), ld_x(a.X + (unsigned)ld_stream(a.col + e, pol)));
    }
  } else {
#pragma unroll 4
    for (long long i = i0 + threadIdx.x; i < i1; i += 256) {
      const unsigned q = (unsigned)(i / N), c = (unsigned)(i - (long long)q * N);
      const int e = s + (int)q;
      out[i] = __fmul_rn(a.val[e], ld_x(a.X + (size_t)(unsigned)a.col[e] * N + c));
    }
  }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// W * N <= 256 threads: thread t = l * N + c folds chain l of column c.
__global__ void __launch_bounds__(256) par_rs_hub_fold_kernel(const HubProdArgs a, const int* __restrict__ rid,
                                                              float* __restrict__ Y, int W) {
  extern __shared__ __align__(128) unsigned char fold_smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(fold_smem);  // kFoldStages mbarriers
  float* ring = reinterpret_cast<float*>(fold_smem + 128);
  const int h = blockIdx.x;
  const int r = a.hubs[h];
  const int len = a.crp[r + 1] - a.crp[r];
  const int N = a.N;
  const int t = threadIdx.x;
  const int l = t / N, c = t - l * N;
  // chunk = CQ positions (a multiple of W, CQ * N * 4 <= stage bytes, CQ*N % 4 == 0)
  const int CQ = (kFoldStageBytes / 4 / N) / max(W, 4) * max(W, 4);  // CQ * N % 4 == 0: 16-B chunks
  const int nch = (len + CQ - 1) / CQ;
  const float* src = a.prod + a.po[h];
  auto issue = [&](int k) {
    const int q0 = k * CQ;
    const int q1 = min(q0 + CQ, len);
    const unsigned bytes = (unsigned)(((q1 - q0) * N * 4 + 15) & ~15);
    uint64_t* bar = bars + (k % kFoldStages);
    mbar_expect_tx(bar, bytes);
    bulk_g2s(ring + (size_t)(k % kFoldStages) * (kFoldStageBytes / 4), src + (size_t)q0 * N, bytes, bar);
  };
  if (t == 0) {
    for (int i = 0; i < kFoldStages; ++i) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0)
    for (int k = 0; k < min(nch, kFoldStages); ++k) issue(k);
  float acc = 0.f;
  for (int k = 0; k < nch; ++k) {
    mbar_wait(bars + (k % kFoldStages), (unsigned)(k / kFoldStages) & 1u);
    const float* b = ring + (size_t)(k % kFoldStages) * (kFoldStageBytes / 4);
    const int q0 = k * CQ;
    const int steps = (min(q0 + CQ, len) - q0 + W - 1) / W;  // chain steps in this chunk
    if (l < W) {
      const int stepf = W * N;  // floats per chain step
      if (q0 + CQ <= len) {
#pragma unroll 8
        for (int j = 0; j < CQ / W; ++j) acc = __fadd_rn(acc, b[j * stepf + t]);
      } else {
        for (int j = 0; j < steps; ++j)
          if (q0 + j * W + l < len) acc = __fadd_rn(acc, b[j * stepf + t]);
      }
    }
    __syncthreads();  // stage k % S free
    if (t == 0 && k + kFoldStages < nch) issue(k + kFoldStages);
  }
  // tree acc[l] = acc[2l+1] + acc[2l] per column (kernels.hpp:193-199)
  float* sacc = ring;  // reuse stage 0 (all copies consumed)
  if (l < W) sacc[t] = acc;
  __syncthreads();
  if (l == 0) {
#pragma unroll 1
    for (int ln = W; ln > 1; ln >>= 1)
#pragma unroll 1
      for (int i = 0; i < ln / 2; ++i) sacc[i * N + c] = __fadd_rn(sacc[(2 * i + 1) * N + c], sacc[2 * i * N + c]);
    Y[(size_t)(unsigned)rid[r] * (unsigned)N + c] = sacc[c];
  }
}

}  // namespace spmk_dev
