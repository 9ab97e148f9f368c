// iter_kernels.cuh — iterative SpMV (PageRank-style, BASELINE cfg5) support:
// column counts (out-degrees of the transposed graph), column-stochastic
// values, and the per-iteration update with deterministic reductions.
// None of this is on the reference's path (the reference has no iterative
// driver); it is the SURVEY §8f row 1 "next" item built on spmm(par-ws).
#pragma once
#include <stdint.h>

namespace spmk_dev {

// counts[c] = number of nonzeros in column c (integer atomics: deterministic).
__global__ void column_counts_kernel(const int* __restrict__ col, long long nnz, int* __restrict__ counts) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x)
    atomicAdd(counts + col[e], 1);
}

// val[e] = 1 / counts[col[e]]  (column-stochastic A: A x = sum_j x_j / outdeg_j).
__global__ void inv_count_values_kernel(const int* __restrict__ col, long long nnz,
                                        const int* __restrict__ counts, float* __restrict__ val) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x)
    val[e] = 1.0f / (float)counts[col[e]];
}

// r_new[i] = alpha * y[i] + base, base = st[0] (device scalar).  Per block:
// partial sums (fp64) of |r_new - r_old| and of r_new over dangling columns
// (counts == 0), written to part[blockIdx.x * 2 + {0,1}] for the ordered
// finalize below (no floating-point atomics: run-to-run bit-identical).
constexpr int kIterThreads = 256;
__device__ __forceinline__ void pr_elem(float yv, float& rv, int cnt, float alpha, float base, double& l1,
                                        double& dang) {
  const float rn = __fadd_rn(__fmul_rn(alpha, yv), base);
  l1 += fabs((double)rn - (double)rv);
  if (cnt == 0) dang += (double)rn;
  rv = rn;
}
__global__ void __launch_bounds__(kIterThreads)
pagerank_update_kernel(const float* __restrict__ y, float* __restrict__ r, const int* __restrict__ counts,
                       long long m, float alpha, const double* __restrict__ st, double* __restrict__ part) {
  __shared__ double s1[kIterThreads / 32], s2[kIterThreads / 32];
  const float base = (float)st[0];
  double l1 = 0.0, dang = 0.0;
  // 16-byte vectors when all three arrays are 16-byte aligned, scalar tail
  const bool vec = ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(r) |
                     reinterpret_cast<uintptr_t>(counts)) & 15) == 0;
  const long long m4 = vec ? (m & ~3LL) : 0;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  // two 16-byte groups per thread per step, all six loads issued first
  // (HBM-bound: more bytes in flight per thread)
  long long i = 4 * tid;
  for (; i + 4 * nth < m4; i += 8 * nth) {
    const long long i2 = i + 4 * nth;
    const float4 yv = *reinterpret_cast<const float4*>(y + i), yv2 = *reinterpret_cast<const float4*>(y + i2);
    float4 rv = *reinterpret_cast<const float4*>(r + i), rv2 = *reinterpret_cast<const float4*>(r + i2);
    const int4 cv = *reinterpret_cast<const int4*>(counts + i), cv2 = *reinterpret_cast<const int4*>(counts + i2);
    pr_elem(yv.x, rv.x, cv.x, alpha, base, l1, dang);
    pr_elem(yv.y, rv.y, cv.y, alpha, base, l1, dang);
    pr_elem(yv.z, rv.z, cv.z, alpha, base, l1, dang);
    pr_elem(yv.w, rv.w, cv.w, alpha, base, l1, dang);
    pr_elem(yv2.x, rv2.x, cv2.x, alpha, base, l1, dang);
    pr_elem(yv2.y, rv2.y, cv2.y, alpha, base, l1, dang);
    pr_elem(yv2.z, rv2.z, cv2.z, alpha, base, l1, dang);
    pr_elem(yv2.w, rv2.w, cv2.w, alpha, base, l1, dang);
    *reinterpret_cast<float4*>(r + i) = rv;
    *reinterpret_cast<float4*>(r + i2) = rv2;
  }
  for (; i < m4; i += 4 * nth) {
    const float4 yv = *reinterpret_cast<const float4*>(y + i);
    float4 rv = *reinterpret_cast<const float4*>(r + i);
    const int4 cv = *reinterpret_cast<const int4*>(counts + i);
    pr_elem(yv.x, rv.x, cv.x, alpha, base, l1, dang);
    pr_elem(yv.y, rv.y, cv.y, alpha, base, l1, dang);
    pr_elem(yv.z, rv.z, cv.z, alpha, base, l1, dang);
    pr_elem(yv.w, rv.w, cv.w, alpha, base, l1, dang);
    *reinterpret_cast<float4*>(r + i) = rv;
  }
  for (long long i = m4 + tid; i < m; i += nth) {
    float rv = r[i];
    pr_elem(y[i], rv, counts[i], alpha, base, l1, dang);
    r[i] = rv;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    dang += __shfl_xor_sync(0xffffffffu, dang, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s1[threadIdx.x >> 5] = l1;
    s2[threadIdx.x >> 5] = dang;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kIterThreads / 32; ++w) {
      a += s1[w];
      b += s2[w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// Fused update + exchange of the row-partitioned iterative SpMV: this rank's
// slice x_next[row0 + i] = alpha*y[i] + base is stored into every replica of
// x_next — this GPU's own and its peers' (CUDA-IPC-mapped buffers reached
// over NVLink with plain P2P stores) — in the same pass that computes the
// residual against x_cur and the dangling mass.  The replicas are complete
// once every rank's kernel has finished (the residual all-reduce that follows
// is the barrier), so no separate all-gather is needed.
constexpr int kMaxPeers = 8;
struct PeerPtrs {
  float* p[kMaxPeers];
};
__global__ void __launch_bounds__(kIterThreads)
pagerank_update_p2p_kernel(const float* __restrict__ y, const float* __restrict__ xcur,
                           const int* __restrict__ counts, long long row0, long long m, float alpha,
                           const double* __restrict__ st, PeerPtrs peers, int npeers,
                           double* __restrict__ part) {
  __shared__ double s1[kIterThreads / 32], s2[kIterThreads / 32];
  const float base = (float)st[0];
  double l1 = 0.0, dang = 0.0;
  // four rows per thread per step with every load issued first (the same
  // per-thread element order as one row per step: the residual bits match)
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * nth < m; i += 4 * nth) {
    float yv[4], rv[4];
    int cv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      yv[u] = y[i + u * nth];
      rv[u] = xcur[row0 + i + u * nth];  // old value in, new value out (residual inside)
      cv[u] = counts[row0 + i + u * nth];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      pr_elem(yv[u], rv[u], cv[u], alpha, base, l1, dang);
#pragma unroll
      for (int q = 0; q < kMaxPeers; ++q)
        if (q < npeers) peers.p[q][row0 + i + u * nth] = rv[u];
    }
  }
  for (; i < m; i += nth) {
    float rv = xcur[row0 + i];
    pr_elem(y[i], rv, counts[row0 + i], alpha, base, l1, dang);
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
      if (q < npeers) peers.p[q][row0 + i] = rv;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    dang += __shfl_xor_sync(0xffffffffu, dang, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s1[threadIdx.x >> 5] = l1;
    s2[threadIdx.x >> 5] = dang;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kIterThreads / 32; ++w) {
      a += s1[w];
      b += s2[w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// Ordered sum of the block partials; st = {base for the next step, l1,
// dangling mass}; hist[t] = l1 of step t.  One warp, fixed order.
__global__ void pagerank_finalize_kernel(const double* __restrict__ part, int nblocks, long long m_total,
                                         double alpha, double* __restrict__ st, double* __restrict__ hist,
                                         int t) {
  double l1 = 0.0, dang = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += 32) {
    l1 += part[2 * b];
    dang += part[2 * b + 1];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    dang += __shfl_xor_sync(0xffffffffu, dang, o);
  }
  if (threadIdx.x == 0) {
    st[0] = (1.0 - alpha) / (double)m_total + alpha * dang / (double)m_total;
    st[1] = l1;
    st[2] = dang;
    if (hist) hist[t] = l1;
  }
}

// Dangling mass of an initial vector (same ordered reduction).
__global__ void __launch_bounds__(kIterThreads)
dangling_mass_kernel(const float* __restrict__ r, const int* __restrict__ counts, long long m,
                     double* __restrict__ part) {
  __shared__ double s2[kIterThreads / 32];
  double dang = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    if (counts[i] == 0) dang += (double)r[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dang += __shfl_xor_sync(0xffffffffu, dang, o);
  if ((threadIdx.x & 31) == 0) s2[threadIdx.x >> 5] = dang;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < kIterThreads / 32; ++w) b += s2[w];
    part[2 * blockIdx.x] = 0.0;
    part[2 * blockIdx.x + 1] = b;
  }
}

}  // namespace spmk_dev
