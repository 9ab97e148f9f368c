// gen_kernels.cuh — bit-exact device generators for the synthetic inputs.
//
// SplitMix64 (rmat.hpp:15-29) is counter-based: the k-th call (k >= 1) of a
// stream seeded with s returns mix(s + k * 0x9e3779b97f4a7c15).  So every
// draw of the reference generators is an independent function of its call
// index and the whole stream parallelises bit-exactly:
//   make_dense  element i        -> call i + 1           (corpus.hpp:116-122)
//   generate_rmat edge e, level l -> call e*scale + l + 1 (rmat.hpp:70-83)
#pragma once
#include <stdint.h>

namespace spmk_dev {

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t k) {
  uint64_t z = seed + k * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double unit_at(uint64_t seed, uint64_t k) {
  return (double)(splitmix_at(seed, k) >> 11) * 0x1.0p-53;
}

// make_dense<float>: float(2u - 1) (double math, then rounded once).
__global__ void make_dense_kernel(float* __restrict__ out, long long total, uint64_t seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (float)(2.0 * unit_at(seed, (uint64_t)i + 1) - 1.0);
}

// R-MAT edge keys (row << scale | col), rmat.hpp:70-83 quadrant descent.
__global__ void rmat_edges_kernel(unsigned long long* __restrict__ keys, long long edges,
                                  int scale, uint64_t seed, double t_a, double t_ab,
                                  double t_abc) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < edges;
       e += (long long)gridDim.x * blockDim.x) {
    unsigned long long row = 0, col = 0;
    const uint64_t base = (uint64_t)e * (uint64_t)scale + 1;
    for (int l = 0; l < scale; ++l) {
      const double u = unit_at(seed, base + l);
      const unsigned rbit = u >= t_ab;
      const unsigned cbit = (u >= t_a && u < t_ab) || u >= t_abc;
      row = (row << 1) | rbit;
      col = (col << 1) | cbit;
    }
    keys[e] = (row << scale) | col;
  }
}

// After sort: keep first of each equal run (duplicates collapse, csr.hpp:147-157).
__global__ void unique_flag_kernel(const unsigned long long* __restrict__ keys, long long n,
                                   int* __restrict__ flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}
__global__ void unique_scatter_kernel(const unsigned long long* __restrict__ keys, long long n,
                                      const int* __restrict__ flag, const int* __restrict__ pos,
                                      int scale, int* __restrict__ col, float* __restrict__ val,
                                      unsigned long long* __restrict__ ukeys) {
  const unsigned long long mask = (1ull << scale) - 1ull;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (flag[i]) {
      const int p = pos[i];
      col[p] = (int)(keys[i] & mask);
      val[p] = 1.0f;  // pattern values (rmat.hpp:85-86)
      ukeys[p] = keys[i] >> scale;  // row
    }
  }
}
// rowPtr[i] = lower_bound(rows, i) over the sorted unique row ids.
__global__ void rowptr_from_rows_kernel(const unsigned long long* __restrict__ rows, long long nnz,
                                        long long m, int* __restrict__ rp) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= m;
       i += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = nnz;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (rows[mid] < (unsigned long long)i) lo = mid + 1; else hi = mid;
    }
    rp[i] = (int)lo;
  }
}

}  // namespace spmk_dev
