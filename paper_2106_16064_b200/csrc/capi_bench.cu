// capi_bench.cu — the selection harness's per-cell measurement on the device
// (bench.hpp:65-98 measure_kernel): X generated in HBM, CUDA-event timing,
// median of `repeats`, and the reference's correctness flag
// (matches_oracle, bench.hpp:47-58, tolerance kernel_tolerance<float>) checked
// against an fp64 product computed by an independent row-parallel kernel —
// none of the four variants' code is on the checking side.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "internal.h"

using namespace spmk_host;

namespace {

// One warp per row: the fp64 sum of v*x (csr.hpp:185-205 in double) for each
// column, compared with y under |y - o| <= tol * max(1, |o|).
__global__ void check_fp64_kernel(const int* __restrict__ rp, const int* __restrict__ col,
                                  const float* __restrict__ val, const float* __restrict__ x,
                                  const float* __restrict__ y, long long m, int n, double tol,
                                  unsigned long long* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  for (long long r = blockIdx.x * (long long)(blockDim.x / 32) + threadIdx.x / 32; r < m; r += warps) {
    const int s = rp[r], e = rp[r + 1];
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int c = c0 + lane;
      double acc = 0.0;
      if (c < n)
        for (int p = s; p < e; ++p) acc += (double)val[p] * (double)x[(size_t)col[p] * n + c];
      if (c < n) {
        const double d = fabs((double)y[(size_t)r * n + c] - acc);
        if (!(d <= tol * fmax(1.0, fabs(acc)))) atomicAdd(bad, 1ull);
      }
    }
  }
}

}  // namespace

extern "C" {

spmk_status spmk_measure_kernel(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg, int64_t n,
                                uint64_t x_seed, int64_t repeats, int64_t warmup, int flush_l2,
                                double* median_seconds, int* correct) {
  if (!a || !median_seconds || n < 0) return fail(SPMK_EINVAL, "bad argument");
  if (repeats < 1) return fail(SPMK_EINVAL, "repeats must be >= 1");
  DeviceGuard g(a->device);
  float *x = nullptr, *y = nullptr;
  unsigned char* flush = nullptr;
  unsigned long long* bad = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  spmk_status st = SPMK_OK;
  try {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    x = dev_alloc<float>((size_t)(a->k * n));
    y = dev_alloc<float>((size_t)(a->m * n));
    if (flush_l2) flush = dev_alloc<unsigned char>((size_t)256 << 20);
    st = spmk_make_dense(a->k, n, x_seed, x, s);
    for (int64_t i = 0; st == SPMK_OK && i < warmup; ++i) st = spmk_spmm(a, id, cfg, x, n, y, s);
    std::vector<double> t;
    for (int64_t i = 0; st == SPMK_OK && i < repeats; ++i) {
      if (flush) CK(cudaMemsetAsync(flush, i & 0xff, (size_t)256 << 20, s));
      CK(cudaEventRecord(e0, s));
      st = spmk_spmm(a, id, cfg, x, n, y, s);
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      t.push_back(ms * 1e-3);
    }
    if (st == SPMK_OK) {
      std::sort(t.begin(), t.end());
      const size_t h = t.size() / 2;
      *median_seconds = std::max(t.size() % 2 ? t[h] : 0.5 * (t[h - 1] + t[h]), 1e-9);
      if (correct) {
        bad = dev_alloc<unsigned long long>(1);
        CK(cudaMemsetAsync(bad, 0, 8, s));
        if (a->m && n) {
          check_fp64_kernel<<<grid_for(a->m * 32, 256, 148 * 32), 256, 0, s>>>(
              a->rp, a->col, a->val, x, y, a->m, (int)n, spmk_kernel_tolerance(a->max_row), bad);
          LAUNCHED(1);
          CK(cudaGetLastError());
        }
        unsigned long long nb = 0;
        CK(cudaMemcpyAsync(&nb, bad, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        *correct = nb == 0;
      }
    }
  } catch (const CudaError& e) {
    st = fail(e.st, e.msg);
  }
  if (s) cudaStreamSynchronize(s);
  cudaFree(x);
  cudaFree(y);
  cudaFree(flush);
  cudaFree(bad);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (s) cudaStreamDestroy(s);
  return st;
}

spmk_status spmk_make_dense_host(int64_t rows, int64_t cols, uint64_t seed, float* out, int device) {
  if (rows < 0 || cols < 0 || (!out && rows * cols)) return fail(SPMK_EINVAL, "bad argument");
  if (rows * cols == 0) return SPMK_OK;
  DeviceGuard g(device);
  float* d = nullptr;
  try {
    d = dev_alloc<float>((size_t)(rows * cols));
    spmk_status st = spmk_make_dense(rows, cols, seed, d, nullptr);
    if (st != SPMK_OK) {
      cudaFree(d);
      return st;
    }
    CK(cudaMemcpy(out, d, (size_t)(rows * cols) * 4, cudaMemcpyDeviceToHost));
  } catch (const CudaError& e) {
    cudaFree(d);
    return fail(e.st, e.msg);
  }
  cudaFree(d);
  return SPMK_OK;
}

}  // extern "C"
