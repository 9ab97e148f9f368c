// capi_iter.cu — iterative SpMV / PageRank support (BASELINE cfg5; SURVEY
// §8f row 1) and the CUDA IPC helpers of its fused multi-GPU exchange.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "internal.h"
#include "iter_kernels.cuh"

using namespace spmk_dev;
using namespace spmk_host;

extern "C" {

// ------------------------------------------------------------ iterative SpMV
spmk_status spmk_column_counts(spmk_csr_t a, int32_t* d_counts, void* stream) {
  if (!a || !d_counts) return fail(SPMK_EINVAL, "null argument");
  DeviceGuard g(a->device);
  cudaStream_t s = (cudaStream_t)stream;
  try {
    CK(cudaMemsetAsync(d_counts, 0, (size_t)a->k * 4, s));
    if (a->nnz) {
      column_counts_kernel<<<grid_for(a->nnz), 256, 0, s>>>(a->col, a->nnz, d_counts); LAUNCHED(1);
    }
    CK(cudaGetLastError());
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_csr_values_inv_column_counts(spmk_csr_t a, const int32_t* d_counts, void* stream) {
  if (!a || !d_counts) return fail(SPMK_EINVAL, "null argument");
  if (!a->own_val) return fail(SPMK_EINVAL, "handle borrows its values; create it with copy=1");
  DeviceGuard g(a->device);
  try {
    if (a->nnz) {
      inv_count_values_kernel<<<grid_for(a->nnz), 256, 0, (cudaStream_t)stream>>>(a->col, a->nnz, d_counts, a->val);
      LAUNCHED(1);
    }
    CK(cudaGetLastError());
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

static const int kIterBlocks = 148 * 8;

int64_t spmk_pagerank_scratch_doubles(void) { return 2 * kIterBlocks; }

spmk_status spmk_pagerank_init(const float* d_r, const int32_t* d_counts, int64_t m, int64_t m_total,
                               double alpha, double* d_state, double* d_scratch, void* stream) {
  if (!d_r || !d_counts || !d_state || !d_scratch || m < 0 || m_total < 1) return fail(SPMK_EINVAL, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  dangling_mass_kernel<<<kIterBlocks, kIterThreads, 0, s>>>(d_r, d_counts, m, d_scratch); LAUNCHED(1);
  pagerank_finalize_kernel<<<1, 32, 0, s>>>(d_scratch, kIterBlocks, m_total, alpha, d_state, nullptr, 0); LAUNCHED(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPMK_OK : fail(SPMK_ECUDA, cudaGetErrorString(e));
}

spmk_status spmk_pagerank_step(const float* d_y, float* d_r, const int32_t* d_counts, int64_t m,
                               int64_t m_total, double alpha, double* d_state, double* d_scratch,
                               double* d_hist, int32_t t, void* stream) {
  if (!d_y || !d_r || !d_counts || !d_state || !d_scratch || m < 0 || m_total < 1)
    return fail(SPMK_EINVAL, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  pagerank_update_kernel<<<kIterBlocks, kIterThreads, 0, s>>>(d_y, d_r, d_counts, m, (float)alpha, d_state,
                                                              d_scratch); LAUNCHED(1);
  pagerank_finalize_kernel<<<1, 32, 0, s>>>(d_scratch, kIterBlocks, m_total, alpha, d_state, d_hist, t); LAUNCHED(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPMK_OK : fail(SPMK_ECUDA, cudaGetErrorString(e));
}

spmk_status spmk_pagerank_step_p2p(const float* d_y, const float* d_x_cur, float* const* peer_x_next,
                                   int32_t npeers, const int32_t* d_counts, int64_t row0, int64_t m,
                                   int64_t m_total, double alpha, double* d_state, double* d_scratch,
                                   void* stream) {
  if (!d_y || !d_x_cur || !peer_x_next || !d_counts || !d_state || !d_scratch || m < 0 || m_total < 1 ||
      row0 < 0 || npeers < 1 || npeers > kMaxPeers)
    return fail(SPMK_EINVAL, "bad argument");
  PeerPtrs pp{};
  for (int q = 0; q < npeers; ++q) {
    if (!peer_x_next[q]) return fail(SPMK_EINVAL, "null peer buffer");
    pp.p[q] = peer_x_next[q];
  }
  cudaStream_t s = (cudaStream_t)stream;
  pagerank_update_p2p_kernel<<<kIterBlocks, kIterThreads, 0, s>>>(d_y, d_x_cur, d_counts, row0, m, (float)alpha,
                                                                  d_state, pp, npeers, d_scratch); LAUNCHED(1);
  pagerank_finalize_kernel<<<1, 32, 0, s>>>(d_scratch, kIterBlocks, m_total, alpha, d_state, nullptr, 0); LAUNCHED(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPMK_OK : fail(SPMK_ECUDA, cudaGetErrorString(e));
}

spmk_status spmk_ipc_handle(const void* d_ptr, void* handle64) {
  if (!d_ptr || !handle64) return fail(SPMK_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr));
  if (e != cudaSuccess) return fail(SPMK_ECUDA, cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  std::memcpy(handle64, &h, 64);
  return SPMK_OK;
}

spmk_status spmk_ipc_open(const void* handle64, void** d_ptr) {
  if (!handle64 || !d_ptr) return fail(SPMK_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(SPMK_ECUDA, cudaGetErrorString(e));
  return SPMK_OK;
}

spmk_status spmk_ipc_close(void* d_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  return e == cudaSuccess ? SPMK_OK : fail(SPMK_ECUDA, cudaGetErrorString(e));
}

}  // extern "C"
