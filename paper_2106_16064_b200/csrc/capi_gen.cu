// capi_gen.cu — device input generators, bit-identical to the reference's
// host generators (counter form of SplitMix64, rmat.hpp:15-29):
// generate_rmat<float> (rmat.hpp:61-88 + csr_from_coo csr.hpp:123-164) and
// make_dense<float> (corpus.hpp:116-122).
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <cmath>
#include <cstdint>

#include "gen_kernels.cuh"
#include "internal.h"

using namespace spmk_dev;
using namespace spmk_host;

extern "C" {

spmk_status spmk_make_dense(int64_t rows, int64_t cols, uint64_t seed, float* d_out, void* stream) {
  const long long total = rows * cols;
  if (total <= 0) return SPMK_OK;
  make_dense_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(d_out, total, seed); LAUNCHED(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SPMK_ECUDA, cudaGetErrorString(e));
  return SPMK_OK;
}

spmk_status spmk_generate_rmat(uint32_t scale, uint64_t edge_factor, double a, double b, double c,
                               double d, uint64_t seed, int device, spmk_csr_t* out) {
  // rmat.hpp:46-59 validate
  if (scale < 1 || scale > 30) return fail(SPMK_EINVAL, "rmat scale must be in [1, 30]");
  if (edge_factor < 1) return fail(SPMK_EINVAL, "rmat edge_factor must be >= 1");
  const double pr[4] = {a, b, c, d};
  double sum = 0.0;
  for (double q : pr) {
    if (q < 0.0 || q > 1.0) return fail(SPMK_EINVAL, "rmat quadrant probability outside [0, 1]");
    sum += q;
  }
  if (std::abs(sum - 1.0) > 1e-9) return fail(SPMK_EINVAL, "rmat quadrant probabilities must sum to 1");
  if (scale > 30 || (edge_factor << scale) >= (1ull << 31))
    return fail(SPMK_EUNSUPPORTED, "edge count must be < 2^31 on the device path");
  DeviceGuard g(device);
  const long long m = 1LL << scale;
  const long long edges = (long long)(edge_factor << scale);
  const double t_a = a, t_ab = a + b, t_abc = a + b + c;  // rmat.hpp:66-68
  cudaStream_t s = nullptr;
  try {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    unsigned long long* keys = dev_alloc<unsigned long long>((size_t)edges);
    unsigned long long* sorted = dev_alloc<unsigned long long>((size_t)edges);
    rmat_edges_kernel<<<grid_for(edges, 256, 148 * 64), 256, 0, s>>>(keys, edges, (int)scale, seed,
                                                                     t_a, t_ab, t_abc); LAUNCHED(1);
    CK(cudaGetLastError());
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, edges, 0, 2 * (int)scale, s);
    void* tmp = dev_alloc<char>(tb);
    cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, edges, 0, 2 * (int)scale, s);
    cudaFree(tmp);
    int* flag = reinterpret_cast<int*>(keys);  // reuse: edges*8 bytes >= 2*edges ints
    int* pos = flag + edges;
    unique_flag_kernel<<<grid_for(edges), 256, 0, s>>>(sorted, edges, flag); LAUNCHED(1);
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, flag, pos, edges, s);
    tmp = dev_alloc<char>(sb);
    cub::DeviceScan::ExclusiveSum(tmp, sb, flag, pos, edges, s);
    int last_flag = 0, last_pos = 0;
    CK(cudaMemcpyAsync(&last_flag, flag + edges - 1, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&last_pos, pos + edges - 1, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(tmp);
    const long long nnz = (long long)last_pos + last_flag;
    int* col = dev_alloc<int>((size_t)nnz);
    float* val = dev_alloc<float>((size_t)nnz);
    unsigned long long* rows = dev_alloc<unsigned long long>((size_t)nnz);
    unique_scatter_kernel<<<grid_for(edges), 256, 0, s>>>(sorted, edges, flag, pos, (int)scale, col,
                                                           val, rows); LAUNCHED(1);
    cudaFree(keys);
    cudaFree(sorted);
    int* rp = dev_alloc<int>((size_t)m + 1);
    rowptr_from_rows_kernel<<<grid_for(m + 1), 256, 0, s>>>(rows, nnz, m, rp); LAUNCHED(1);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    cudaFree(rows);
    spmk_status st = create_from_device32(m, m, nnz, rp, col, val, true, device, out, s);
    cudaStreamDestroy(s);
    return st;
  } catch (const CudaError& e) {
    if (s) cudaStreamDestroy(s);
    return fail(e.st, e.msg);
  }
}

}  // extern "C"
