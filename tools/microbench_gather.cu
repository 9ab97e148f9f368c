// Dev microbenchmark (not product): random 128-B row gathers on B200.
//   ./mb  -> prints gathered GB/s for L2-resident and HBM-resident X, with
//            register-only loads vs prefetch.global.L1 staging.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench_gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void pf_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Each warp: for its slice of idx[], lane l reads X[idx[j]*32 + l] and sums.
template <int UNROLL>
__global__ void gather_reg(const float* __restrict__ X, const int* __restrict__ idx, long long n,
                           float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (long long j0 = w * UNROLL; j0 < n; j0 += nw * UNROLL) {
    int c[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) c[u] = (j0 + u < n) ? __ldg(idx + j0 + u) : 0;
    float x[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) x[u] = __ldg(X + (size_t)c[u] * 32 + lane);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += x[u];
  }
  if (acc == 12345.f) out[0] = acc;
}

// Contiguous per-warp streams with prefetch distance D (in batches of UNROLL).
template <int UNROLL, int D>
__global__ void gather_pf(const float* __restrict__ X, const int* __restrict__ idx, long long n,
                          float* __restrict__ out, long long per_warp) {
  const int lane = threadIdx.x & 31;
  long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  long long s = w * per_warp, e = s + per_warp;
  if (e > n) e = n;
  float acc = 0.f;
  for (long long j0 = s; j0 < e; j0 += UNROLL) {
    // prefetch batch j0 + D*UNROLL
    const long long jp = j0 + (long long)D * UNROLL;
    if (jp + lane < e && lane < UNROLL) pf_l1(X + (size_t)__ldg(idx + jp + lane) * 32);
    int c[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) c[u] = (j0 + u < e) ? __ldg(idx + j0 + u) : 0;
    float x[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) x[u] = __ldg(X + (size_t)c[u] * 32 + lane);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += x[u];
  }
  if (acc == 12345.f) out[0] = acc;
}

// 4-byte random gathers: every lane its own index (SpMV x[col] pattern).
template <int UNROLL>
__global__ void gather_word(const float* __restrict__ X, const int* __restrict__ idx, long long n,
                            float* __restrict__ out) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long nt = (long long)gridDim.x * blockDim.x;
  float acc = 0.f;
  for (long long j0 = t; j0 < n; j0 += nt * UNROLL) {
    int c[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) c[u] = (j0 + u * nt < n) ? __ldg(idx + j0 + u * nt) : 0;
    float x[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) x[u] = __ldg(X + c[u]);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += x[u];
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void fill_idx(int* idx, long long n, long long rows, unsigned long long seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = seed + i * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    idx[i] = (int)((z ^ (z >> 31)) % rows);
  }
}

int main() {
  const long long n = 16 << 20;  // gathers
  int* idx;
  float *X, *out;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&out, 4);
  const long long maxrows = (2048LL << 20) / 128;  // 2 GB of X
  cudaMalloc(&X, maxrows * 128);
  cudaMemset(X, 0, maxrows * 128);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (long long mb : {4LL, 16LL, 64LL}) {  // 4-byte gathers: request rate
    const long long words = (mb << 20) / 4;
    fill_idx<<<1184, 256>>>(idx, n, words, 7);
    for (int blocks : {148 * 8, 148 * 16, 148 * 32}) {
      gather_word<8><<<blocks, 256>>>(X, idx, n, out);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) gather_word<8><<<blocks, 256>>>(X, idx, n, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      printf("x=%5lld MB word gathers blocks=%d  %8.1f us  %7.1f G req/s\n", mb, blocks, ms * 1e3, n / (ms * 1e-3) / 1e9);
    }
  }
  for (long long mb : {16LL, 48LL, 96LL, 2048LL}) {
    const long long rows = (mb << 20) / 128;
    fill_idx<<<1184, 256>>>(idx, n, rows, 7);
    auto run = [&](const char* name, auto launch) {
      launch();
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      printf("X=%5lld MB %-28s %8.1f us  %7.1f GB/s gathered\n", mb, name, ms * 1e3, n * 128.0 / (ms * 1e-3) / 1e9);
    };
    for (int blocks : {148 * 8, 148 * 16, 148 * 32}) {
      char nm[64];
      snprintf(nm, 64, "reg U8 blocks=%d", blocks);
      run(nm, [&] { gather_reg<8><<<blocks, 256>>>(X, idx, n, out); });
      snprintf(nm, 64, "reg U32 blocks=%d", blocks);
      run(nm, [&] { gather_reg<32><<<blocks, 256>>>(X, idx, n, out); });
    }
    for (int blocks : {148 * 4, 148 * 8}) {
      const long long warps = blocks * 8LL;
      const long long pw = (n + warps - 1) / warps;
      char nm[64];
      snprintf(nm, 64, "pf U8 D2 blocks=%d", blocks);
      run(nm, [&] { gather_pf<8, 2><<<blocks, 256>>>(X, idx, n, out, pw); });
      snprintf(nm, 64, "pf U8 D4 blocks=%d", blocks);
      run(nm, [&] { gather_pf<8, 4><<<blocks, 256>>>(X, idx, n, out, pw); });
      snprintf(nm, 64, "pf U16 D4 blocks=%d", blocks);
      run(nm, [&] { gather_pf<16, 4><<<blocks, 256>>>(X, idx, n, out, pw); });
    }
  }
  // plain copy bandwidth for reference
  float* Y;
  cudaMalloc(&Y, 1LL << 30);
  cudaMemcpy(Y, X, 1LL << 30, cudaMemcpyDeviceToDevice);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) cudaMemcpy(Y, X, 1LL << 30, cudaMemcpyDeviceToDevice);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("memcpy 1GiB: %.1f GB/s (r+w)\n", 2.0 * (1 << 30) / (ms / 5 * 1e-3) / 1e9);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
