// Does ptxas's FFMA2 (formed from mul.rn.f32x2 + add.rn.f32x2) round twice?
// Prints the number of mismatches against the two-rounding host result.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) { u64 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) { u64 d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__global__ void k(const float* a, const float* b, const float* c, u64* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = fadd2(pk(c[2 * i], c[2 * i + 1]), fmul2(pk(a[2 * i], a[2 * i + 1]), pk(b[2 * i], b[2 * i + 1])));
}
int main() {
  const int n = 1 << 20;
  float *a = new float[2 * n], *b = new float[2 * n], *c = new float[2 * n];
  uint64_t s = 88172645463325252ull;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (float)((double)(s >> 11) / 9007199254740992.0 * 2.0 - 1.0); };
  for (int i = 0; i < 2 * n; ++i) { a[i] = rnd(); b[i] = rnd(); c[i] = rnd(); }
  float *da, *db, *dc; u64* dout;
  cudaMalloc(&da, 8 * n); cudaMalloc(&db, 8 * n); cudaMalloc(&dc, 8 * n); cudaMalloc(&dout, 8 * n);
  cudaMemcpy(da, a, 8 * n, cudaMemcpyHostToDevice); cudaMemcpy(db, b, 8 * n, cudaMemcpyHostToDevice); cudaMemcpy(dc, c, 8 * n, cudaMemcpyHostToDevice);
  k<<<n / 256, 256>>>(da, db, dc, dout, n);
  float* out = new float[2 * n];
  cudaMemcpy(out, dout, 8 * n, cudaMemcpyDeviceToHost);
  long two = 0, fused = 0;
  for (int i = 0; i < 2 * n; ++i) {
    volatile float p = a[i] * b[i];
    float r2 = c[i] + p;
    float rf = __builtin_fmaf(a[i], b[i], c[i]);
    if (memcmp(&out[i], &r2, 4)) ++two;
    if (memcmp(&out[i], &rf, 4)) ++fused;
  }
  printf("f32x2 mul+add: mismatches vs two roundings %ld, vs fused %ld (of %d)\n", two, fused, 2 * n);
  return 0;
}
