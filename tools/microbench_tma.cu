// Dev microbenchmark (not product): 128-B dense-row gathers (the seq sweep's
// X[col, 0:32] fetch at N=32) through three paths on B200:
//   tma   cp.async.bulk.tensor.2d.tile::gather4 (TMA, 4 rows per instruction,
//         mbarrier completion) into a per-warp shared-memory ring
//   ldgsts cp.async 16 B per lane (8 lanes per row) into the same ring shape
//   reg   plain LDG of 4 B per lane
// over uniform and R-MAT-distributed (Graph500 skew) row indices, X = 2^20 x 32
// fp32 (134 MB, the cfg2 X).  Prints gathered GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbt microbench_tma.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int c0, int4 r, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
      "l"(tm), "r"(c0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(su32(b))
      : "memory");
}
__device__ __forceinline__ void cp16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

// Each warp: a contiguous slice of idx; G rows per stage, S stages.
template <int S, int G>
__global__ void gather_tma(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, long long per_warp,
                           float* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  float4* ring = reinterpret_cast<float4*>(sm) + (size_t)warp * S * G * 8;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)wpb * S * G * 128) + warp * S;
  if (lane == 0)
    for (int s = 0; s < S; ++s) bar_init(bar + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long gw = blockIdx.x * (long long)wpb + warp;
  const int* ip = idx + gw * per_warp;
  const int nb = (int)(per_warp / G);
  auto issue = [&](int b, int s) {
    if (lane == 0) bar_expect(bar + s, G * 128);
    __syncwarp();
    if (lane < G / 4) {
      const int4 r = __ldg(reinterpret_cast<const int4*>(ip + (size_t)b * G) + lane);
      tma_gather4(ring + (s * G + 4 * lane) * 8, &tm, 0, r, bar + s);
    }
  };
  for (int s = 0; s < S - 1 && s < nb; ++s) issue(s, s);
  float acc = 0.f;
  unsigned ph = 0;
  for (int b = 0; b < nb; ++b) {
    const int s = b % S;
    if (b + S - 1 < nb) issue(b + S - 1, (b + S - 1) % S);
    bar_wait(bar + s, (ph >> s) & 1);
    ph ^= 1u << s;
#pragma unroll
    for (int i = 0; i < G / 4; ++i) {
      const float4 v = ring[(s * G) * 8 + i * 32 + lane];
      acc += v.x + v.y + v.z + v.w;
    }
    __syncwarp();
  }
  if (acc == 12345.f) out[0] = acc;
}

template <int S, int G>
__global__ void gather_ldgsts(const float* __restrict__ X, const int* __restrict__ idx, long long per_warp,
                              float* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  float4* ring = reinterpret_cast<float4*>(sm) + (size_t)warp * S * G * 8;
  const long long gw = blockIdx.x * (long long)wpb + warp;
  const int* ip = idx + gw * per_warp;
  const int nb = (int)(per_warp / G);
  const unsigned r0 = su32(ring) + lane * 16;
  const char* xg = reinterpret_cast<const char*>(X) + (lane & 7) * 16;
  auto issue = [&](int b, int s) {
    int c = lane < G ? __ldg(ip + (size_t)b * G + lane) : 0;
#pragma unroll
    for (int i = 0; i < G / 4; ++i) {
      const int ci = __shfl_sync(0xffffffffu, c, 4 * i + (lane >> 3));
      cp16(r0 + (s * G * 8 + i * 32) * 16, xg + (size_t)ci * 128);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < S - 1 && s < nb; ++s) issue(s, s);
  float acc = 0.f;
  for (int b = 0; b < nb; ++b) {
    const int s = b % S;
    if (b + S - 1 < nb) issue(b + S - 1, (b + S - 1) % S);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
#pragma unroll
    for (int i = 0; i < G / 4; ++i) {
      const float4 v = ring[(s * G) * 8 + i * 32 + lane];
      acc += v.x + v.y + v.z + v.w;
    }
    __syncwarp();
  }
  if (acc == 12345.f) out[0] = acc;
}

__device__ __forceinline__ unsigned long long smix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// mode 0 uniform, 1 R-MAT column (a .57 b .19 c .19 d .05: column bit 1 w.p. .24)
__global__ void fill_idx(int* idx, long long n, int scale, int mode, unsigned long long seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = smix(seed + i * 0x9e3779b97f4a7c15ULL);
    if (mode == 0) {
      idx[i] = (int)(z & ((1ull << scale) - 1));
    } else {
      int c = 0;
      for (int l = 0; l < scale; ++l) {
        z = smix(z + l);
        const double u = (z >> 11) * (1.0 / 9007199254740992.0);
        c = (c << 1) | (u >= 0.76 ? 1 : 0);
      }
      idx[i] = c;
    }
  }
}

int main() {
  const int scale = 20;
  const long long K = 1LL << scale;
  const long long n = 16LL << 20;
  int* idx;
  float *X, *out;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&out, 4);
  cudaMalloc(&X, K * 128);
  cudaMemset(X, 0, K * 128);
  float* flush;
  cudaMalloc(&flush, 256 << 20);

  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  for (int box1 : {1}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {32, (cuuint64_t)K};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32, (cuuint32_t)box1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode box1=%d -> %d\n", box1, (int)r);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode : {0, 1}) {
      fill_idx<<<1184, 256>>>(idx, n, scale, mode, 7);
      auto run = [&](const char* name, auto launch) {
        launch();
        float tot = 0;
        for (int rep = 0; rep < 5; ++rep) {
          cudaMemsetAsync(flush, rep, 256 << 20);
          cudaEventRecord(a);
          launch();
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          tot += ms;
        }
        const float ms = tot / 5;
        printf("%s %-34s %8.1f us  %7.1f GB/s gathered  (%s)\n", mode ? "rmat" : "unif", name, ms * 1e3,
               n * 128.0 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      };
#define RUN_TMA(S, G, WPB, BPS)                                                                    \
  {                                                                                               \
    const int blocks = 148 * BPS;                                                                 \
    const long long warps = (long long)blocks * WPB;                                              \
    long long pw = (n / warps) / G * G;                                                           \
    const int smem = WPB * S * G * 128 + WPB * S * 8;                                             \
    cudaFuncSetAttribute(gather_tma<S, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);    \
    char nm[96];                                                                                  \
    snprintf(nm, 96, "tma S%d G%d wpb%d bps%d", S, G, WPB, BPS);                                  \
    run(nm, [&] { gather_tma<S, G><<<blocks, WPB * 32, smem>>>(tm, idx, pw, out); });             \
  }
#define RUN_LDG(S, G, WPB, BPS)                                                                    \
  {                                                                                               \
    const int blocks = 148 * BPS;                                                                 \
    const long long warps = (long long)blocks * WPB;                                              \
    long long pw = (n / warps) / G * G;                                                           \
    const int smem = WPB * S * G * 128;                                                           \
    cudaFuncSetAttribute(gather_ldgsts<S, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    char nm[96];                                                                                  \
    snprintf(nm, 96, "ldgsts S%d G%d wpb%d bps%d", S, G, WPB, BPS);                               \
    run(nm, [&] { gather_ldgsts<S, G><<<blocks, WPB * 32, smem>>>(X, idx, pw, out); });           \
  }
      RUN_LDG(2, 32, 4, 8)
      RUN_LDG(2, 32, 8, 4)
      RUN_LDG(4, 16, 8, 4)
      RUN_TMA(2, 32, 4, 4)
      RUN_TMA(2, 32, 8, 2)
      RUN_TMA(4, 32, 4, 4)
      RUN_TMA(4, 32, 8, 2)
      RUN_TMA(4, 16, 8, 4)
      RUN_TMA(8, 16, 8, 2)
      RUN_TMA(4, 32, 16, 1)
      RUN_TMA(8, 32, 8, 1)
      RUN_TMA(3, 64, 4, 2)
      RUN_TMA(6, 32, 2, 8)
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
