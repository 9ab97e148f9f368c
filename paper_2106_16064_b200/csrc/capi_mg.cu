// capi_mg.cu — multi-GPU layer (spmk_mg_*): one process (or thread) per GPU,
// NCCL over NVLink 5 / NVSwitch.  SURVEY §8e: the row-partitioned configs
// (cfg4 SpMM, cfg5 iterative SpMV) cut A into equal-nnz row slices (the
// reference's static partition, kernels.hpp:124-129, applied to nonzeros),
// replicate X once, and let every rank write its own Y slice with the
// per-slice rule; only the iterative driver exchanges Y.  This replaces the
// reference's single-process parallel substrate (thread_pool.hpp:51-76).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2": the copy already in
// the process — torch's — or the system one), so the library loads and every
// single-GPU entry point works on hosts without NCCL; spmk_mg_* then return
// SPMK_ENCCL.  Types come from the system nccl.h (ABI-stable across 2.2x).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

using namespace spmk_host;

namespace {

struct NcclApi {
  void* so = nullptr;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      api.so = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.so) break;
    }
    if (!api.so) {
      api.err = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
#define SYM(field, name)                                                  \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.so, name)); \
  if (!api.field) {                                                       \
    api.err = std::string("NCCL symbol missing: ") + name;                \
    api.so = nullptr;                                                     \
    return;                                                               \
  }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Broadcast, "ncclBroadcast");
    SYM(AllReduce, "ncclAllReduce");
    SYM(AllGather, "ncclAllGather");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
    SYM(GetVersion, "ncclGetVersion");
#undef SYM
  });
  return api;
}

NcclApi* nccl() {
  NcclApi& api = nccl_api();
  return api.so ? &api : nullptr;
}

spmk_status nccl_missing() {
  return fail(SPMK_ENCCL, "NCCL unavailable: " + nccl_api().err);
}

struct NcclError {
  std::string msg;
};

#define NK(expr)                                                                        \
  do {                                                                                  \
    ncclResult_t _r = (expr);                                                           \
    if (_r != ncclSuccess) throw NcclError{std::string(#expr) + ": " + api->GetErrorString(_r)}; \
  } while (0)

}  // namespace

struct spmk_mg_s {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
};

extern "C" {

spmk_status spmk_mg_available(int* nccl_version) {
  NcclApi* api = nccl();
  if (!api) return nccl_missing();
  int v = 0;
  api->GetVersion(&v);
  if (nccl_version) *nccl_version = v;
  return SPMK_OK;
}

spmk_status spmk_mg_unique_id(void* id128) {
  if (!id128) return fail(SPMK_EINVAL, "null argument");
  NcclApi* api = nccl();
  if (!api) return nccl_missing();
  try {
    ncclUniqueId id;
    NK(api->GetUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id));
  } catch (const NcclError& e) {
    return fail(SPMK_ENCCL, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_mg_init(const void* id128, int nranks, int rank, int device, spmk_mg_t* out) {
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(SPMK_EINVAL, "bad argument");
  NcclApi* api = nccl();
  if (!api) return nccl_missing();
  DeviceGuard g(device);
  auto* mg = new spmk_mg_s;
  mg->rank = rank;
  mg->nranks = nranks;
  mg->device = device;
  try {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    NK(api->CommInitRank(&mg->comm, nranks, id, rank));
  } catch (const NcclError& e) {
    delete mg;
    return fail(SPMK_ENCCL, e.msg);
  }
  *out = mg;
  return SPMK_OK;
}

spmk_status spmk_mg_destroy(spmk_mg_t mg) {
  if (!mg) return SPMK_OK;
  NcclApi* api = nccl();
  if (api && mg->comm) {
    DeviceGuard g(mg->device);
    api->CommDestroy(mg->comm);
  }
  delete mg;
  return SPMK_OK;
}

spmk_status spmk_mg_info(spmk_mg_t mg, int* rank, int* nranks, int* device) {
  if (!mg) return fail(SPMK_EINVAL, "null communicator");
  if (rank) *rank = mg->rank;
  if (nranks) *nranks = mg->nranks;
  if (device) *device = mg->device;
  return SPMK_OK;
}

spmk_status spmk_mg_slice(spmk_mg_t mg, spmk_csr_t full, spmk_csr_t* slice, int64_t* row_begin,
                          int64_t* row_end) {
  if (!mg || !full || !slice) return fail(SPMK_EINVAL, "null argument");
  std::vector<int64_t> b((size_t)mg->nranks + 1);
  spmk_status st = spmk_row_slices(full, mg->nranks, b.data());
  if (st != SPMK_OK) return st;
  if (row_begin) *row_begin = b[mg->rank];
  if (row_end) *row_end = b[mg->rank + 1];
  return spmk_csr_slice(full, b[mg->rank], b[mg->rank + 1], mg->device, slice);
}

spmk_status spmk_mg_broadcast(spmk_mg_t mg, float* d_buf, int64_t count, int root, void* stream) {
  if (!mg || (!d_buf && count) || count < 0 || root < 0 || root >= mg->nranks)
    return fail(SPMK_EINVAL, "bad argument");
  NcclApi* api = nccl();
  if (!api) return nccl_missing();
  DeviceGuard g(mg->device);
  try {
    if (count) NK(api->Broadcast(d_buf, d_buf, (size_t)count, ncclFloat32, root, mg->comm, (cudaStream_t)stream));
  } catch (const NcclError& e) {
    return fail(SPMK_ENCCL, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_mg_allgather_x(spmk_mg_t mg, float* d_x, int64_t chunk, void* stream) {
  if (!mg || (!d_x && chunk) || chunk < 0) return fail(SPMK_EINVAL, "bad argument");
  NcclApi* api = nccl();
  if (!api) return nccl_missing();
  DeviceGuard g(mg->device);
  try {
    if (chunk)
      NK(api->AllGather(d_x + (size_t)mg->rank * (size_t)chunk, d_x, (size_t)chunk, ncclFloat32, mg->comm,
                        (cudaStream_t)stream));
  } catch (const NcclError& e) {
    return fail(SPMK_ENCCL, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_mg_allgather_rows(spmk_mg_t mg, float* d_y, const int64_t* row_bounds, int64_t n,
                                   void* stream) {
  if (!mg || !row_bounds || n < 0) return fail(SPMK_EINVAL, "bad argument");
  for (int g2 = 0; g2 < mg->nranks; ++g2)
    if (row_bounds[g2 + 1] < row_bounds[g2] || row_bounds[0] < 0)
      return fail(SPMK_EINVAL, "row_bounds must be non-decreasing");
  if (!d_y && row_bounds[mg->nranks] > 0 && n) return fail(SPMK_EINVAL, "null Y");
  NcclApi* api = nccl();
  if (!api) return nccl_missing();
  DeviceGuard g(mg->device);
  try {
    // one group: every rank's rows broadcast from their owner (slices are
    // unequal, so a padded all-gather would move up to 3.5x the bytes)
    NK(api->GroupStart());
    ncclResult_t first = ncclSuccess;
    for (int src = 0; src < mg->nranks; ++src) {
      const size_t cnt = (size_t)(row_bounds[src + 1] - row_bounds[src]) * (size_t)n;
      if (!cnt) continue;
      float* p = d_y + (size_t)row_bounds[src] * (size_t)n;
      ncclResult_t r = api->Broadcast(p, p, cnt, ncclFloat32, src, mg->comm, (cudaStream_t)stream);
      if (r != ncclSuccess && first == ncclSuccess) first = r;
    }
    NK(api->GroupEnd());
    NK(first);
  } catch (const NcclError& e) {
    return fail(SPMK_ENCCL, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_mg_allreduce_f64(spmk_mg_t mg, double* d_buf, int64_t count, void* stream) {
  if (!mg || (!d_buf && count) || count < 0) return fail(SPMK_EINVAL, "bad argument");
  NcclApi* api = nccl();
  if (!api) return nccl_missing();
  DeviceGuard g(mg->device);
  try {
    if (count) NK(api->AllReduce(d_buf, d_buf, (size_t)count, ncclFloat64, ncclSum, mg->comm, (cudaStream_t)stream));
  } catch (const NcclError& e) {
    return fail(SPMK_ENCCL, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_mg_allreduce_i32(spmk_mg_t mg, int32_t* d_buf, int64_t count, void* stream) {
  if (!mg || (!d_buf && count) || count < 0) return fail(SPMK_EINVAL, "bad argument");
  NcclApi* api = nccl();
  if (!api) return nccl_missing();
  DeviceGuard g(mg->device);
  try {
    if (count) NK(api->AllReduce(d_buf, d_buf, (size_t)count, ncclInt32, ncclSum, mg->comm, (cudaStream_t)stream));
  } catch (const NcclError& e) {
    return fail(SPMK_ENCCL, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_mg_barrier(spmk_mg_t mg, void* stream) {
  if (!mg) return fail(SPMK_EINVAL, "null communicator");
  DeviceGuard g(mg->device);
  int32_t* d = nullptr;
  try {
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMallocAsync(&d, 4, s));
    CK(cudaMemsetAsync(d, 0, 4, s));
    spmk_status st = spmk_mg_allreduce_i32(mg, d, 1, stream);
    CK(cudaFreeAsync(d, s));
    if (st != SPMK_OK) return st;
    CK(cudaStreamSynchronize(s));
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_mg_spmm(spmk_mg_t mg, spmk_csr_t slice, const spmk_thresholds* t, const spmk_kernel_config* cfg,
                         const float* d_x, int64_t n, float* d_y, void* stream, spmk_kernel_id* chosen) {
  if (!mg || !slice) return fail(SPMK_EINVAL, "null argument");
  if (slice->device != mg->device) return fail(SPMK_EINVAL, "slice is not on the communicator's device");
  // no collective: the slice's rows are this rank's alone (X already replicated)
  return spmk_spmm_auto(slice, t, cfg, d_x, n, d_y, stream, chosen);
}

}  // extern "C"
