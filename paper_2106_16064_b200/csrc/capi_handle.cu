// capi_handle.cu — the A operand handle (spmk_csr_t): upload, validation,
// resident row metadata, cached plans, features, selection and partition.
// Reference interfaces: CsrMatrix / validate / extract_features (csr.hpp),
// plan_balanced / partition / check_config / KernelStats (kernels.hpp),
// select_kernel (selector.hpp).  See include/spmk_capi.h.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "aux_kernels.cuh"
#include "internal.h"

using namespace spmk_dev;

namespace spmk_host {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

spmk_status fail(spmk_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

// ------------------------------------------------------------ tuning state
namespace {
struct Knob {
  const char* key;
  const char* env;
  long long Tuning::*field;
};
const Knob kKnobs[] = {
    {"seq_tile_nnz", "SPMK_SEQ_TILE_NNZ", &Tuning::seq_tile_nnz},
    {"seq_ext", "SPMK_SEQ_EXT", &Tuning::seq_ext},
    {"parws_ext", "SPMK_PARWS_EXT", &Tuning::parws_ext},
    {"parws_t", "SPMK_PARWS_T", &Tuning::parws_t},
    {"parrs_vl", "SPMK_PARRS_VL", &Tuning::parrs_vl},
    {"hub_nnz", "SPMK_HUB_NNZ", &Tuning::hub_nnz},
    {"hub_two_pass", "SPMK_HUB_TWO_PASS", &Tuning::hub_two_pass},
    {"hub_smem", "SPMK_HUB_SMEM", &Tuning::hub_smem},
    {"l2_persist", "SPMK_L2_PERSIST", &Tuning::l2_persist},
    {"parws_impl", "SPMK_PARWS_IMPL", &Tuning::parws_impl},
    {"parws_cpt", "SPMK_PARWS_CPT", &Tuning::parws_cpt},
    {"parws3", "SPMK_PARWS3", &Tuning::parws3},
    {"seq_impl", "SPMK_SEQ_IMPL", &Tuning::seq_impl},
    {"sell_cfg", "SPMK_SELL_CFG", &Tuning::sell_cfg},
};
}  // namespace

void Tuning::from_env() {
  for (const Knob& k : kKnobs) {
    const char* v = std::getenv(k.env);
    if (v && *v) this->*(k.field) = std::atoll(v);
  }
}
bool Tuning::set(const std::string& key, long long v) {
  for (const Knob& k : kKnobs)
    if (key == k.key) {
      this->*(k.field) = v;
      return true;
    }
  return false;
}
bool Tuning::get(const std::string& key, long long* v) const {
  for (const Knob& k : kKnobs)
    if (key == k.key) {
      *v = this->*(k.field);
      return true;
    }
  return false;
}

float* GrowBuffer::get(size_t n) {
  if (n > floats) {
    if (ptr) retired.push_back(ptr);
    ptr = nullptr;
    floats = 0;
    ptr = dev_alloc<float>(n);
    floats = n;
  }
  return ptr;
}
void GrowBuffer::release() {
  for (float* p : retired) cudaFree(p);
  retired.clear();
  cudaFree(ptr);
  ptr = nullptr;
  floats = 0;
}

namespace {

void free_handle(spmk_csr_s* h) {
  DeviceGuard g(h->device);
  if (h->side) cudaStreamSynchronize(h->side);
  if (h->has_last) cudaEventSynchronize(h->ev_last);
  if (h->own_rp) cudaFree(h->rp);
  if (h->own_col) cudaFree(h->col);
  if (h->own_val) cudaFree(h->val);
  cudaFree(h->hflag32);
  cudaFree(h->crp);
  cudaFree(h->rid);
  cudaFree(h->erow);
  for (auto& kv : h->plans) {
    cudaFree(kv.second.rlo);
    cudaFree(kv.second.desc);
    cudaFree(kv.second.longrows);
    cudaFree(kv.second.longinfo);
  }
  for (auto& kv : h->sell_plans) free_sell_plan(kv.second);
  h->scratch.release();
  for (auto& kv : h->hub_layouts) {
    cudaFree(kv.second.po);
    cudaFree(kv.second.segs);
  }
  h->hub_prod.release();
  if (h->side) {
    cudaStreamDestroy(h->side);
    cudaEventDestroy(h->ev_fork);
    cudaEventDestroy(h->ev_join);
  }
  if (h->ev_last) cudaEventDestroy(h->ev_last);
  for (int i = 0; i < spmk_csr_s::kStageSlots; ++i) {
    cudaFree(h->stage_x[i]);
    cudaFree(h->stage_y[i]);
    if (h->slot_done[i]) cudaEventDestroy(h->slot_done[i]);
  }
  delete h;
}

// Row metadata: non-empty compaction + moments (one-time, at create).
void build_meta(spmk_csr_s* h, cudaStream_t s) {
  const int m = (int)h->m;
  h->crp = dev_alloc<int>((size_t)m + 1);
  h->rid = dev_alloc<int>((size_t)m);
  h->erow = dev_alloc<int>((size_t)m);
  int* flag = dev_alloc<int>((size_t)m + 1);
  int* pos = dev_alloc<int>((size_t)m + 1);
  unsigned long long* mom = dev_alloc<unsigned long long>(4);
  CK(cudaMemsetAsync(mom, 0, 4 * sizeof(unsigned long long), s));
  if (m > 0) {
    nonempty_flag_kernel<<<grid_for(m), 256, 0, s>>>(h->rp, m, flag); LAUNCHED(1);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flag, pos, m + 1, s);
    void* tmp = dev_alloc<char>(tmp_bytes);
    CK(cudaMemsetAsync(flag + m, 0, sizeof(int), s));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, pos, m + 1, s);
    compact_scatter_kernel<<<grid_for(m), 256, 0, s>>>(h->rp, m, pos, h->crp, h->rid, h->erow); LAUNCHED(1);
    row_moments_kernel<<<grid_for(m), 256, 0, s>>>(h->rp, m, mom); LAUNCHED(1);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&h->mne, pos + m, sizeof(int), cudaMemcpyDeviceToHost, s));
    unsigned long long hm[4];
    CK(cudaMemcpyAsync(hm, mom, sizeof(hm), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(tmp);
    h->sum_len2 = hm[1];
    h->max_row = (long long)hm[2];
    h->nempty = m - h->mne;
  }
  // crp[mne] = nnz
  const int nnz32 = (int)h->nnz;
  CK(cudaMemcpyAsync(h->crp + h->mne, &nnz32, sizeof(int), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  cudaFree(flag);
  cudaFree(pos);
  cudaFree(mom);
}

}  // namespace

// Plan for a nonzero-split kernel: tiles of TS nonzeros made of CH-chunks.
// Segment-head flags of the 32-nonzero chunks (par_ws2.cuh), once per handle.
const unsigned* get_head_flags32(spmk_csr_s* h, cudaStream_t s) {
  if (h->hflag32) return h->hflag32;
  const long long words = (h->nnz + 31) / 32 + 1;
  unsigned* f = dev_alloc<unsigned>((size_t)words);
  CK(cudaMemsetAsync(f, 0, (size_t)words * 4, s));
  head_flags_kernel<<<grid_for((long long)h->mne + 1), 256, 0, s>>>(h->crp, h->mne, f); LAUNCHED(1);
  CK(cudaGetLastError());
  h->hflag32 = f;
  return f;
}

Plan& get_plan(spmk_csr_s* h, int kind, long long TS, long long CH, long long EXT, cudaStream_t s) {
  EXT = std::max(1LL, std::min(EXT, TS));
  auto key = std::make_tuple(kind, TS, CH, EXT);
  auto it = h->plans.find(key);
  if (it != h->plans.end()) return it->second;
  Plan p;
  p.TS = TS;
  p.CH = CH;
  p.EXT = EXT;
  p.ntiles = (h->nnz + TS - 1) / TS;
  p.rlo = dev_alloc<int>((size_t)p.ntiles + 1);
  tile_plan_kernel<<<grid_for(p.ntiles + 1), 256, 0, s>>>(h->crp, h->mne, p.ntiles, TS, p.rlo); LAUNCHED(1);
  p.desc = dev_alloc<int4>((size_t)p.ntiles);
  ws_tile_desc_kernel<<<grid_for(p.ntiles), 256, 0, s>>>(h->crp, p.rlo, p.ntiles, TS, EXT, h->nnz, p.desc); LAUNCHED(1);
  int* cnt = dev_alloc<int>(1);
  CK(cudaMemsetAsync(cnt, 0, sizeof(int), s));
  // upper bound on long rows: every long row crosses a tile boundary
  const long long cap = p.ntiles + 1;
  p.longrows = dev_alloc<int>((size_t)cap);
  if (h->mne > 0)
    long_rows_kernel<<<grid_for(h->mne), 256, 0, s>>>(h->crp, h->mne, TS, EXT, p.longrows, cnt); LAUNCHED(1);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&p.nlong, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  cudaFree(cnt);
  if (p.nlong > 0) {
    p.longinfo = dev_alloc<int4>((size_t)p.nlong);
    long_info_kernel<<<grid_for(p.nlong), 256, 0, s>>>(p.longrows, p.nlong, h->crp, h->rid, TS, CH, p.longinfo); LAUNCHED(1);
    CK(cudaGetLastError());
    // big rows first (stable partition on the host, once per plan)
    std::vector<int4> info((size_t)p.nlong);
    CK(cudaMemcpyAsync(info.data(), p.longinfo, sizeof(int4) * info.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    auto it2 = std::stable_partition(info.begin(), info.end(),
                                     [](const int4& d) { return d.w - d.z >= kFixupLaneMax; });
    p.nbig = (int)(it2 - info.begin());
    CK(cudaMemcpyAsync(p.longinfo, info.data(), sizeof(int4) * info.size(), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  return h->plans.emplace(key, p).first->second;
}

// Hub rows of the row-split variants (rows with >= L nonzeros, hub_kernels.cuh):
// device list longest first (launch order), host copy ascending.
Plan& get_hub_plan(spmk_csr_s* h, int L, cudaStream_t s) {
  auto key = std::make_tuple(4, (long long)L, 0LL, 0LL);
  auto it = h->plans.find(key);
  if (it != h->plans.end()) return it->second;
  Plan p;
  const long long cap = h->nnz / L + 1;
  int2* list = dev_alloc<int2>((size_t)cap);
  int* cnt = dev_alloc<int>(1);
  CK(cudaMemsetAsync(cnt, 0, sizeof(int), s));
  hub_rows_kernel<<<grid_for(h->mne), 256, 0, s>>>(h->crp, h->mne, L, list, cnt); LAUNCHED(1);
  CK(cudaGetLastError());
  int n = 0;
  CK(cudaMemcpyAsync(&n, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (n > 0) {
    std::vector<int2> hl((size_t)n);
    CK(cudaMemcpyAsync(hl.data(), list, sizeof(int2) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::sort(hl.begin(), hl.end(), [](int2 x, int2 y) { return x.y != y.y ? x.y > y.y : x.x < y.x; });
    std::vector<int> rows((size_t)n);
    for (int i = 0; i < n; ++i) rows[i] = hl[i].x;
    p.hlen.resize((size_t)n);
    for (int i = 0; i < n; ++i) p.hlen[i] = hl[i].y;
    p.longrows = dev_alloc<int>((size_t)n);
    CK(cudaMemcpyAsync(p.longrows, rows.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    std::sort(rows.begin(), rows.end());
    p.hrows = std::move(rows);
    CK(cudaStreamSynchronize(s));
  }
  p.nlong = n;
  cudaFree(list);
  cudaFree(cnt);
  return h->plans.emplace(key, p).first->second;
}

// Row-split tile descriptors, cached like a plan: tile t holds the whole rows
// that start in [t*TS, (t+1)*TS) (rlo of tile_plan_kernel), so tiles are
// nnz-balanced without ever splitting a row (the row-split contract).  With
// hub rows (hub plan `hub`), a tile holding hubs is cut into the runs of
// non-hub rows between them: the first run keeps the tile's slot, the others
// are appended; hub rows belong to no tile.
Plan& get_rs_desc(spmk_csr_s* h, long long TS, int L, const Plan* hub, cudaStream_t s) {
  auto key = std::make_tuple(3, TS, (long long)L, 0LL);
  auto it = h->plans.find(key);
  if (it != h->plans.end()) return it->second;
  Plan p;
  p.TS = TS;
  p.ntiles = (h->nnz + TS - 1) / TS;
  p.rlo = dev_alloc<int>((size_t)p.ntiles + 1);
  tile_plan_kernel<<<grid_for(p.ntiles + 1), 256, 0, s>>>(h->crp, h->mne, p.ntiles, TS, p.rlo); LAUNCHED(1);
  p.desc = dev_alloc<int4>((size_t)p.ntiles);
  rs_tile_desc_kernel<<<grid_for(p.ntiles), 256, 0, s>>>(h->crp, p.rlo, p.ntiles, p.desc); LAUNCHED(1);
  CK(cudaGetLastError());
  if (hub && !hub->hrows.empty()) {
    // one round trip: row metadata and descriptors down, edited, back up
    const std::vector<int>& hr = hub->hrows;
    std::vector<int> rlo((size_t)p.ntiles + 1), rp((size_t)h->mne + 1);
    std::vector<int4> desc((size_t)p.ntiles);
    CK(cudaMemcpyAsync(rlo.data(), p.rlo, sizeof(int) * rlo.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(rp.data(), h->crp, sizeof(int) * rp.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(desc.data(), p.desc, sizeof(int4) * desc.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (size_t i = 0; i < hr.size();) {
      // the tile whose rows [rlo[t], rlo[t+1]) contain hub row hr[i]
      const long long t = (long long)(std::upper_bound(rlo.begin(), rlo.end(), hr[i]) - rlo.begin()) - 1;
      const int r0 = rlo[t], r1 = rlo[t + 1];
      std::vector<int4> pieces;
      int a0 = r0;
      for (; i < hr.size() && hr[i] < r1; ++i) {
        if (hr[i] > a0) pieces.push_back(make_int4(a0, rp[a0], rp[hr[i]], MODE_NORMAL));
        a0 = hr[i] + 1;
      }
      if (a0 < r1) pieces.push_back(make_int4(a0, rp[a0], rp[r1], MODE_NORMAL));
      // an empty first run keeps the slot as an idle tile (start == end)
      desc[t] = pieces.empty() ? make_int4(r0, 0, 0, MODE_NORMAL) : pieces[0];
      for (size_t k = 1; k < pieces.size(); ++k) desc.push_back(pieces[k]);
    }
    if ((long long)desc.size() != p.ntiles) {
      cudaFree(p.desc);
      p.desc = nullptr;
      p.desc = dev_alloc<int4>(desc.size());
      p.ntiles = (long long)desc.size();
    }
    CK(cudaMemcpyAsync(p.desc, desc.data(), sizeof(int4) * desc.size(), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  return h->plans.emplace(key, p).first->second;
}

void launch_zero_all(float* y, long long total, cudaStream_t s) {
  zero_all_kernel<<<grid_for(total), 256, 0, s>>>(y, total); LAUNCHED(1);
}

void launch_zero_rows(const spmk_csr_s* h, int N, float* y, bool vec4, cudaStream_t s) {
  if (vec4) {
    zero_rows_kernel<4><<<grid_for((long long)h->nempty * N / 4), 256, 0, s>>>(h->erow, h->nempty, N, y); LAUNCHED(1);
  } else {
    zero_rows_kernel<1><<<grid_for((long long)h->nempty * N), 256, 0, s>>>(h->erow, h->nempty, N, y); LAUNCHED(1);
  }
}

void launch_fixup(const Plan& p, const float* H, const float* Tsl, float* y, int N, cudaStream_t s) {
  fixup_kernel<<<fixup_blocks(p.nlong, p.nbig, N), kFixupWarps * 32, 0, s>>>(p.longinfo, p.nlong, p.nbig, H, Tsl,
                                                                              y, N); LAUNCHED(1);
}

spmk_status create_from_device32(long long m, long long k, long long nnz, int* rp, int* col, float* val,
                                 bool own, int device, spmk_csr_t* out, cudaStream_t s) {
  auto* h = new spmk_csr_s;
  h->device = device;
  h->m = m;
  h->k = k;
  h->nnz = nnz;
  h->rp = rp;
  h->col = col;
  h->val = val;
  h->own_rp = h->own_col = h->own_val = own;
  h->tune.from_env();
  try {
    int* err = dev_alloc<int>(1);
    unsigned* starts = dev_alloc<unsigned>((size_t)(nnz + 31) / 32);
    CK(cudaMemsetAsync(err, 0, sizeof(int), s));
    CK(cudaMemsetAsync(starts, 0, sizeof(unsigned) * (size_t)((nnz + 31) / 32 ? (nnz + 31) / 32 : 1), s));
    validate_rows_kernel<<<grid_for(std::max(m, 1LL)), 256, 0, s>>>(rp, (int)m, nnz, starts, err); LAUNCHED(1);
    if (nnz > 0) {
      validate_cols_kernel<<<grid_for(nnz, 256, 148 * 32), 256, 0, s>>>(col, nnz, (int)k, starts, err); LAUNCHED(1);
    }
    CK(cudaGetLastError());
    int herr = 0;
    CK(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(err);
    cudaFree(starts);
    // Safety (row_ptr shape, column range) is required by the device path; the
    // strict column order of csr.hpp:95-119 is not (every kernel follows
    // position order, as the reference's spmm_* do on non-canonical input), so
    // it is recorded and reported by spmk_csr_validate instead.
    if (herr & 3) {
      free_handle(h);
      return fail(SPMK_EINVAL, (herr & 1) ? "row_ptr malformed (csr.hpp:95-119)" : "column index out of range");
    }
    h->canonical = !(herr & 4);
    build_meta(h, s);
  } catch (const CudaError& e) {
    free_handle(h);
    return fail(e.st, e.msg);
  }
  *out = h;
  return SPMK_OK;
}

}  // namespace spmk_host

using namespace spmk_host;

// =============================================================== C ABI
extern "C" {

const char* spmk_last_error(void) { return g_err.c_str(); }
int spmk_version(void) { return SPMK_CAPI_VERSION; }
uint64_t spmk_launch_count(void) { return g_launches.load(); }

void spmk_default_config(spmk_kernel_config* cfg) {
  cfg->lane_width = 32;
  cfg->vdl_group = 0;
  cfg->seq_chunk = 256;
  cfg->worker_count = 0;
}
void spmk_default_thresholds(spmk_thresholds* t) {
  t->n_parallel_max = 4;
  t->t_parallel_avg = 32.0;
  t->t_cv = 1.0;
}

spmk_status spmk_check_config(const spmk_kernel_config* cfg) {
  if (!cfg) return SPMK_OK;
  if (!is_pow2(cfg->lane_width) || cfg->lane_width < 2 || cfg->lane_width > 64)
    return fail(SPMK_EINVAL, "lane_width must be a power of two in [2, 64]");
  if (cfg->vdl_group != 0 && cfg->vdl_group != 1 && cfg->vdl_group != 2 && cfg->vdl_group != 4)
    return fail(SPMK_EINVAL, "vdl_group must be 0 (auto), 1, 2 or 4");
  if (cfg->seq_chunk < 1) return fail(SPMK_EINVAL, "seq_chunk must be >= 1");
  if (cfg->seq_chunk > (1ull << 30)) return fail(SPMK_EUNSUPPORTED, "seq_chunk too large for the device path");
  return SPMK_OK;
}

const char* spmk_kernel_name(spmk_kernel_id id) {
  switch (id) {
    case SPMK_PAR_ROWSPLIT: return "par-rs";
    case SPMK_PAR_BALANCED: return "par-ws";
    case SPMK_SEQ_ROWSPLIT: return "seq-rs";
    default: return "seq-ws";
  }
}

spmk_status spmk_parse_kernel(const char* name, spmk_kernel_id* out) {
  for (int i = 0; i < 4; ++i) {
    if (std::strcmp(name, spmk_kernel_name((spmk_kernel_id)i)) == 0) {
      *out = (spmk_kernel_id)i;
      return SPMK_OK;
    }
  }
  return fail(SPMK_EINVAL, std::string("unknown kernel name: ") + name);
}

spmk_status spmk_csr_create(int64_t num_rows, int64_t num_cols, int64_t nnz,
                            const int64_t* row_ptr, const int64_t* col_idx,
                            const float* values, int device, spmk_csr_t* out) {
  if (!out || !row_ptr || (nnz > 0 && (!col_idx || !values)))
    return fail(SPMK_EINVAL, "null argument");
  if (num_rows < 0 || num_cols < 0 || nnz < 0) return fail(SPMK_EINVAL, "negative dimension");
  if (num_rows >= INT32_MAX || num_cols >= INT32_MAX || nnz >= INT32_MAX)
    return fail(SPMK_EUNSUPPORTED, "device path narrows indices to int32 (need < 2^31)");
  if (row_ptr[0] != 0 || row_ptr[num_rows] != nnz)
    return fail(SPMK_EINVAL, "row_ptr[0] must be 0 and row_ptr[M] must equal nnz");
  DeviceGuard g(device);
  cudaStream_t s = nullptr;
  int *rp = nullptr, *col = nullptr;
  float* val = nullptr;
  long long* tmp = nullptr;
  int* bad = nullptr;
  try {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    rp = dev_alloc<int>((size_t)num_rows + 1);
    col = dev_alloc<int>((size_t)nnz);
    val = dev_alloc<float>((size_t)nnz);
    const long long chunk = 1LL << 24;
    tmp = dev_alloc<long long>((size_t)std::min<long long>(chunk, std::max<long long>(nnz, num_rows + 1)));
    bad = dev_alloc<int>(1);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
    auto narrow = [&](const int64_t* src, int* dst, long long n) {
      for (long long o = 0; o < n; o += chunk) {
        const long long c = std::min(chunk, n - o);
        CK(cudaMemcpyAsync(tmp, src + o, c * 8, cudaMemcpyHostToDevice, s));
        narrow_kernel<<<grid_for(c), 256, 0, s>>>(tmp, dst + o, c, bad); LAUNCHED(1);
        CK(cudaGetLastError());
      }
    };
    narrow(row_ptr, rp, num_rows + 1);
    narrow(col_idx, col, nnz);
    if (nnz) CK(cudaMemcpyAsync(val, values, nnz * 4, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    int hbad = 0;
    CK(cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(tmp);
    cudaFree(bad);
    tmp = nullptr;
    bad = nullptr;
    if (hbad) {
      cudaFree(rp);
      cudaFree(col);
      cudaFree(val);
      cudaStreamDestroy(s);
      return fail(SPMK_EINVAL, "index out of int32 range");
    }
    spmk_status st = create_from_device32(num_rows, num_cols, nnz, rp, col, val, true, device, out, s);
    cudaStreamDestroy(s);
    return st;
  } catch (const CudaError& e) {
    cudaFree(rp);
    cudaFree(col);
    cudaFree(val);
    cudaFree(tmp);
    cudaFree(bad);
    if (s) cudaStreamDestroy(s);
    return fail(e.st, e.msg);
  }
}

spmk_status spmk_csr_create_device(int64_t num_rows, int64_t num_cols, int64_t nnz,
                                   const int32_t* d_row_ptr, const int32_t* d_col_idx,
                                   const float* d_values, int copy, spmk_csr_t* out) {
  if (!out || !d_row_ptr) return fail(SPMK_EINVAL, "null argument");
  if (num_rows < 0 || num_cols < 0 || nnz < 0) return fail(SPMK_EINVAL, "negative dimension");
  if (num_rows >= INT32_MAX || num_cols >= INT32_MAX || nnz >= INT32_MAX)
    return fail(SPMK_EUNSUPPORTED, "device path needs indices < 2^31");
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, d_row_ptr) != cudaSuccess || attr.type != cudaMemoryTypeDevice)
    return fail(SPMK_EINVAL, "d_row_ptr is not device memory");
  const int device = attr.device;
  DeviceGuard g(device);
  cudaStream_t s = nullptr;
  try {
    // the arrays may still be in flight on any of the caller's streams
    CK(cudaDeviceSynchronize());
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int* rp = const_cast<int*>(d_row_ptr);
    int* col = const_cast<int*>(d_col_idx);
    float* val = const_cast<float*>(d_values);
    if (copy) {
      rp = dev_alloc<int>((size_t)num_rows + 1);
      col = dev_alloc<int>((size_t)nnz);
      val = dev_alloc<float>((size_t)nnz);
      CK(cudaMemcpyAsync(rp, d_row_ptr, (num_rows + 1) * 4, cudaMemcpyDeviceToDevice, s));
      if (nnz) {
        CK(cudaMemcpyAsync(col, d_col_idx, nnz * 4, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(val, d_values, nnz * 4, cudaMemcpyDeviceToDevice, s));
      }
    }
    spmk_status st = create_from_device32(num_rows, num_cols, nnz, rp, col, val, copy != 0, device, out, s);
    cudaStreamDestroy(s);
    return st;
  } catch (const CudaError& e) {
    if (s) cudaStreamDestroy(s);
    return fail(e.st, e.msg);
  }
}

spmk_status spmk_csr_slice(spmk_csr_t a, int64_t row_begin, int64_t row_end, int device,
                           spmk_csr_t* out) {
  if (!a || !out || row_begin < 0 || row_end < row_begin || row_end > a->m)
    return fail(SPMK_EINVAL, "bad slice");
  try {
    int rp_b = 0, rp_e = 0;
    {
      DeviceGuard g(a->device);
      CK(cudaMemcpy(&rp_b, a->rp + row_begin, 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&rp_e, a->rp + row_end, 4, cudaMemcpyDeviceToHost));
    }
    const long long rows = row_end - row_begin, nnz = rp_e - rp_b;
    DeviceGuard g(device);
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int* rp = dev_alloc<int>((size_t)rows + 1);
    int* col = dev_alloc<int>((size_t)nnz);
    float* val = dev_alloc<float>((size_t)nnz);
    int* rpsrc = a->rp;
    int* tmp = nullptr;
    if (device != a->device) {
      tmp = dev_alloc<int>((size_t)rows + 1);
      CK(cudaMemcpyPeerAsync(tmp, device, a->rp + row_begin, a->device, (rows + 1) * 4, s));
      CK(cudaMemcpyPeerAsync(col, device, a->col + rp_b, a->device, nnz * 4, s));
      CK(cudaMemcpyPeerAsync(val, device, a->val + rp_b, a->device, nnz * 4, s));
      rebase_kernel<<<grid_for(rows + 1), 256, 0, s>>>(tmp, 0, rows, rp); LAUNCHED(1);
    } else {
      CK(cudaMemcpyAsync(col, a->col + rp_b, nnz * 4, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(val, a->val + rp_b, nnz * 4, cudaMemcpyDeviceToDevice, s));
      rebase_kernel<<<grid_for(rows + 1), 256, 0, s>>>(rpsrc, row_begin, rows, rp); LAUNCHED(1);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    if (tmp) cudaFree(tmp);
    spmk_status st = create_from_device32(rows, a->k, nnz, rp, col, val, true, device, out, s);
    if (st == SPMK_OK) (*out)->tune = a->tune;  // a slice keeps its parent's knobs
    cudaStreamDestroy(s);
    return st;
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
}

spmk_status spmk_csr_abs_copy(spmk_csr_t a, spmk_csr_t* out) {
  if (!a || !out) return fail(SPMK_EINVAL, "null argument");
  DeviceGuard g(a->device);
  cudaStream_t s = nullptr;
  try {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int* rp = dev_alloc<int>((size_t)a->m + 1);
    int* col = dev_alloc<int>((size_t)a->nnz);
    float* val = dev_alloc<float>((size_t)a->nnz);
    CK(cudaMemcpyAsync(rp, a->rp, (a->m + 1) * 4, cudaMemcpyDeviceToDevice, s));
    if (a->nnz) {
      CK(cudaMemcpyAsync(col, a->col, a->nnz * 4, cudaMemcpyDeviceToDevice, s));
      abs_copy_kernel<<<grid_for(a->nnz), 256, 0, s>>>(a->val, val, a->nnz); LAUNCHED(1);
      CK(cudaGetLastError());
    }
    spmk_status st = create_from_device32(a->m, a->k, a->nnz, rp, col, val, true, a->device, out, s);
    if (st == SPMK_OK) (*out)->tune = a->tune;
    cudaStreamDestroy(s);
    return st;
  } catch (const CudaError& e) {
    if (s) cudaStreamDestroy(s);
    return fail(e.st, e.msg);
  }
}

spmk_status spmk_csr_destroy(spmk_csr_t a) {
  if (a) free_handle(a);
  return SPMK_OK;
}

spmk_status spmk_csr_validate(spmk_csr_t a) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  if (!a->canonical) return fail(SPMK_EINVAL, "columns not strictly increasing within a row (csr.hpp:95-119)");
  return SPMK_OK;
}

spmk_status spmk_csr_set_tuning(spmk_csr_t a, const char* key, int64_t value) {
  if (!a || !key) return fail(SPMK_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(a->mu);
  if (!a->tune.set(key, value)) return fail(SPMK_EINVAL, std::string("unknown tuning key: ") + key);
  return SPMK_OK;
}

spmk_status spmk_csr_get_tuning(spmk_csr_t a, const char* key, int64_t* value) {
  if (!a || !key || !value) return fail(SPMK_EINVAL, "null argument");
  long long v = 0;
  if (!a->tune.get(key, &v)) return fail(SPMK_EINVAL, std::string("unknown tuning key: ") + key);
  *value = v;
  return SPMK_OK;
}

spmk_status spmk_csr_info(spmk_csr_t a, int64_t* num_rows, int64_t* num_cols, int64_t* nnz,
                          int64_t* max_row_nnz, int64_t* empty_rows) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  if (num_rows) *num_rows = a->m;
  if (num_cols) *num_cols = a->k;
  if (nnz) *nnz = a->nnz;
  if (max_row_nnz) *max_row_nnz = a->max_row;
  if (empty_rows) *empty_rows = a->nempty;
  return SPMK_OK;
}

spmk_status spmk_csr_device_arrays(spmk_csr_t a, const int32_t** d_row_ptr,
                                   const int32_t** d_col_idx, const float** d_values) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  if (d_row_ptr) *d_row_ptr = a->rp;
  if (d_col_idx) *d_col_idx = a->col;
  if (d_values) *d_values = a->val;
  return SPMK_OK;
}

spmk_status spmk_csr_download(spmk_csr_t a, int64_t* row_ptr, int64_t* col_idx, float* values) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  DeviceGuard g(a->device);
  try {
    auto widen = [&](const int* src, int64_t* dst, long long n) {
      if (!dst || n == 0) return;
      long long* tmp = dev_alloc<long long>((size_t)n);
      widen_kernel<<<grid_for(n), 256>>>(src, tmp, n); LAUNCHED(1);
      CK(cudaGetLastError());
      CK(cudaMemcpy(dst, tmp, n * 8, cudaMemcpyDeviceToHost));
      cudaFree(tmp);
    };
    widen(a->rp, row_ptr, a->m + 1);
    widen(a->col, col_idx, a->nnz);
    if (values && a->nnz) CK(cudaMemcpy(values, a->val, a->nnz * 4, cudaMemcpyDeviceToHost));
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

// csr.hpp:166-181, sequential double sum (the reference order).
spmk_status spmk_features_host(int64_t num_rows, const int64_t* row_ptr, spmk_features* out) {
  if (num_rows < 1) return fail(SPMK_EINVAL, "extract_features requires num_rows >= 1");
  const long long nnz = row_ptr[num_rows];
  out->num_rows = num_rows;
  out->nnz = nnz;
  out->avg_row = (double)nnz / (double)num_rows;
  double ss = 0.0;
  for (long long i = 0; i < num_rows; ++i) {
    const double d = (double)(row_ptr[i + 1] - row_ptr[i]) - out->avg_row;
    ss += d * d;
  }
  out->stdv_row = std::sqrt(ss / (double)num_rows);
  out->cv = out->avg_row == 0.0 ? 0.0 : out->stdv_row / out->avg_row;
  return SPMK_OK;
}

spmk_status spmk_features_compute(spmk_csr_t a, spmk_features* out) {
  if (!a || !out) return fail(SPMK_EINVAL, "null argument");
  if (a->m < 1) return fail(SPMK_EINVAL, "extract_features requires num_rows >= 1");
  // exact integer moments (computed at create); host finalize
  const long double m = (long double)a->m, nnz = (long double)a->nnz;
  out->num_rows = a->m;
  out->nnz = a->nnz;
  out->avg_row = (double)a->nnz / (double)a->m;  // bit-identical to csr.hpp:170
  long double ss = (long double)a->sum_len2 - nnz * nnz / m;
  if (ss < 0) ss = 0;
  out->stdv_row = (double)std::sqrt(ss / m);
  out->cv = out->avg_row == 0.0 ? 0.0 : out->stdv_row / out->avg_row;
  return SPMK_OK;
}

spmk_kernel_id spmk_select(const spmk_features* f, uint64_t n, const spmk_thresholds* t) {
  spmk_thresholds d;
  spmk_default_thresholds(&d);
  const spmk_thresholds& th = t ? *t : d;
  if (n <= th.n_parallel_max) return f->avg_row < th.t_parallel_avg ? SPMK_PAR_BALANCED : SPMK_PAR_ROWSPLIT;
  return f->cv > th.t_cv ? SPMK_SEQ_BALANCED : SPMK_SEQ_ROWSPLIT;
}

spmk_status spmk_select_for(spmk_csr_t a, uint64_t n, const spmk_thresholds* t,
                            spmk_kernel_id* out) {
  spmk_features f;
  spmk_status st = spmk_features_compute(a, &f);
  if (st != SPMK_OK) return st;
  spmk_thresholds d;
  spmk_default_thresholds(&d);
  const spmk_thresholds& th = t ? *t : d;
  // tie-guard: near a threshold recompute in the reference's exact order
  if (std::fabs(f.cv - th.t_cv) <= 1e-9 * std::fabs(th.t_cv)) {
    std::vector<int64_t> rp((size_t)a->m + 1);
    st = spmk_csr_download(a, rp.data(), nullptr, nullptr);
    if (st != SPMK_OK) return st;
    spmk_features_host(a->m, rp.data(), &f);
  }
  *out = spmk_select(&f, n, &th);
  return SPMK_OK;
}

spmk_status spmk_plan(spmk_csr_t a, int64_t chunk, int64_t* chunk_first_row, int64_t* num_chunks) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  if (chunk < 1) return fail(SPMK_EINVAL, "chunk_size must be >= 1");
  const long long nch = (a->nnz + chunk - 1) / chunk;
  if (num_chunks) *num_chunks = nch;
  if (!chunk_first_row || nch == 0) return SPMK_OK;
  DeviceGuard g(a->device);
  try {
    long long* d = dev_alloc<long long>((size_t)nch);
    chunk_first_row_kernel<<<grid_for(nch), 256>>>(a->rp, (int)a->m, nch, chunk, d); LAUNCHED(1);
    CK(cudaGetLastError());
    CK(cudaMemcpy(chunk_first_row, d, nch * 8, cudaMemcpyDeviceToHost));
    cudaFree(d);
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_plan_elem_row(spmk_csr_t a, int64_t* elem_row) {
  if (!a || !elem_row) return fail(SPMK_EINVAL, "null argument");
  if (a->nnz == 0) return SPMK_OK;
  DeviceGuard g(a->device);
  try {
    long long* d = dev_alloc<long long>((size_t)a->nnz);
    elem_row_kernel<<<grid_for(a->nnz), 256>>>(a->rp, (int)a->m, a->nnz, d); LAUNCHED(1);
    CK(cudaGetLastError());
    CK(cudaMemcpy(elem_row, d, a->nnz * 8, cudaMemcpyDeviceToHost));
    cudaFree(d);
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

void spmk_partition(int64_t items, int64_t parts, int64_t w, int64_t* lo, int64_t* hi) {
  *lo = items * w / parts;
  *hi = items * (w + 1) / parts;
}

spmk_status spmk_row_slices(spmk_csr_t a, int64_t parts, int64_t* bounds) {
  if (!a || !bounds || parts < 1) return fail(SPMK_EINVAL, "bad argument");
  DeviceGuard g(a->device);
  try {
    long long* d = dev_alloc<long long>((size_t)parts + 1);
    row_slices_kernel<<<grid_for(parts + 1), 256>>>(a->rp, (int)a->m, a->nnz, parts, d); LAUNCHED(1);
    CK(cudaGetLastError());
    CK(cudaMemcpy(bounds, d, (parts + 1) * 8, cudaMemcpyDeviceToHost));
    cudaFree(d);
    for (int64_t g2 = 1; g2 <= parts; ++g2)
      if (bounds[g2] < bounds[g2 - 1]) bounds[g2] = bounds[g2 - 1];
  } catch (const CudaError& e) {
    return fail(e.st, e.msg);
  }
  return SPMK_OK;
}

spmk_status spmk_kernel_stats(spmk_csr_t a, spmk_kernel_id id, const spmk_kernel_config* cfg,
                              int64_t n, uint64_t* lane_multiplies, uint64_t* scan_ops) {
  if (!a) return fail(SPMK_EINVAL, "null handle");
  spmk_status st = spmk_check_config(cfg);
  if (st != SPMK_OK) return st;
  spmk_kernel_config c;
  spmk_default_config(&c);
  if (cfg) c = *cfg;
  *lane_multiplies = 0;
  *scan_ops = 0;
  if (n == 0 || id == SPMK_SEQ_ROWSPLIT || id == SPMK_SEQ_BALANCED) return SPMK_OK;
  const uint64_t w = c.lane_width;
  uint64_t levels = 0;
  for (uint64_t off = 1; off < w; off <<= 1) ++levels;
  int64_t group = c.vdl_group ? (int64_t)c.vdl_group : (n >= 4 ? 4 : n >= 2 ? 2 : 1);
  if (group > n) group = n;
  const uint64_t wc_sum = (uint64_t)((n / group) * group + (n % group));
  if (id == SPMK_PAR_ROWSPLIT) {
    // sum over non-empty rows of ceil(len/W) * W (kernels.hpp:187)
    std::vector<int64_t> rp((size_t)a->m + 1);
    st = spmk_csr_download(a, rp.data(), nullptr, nullptr);
    if (st != SPMK_OK) return st;
    uint64_t lm = 0, rows = 0;
    for (int64_t i = 0; i < a->m; ++i) {
      const uint64_t len = (uint64_t)(rp[i + 1] - rp[i]);
      if (!len) continue;
      lm += (len + w - 1) / w * w;
      ++rows;
    }
    *lane_multiplies = lm * wc_sum;
    *scan_ops = rows * levels * w * wc_sum;
  } else {
    if (a->nnz == 0) return SPMK_OK;
    const uint64_t chunks = ((uint64_t)a->nnz + w - 1) / w;
    *lane_multiplies = chunks * w * wc_sum;
    *scan_ops = chunks * levels * w * wc_sum;
  }
  return SPMK_OK;
}

double spmk_kernel_tolerance(int64_t max_row_nnz) {
  return 1e-5 * std::log2((double)max_row_nnz + 2.0);
}

}  // extern "C"
