// aux_kernels.cuh — partition, features, row metadata, fix-up, zero-fill and
// validation kernels (integer work; bit-exact by construction).
#pragma once
#include "common.cuh"

namespace spmk_dev {

__device__ __forceinline__ long long lower_bound_i32(const int* __restrict__ a,
                                                     long long n, long long v) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if ((long long)a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ long long upper_bound_i32(const int* __restrict__ a,
                                                     long long n, long long v) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if ((long long)a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// int64 (reference Index) -> int32 device narrowing, with overflow flag.
__global__ void narrow_kernel(const long long* __restrict__ in, int* __restrict__ out,
                              long long n, int* __restrict__ bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long v = in[i];
    if (v < INT32_MIN || v > INT32_MAX) *bad = 1;
    out[i] = (int)v;
  }
}
__global__ void widen_kernel(const int* __restrict__ in, long long* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i];
}

// validate (csr.hpp:95-119) on the device, nonzero-parallel.  err bits:
// 1 row_ptr, 2 column range, 4 column order.  Pass 1 (one thread per row)
// checks row_ptr and marks every row start in a bitmap; pass 2 (one thread per
// nonzero) checks the column range and, unless the position starts a row, the
// strict order against its predecessor.  Work is O(M + nnz) with no serial
// per-row loop, so hub rows cost nothing extra.
__global__ void validate_rows_kernel(const int* __restrict__ rp, int m, long long nnz,
                                     unsigned* __restrict__ starts, int* __restrict__ err) {
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = rp[i], f = rp[i + 1];
    if (s > f || s < 0 || f > nnz) {
      bad |= 1;
    } else if (s < f) {
      atomicOr(starts + (s >> 5), 1u << (s & 31));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (rp[0] != 0 || (long long)rp[m] != nnz) bad |= 1;
  }
  if (bad) atomicOr(err, bad);
}
__global__ void validate_cols_kernel(const int* __restrict__ col, long long nnz, int k,
                                     const unsigned* __restrict__ starts, int* __restrict__ err) {
  int bad = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = col[e];
    if (c < 0 || c >= k) bad |= 2;
    if (e > 0 && !((starts[e >> 5] >> (e & 31)) & 1u) && c <= col[e - 1]) bad |= 4;
  }
  if (bad) atomicOr(err, bad);
}

// row-length moments for extract_features (csr.hpp:166-181): exact integer
// sums sum(len), sum(len^2), max(len).  Order-independent => deterministic.
__global__ void row_moments_kernel(const int* __restrict__ rp, int m,
                                   unsigned long long* __restrict__ out /*3*/) {
  unsigned long long s1 = 0, s2 = 0, mx = 0, ne = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long l = (unsigned long long)(rp[i + 1] - rp[i]);
    s1 += l;
    s2 += l * l;
    mx = l > mx ? l : mx;
    ne += l == 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
    ne += __shfl_xor_sync(0xffffffffu, ne, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out + 0, s1);
    atomicAdd(out + 1, s2);
    atomicMax(out + 2, mx);
    atomicAdd(out + 3, ne);
  }
}

// Non-empty row compaction: flags -> (exclusive scan on host-driven CUB) ->
// scatter.  crp[pos] = rp[i] for non-empty rows, erow = empty rows.
__global__ void nonempty_flag_kernel(const int* __restrict__ rp, int m, int* __restrict__ flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    flag[i] = rp[i + 1] > rp[i] ? 1 : 0;
}
__global__ void compact_scatter_kernel(const int* __restrict__ rp, int m,
                                       const int* __restrict__ pos /*exclusive scan*/,
                                       int* __restrict__ crp, int* __restrict__ rid,
                                       int* __restrict__ erow) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const int p = pos[i];
    if (rp[i + 1] > rp[i]) {
      crp[p] = rp[i];
      rid[p] = (int)i;
    } else {
      erow[i - p] = (int)i;
    }
  }
}

// Segment heads of the 32-nonzero chunks: bit (p & 31) of word p >> 5 for
// every row start p = crp[r] (non-empty rows, so distinct positions), plus a
// phantom head at p = nnz = crp[mne] closing the last row.
__global__ void head_flags_kernel(const int* __restrict__ crp, int mne, unsigned* __restrict__ f) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r <= mne;
       r += (long long)gridDim.x * blockDim.x) {
    const unsigned p = (unsigned)crp[r];
    atomicOr(f + (p >> 5), 1u << (p & 31));
  }
}

// Tile plan: rlo[t] = lower_bound(crp, t*TS) for t < ntiles, rlo[ntiles] = mne.
__global__ void tile_plan_kernel(const int* __restrict__ crp, int mne, long long ntiles,
                                 long long TS, int* __restrict__ rlo) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t <= ntiles;
       t += (long long)gridDim.x * blockDim.x) {
    rlo[t] = (t == ntiles) ? mne : (int)lower_bound_i32(crp, (long long)mne + 1, t * TS);
  }
}
// Per-tile start descriptors (the "K-p" partition plan, computed once per
// handle and tile shape).  {cur, start, hard_end, mode}:
//   nonzero-split tiles [t*TS, min((t+1)*TS, nnz)):
//     cur      compact row containing the first position swept
//     start    first position swept (> tile start when the entering row is
//              short and therefore finished by the tile that owns its start)
//     hard_end last position+1 swept: the tile end, or the end of the row
//              crossing it when that row ends in the next tile (owner extends)
//     mode     MODE_ENTER_LONG when the entering row spans >= 2 tile
//              boundaries (its per-chunk partials go to the H slots), else 0;
//              start == hard_end marks an empty tile.
//   row-split tiles (RB compact rows each): {r0, crp[r0], crp[r1], 0}.
// A row crossing exactly one tile boundary B and ending at f <= B + EXT is
// finished by the tile that owns its start ("owner extends"); every other
// boundary-crossing row is "long" (per-chunk partials + owner prefix, merged
// by fixup_kernel).  EXT <= TS; EXT bounds the extra work of one unit.
__device__ __forceinline__ bool row_is_long(long long s, long long f, long long TS, long long EXT) {
  const long long b0 = s / TS, b1 = (f - 1) / TS;
  return b1 - b0 >= 2 || (b1 - b0 == 1 && f > (b0 + 1) * TS + EXT);
}
__global__ void ws_tile_desc_kernel(const int* __restrict__ crp, const int* __restrict__ rlo,
                                    long long ntiles, long long TS, long long EXT, long long nnz,
                                    int4* __restrict__ desc) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ntiles;
       t += (long long)gridDim.x * blockDim.x) {
    const long long tb = t * TS;
    const long long te = min(tb + TS, nnz);
    const int r = rlo[t];
    long long hard_end = te;
    if (te < nnz) {
      const int r2 = rlo[t + 1];
      const long long c2 = crp[r2];
      if (c2 > te && crp[r2 - 1] >= tb && c2 <= te + EXT) hard_end = c2;
    }
    int cur = r, mode = MODE_NORMAL;
    long long start = tb;
    const long long cr = crp[r];
    if (cr > tb) {  // row r-1 enters from the left
      const long long rs = crp[r - 1];
      if (row_is_long(rs, cr, TS, EXT)) {
        cur = r - 1;
        mode = MODE_ENTER_LONG;
      } else {
        start = cr;
        if (start >= te) hard_end = start;  // nothing to do
      }
    }
    desc[t] = make_int4(cur, (int)start, (int)hard_end, mode);
  }
}
__global__ void rs_tile_desc_kernel(const int* __restrict__ crp, const int* __restrict__ rlo, long long ntiles,
                                    int4* __restrict__ desc) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ntiles;
       t += (long long)gridDim.x * blockDim.x) {
    const int r0 = rlo[t], r1 = rlo[t + 1];
    desc[t] = make_int4(r0, crp[r0], crp[r1], MODE_NORMAL);
  }
}
// Long rows for a tile size: rows spanning >= 2 tile boundaries past their own.
__global__ void long_rows_kernel(const int* __restrict__ crp, int mne, long long TS, long long EXT,
                                 int* __restrict__ list, int* __restrict__ count) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < mne;
       c += (long long)gridDim.x * blockDim.x) {
    if (row_is_long(crp[c], crp[c + 1], TS, EXT)) list[atomicAdd(count, 1)] = (int)c;
  }
}
// plan_balanced (kernels.hpp:133-149) chunk starts: elem_row[q*chunk] =
// upper_bound(rowPtr, q*chunk) - 1.
__global__ void chunk_first_row_kernel(const int* __restrict__ rp, int m, long long nchunks,
                                       long long chunk, long long* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nchunks;
       q += (long long)gridDim.x * blockDim.x)
    out[q] = upper_bound_i32(rp, (long long)m + 1, q * chunk) - 1;
}
// Full elem_row expansion (parity tests only).
__global__ void elem_row_kernel(const int* __restrict__ rp, int m, long long nnz,
                                long long* __restrict__ out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = upper_bound_i32(rp, (long long)m + 1, e) - 1;
}
// Multi-GPU equal-nnz row slices (partition kernels.hpp:124-129).
__global__ void row_slices_kernel(const int* __restrict__ rp, int m, long long nnz,
                                  long long parts, long long* __restrict__ bounds) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g > parts) return;
  if (g == 0) { bounds[0] = 0; return; }
  if (g == parts) { bounds[parts] = m; return; }
  const long long target = nnz * g / parts;
  long long b = lower_bound_i32(rp, (long long)m + 1, target);
  bounds[g] = b > m ? m : b;
}

// Zero the empty rows of Y (reference: Y zero-allocated, csr.hpp:66-72).
// V = 4 when N % 4 == 0 and Y is 16-byte aligned (float4 stores).
template <int V>
__global__ void zero_rows_kernel(const int* __restrict__ erow, int ne, int N,
                                 float* __restrict__ Y) {
  const int per_row = N / V;
  const long long total = (long long)ne * per_row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = erow[i / per_row];
    float* p = Y + r * N + (i % per_row) * V;
    if constexpr (V == 4) {
      __stcs(reinterpret_cast<float4*>(p), make_float4(0.f, 0.f, 0.f, 0.f));
    } else {
      __stcs(p, 0.f);
    }
  }
}
// All of Y zero (nnz == 0 or every row empty).
// Rows with >= L nonzeros: {compact row, length}.
__global__ void hub_rows_kernel(const int* __restrict__ crp, int mne, int L, int2* __restrict__ out,
                                int* __restrict__ count) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < mne;
       c += (long long)gridDim.x * blockDim.x) {
    const int len = crp[c + 1] - crp[c];
    if (len >= L) out[atomicAdd(count, 1)] = make_int2((int)c, len);
  }
}

__global__ void zero_all_kernel(float* __restrict__ Y, long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    Y[i] = 0.f;
}

// Long-row fix-up: Y[r] = (((T[t1] + H[q0]) + H[q0+1]) + ... ) + H[q1] in
// ascending order (the reference's serial boundary merge, kernels.hpp:316-323
// / :448-453, restricted to rows whose partials were not merged in
// registers).  One warp per long row: the row's partials H[q0..q1][cols] are
// one contiguous range, staged into the warp's shared-memory buffer by
// coalesced loads, then lane j folds column j sequentially (the order is the
// contract; the adds are the only serial part).
constexpr int kFixupWarps = 8;
constexpr int kFixupBuf = 1024;  // floats per warp per batch

// Per long row, precomputed with the plan: {output row, owner tile t1, first
// and last partial slot q0..q1} — the fixup then starts with one 16-byte load
// instead of the list -> rowPtr -> rid chain (most long rows have 1-2
// partials, so that chain was most of the fixup's time).
__global__ void long_info_kernel(const int* __restrict__ list, int nlong, const int* __restrict__ crp,
                                 const int* __restrict__ rid, long long TS, long long CH,
                                 int4* __restrict__ info) {
  for (long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x; li < nlong;
       li += (long long)gridDim.x * blockDim.x) {
    const int c = list[li];
    const long long s = crp[c], f = crp[c + 1];
    const long long t1 = s / TS;
    info[li] = make_int4(rid[c], (int)t1, (int)((t1 + 1) * (TS / CH)), (int)((f - 1) / CH));
  }
}

// One long row folded by the whole warp (all lanes converged).
__device__ __forceinline__ void fixup_row(const int4 d, int lane, float* buf, const float* __restrict__ H,
                                          const float* __restrict__ Tsl, float* __restrict__ Y, int N) {
  const long long t1 = d.y, q0 = d.z, q1 = d.w;
  const long long yrow = (long long)d.x * N;
  for (int j0 = 0; j0 < N; j0 += 32) {
    const int ncol = min(32, N - j0);
    float acc = (lane < ncol) ? Tsl[t1 * N + j0 + lane] : 0.f;
    if (ncol == 32) {
      // 32 columns: lane j reads column j of every partial directly (one
      // 128-B line per partial), 16 partials in flight ahead of the adds
      // (measured: N=64 whole call 461 -> 417 us, N=32 291 -> 287 us;
      // prefetching the next 16 before the adds was slower)
      const float* src = H + j0 + lane;
      long long q = q0;
      for (; q + 16 <= q1 + 1; q += 16) {
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = src[(q + u) * N];
#pragma unroll
        for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, v[u]);
      }
      for (; q <= q1; ++q) acc = __fadd_rn(acc, src[q * N]);
      Y[yrow + j0 + lane] = acc;
      continue;
    }
    const long long qpb = kFixupBuf / ncol;  // partials per batch
    for (long long qb = q0; qb <= q1; qb += qpb) {
      const int nqb = (int)min(qpb, q1 + 1 - qb);
      const int cnt = nqb * ncol;
      __syncwarp();
      if (ncol == N) {  // whole rows of H: one contiguous range
        const float* src = H + qb * N;
#pragma unroll 8
        for (int i = lane; i < cnt; i += 32) buf[i] = src[i];
      } else {
#pragma unroll 4
        for (int i = lane; i < cnt; i += 32) buf[i] = H[(qb + i / ncol) * N + j0 + i % ncol];
      }
      __syncwarp();
      if (lane < ncol) {
#pragma unroll 8
        for (int qq = 0; qq < nqb; ++qq) acc = __fadd_rn(acc, buf[qq * ncol + lane]);
      }
    }
    if (lane < ncol) Y[yrow + j0 + lane] = acc;
  }
}

// Rows with more than kFixupLaneMax partials are "big": the plan puts them
// first in the descriptor list (nbig of them) so they spread over warps.
constexpr int kFixupLaneMax = 32;
inline int fixup_blocks(int nlong, int nbig, int N) {
  if (N > 16) return (nlong + kFixupWarps - 1) / kFixupWarps;
  const int rpw = 32 / N;
  const int b_big = (nbig + kFixupWarps - 1) / kFixupWarps;
  const int b_small = (nlong - nbig + kFixupWarps * rpw - 1) / (kFixupWarps * rpw);
  return b_big > b_small ? b_big : (b_small > 0 ? b_small : 1);
}

__global__ void __launch_bounds__(kFixupWarps * 32)
fixup_kernel(const int4* __restrict__ info, int nlong, int nbig, const float* __restrict__ H,
             const float* __restrict__ Tsl, float* __restrict__ Y, int N) {
  __shared__ float sm[kFixupWarps][kFixupBuf];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* buf = sm[w];
  if (N == 1) {
    // One column: the big rows one per warp (the chain of adds is the serial
    // part), then every other row folded by one lane, 32 rows per warp (most
    // long rows have 1-2 partials).
    const long long gw = (long long)blockIdx.x * kFixupWarps + w, nw = (long long)gridDim.x * kFixupWarps;
    for (long long li = gw; li < nbig; li += nw) fixup_row(info[li], lane, buf, H, Tsl, Y, N);
    for (long long l0 = nbig + gw * 32; l0 < nlong; l0 += nw * 32) {
      const long long li = l0 + lane;
      const bool mine = li < nlong;
      const int4 d = mine ? info[li] : make_int4(0, 0, 0, -1);
      const bool small = mine && d.w - d.z < kFixupLaneMax;
      if (small) {
        float acc = Tsl[d.y];
        int q = d.z;
        for (; q + 4 <= d.w + 1; q += 4) {
          const float v0 = H[q], v1 = H[q + 1], v2 = H[q + 2], v3 = H[q + 3];
          acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, v0), v1), v2), v3);
        }
        for (; q <= d.w; ++q) acc = __fadd_rn(acc, H[q]);
        Y[d.x] = acc;
      }
      unsigned big = __ballot_sync(0xffffffffu, mine && !small);
      while (big) {
        const int src = __ffs(big) - 1;
        big &= big - 1;
        const int4 db = make_int4(__shfl_sync(0xffffffffu, d.x, src), __shfl_sync(0xffffffffu, d.y, src),
                                  __shfl_sync(0xffffffffu, d.z, src), __shfl_sync(0xffffffffu, d.w, src));
        fixup_row(db, lane, buf, H, Tsl, Y, N);
      }
    }
    return;
  }
  if (N <= 16) {
    // Narrow Y (2 <= N <= 16): the same with N lanes per small row (lane = row
    // slot x column), 32/N rows per warp — most long rows have 1-2 partials.
    const int rpw = 32 / N;                 // rows per warp
    const int rs = lane / N, c = lane - rs * N;
    const long long gw = (long long)blockIdx.x * kFixupWarps + w, nw = (long long)gridDim.x * kFixupWarps;
    for (long long li = gw; li < nbig; li += nw) fixup_row(info[li], lane, buf, H, Tsl, Y, N);
    for (long long l0 = nbig + gw * rpw; l0 < nlong; l0 += nw * rpw) {
      const long long li = l0 + rs;
      const bool mine = rs < rpw && li < nlong;
      const int4 d = mine ? info[li] : make_int4(0, 0, 0, -1);
      const bool small = mine && d.w - d.z < kFixupLaneMax;
      if (small) {
        const float* hc = H + c;
        float acc = Tsl[(long long)d.y * N + c];
        long long q = d.z;
        for (; q + 4 <= d.w + 1; q += 4) {
          const float v0 = hc[q * N], v1 = hc[(q + 1) * N], v2 = hc[(q + 2) * N], v3 = hc[(q + 3) * N];
          acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, v0), v1), v2), v3);
        }
        for (; q <= d.w; ++q) acc = __fadd_rn(acc, hc[q * N]);
        Y[(long long)d.x * N + c] = acc;
      }
      // (rows past nbig are small by construction; kept for safety)
      unsigned big = __ballot_sync(0xffffffffu, mine && !small && c == 0);
      while (big) {
        const int src = __ffs(big) - 1;
        big &= big - 1;
        const int4 db = make_int4(__shfl_sync(0xffffffffu, d.x, src), __shfl_sync(0xffffffffu, d.y, src),
                                  __shfl_sync(0xffffffffu, d.z, src), __shfl_sync(0xffffffffu, d.w, src));
        fixup_row(db, lane, buf, H, Tsl, Y, N);
      }
    }
    return;
  }
  for (long long li = (long long)blockIdx.x * kFixupWarps + w; li < nlong;
       li += (long long)gridDim.x * kFixupWarps)
    fixup_row(info[li], lane, buf, H, Tsl, Y, N);
}

// |val| (for the north-star bound sum_j |a_ij x_j| computed on the device).
__global__ void abs_copy_kernel(const float* __restrict__ in, float* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = fabsf(in[i]);
}

// Row slice [r0, r1) rebased: rp_out[i] = rp[r0+i] - rp[r0].
__global__ void rebase_kernel(const int* __restrict__ rp, long long r0, long long rows,
                              int* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= rows;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = rp[r0 + i] - rp[r0];
}

}  // namespace spmk_dev
