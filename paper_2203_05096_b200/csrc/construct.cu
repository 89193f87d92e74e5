// Device-side CSR-k construction: symmetric permutation, group pointers,
// vector permutation, matrix statistics and the synthetic stencil generator.
//
//   csrk_pack        pack_csrk (reference format.py:347-393) with
//                    _permute_symmetric (format.py:318-344)
//   csrk_gather_f64  permute_vector / unpermute_vector (format.py:396-409)
//   csrk_stats       the integer reductions of compute_stats (tuning.py:108-134)
//   csrk_stencil     synthetic grid Laplacians in canonical CSR
//
// All integer outputs are exact: the permuted matrix only moves entries, and
// every row's columns are unique, so "sort the row by new column" has one
// answer whatever the sorting algorithm (format.py:336-340 lexsort).

#include <algorithm>
#include <cstdint>
#include <vector>

#include "internal.h"

namespace csrk {
namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int64_t kScanTile = int64_t(kScanThreads) * kScanItems;

// ---- exclusive scan of int64 (3-phase, recursive over block sums) ---------

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t *tmp,
                                                        int64_t *total) {
  // warp scan then scan of warp sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) tmp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    int64_t w = lane < nw ? tmp[lane] : 0;
    int64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < nw) tmp[lane] = wi - w;
    if (lane == nw - 1) *total = wi;
  }
  __syncthreads();
  const int64_t res = incl - v + tmp[warp];
  __syncthreads();
  return res;
}

__global__ void scan_reduce_kernel(const int64_t *__restrict__ in, int64_t n,
                                   int64_t *__restrict__ sums) {
  __shared__ int64_t tmp[32];
  __shared__ int64_t total;
  const int64_t base = blockIdx.x * kScanTile;
  int64_t s = 0;
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + threadIdx.x * int64_t(kScanItems) + j;
    if (i < n) s += in[i];
  }
  block_exclusive_scan(s, tmp, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void scan_apply_kernel(const int64_t *__restrict__ in, int64_t n,
                                  const int64_t *__restrict__ offs,
                                  int64_t *__restrict__ out) {
  __shared__ int64_t tmp[32];
  __shared__ int64_t total;
  const int64_t base = blockIdx.x * kScanTile;
  int64_t v[kScanItems];
  int64_t s = 0;
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + threadIdx.x * int64_t(kScanItems) + j;
    v[j] = i < n ? in[i] : 0;
    s += v[j];
  }
  int64_t run = block_exclusive_scan(s, tmp, &total) + (offs ? offs[blockIdx.x] : 0);
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + threadIdx.x * int64_t(kScanItems) + j;
    if (i < n) out[i] = run;
    run += v[j];
  }
}

// out[i] = sum(in[0..i)) for i in [0, n]; out has n + 1 entries
int exclusive_scan(const int64_t *in, int64_t n, int64_t *out, cudaStream_t s) {
  if (n == 0) {
    CSRK_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
    return CSRK_OK;
  }
  const int64_t blocks = (n + kScanTile - 1) / kScanTile;
  int64_t *sums = nullptr, *offs = nullptr;
  keep_async_pool();

  CSRK_CUDA_TRY(cudaMallocAsync(&sums, (blocks + 1) * sizeof(int64_t), s));
  keep_async_pool();

  CSRK_CUDA_TRY(cudaMallocAsync(&offs, (blocks + 1) * sizeof(int64_t), s));
  scan_reduce_kernel<<<static_cast<unsigned>(blocks), kScanThreads, 0, s>>>(in, n,
                                                                            sums);
  CSRK_CUDA_TRY(cudaGetLastError());
  int rc = CSRK_OK;
  if (blocks == 1) {
    CSRK_CUDA_TRY(cudaMemsetAsync(offs, 0, sizeof(int64_t), s));
    CSRK_CUDA_TRY(cudaMemcpyAsync(offs + 1, sums, sizeof(int64_t),
                                  cudaMemcpyDeviceToDevice, s));
  } else {
    rc = exclusive_scan(sums, blocks, offs, s);
  }
  if (rc == CSRK_OK) {
    scan_apply_kernel<<<static_cast<unsigned>(blocks), kScanThreads, 0, s>>>(
        in, n, offs, out);
    CSRK_CUDA_TRY(cudaGetLastError());
    // total
    CSRK_CUDA_TRY(cudaMemcpyAsync(out + n, offs + blocks, sizeof(int64_t),
                                  cudaMemcpyDeviceToDevice, s));
  }
  cudaFreeAsync(sums, s);
  cudaFreeAsync(offs, s);
  return rc;
}

__global__ void i64_to_u32_kernel(const int64_t *__restrict__ in,
                                  uint32_t *__restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint32_t>(in[i]);
}

// ---- symmetric permutation -----------------------------------------------

__global__ void new_lens_kernel(const uint32_t *__restrict__ row_ptr,
                                const int64_t *__restrict__ inv, int64_t n,
                                int64_t *__restrict__ lens) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t src = inv[i];
    lens[i] = int64_t(row_ptr[src + 1]) - row_ptr[src];
  }
}

// Rows of at most 32 entries: one warp per row; every lane holds one entry
// and its destination is its rank among the row's (unique) new columns.
__global__ void permute_short_rows_kernel(
    const uint32_t *__restrict__ row_ptr, const uint32_t *__restrict__ col_idx,
    const double *__restrict__ vals, const int64_t *__restrict__ fwd,
    const int64_t *__restrict__ inv, const int64_t *__restrict__ new_ptr,
    int64_t n, uint32_t *__restrict__ out_cols, double *__restrict__ out_vals,
    int *__restrict__ long_rows, int *__restrict__ n_long) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    const int64_t src = inv[i];
    const uint32_t s = row_ptr[src];
    const uint32_t len = row_ptr[src + 1] - s;
    if (len > 32) {
      if (lane == 0) long_rows[atomicAdd(n_long, 1)] = static_cast<int>(i);
      continue;
    }
    uint32_t key = 0xffffffffu;
    double v = 0.0;
    if (lane < static_cast<int>(len)) {
      key = static_cast<uint32_t>(fwd[col_idx[s + lane]]);
      v = vals[s + lane];
    }
    int rank = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t o = __shfl_sync(0xffffffffu, key, j);
      rank += (o < key);
    }
    if (lane < static_cast<int>(len)) {
      const int64_t dst = new_ptr[i] + rank;
      out_cols[dst] = key;
      out_vals[dst] = v;
    }
  }
}

// Rows longer than a warp: one block per row, bitonic sort of
// (new column, source slot) pairs in `buf` (shared memory when it fits,
// otherwise a global scratch slice), then the values follow their slots.
__global__ void permute_long_rows_kernel(
    const uint32_t *__restrict__ row_ptr, const uint32_t *__restrict__ col_idx,
    const double *__restrict__ vals, const int64_t *__restrict__ fwd,
    const int64_t *__restrict__ inv, const int64_t *__restrict__ new_ptr,
    const int *__restrict__ long_rows, uint64_t *__restrict__ gscratch,
    const int64_t *__restrict__ scratch_off, uint32_t *__restrict__ out_cols,
    double *__restrict__ out_vals) {
  extern __shared__ uint64_t sbuf[];
  const int64_t i = long_rows[blockIdx.x];
  const int64_t src = inv[i];
  const uint32_t s = row_ptr[src];
  const uint32_t len = row_ptr[src + 1] - s;
  uint32_t pw = 1;
  while (pw < len) pw <<= 1;
  uint64_t *buf = scratch_off[blockIdx.x] < 0 ? sbuf : gscratch + scratch_off[blockIdx.x];
  for (uint32_t j = threadIdx.x; j < pw; j += blockDim.x)
    buf[j] = j < len ? (static_cast<uint64_t>(fwd[col_idx[s + j]]) << 32) | j
                     : ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= pw; k <<= 1)
    for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
      for (uint32_t t = threadIdx.x; t < pw; t += blockDim.x) {
        const uint32_t p = t ^ jj;
        if (p > t) {
          const uint64_t a = buf[t], b = buf[p];
          const bool up = (t & k) == 0;
          if ((a > b) == up) {
            buf[t] = b;
            buf[p] = a;
          }
        }
      }
      __syncthreads();
    }
  const int64_t d0 = new_ptr[i];
  for (uint32_t j = threadIdx.x; j < len; j += blockDim.x) {
    const uint64_t e = buf[j];
    out_cols[d0 + j] = static_cast<uint32_t>(e >> 32);
    out_vals[d0 + j] = vals[s + static_cast<uint32_t>(e & 0xffffffffu)];
  }
}

__global__ void gather_f64_kernel(const double *__restrict__ in,
                                  const int64_t *__restrict__ idx, int64_t n,
                                  double *__restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = in[idx[i]];
}

// ---- statistics -----------------------------------------------------------

__global__ void stats_kernel(const uint32_t *__restrict__ row_ptr,
                             const uint32_t *__restrict__ col_idx,
                             int64_t n_rows, unsigned long long *out) {
  unsigned long long s = 0, s2 = 0, mx = 0, off = 0, sym = 0;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t a = row_ptr[r], b = row_ptr[r + 1];
    const unsigned long long c = b - a;
    s += c;
    s2 += c * c;
    mx = c > mx ? c : mx;
    for (uint32_t p = a; p < b; ++p) {
      const uint32_t col = col_idx[p];
      if (col == r) continue;
      ++off;
      if (col >= n_rows) continue;
      // binary search r in row `col` (columns strictly increasing)
      uint32_t lo = row_ptr[col], hi = row_ptr[col + 1];
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        const uint32_t v = col_idx[mid];
        if (v < r)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo < row_ptr[col + 1] && col_idx[lo] == r) ++sym;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    s2 += __shfl_down_sync(0xffffffffu, s2, o);
    const unsigned long long m2 = __shfl_down_sync(0xffffffffu, mx, o);
    mx = m2 > mx ? m2 : mx;
    off += __shfl_down_sync(0xffffffffu, off, o);
    sym += __shfl_down_sync(0xffffffffu, sym, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out + 0, s);
    atomicAdd(out + 1, s2);
    atomicMax(out + 2, mx);
    atomicAdd(out + 3, off);
    atomicAdd(out + 4, sym);
  }
}

// ---- numpy-exact variance of the row counts --------------------------------
// np.var(int64 counts) == pairwise_sum((c - mean)^2) / n, where pairwise_sum
// is numpy's: blocks of <= 128 summed with 8 accumulators, larger spans
// split at n/2 rounded down to a multiple of 8.  Leaves are summed on the
// device, the tree is folded on the host in the same order.

__global__ void variance_leaf_kernel(const uint32_t *__restrict__ row_ptr,
                                     double mean, const int64_t *__restrict__ leaf_lo,
                                     const int32_t *__restrict__ leaf_n,
                                     int64_t n_leaves, double *__restrict__ out) {
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < n_leaves;
       l += int64_t(gridDim.x) * blockDim.x) {
    const int64_t lo = leaf_lo[l];
    const int n = leaf_n[l];
    auto val = [&](int64_t i) {
      const double d = __dsub_rn(static_cast<double>(row_ptr[i + 1] - row_ptr[i]), mean);
      return __dmul_rn(d, d);
    };
    double res;
    if (n < 8) {
      res = 0.0;
      for (int i = 0; i < n; ++i) res = __dadd_rn(res, val(lo + i));
    } else {
      double r[8];
      for (int j = 0; j < 8; ++j) r[j] = val(lo + j);
      int i = 8;
      for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], val(lo + i + j));
      res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      for (; i < n; ++i) res = __dadd_rn(res, val(lo + i));
    }
    out[l] = res;
  }
}

void pairwise_leaves(int64_t lo, int64_t n, std::vector<int64_t> &los,
                     std::vector<int32_t> &ns) {
  if (n <= 128) {
    los.push_back(lo);
    ns.push_back(static_cast<int32_t>(n));
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  pairwise_leaves(lo, n2, los, ns);
  pairwise_leaves(lo + n2, n - n2, los, ns);
}

double pairwise_fold(int64_t n, const double *leaf, size_t &cursor) {
  if (n <= 128) return leaf[cursor++];
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  const double a = pairwise_fold(n2, leaf, cursor);
  const double b = pairwise_fold(n - n2, leaf, cursor);
  return a + b;
}

// ---- stencil generator ----------------------------------------------------

struct Stencil {
  int n;
  int dz[27], dy[27], dx[27];
};

__host__ bool make_stencil(int64_t nz, int points, Stencil &st) {
  st.n = 0;
  auto add = [&](int z, int y, int x) {
    st.dz[st.n] = z;
    st.dy[st.n] = y;
    st.dx[st.n] = x;
    ++st.n;
  };
  if (nz == 1 && points == 5) {
    add(0, -1, 0); add(0, 0, -1); add(0, 0, 0); add(0, 0, 1); add(0, 1, 0);
  } else if (nz == 1 && points == 9) {
    for (int y = -1; y <= 1; ++y)
      for (int x = -1; x <= 1; ++x) add(0, y, x);
  } else if (points == 7) {
    add(-1, 0, 0); add(0, -1, 0); add(0, 0, -1); add(0, 0, 0);
    add(0, 0, 1); add(0, 1, 0); add(1, 0, 0);
  } else if (points == 27) {
    for (int z = -1; z <= 1; ++z)
      for (int y = -1; y <= 1; ++y)
        for (int x = -1; x <= 1; ++x) add(z, y, x);
  } else {
    return false;
  }
  return true;
}

// Rows of planes [z0, z0 + nzl) of an nz x ny x nx grid (the whole grid:
// z0 = 0, nzl = nz); columns are global indices minus col_base.
__global__ void stencil_count_kernel(Stencil st, int64_t nz, int64_t ny,
                                     int64_t nx, int64_t z0, int64_t nzl,
                                     int64_t *__restrict__ counts) {
  const int64_t n = nzl * ny * nx;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t x = i % nx, y = (i / nx) % ny, z = z0 + i / (nx * ny);
    int64_t c = 0;
    for (int j = 0; j < st.n; ++j) {
      const int64_t zz = z + st.dz[j], yy = y + st.dy[j], xx = x + st.dx[j];
      c += (zz >= 0 && zz < nz && yy >= 0 && yy < ny && xx >= 0 && xx < nx);
    }
    counts[i] = c;
  }
}

__global__ void stencil_fill_kernel(Stencil st, int64_t nz, int64_t ny,
                                    int64_t nx, int64_t z0, int64_t nzl,
                                    int64_t col_base, const int64_t *__restrict__ ptr,
                                    uint32_t *__restrict__ row_ptr,
                                    uint32_t *__restrict__ cols,
                                    double *__restrict__ vals) {
  const int64_t n = nzl * ny * nx;
  const double diag = static_cast<double>(st.n - 1);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= n;
       i += int64_t(gridDim.x) * blockDim.x) {
    row_ptr[i] = static_cast<uint32_t>(ptr[i]);
    if (i == n) continue;
    const int64_t x = i % nx, y = (i / nx) % ny, z = z0 + i / (nx * ny);
    int64_t p = ptr[i];
    for (int j = 0; j < st.n; ++j) {
      const int64_t zz = z + st.dz[j], yy = y + st.dy[j], xx = x + st.dx[j];
      if (zz >= 0 && zz < nz && yy >= 0 && yy < ny && xx >= 0 && xx < nx) {
        cols[p] = static_cast<uint32_t>((zz * ny + yy) * nx + xx - col_base);
        vals[p] = (st.dz[j] == 0 && st.dy[j] == 0 && st.dx[j] == 0) ? diag : -1.0;
        ++p;
      }
    }
  }
}

inline unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 64) b = 148 * 64;
  return static_cast<unsigned>(b);
}

template <typename T>
struct DevBuf {
  T *p = nullptr;
  ~DevBuf() { cudaFree(p); }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, (n ? n : 1) * sizeof(T)); }
};

}  // namespace

int exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, cudaStream_t s) {
  return exclusive_scan(in, n, out, s);
}

int pack_device(int device, int64_t n, int64_t nnz, const uint32_t *row_ptr_h,
                const uint32_t *col_idx_h, const double *vals_h,
                const int64_t *fwd_h, const int64_t *inv_h, int n_levels,
                int64_t n1, const int64_t *sizes1, int64_t n2,
                const int64_t *sizes2, csrk_matrix **out) {
  *out = nullptr;
  if (n_levels != 1 && n_levels != 2) {
    set_error("groups must hold 1 or 2 levels (k = 2 or 3)");
    return CSRK_EINVAL;
  }
  if (nnz > 2147483647LL) {
    set_error("nnz %lld exceeds the 32-bit index limit 2147483647",
              static_cast<long long>(nnz));
    return CSRK_EINVAL;
  }
  // group sizes (format.py:373-386)
  const int64_t *sz[2] = {sizes1, sizes2};
  const int64_t len[2] = {n1, n2};
  int64_t below = n;
  for (int level = 1; level <= n_levels; ++level) {
    const int64_t *s = sz[level - 1];
    const int64_t l = len[level - 1];
    bool ok = l > 0 && s != nullptr;
    int64_t total = 0;
    for (int64_t i = 0; ok && i < l; ++i) {
      if (s[i] < 1) ok = false;
      total += s[i];
    }
    if (!ok) {
      set_error("level %d group sizes must be positive", level);
      return CSRK_EINVAL;
    }
    if (total != below) {
      set_error("level %d group sizes sum to %lld, expected %lld", level,
                static_cast<long long>(total), static_cast<long long>(below));
      return CSRK_EINVAL;
    }
    below = l;
  }
  CSRK_CUDA_TRY(cudaSetDevice(device));
  csrk_matrix *m = new csrk_matrix();
  m->device = device;
  m->n_rows = n;
  m->n_cols = n;
  m->nnz = nnz;
  m->k = n_levels + 1;
  m->n_sr = n1;
  m->n_ssr = n_levels == 2 ? n2 : 0;
  auto bail = [&](int rc) {
    csrk_matrix_free(m);
    return rc;
  };
  int rc = alloc_matrix_arrays(m, true, false);
  if (rc != CSRK_OK) return bail(rc);
  cudaStream_t s = m->stream;

  DevBuf<uint32_t> a_ptr, a_cols;
  DevBuf<double> a_vals;
  DevBuf<int64_t> d_fwd, d_inv, lens, nptr, gsz, gptr, scratch_off;
  DevBuf<int> long_rows, n_long;
  DevBuf<uint64_t> gscratch;
#define PACK_CUDA(expr)                                                   \
  do {                                                                    \
    cudaError_t e_ = (expr);                                              \
    if (e_ != cudaSuccess) {                                              \
      set_error("CUDA error %s in pack: %s", cudaGetErrorName(e_),        \
                cudaGetErrorString(e_));                                  \
      return bail(e_ == cudaErrorMemoryAllocation ? CSRK_ENOMEM : CSRK_ECUDA); \
    }                                                                     \
  } while (0)
  PACK_CUDA(a_ptr.alloc(n + 1));
  PACK_CUDA(a_cols.alloc(nnz));
  PACK_CUDA(a_vals.alloc(nnz));
  PACK_CUDA(d_fwd.alloc(n));
  PACK_CUDA(d_inv.alloc(n));
  PACK_CUDA(lens.alloc(n));
  PACK_CUDA(nptr.alloc(n + 1));
  PACK_CUDA(long_rows.alloc(n));
  PACK_CUDA(n_long.alloc(1));
  PACK_CUDA(cudaMemcpyAsync(a_ptr.p, row_ptr_h, (n + 1) * sizeof(uint32_t),
                            cudaMemcpyHostToDevice, s));
  if (nnz) {
    PACK_CUDA(cudaMemcpyAsync(a_cols.p, col_idx_h, nnz * sizeof(uint32_t),
                              cudaMemcpyHostToDevice, s));
    PACK_CUDA(cudaMemcpyAsync(a_vals.p, vals_h, nnz * sizeof(double),
                              cudaMemcpyHostToDevice, s));
  }
  PACK_CUDA(cudaMemcpyAsync(d_fwd.p, fwd_h, n * sizeof(int64_t),
                            cudaMemcpyHostToDevice, s));
  PACK_CUDA(cudaMemcpyAsync(d_inv.p, inv_h, n * sizeof(int64_t),
                            cudaMemcpyHostToDevice, s));
  PACK_CUDA(cudaMemsetAsync(n_long.p, 0, sizeof(int), s));
  new_lens_kernel<<<grid_for(n, 256), 256, 0, s>>>(a_ptr.p, d_inv.p, n, lens.p);
  PACK_CUDA(cudaGetLastError());
  rc = exclusive_scan(lens.p, n, nptr.p, s);
  if (rc != CSRK_OK) return bail(rc);
  i64_to_u32_kernel<<<grid_for(n + 1, 256), 256, 0, s>>>(nptr.p, m->row_ptr, n + 1);
  PACK_CUDA(cudaGetLastError());
  permute_short_rows_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(
      a_ptr.p, a_cols.p, a_vals.p, d_fwd.p, d_inv.p, nptr.p, n, m->col_idx,
      m->vals64, long_rows.p, n_long.p);
  PACK_CUDA(cudaGetLastError());
  int h_long = 0;
  PACK_CUDA(cudaMemcpyAsync(&h_long, n_long.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  PACK_CUDA(cudaStreamSynchronize(s));
  if (h_long > 0) {
    // per long row: shared buffer when the padded row fits, else global
    std::vector<int> rows(h_long);
    PACK_CUDA(cudaMemcpy(rows.data(), long_rows.p, h_long * sizeof(int),
                         cudaMemcpyDeviceToHost));
    std::vector<int64_t> off(h_long);
    int64_t gtotal = 0;
    constexpr uint32_t kSmemEntries = 4096;
    for (int j = 0; j < h_long; ++j) {
      const int64_t src = inv_h[rows[j]];
      const uint32_t l = row_ptr_h[src + 1] - row_ptr_h[src];
      uint64_t pw = 1;
      while (pw < l) pw <<= 1;
      if (pw <= kSmemEntries) {
        off[j] = -1;
      } else {
        off[j] = gtotal;
        gtotal += static_cast<int64_t>(pw);
      }
    }
    PACK_CUDA(scratch_off.alloc(h_long));
    PACK_CUDA(cudaMemcpyAsync(scratch_off.p, off.data(), h_long * sizeof(int64_t),
                              cudaMemcpyHostToDevice, s));
    PACK_CUDA(gscratch.alloc(gtotal));
    permute_long_rows_kernel<<<h_long, 512, kSmemEntries * sizeof(uint64_t), s>>>(
        a_ptr.p, a_cols.p, a_vals.p, d_fwd.p, d_inv.p, nptr.p, long_rows.p,
        gscratch.p, scratch_off.p, m->col_idx, m->vals64);
    PACK_CUDA(cudaGetLastError());
  }
  // group pointers as prefix sums of the sizes (format.py:386-388)
  for (int level = 1; level <= n_levels; ++level) {
    const int64_t l = len[level - 1];
    PACK_CUDA(gsz.alloc(l));
    PACK_CUDA(gptr.alloc(l + 1));
    PACK_CUDA(cudaMemcpyAsync(gsz.p, sz[level - 1], l * sizeof(int64_t),
                              cudaMemcpyHostToDevice, s));
    rc = exclusive_scan(gsz.p, l, gptr.p, s);
    if (rc != CSRK_OK) return bail(rc);
    uint32_t *dst = level == 1 ? m->sr_ptr : m->ssr_ptr;
    i64_to_u32_kernel<<<grid_for(l + 1, 256), 256, 0, s>>>(gptr.p, dst, l + 1);
    PACK_CUDA(cudaGetLastError());
    PACK_CUDA(cudaStreamSynchronize(s));
    cudaFree(gsz.p);
    cudaFree(gptr.p);
    gsz.p = nullptr;
    gptr.p = nullptr;
  }
  rc = ensure_plan(m, 0, 0, 0, s);
  if (rc != CSRK_OK) return bail(rc);
  PACK_CUDA(cudaStreamSynchronize(s));
#undef PACK_CUDA
  *out = m;
  return CSRK_OK;
}

int gather_f64(int64_t n, const double *in, const int64_t *idx, double *out,
               cudaStream_t s) {
  if (n == 0) return CSRK_OK;
  gather_f64_kernel<<<grid_for(n, 256), 256, 0, s>>>(in, idx, n, out);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

int stats_device(const csrk_matrix *m, int64_t out[5]) {
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  unsigned long long *d = nullptr;
  CSRK_CUDA_TRY(cudaMalloc(&d, 5 * sizeof(unsigned long long)));
  cudaError_t e = cudaMemsetAsync(d, 0, 5 * sizeof(unsigned long long), m->stream);
  if (e == cudaSuccess && m->n_rows > 0) {
    stats_kernel<<<grid_for(m->n_rows, 256), 256, 0, m->stream>>>(
        m->row_ptr, m->col_idx, m->n_rows, d);
    e = cudaGetLastError();
  }
  unsigned long long h[5] = {0, 0, 0, 0, 0};
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, m->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(m->stream);
  cudaFree(d);
  if (e != cudaSuccess) {
    set_error("CUDA error %s in stats: %s", cudaGetErrorName(e),
              cudaGetErrorString(e));
    return CSRK_ECUDA;
  }
  for (int i = 0; i < 5; ++i) out[i] = static_cast<int64_t>(h[i]);
  return CSRK_OK;
}

__global__ void uniform_ptr_kernel(uint32_t *ptr, int64_t count, int64_t size,
                                   int64_t total) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = i * size;
    ptr[i] = static_cast<uint32_t>(v < total ? v : total);
  }
}

int group_uniform(csrk_matrix *m, int64_t srs, int64_t ssrs) {
  if (srs < 1 || ssrs < 1) {
    set_error("group sizes must be at least 1");
    return CSRK_EINVAL;
  }
  if (m->n_rows == 0) {
    set_error("cannot group an empty matrix");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  const int64_t n_sr = (m->n_rows + srs - 1) / srs;
  const int64_t n_ssr = (n_sr + ssrs - 1) / ssrs;
  uint32_t *sr = nullptr, *ssr = nullptr;
  CSRK_CUDA_TRY(cudaMalloc(&sr, (n_sr + 1) * sizeof(uint32_t)));
  cudaError_t e = cudaMalloc(&ssr, (n_ssr + 1) * sizeof(uint32_t));
  if (e != cudaSuccess) {
    cudaFree(sr);
    set_error("out of device memory");
    return CSRK_ENOMEM;
  }
  uniform_ptr_kernel<<<grid_for(n_sr + 1, 256), 256, 0, m->stream>>>(sr, n_sr, srs,
                                                                     m->n_rows);
  uniform_ptr_kernel<<<grid_for(n_ssr + 1, 256), 256, 0, m->stream>>>(ssr, n_ssr, ssrs,
                                                                      n_sr);
  CSRK_CUDA_TRY(cudaGetLastError());
  cudaFree(m->sr_ptr);
  cudaFree(m->ssr_ptr);
  m->sr_ptr = sr;
  m->ssr_ptr = ssr;
  m->k = 3;
  m->n_sr = n_sr;
  m->n_ssr = n_ssr;
  // force a new plan for the new grouping
  const int64_t tc = m->plan.tile_cost, cap = m->plan.cap, st = m->plan.stages;
  cudaFree(m->plan.tile_row);
  m->plan.tile_row = nullptr;
  m->plan.tile_ptr = m->plan.tile_long = nullptr;
  m->pipe.plan_tiles = -1;
  CSRK_TRY(ensure_plan(m, tc, cap, st, m->stream));
  CSRK_CUDA_TRY(cudaStreamSynchronize(m->stream));
  return CSRK_OK;
}

int row_variance(const csrk_matrix *m, double mean, double *out) {
  const int64_t n = m->n_rows;
  if (n == 0) {
    *out = 0.0;
    return CSRK_OK;
  }
  std::vector<int64_t> los;
  std::vector<int32_t> ns;
  pairwise_leaves(0, n, los, ns);
  const int64_t nl = static_cast<int64_t>(los.size());
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  DevBuf<int64_t> dlo;
  DevBuf<int32_t> dn;
  DevBuf<double> dsum;
  CSRK_CUDA_TRY(dlo.alloc(nl));
  CSRK_CUDA_TRY(dn.alloc(nl));
  CSRK_CUDA_TRY(dsum.alloc(nl));
  CSRK_CUDA_TRY(cudaMemcpyAsync(dlo.p, los.data(), nl * sizeof(int64_t),
                                cudaMemcpyHostToDevice, m->stream));
  CSRK_CUDA_TRY(cudaMemcpyAsync(dn.p, ns.data(), nl * sizeof(int32_t),
                                cudaMemcpyHostToDevice, m->stream));
  variance_leaf_kernel<<<grid_for(nl, 128), 128, 0, m->stream>>>(
      m->row_ptr, mean, dlo.p, dn.p, nl, dsum.p);
  CSRK_CUDA_TRY(cudaGetLastError());
  std::vector<double> leaf(nl);
  CSRK_CUDA_TRY(cudaMemcpyAsync(leaf.data(), dsum.p, nl * sizeof(double),
                                cudaMemcpyDeviceToHost, m->stream));
  CSRK_CUDA_TRY(cudaStreamSynchronize(m->stream));
  size_t cursor = 0;
  // the fold's additions are plain host IEEE double adds (no contraction)
  *out = pairwise_fold(n, leaf.data(), cursor) / static_cast<double>(n);
  return CSRK_OK;
}

// ---- coordinate triplets -> canonical CSR (reference format.py:233-284) ---
//
// csr_from_arrays sorts the triplets stably by (row, col) (np.lexsort) and
// sums duplicate coordinates with np.add.reduceat, whose float64 reduction
// is v0 + pairwise_sum(v1 .. v_{L-1}) with numpy's pairwise_sum (blocks of
// 8 accumulators up to 128 elements, halves above; sequential from -0.0
// below 8).  Here: a stable LSD radix sort of (row << cb | col, input index)
// pairs, run heads, and one thread per run summing in exactly that order.

__global__ void coo_key_kernel(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols,
                               int64_t count, int cb, uint64_t *__restrict__ keys,
                               uint32_t *__restrict__ idx) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    keys[i] = (static_cast<uint64_t>(rows[i]) << cb) | static_cast<uint64_t>(cols[i]);
    idx[i] = static_cast<uint32_t>(i);
  }
}

__global__ void coo_head_kernel(const uint64_t *__restrict__ keys, int64_t count,
                                int64_t *__restrict__ head) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x)
    head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// numpy's pairwise_sum over v[idx[a .. a+n)] (loops_utils.h.src)
__device__ double np_pairwise(const double *__restrict__ v, const uint32_t *__restrict__ idx,
                              int64_t a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res += v[idx[a + i]];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = v[idx[a + j]];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += v[idx[a + i + j]];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += v[idx[a + i]];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(v, idx, a, n2) + np_pairwise(v, idx, a + n2, n - n2);
}

__global__ void coo_runs_kernel(const uint64_t *__restrict__ keys,
                                const uint32_t *__restrict__ idx, const double *__restrict__ v,
                                const int64_t *__restrict__ head, const int64_t *__restrict__ pos,
                                int64_t count, int cb, uint32_t *__restrict__ col_idx,
                                double *__restrict__ vals, int64_t *__restrict__ row_count) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (!head[i]) continue;
    int64_t e = i + 1;
    while (e < count && !head[e]) ++e;
    const int64_t u = pos[i];
    const uint64_t k = keys[i];
    col_idx[u] = static_cast<uint32_t>(k & ((uint64_t(1) << cb) - 1));
    double s = v[idx[i]];
    if (e - i > 1) s += np_pairwise(v, idx, i + 1, e - i - 1);
    vals[u] = s;
    atomicAdd(reinterpret_cast<unsigned long long *>(&row_count[k >> cb]), 1ull);
  }
}

int coo_to_csr_device(int device, int64_t n_rows, int64_t n_cols, int64_t count,
                      const int64_t *rows_h, const int64_t *cols_h, const double *vals_h,
                      csrk_matrix **out) {
  *out = nullptr;
  if (n_rows < 0 || n_cols < 0 || count < 0 || n_rows > 4294967295LL ||
      n_cols > 4294967295LL) {
    set_error("invalid shape %lld x %lld", static_cast<long long>(n_rows),
              static_cast<long long>(n_cols));
    return CSRK_EINVAL;
  }
  if (count > 2147483647LL) {
    set_error("entry count %lld exceeds the 32-bit index limit",
              static_cast<long long>(count));
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(device));
  csrk_matrix *m = new csrk_matrix();
  m->device = device;
  m->n_rows = n_rows;
  m->n_cols = n_cols;
  m->k = 1;
  cudaStream_t s = nullptr;
  int rc = CSRK_OK;
  auto fail = [&](int code, const char *what) {
    if (code == CSRK_ECUDA || code == CSRK_ENOMEM) set_error("%s failed", what);
    csrk_matrix_free(m);
    return code;
  };
  int cb = 1;
  while ((int64_t(1) << cb) < n_cols) ++cb;
  int rb = 1;
  while ((int64_t(1) << rb) < n_rows) ++rb;
  const int key_bits = ((cb + rb + 7) / 8) * 8;
  DevBuf<int64_t> r, c, head, pos, rcount, rptr;
  DevBuf<double> v;
  DevBuf<uint64_t> keys, tkeys;
  DevBuf<uint32_t> idx, tidx;
  if (r.alloc(count) || c.alloc(count) || v.alloc(count) || keys.alloc(count) ||
      tkeys.alloc(count) || idx.alloc(count) || tidx.alloc(count) || head.alloc(count) ||
      pos.alloc(count + 1) || rcount.alloc(n_rows) || rptr.alloc(n_rows + 1))
    return fail(CSRK_ENOMEM, "device memory for the triplets");
  if (count) {
    if (cudaMemcpy(r.p, rows_h, count * 8, cudaMemcpyHostToDevice) ||
        cudaMemcpy(c.p, cols_h, count * 8, cudaMemcpyHostToDevice) ||
        cudaMemcpy(v.p, vals_h, count * 8, cudaMemcpyHostToDevice))
      return fail(CSRK_ECUDA, "triplet upload");
    coo_key_kernel<<<grid_for(count, 256), 256, 0, s>>>(r.p, c.p, count, cb, keys.p, idx.p);
    rc = radix_sort_pairs(keys.p, idx.p, tkeys.p, tidx.p, count, 0, key_bits, s);
    if (rc != CSRK_OK) return fail(rc, "triplet sort");
    coo_head_kernel<<<grid_for(count, 256), 256, 0, s>>>(keys.p, count, head.p);
    rc = exclusive_scan(head.p, count, pos.p, s);
    if (rc != CSRK_OK) return fail(rc, "run scan");
  } else if (cudaMemset(pos.p, 0, sizeof(int64_t))) {
    return fail(CSRK_ECUDA, "run scan");
  }
  int64_t nnz = 0;
  if (cudaMemcpy(&nnz, pos.p + count, sizeof(nnz), cudaMemcpyDeviceToHost))
    return fail(CSRK_ECUDA, "run count");
  m->nnz = nnz;
  rc = alloc_matrix_arrays(m, true, false);
  if (rc != CSRK_OK) {
    csrk_matrix_free(m);
    return rc;
  }
  if (cudaMemset(rcount.p, 0, (n_rows > 0 ? n_rows : 1) * sizeof(int64_t)))
    return fail(CSRK_ECUDA, "row counts");
  if (count)
    coo_runs_kernel<<<grid_for(count, 256), 256, 0, s>>>(keys.p, idx.p, v.p, head.p, pos.p,
                                                         count, cb, m->col_idx, m->vals64,
                                                         rcount.p);
  rc = exclusive_scan(rcount.p, n_rows, rptr.p, s);
  if (rc != CSRK_OK) return fail(rc, "row pointer scan");
  i64_to_u32_kernel<<<grid_for(n_rows + 1, 256), 256, 0, s>>>(rptr.p, m->row_ptr, n_rows + 1);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return fail(CSRK_ECUDA, "triplet assembly");
  rc = ensure_plan(m, 0, 0, 0, m->stream);
  if (rc == CSRK_OK && cudaStreamSynchronize(m->stream) != cudaSuccess) rc = CSRK_ECUDA;
  if (rc != CSRK_OK) {
    csrk_matrix_free(m);
    return rc;
  }
  *out = m;
  return CSRK_OK;
}

int stencil_device(int device, int64_t nz, int64_t ny, int64_t nx, int points,
                   int64_t z0, int64_t z1, csrk_matrix **out) {
  *out = nullptr;
  Stencil st;
  if (nz < 1 || ny < 1 || nx < 1 || !make_stencil(nz, points, st)) {
    set_error("unsupported stencil: %d points on %lldx%lldx%lld", points,
              static_cast<long long>(nz), static_cast<long long>(ny),
              static_cast<long long>(nx));
    return CSRK_EINVAL;
  }
  if (z0 < 0 || z1 > nz || z0 >= z1) {
    set_error("slab planes [%lld, %lld) are not a non-empty range of 0..%lld",
              static_cast<long long>(z0), static_cast<long long>(z1),
              static_cast<long long>(nz));
    return CSRK_EINVAL;
  }
  const int64_t plane = ny * nx;
  const int64_t nzl = z1 - z0;
  const int64_t n = nzl * plane;
  // halo planes: one below / above the slab where the stencil reaches them
  const bool reach = st.n == 7 || st.n == 27;
  const int64_t c0 = reach ? (z0 > 0 ? z0 - 1 : 0) : z0;
  const int64_t c1 = reach ? (z1 < nz ? z1 + 1 : nz) : z1;
  const int64_t n_cols = (c1 - c0) * plane;
  CSRK_CUDA_TRY(cudaSetDevice(device));
  // exact nnz on the host: per-axis counts of valid offsets are separable
  // (planes: rows in [z0, z1) whose neighbour plane z + dz is in the grid)
  int64_t nnz = 0;
  for (int j = 0; j < st.n; ++j) {
    const int64_t lo = z0 > -st.dz[j] ? z0 : -st.dz[j];
    const int64_t hi = z1 < nz - st.dz[j] ? z1 : nz - st.dz[j];
    nnz += (hi > lo ? hi - lo : 0) * (ny - (st.dy[j] != 0)) * (nx - (st.dx[j] != 0));
  }
  if (nnz > 2147483647LL || n > 4294967295LL || n_cols > 4294967295LL) {
    set_error("nnz %lld exceeds the 32-bit index limit 2147483647",
              static_cast<long long>(nnz));
    return CSRK_EINVAL;
  }
  csrk_matrix *m = new csrk_matrix();
  m->device = device;
  m->n_rows = n;
  m->n_cols = n_cols;
  m->nnz = nnz;
  m->k = 1;
  int rc = alloc_matrix_arrays(m, true, false);
  if (rc != CSRK_OK) {
    csrk_matrix_free(m);
    return rc;
  }
  DevBuf<int64_t> counts, ptr;
  cudaError_t e = counts.alloc(n);
  if (e == cudaSuccess) e = ptr.alloc(n + 1);
  if (e != cudaSuccess) {
    csrk_matrix_free(m);
    set_error("out of device memory in stencil generator");
    return CSRK_ENOMEM;
  }
  stencil_count_kernel<<<grid_for(n, 256), 256, 0, m->stream>>>(st, nz, ny, nx, z0,
                                                                 nzl, counts.p);
  rc = exclusive_scan(counts.p, n, ptr.p, m->stream);
  if (rc == CSRK_OK) {
    stencil_fill_kernel<<<grid_for(n + 1, 256), 256, 0, m->stream>>>(
        st, nz, ny, nx, z0, nzl, c0 * plane, ptr.p, m->row_ptr, m->col_idx, m->vals64);
    if (cudaGetLastError() != cudaSuccess) rc = CSRK_ECUDA;
  }
  if (rc == CSRK_OK) rc = ensure_plan(m, 0, 0, 0, m->stream);
  if (rc == CSRK_OK && cudaStreamSynchronize(m->stream) != cudaSuccess) {
    set_error("stencil generator failed");
    rc = CSRK_ECUDA;
  }
  if (rc != CSRK_OK) {
    csrk_matrix_free(m);
    return rc;
  }
  *out = m;
  return CSRK_OK;
}

}  // namespace csrk

extern "C" {

int csrk_pack(int device, int64_t n, int64_t nnz, const uint32_t *row_ptr,
              const uint32_t *col_idx, const double *vals, const int64_t *fwd,
              const int64_t *inv, int n_levels, int64_t n_sizes1,
              const int64_t *sizes1, int64_t n_sizes2, const int64_t *sizes2,
              csrk_matrix **out) {
  if (!out || !row_ptr || !fwd || !inv || (nnz && (!col_idx || !vals))) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  const int rc = csrk::pack_device(device, n, nnz, row_ptr, col_idx, vals, fwd, inv,
                           n_levels, n_sizes1, sizes1, n_sizes2, sizes2, out);
  csrk::trim_async_pool();
  return rc;
}

int csrk_gather_f64(int64_t n, const double *in, const int64_t *idx,
                    double *out, void *stream) {
  return csrk::gather_f64(n, in, idx, out, static_cast<cudaStream_t>(stream));
}

int csrk_stats(const csrk_matrix *m, int64_t out[5]) {
  if (!m || !out) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  return csrk::stats_device(m, out);
}

int csrk_matrix_group_uniform(csrk_matrix *m, int64_t srs, int64_t ssrs) {
  if (!m) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  return csrk::group_uniform(m, srs, ssrs);
}

int csrk_row_variance(const csrk_matrix *m, double mean, double *out) {
  if (!m || !out) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  return csrk::row_variance(m, mean, out);
}

int csrk_stencil(int device, int64_t nz, int64_t ny, int64_t nx, int points,
                 csrk_matrix **out) {
  if (!out) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  return csrk::stencil_device(device, nz, ny, nx, points, 0, nz, out);
}

int csrk_coo_to_csr(int device, int64_t n_rows, int64_t n_cols, int64_t count,
                    const int64_t *rows, const int64_t *cols, const double *vals,
                    csrk_matrix **out) {
  if (!out || (count > 0 && (!rows || !cols || !vals))) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  const int rc = csrk::coo_to_csr_device(device, n_rows, n_cols, count, rows, cols, vals, out);
  csrk::trim_async_pool();
  return rc;
}

int csrk_stencil_slab(int device, int64_t nz, int64_t ny, int64_t nx, int points,
                      int64_t z0, int64_t z1, csrk_matrix **out) {
  if (!out) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  if (points != 7 && points != 27) {
    csrk::set_error("slabs need a 3D stencil (7 or 27 points), got %d", points);
    return CSRK_EINVAL;
  }
  return csrk::stencil_device(device, nz, ny, nx, points, z0, z1, out);
}

}  // extern "C"
