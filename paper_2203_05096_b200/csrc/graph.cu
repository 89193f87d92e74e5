// Device-side graph construction for Band-k (first stage of moving the
// reordering onto the GPU).
//
// Every operation is "emit (row << 32 | col) keys, stable radix sort, then
// unique or sum runs": the result is the sorted CSR adjacency that the host
// restatement (bandk.cpp) and the reference (reorder.py:87-196) produce, so
// the arrays are bit-identical:
//   csrk_graph_build_dev     build_graph    reorder.py:115-135
//   csrk_graph_relabel_dev   _relabel_graph reorder.py:192-196
//   csrk_graph_contract_dev  _contract      reorder.py:176-184
// A device graph is {n, m, ptr[n+1] int64, idx[m] int32, ew[m] int32,
// nw[n] int32} in device memory, owned by the csrk_dgraph handle.

#include <cstdint>

#include "internal.h"

namespace csrk {
namespace {

inline unsigned blocks_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return static_cast<unsigned>(b);
}

#define GRID_STRIDE(i, n)                                                  \
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < (n); \
       i += int64_t(gridDim.x) * blockDim.x)

// off-diagonal count per matrix row
__global__ void offdiag_count_kernel(const uint32_t *__restrict__ row_ptr,
                                     const uint32_t *__restrict__ col_idx, int64_t n,
                                     int64_t *__restrict__ cnt) {
  GRID_STRIDE(r, n) {
    int64_t c = 0;
    for (uint32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) c += col_idx[p] != r;
    cnt[r] = c;
  }
}

// both directions of every off-diagonal entry as (u << 32 | v)
__global__ void emit_sym_kernel(const uint32_t *__restrict__ row_ptr,
                                const uint32_t *__restrict__ col_idx, int64_t n,
                                const int64_t *__restrict__ off, uint64_t *__restrict__ keys,
                                uint32_t *__restrict__ vals) {
  GRID_STRIDE(r, n) {
    int64_t o = 2 * off[r];
    for (uint32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
      const uint32_t c = col_idx[p];
      if (c == r) continue;
      keys[o] = (static_cast<uint64_t>(r) << 32) | c;
      vals[o] = 1;
      keys[o + 1] = (static_cast<uint64_t>(c) << 32) | static_cast<uint32_t>(r);
      vals[o + 1] = 1;
      o += 2;
    }
  }
}

// relabelled edges (fwd[u] << 32 | fwd[v]) with the edge weight as value
__global__ void emit_relabel_kernel(const int64_t *__restrict__ ptr,
                                    const int32_t *__restrict__ idx,
                                    const int32_t *__restrict__ ew,
                                    const int64_t *__restrict__ fwd, int64_t n,
                                    uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  GRID_STRIDE(u, n) {
    const uint64_t fu = static_cast<uint64_t>(fwd[u]) << 32;
    for (int64_t p = ptr[u]; p < ptr[u + 1]; ++p) {
      keys[p] = fu | static_cast<uint32_t>(fwd[idx[p]]);
      vals[p] = static_cast<uint32_t>(ew[p]);
    }
  }
}

// contracted edges (f2c[u] << 32 | f2c[v]) for f2c[u] != f2c[v]; slots of
// internal edges get an all-ones key and sort to the end
__global__ void emit_contract_kernel(const int64_t *__restrict__ ptr,
                                     const int32_t *__restrict__ idx,
                                     const int32_t *__restrict__ ew,
                                     const int32_t *__restrict__ f2c, int64_t n,
                                     uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  GRID_STRIDE(u, n) {
    const uint32_t cu = static_cast<uint32_t>(f2c[u]);
    for (int64_t p = ptr[u]; p < ptr[u + 1]; ++p) {
      const uint32_t cv = static_cast<uint32_t>(f2c[idx[p]]);
      keys[p] = cu == cv ? ~0ull : ((static_cast<uint64_t>(cu) << 32) | cv);
      vals[p] = static_cast<uint32_t>(ew[p]);
    }
  }
}

// run heads among the first `count` sorted keys (excluding sentinel keys)
__global__ void run_head_kernel(const uint64_t *__restrict__ keys, int64_t count,
                                int64_t *__restrict__ head) {
  GRID_STRIDE(i, count) {
    head[i] = keys[i] != ~0ull && (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
  }
}

// compact runs: run r = [start, next start); sums the weights (or 1)
__global__ void run_compact_kernel(const uint64_t *__restrict__ keys,
                                   const uint32_t *__restrict__ vals, int64_t count,
                                   const int64_t *__restrict__ head_pos, bool unit,
                                   int32_t *__restrict__ idx, int32_t *__restrict__ ew,
                                   uint32_t *__restrict__ src) {
  GRID_STRIDE(i, count) {
    const bool is_head = keys[i] != ~0ull && (i == 0 || keys[i] != keys[i - 1]);
    if (!is_head) continue;
    const int64_t r = head_pos[i];
    int64_t w = 0;
    for (int64_t j = i; j < count && keys[j] == keys[i]; ++j) w += vals[j];
    idx[r] = static_cast<int32_t>(keys[i] & 0xffffffffu);
    ew[r] = unit ? 1 : static_cast<int32_t>(w);
    src[r] = static_cast<uint32_t>(keys[i] >> 32);
  }
}

// ptr[u] = first edge of row u (lower bound of u over the sorted sources)
__global__ void row_ptr_kernel(const uint32_t *__restrict__ src, int64_t m, int64_t n,
                               int64_t *__restrict__ ptr) {
  GRID_STRIDE(u, n + 1) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (src[mid] < u)
        lo = mid + 1;
      else
        hi = mid;
    }
    ptr[u] = lo;
  }
}

__global__ void fill_i32_kernel(int32_t *__restrict__ a, int64_t n, int32_t v) {
  GRID_STRIDE(i, n) { a[i] = v; }
}

__global__ void gather_nw_kernel(const int32_t *__restrict__ nw,
                                 const int64_t *__restrict__ inv, int64_t n,
                                 int32_t *__restrict__ out) {
  GRID_STRIDE(i, n) { out[i] = nw[inv[i]]; }
}

__global__ void contract_nw_kernel(const int32_t *__restrict__ nw,
                                   const int32_t *__restrict__ f2c, int64_t n,
                                   int32_t *__restrict__ out) {
  GRID_STRIDE(v, n) { atomicAdd(&out[f2c[v]], nw[v]); }
}

template <typename T>
struct Buf {
  T *p = nullptr;
  cudaStream_t s = nullptr;
  explicit Buf(cudaStream_t st) : s(st) {}
  ~Buf() {
    if (p) cudaFreeAsync(p, s);
  }
  cudaError_t alloc(int64_t n) {
    keep_async_pool();
    return cudaMallocAsync(&p, (n > 0 ? n : 1) * sizeof(T), s);
  }
};

// sorted keys / vals (count entries, sentinels at the end) -> graph arrays
int finish_graph(csrk_dgraph *g, int64_t n, uint64_t *keys, uint32_t *vals, int64_t count,
                 bool unit, cudaStream_t s) {
  Buf<int64_t> head(s), pos(s);
  Buf<uint32_t> src(s);
  CSRK_CUDA_TRY(head.alloc(count));
  CSRK_CUDA_TRY(pos.alloc(count + 1));
  run_head_kernel<<<blocks_for(count), 256, 0, s>>>(keys, count, head.p);
  CSRK_TRY(exclusive_scan_i64(head.p, count, pos.p, s));
  int64_t m = 0;
  CSRK_CUDA_TRY(cudaMemcpyAsync(&m, pos.p + count, sizeof(m), cudaMemcpyDeviceToHost, s));
  CSRK_CUDA_TRY(cudaStreamSynchronize(s));
  g->n = n;
  g->m = m;
  CSRK_CUDA_TRY(cudaMalloc(&g->ptr, (n + 1) * sizeof(int64_t)));
  CSRK_CUDA_TRY(cudaMalloc(&g->idx, (m > 0 ? m : 1) * sizeof(int32_t)));
  CSRK_CUDA_TRY(cudaMalloc(&g->ew, (m > 0 ? m : 1) * sizeof(int32_t)));
  CSRK_CUDA_TRY(cudaMalloc(&g->nw, (n > 0 ? n : 1) * sizeof(int32_t)));
  CSRK_CUDA_TRY(src.alloc(m));
  run_compact_kernel<<<blocks_for(count), 256, 0, s>>>(keys, vals, count, pos.p, unit,
                                                      g->idx, g->ew, src.p);
  row_ptr_kernel<<<blocks_for(n + 1), 256, 0, s>>>(src.p, m, n, g->ptr);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

int sort_keys(uint64_t *keys, uint32_t *vals, int64_t count, int key_bits,
              cudaStream_t s) {
  Buf<uint64_t> tk(s);
  Buf<uint32_t> tv(s);
  CSRK_CUDA_TRY(tk.alloc(count));
  CSRK_CUDA_TRY(tv.alloc(count));
  return radix_sort_pairs(keys, vals, tk.p, tv.p, count, 0, key_bits, s);
}

int key_bits_for(int64_t n) {
  int b = 0;
  while (b < 32 && (int64_t(1) << b) < n + 1) ++b;
  return 32 + ((b + 7) / 8) * 8;  // low word = column, high word = row
}

void free_graph(csrk_dgraph *g) {
  if (!g) return;
  cudaFree(g->ptr);
  cudaFree(g->idx);
  cudaFree(g->ew);
  cudaFree(g->nw);
  delete g;
}

}  // namespace

int graph_build_dev(const csrk_matrix *a, csrk_dgraph **out) {
  const int64_t n = a->n_rows;
  cudaStream_t s = a->stream;
  Buf<int64_t> cnt(s), off(s);
  CSRK_CUDA_TRY(cnt.alloc(n));
  CSRK_CUDA_TRY(off.alloc(n + 1));
  offdiag_count_kernel<<<blocks_for(n), 256, 0, s>>>(a->row_ptr, a->col_idx, n, cnt.p);
  CSRK_TRY(exclusive_scan_i64(cnt.p, n, off.p, s));
  int64_t n_off = 0;
  CSRK_CUDA_TRY(cudaMemcpyAsync(&n_off, off.p + n, sizeof(n_off), cudaMemcpyDeviceToHost, s));
  CSRK_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t count = 2 * n_off;
  Buf<uint64_t> keys(s);
  Buf<uint32_t> vals(s);
  CSRK_CUDA_TRY(keys.alloc(count));
  CSRK_CUDA_TRY(vals.alloc(count));
  emit_sym_kernel<<<blocks_for(n), 256, 0, s>>>(a->row_ptr, a->col_idx, n, off.p, keys.p,
                                                vals.p);
  CSRK_TRY(sort_keys(keys.p, vals.p, count, key_bits_for(n), s));
  csrk_dgraph *g = new csrk_dgraph();
  g->device = a->device;
  int rc = finish_graph(g, n, keys.p, vals.p, count, /*unit=*/true, s);
  if (rc == CSRK_OK) {
    fill_i32_kernel<<<blocks_for(n), 256, 0, s>>>(g->nw, n, 1);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = CSRK_ECUDA;
  }
  if (rc != CSRK_OK) {
    free_graph(g);
    return rc;
  }
  *out = g;
  return CSRK_OK;
}

int graph_relabel_dev(const csrk_dgraph *g, const int64_t *fwd_dev, const int64_t *inv_dev,
                      cudaStream_t s, csrk_dgraph **out) {
  const int64_t count = g->m;
  Buf<uint64_t> keys(s);
  Buf<uint32_t> vals(s);
  CSRK_CUDA_TRY(keys.alloc(count));
  CSRK_CUDA_TRY(vals.alloc(count));
  emit_relabel_kernel<<<blocks_for(g->n), 256, 0, s>>>(g->ptr, g->idx, g->ew, fwd_dev, g->n,
                                                       keys.p, vals.p);
  CSRK_TRY(sort_keys(keys.p, vals.p, count, key_bits_for(g->n), s));
  csrk_dgraph *r = new csrk_dgraph();
  r->device = g->device;
  int rc = finish_graph(r, g->n, keys.p, vals.p, count, false, s);
  if (rc == CSRK_OK) {
    gather_nw_kernel<<<blocks_for(g->n), 256, 0, s>>>(g->nw, inv_dev, g->n, r->nw);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = CSRK_ECUDA;
  }
  if (rc != CSRK_OK) {
    free_graph(r);
    return rc;
  }
  *out = r;
  return CSRK_OK;
}

int graph_contract_dev(const csrk_dgraph *g, const int32_t *f2c_dev, int64_t m_coarse,
                       cudaStream_t s, csrk_dgraph **out) {
  const int64_t count = g->m;
  Buf<uint64_t> keys(s);
  Buf<uint32_t> vals(s);
  CSRK_CUDA_TRY(keys.alloc(count));
  CSRK_CUDA_TRY(vals.alloc(count));
  emit_contract_kernel<<<blocks_for(g->n), 256, 0, s>>>(g->ptr, g->idx, g->ew, f2c_dev, g->n,
                                                        keys.p, vals.p);
  // sentinel keys (all ones) need every bit sorted
  CSRK_TRY(sort_keys(keys.p, vals.p, count, 64, s));
  csrk_dgraph *r = new csrk_dgraph();
  r->device = g->device;
  int rc = finish_graph(r, m_coarse, keys.p, vals.p, count, false, s);
  if (rc == CSRK_OK) {
    cudaMemsetAsync(r->nw, 0, (m_coarse > 0 ? m_coarse : 1) * sizeof(int32_t), s);
    contract_nw_kernel<<<blocks_for(g->n), 256, 0, s>>>(g->nw, f2c_dev, g->n, r->nw);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = CSRK_ECUDA;
  }
  if (rc != CSRK_OK) {
    free_graph(r);
    return rc;
  }
  *out = r;
  return CSRK_OK;
}

void graph_free_dev(csrk_dgraph *g) { free_graph(g); }

}  // namespace csrk

using namespace csrk;

extern "C" {

int csrk_dgraph_build(const csrk_matrix *a, csrk_dgraph **out) {
  if (!a || !out) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (a->n_rows != a->n_cols) {
    set_error("graph construction requires a square matrix");
    return CSRK_EINVAL;
  }
  if (a->n_rows > 0x7fffffffLL) {
    set_error("graph size out of range");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(a->device));
  *out = nullptr;
  return graph_build_dev(a, out);
}

int csrk_dgraph_relabel(const csrk_dgraph *g, const int64_t *fwd_host, csrk_dgraph **out) {
  if (!g || !fwd_host || !out) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(g->device));
  const int64_t n = g->n;
  std::vector<int64_t> inv(n);
  for (int64_t i = 0; i < n; ++i) inv[fwd_host[i]] = i;
  int64_t *d = nullptr;
  CSRK_CUDA_TRY(cudaMalloc(&d, 2 * (n > 0 ? n : 1) * sizeof(int64_t)));
  cudaMemcpy(d, fwd_host, n * sizeof(int64_t), cudaMemcpyHostToDevice);
  cudaMemcpy(d + n, inv.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice);
  *out = nullptr;
  const int rc = graph_relabel_dev(g, d, d + n, nullptr, out);
  cudaFree(d);
  return rc;
}

int csrk_dgraph_contract(const csrk_dgraph *g, const int64_t *f2c_host, int64_t m,
                         csrk_dgraph **out) {
  if (!g || !f2c_host || !out) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(g->device));
  const int64_t n = g->n;
  std::vector<int32_t> f(n);
  for (int64_t i = 0; i < n; ++i) f[i] = static_cast<int32_t>(f2c_host[i]);
  int32_t *d = nullptr;
  CSRK_CUDA_TRY(cudaMalloc(&d, (n > 0 ? n : 1) * sizeof(int32_t)));
  cudaMemcpy(d, f.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice);
  *out = nullptr;
  const int rc = graph_contract_dev(g, d, m, nullptr, out);
  cudaFree(d);
  return rc;
}

int csrk_dgraph_sizes(const csrk_dgraph *g, int64_t out[2]) {
  if (!g || !out) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  out[0] = g->n;
  out[1] = g->m;
  return CSRK_OK;
}

int csrk_dgraph_download(const csrk_dgraph *g, int64_t *ptr, int64_t *idx, int64_t *ew,
                         int64_t *nw) {
  if (!g) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(g->device));
  if (ptr) CSRK_CUDA_TRY(cudaMemcpy(ptr, g->ptr, (g->n + 1) * 8, cudaMemcpyDeviceToHost));
  std::vector<int32_t> t(g->m > g->n ? g->m : g->n);
  if (idx) {
    CSRK_CUDA_TRY(cudaMemcpy(t.data(), g->idx, g->m * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < g->m; ++i) idx[i] = t[i];
  }
  if (ew) {
    CSRK_CUDA_TRY(cudaMemcpy(t.data(), g->ew, g->m * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < g->m; ++i) ew[i] = t[i];
  }
  if (nw) {
    CSRK_CUDA_TRY(cudaMemcpy(t.data(), g->nw, g->n * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < g->n; ++i) nw[i] = t[i];
  }
  return CSRK_OK;
}

int csrk_dgraph_free(csrk_dgraph *g) {
  graph_free_dev(g);
  return CSRK_OK;
}

}  // extern "C"
