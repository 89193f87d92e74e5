// Device Band-k: the whole of reorder.py:415-469 on the GPU, bit-exact.
//
//   build_graph / relabel / contract   graph.cu (radix-sort based)
//   weighted_bandwidth_order           rcm.cu (level-synchronous exact CM)
//   heavy_edge_matching / coarsen      coarsen.cu (Jacobi fixed point)
//   _expand_level / _order_members     here
//
// _expand_level places the members of each coarse node (a "block") in coarse
// sequence order.  A member's seed key is (anchor, outside_unplaced, key):
// outside_unplaced counts neighbours in later blocks, which is fixed by the
// block order; anchor is the smallest placed position of a neighbour in an
// earlier block, which depends on earlier blocks' internal orders.  Every
// block is ordered by one thread from the previous iteration's positions
// (seeded BFS inside the block with key-sorted frontiers, reorder.py:339-387)
// until no position changes -- the unique fixed point is the sequential
// result because a block only reads positions of earlier blocks.

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.h"

struct csrk_bandk_result {
  std::vector<int64_t> fwd;
  std::vector<int64_t> sizes1, sizes2;
};

namespace csrk {

int graph_build_dev(const csrk_matrix *a, csrk_dgraph **out);
int graph_wbo_dev(const csrk_dgraph *g, int64_t *fwd_dev, cudaStream_t s);
int graph_relabel_dev(const csrk_dgraph *g, const int64_t *fwd_dev, const int64_t *inv_dev,
                      cudaStream_t s, csrk_dgraph **out);
int graph_coarsen_dev(const csrk_dgraph *g, double target, int32_t *f2c, csrk_dgraph **out,
                      cudaStream_t s);
void graph_free_dev(csrk_dgraph *g);

namespace {

inline unsigned nbk(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return static_cast<unsigned>(b);
}

#define GSX(i, n)                                                          \
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < (n); \
       i += int64_t(gridDim.x) * blockDim.x)

constexpr int64_t kInf64 = 0x7fffffffffffffffLL;

template <typename T>
struct DV {  // stream-ordered scratch from the kept pool (keep_async_pool)
  T *p = nullptr;
  cudaStream_t st = nullptr;
  ~DV() {
    if (p) cudaFreeAsync(p, st);
  }
  cudaError_t alloc(int64_t n, cudaStream_t s) {
    keep_async_pool();
    st = s;
    return cudaMallocAsync(&p, (n > 0 ? n : 1) * sizeof(T), s);
  }
};

__global__ void inv64_kernel(const int64_t *__restrict__ fwd, int64_t n,
                             int64_t *__restrict__ inv) {
  GSX(i, n) { inv[fwd[i]] = i; }
}

__global__ void compose_f2c_kernel(int32_t *__restrict__ f2c, const int64_t *__restrict__ fwd,
                                   int64_t n) {
  GSX(i, n) { f2c[i] = static_cast<int32_t>(fwd[f2c[i]]); }
}

__global__ void member_keys_kernel(const int32_t *__restrict__ f2c, int64_t n,
                                   uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  GSX(v, n) {
    keys[v] = static_cast<uint32_t>(f2c[v]);
    vals[v] = static_cast<uint32_t>(v);
  }
}

__global__ void count_kernel(const int32_t *__restrict__ f2c, int64_t n,
                             int64_t *__restrict__ cnt) {
  GSX(v, n) { atomicAdd(reinterpret_cast<unsigned long long *>(&cnt[f2c[v]]), 1ull); }
}

__global__ void key_rank_keys_kernel(const int64_t *__restrict__ ptr,
                                     const int32_t *__restrict__ nw, int64_t n,
                                     uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  GSX(v, n) {
    keys[v] = (static_cast<uint64_t>(ptr[v + 1] - ptr[v]) << 32) | static_cast<uint32_t>(nw[v]);
    vals[v] = static_cast<uint32_t>(v);
  }
}

__global__ void scatter_rank_kernel(const uint32_t *__restrict__ order, int64_t n,
                                    uint32_t *__restrict__ krank) {
  GSX(i, n) { krank[order[i]] = static_cast<uint32_t>(i); }
}

// block sizes in sequence order and each member's block index
__global__ void block_size_kernel(const int64_t *__restrict__ seq,
                                  const int64_t *__restrict__ mptr, int64_t nb,
                                  int64_t *__restrict__ bsize) {
  GSX(i, nb) { bsize[i] = mptr[seq[i] + 1] - mptr[seq[i]]; }
}

__global__ void block_of_kernel(const int64_t *__restrict__ seq,
                                const int64_t *__restrict__ mptr,
                                const uint32_t *__restrict__ mem,
                                const int64_t *__restrict__ off, int64_t nb,
                                int64_t *__restrict__ blk, int64_t *__restrict__ pos) {
  GSX(i, nb) {
    const int64_t c = seq[i];
    for (int64_t j = mptr[c]; j < mptr[c + 1]; ++j) {
      blk[mem[j]] = i;
      pos[mem[j]] = off[i] + (j - mptr[c]);
    }
  }
}

__global__ void outside_kernel(const int64_t *__restrict__ ptr, const int32_t *__restrict__ idx,
                               const int64_t *__restrict__ blk, int64_t n,
                               int64_t *__restrict__ outside) {
  GSX(v, n) {
    int64_t c = 0;
    for (int64_t p = ptr[v]; p < ptr[v + 1]; ++p) c += blk[idx[p]] > blk[v];
    outside[v] = c;
  }
}

// One Jacobi step: every block (one thread) orders its members from the
// previous positions and writes their new positions.
__global__ void order_blocks_kernel(const int64_t *__restrict__ ptr,
                                    const int32_t *__restrict__ idx,
                                    const uint32_t *__restrict__ krank,
                                    const int64_t *__restrict__ seq,
                                    const int64_t *__restrict__ mptr,
                                    const uint32_t *__restrict__ mem,
                                    const int64_t *__restrict__ off,
                                    const int64_t *__restrict__ blk,
                                    const int64_t *__restrict__ outside, int64_t nb,
                                    const int64_t *__restrict__ pos_prev,
                                    int64_t *__restrict__ pos_next,
                                    int64_t *__restrict__ anchor, int32_t *__restrict__ cand,
                                    int32_t *__restrict__ queue, int8_t *__restrict__ state) {
  GSX(i, nb) {
    const int64_t c = seq[i];
    const int64_t m0 = mptr[c], size = mptr[c + 1] - m0, base = off[i];
    int32_t *cd = cand + base;
    int32_t *q = queue + base;
    // seed keys
    for (int64_t j = 0; j < size; ++j) {
      const int32_t v = static_cast<int32_t>(mem[m0 + j]);
      int64_t a = kInf64;
      for (int64_t p = ptr[v]; p < ptr[v + 1]; ++p) {
        const int32_t u = idx[p];
        if (blk[u] < i) a = min(a, pos_prev[u]);
      }
      anchor[v] = a;
      state[v] = 1;  // remaining
      // insertion sort of candidates by (anchor, outside, krank)
      int64_t k = j;
      while (k > 0) {
        const int32_t w = cd[k - 1];
        const bool less = a != anchor[w] ? a < anchor[w]
                          : outside[v] != outside[w] ? outside[v] < outside[w]
                                                     : krank[v] < krank[w];
        if (!less) break;
        cd[k] = w;
        --k;
      }
      cd[k] = v;
    }
    int64_t qlen = 0, next_seed = 0;
    while (qlen < size) {
      while (state[cd[next_seed]] != 1) ++next_seed;
      const int32_t seed = cd[next_seed];
      state[seed] = 2;
      q[qlen++] = seed;
      for (int64_t h = qlen - 1; h < qlen; ++h) {
        const int32_t v = q[h];
        const int64_t fresh0 = qlen;
        for (int64_t p = ptr[v]; p < ptr[v + 1]; ++p) {
          const int32_t u = idx[p];
          if (blk[u] == i && state[u] == 1) {
            state[u] = 2;
            // insert u keeping q[fresh0..qlen) sorted by key rank
            int64_t k = qlen++;
            while (k > fresh0 && krank[q[k - 1]] > krank[u]) {
              q[k] = q[k - 1];
              --k;
            }
            q[k] = u;
          }
        }
      }
    }
    for (int64_t j = 0; j < size; ++j) {
      pos_next[q[j]] = base + j;
      state[q[j]] = 0;
    }
  }
}

__global__ void pos_diff_kernel(const int64_t *__restrict__ a, const int64_t *__restrict__ b,
                                int64_t n, int *__restrict__ changed) {
  GSX(i, n) {
    if (a[i] != b[i]) *changed = 1;
  }
}

__global__ void seq_from_pos_kernel(const int64_t *__restrict__ pos, int64_t n,
                                    int64_t *__restrict__ seq) {
  GSX(v, n) { seq[pos[v]] = v; }
}

__global__ void iota64_kernel(int64_t *__restrict__ a, int64_t n) {
  GSX(i, n) { a[i] = i; }
}

__global__ void final_perm_kernel(const int64_t *__restrict__ seq,
                                  const int64_t *__restrict__ base_inv, int64_t n,
                                  int64_t *__restrict__ fwd) {
  GSX(i, n) { fwd[base_inv[seq[i]]] = i; }
}

struct Level {
  int64_t n_coarse = 0;
  int64_t *mptr = nullptr;  // device, n_coarse + 1
  uint32_t *mem = nullptr;  // device, fine nodes grouped by coarse node
};

int make_level(const int32_t *f2c, int64_t n_fine, int64_t n_coarse, Level &lv,
               cudaStream_t s) {
  DV<uint64_t> keys, tk;
  DV<uint32_t> tv;
  DV<int64_t> cnt;
  CSRK_CUDA_TRY(keys.alloc(n_fine, s));
  CSRK_CUDA_TRY(tk.alloc(n_fine, s));
  CSRK_CUDA_TRY(tv.alloc(n_fine, s));
  CSRK_CUDA_TRY(cnt.alloc(n_coarse, s));
  CSRK_CUDA_TRY(cudaMalloc(&lv.mem, (n_fine > 0 ? n_fine : 1) * sizeof(uint32_t)));
  CSRK_CUDA_TRY(cudaMalloc(&lv.mptr, (n_coarse + 1) * sizeof(int64_t)));
  member_keys_kernel<<<nbk(n_fine), 256, 0, s>>>(f2c, n_fine, keys.p, lv.mem);
  CSRK_TRY(radix_sort_pairs(keys.p, lv.mem, tk.p, tv.p, n_fine, 0, 32, s));
  CSRK_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, n_coarse * sizeof(int64_t), s));
  count_kernel<<<nbk(n_fine), 256, 0, s>>>(f2c, n_fine, cnt.p);
  CSRK_TRY(exclusive_scan_i64(cnt.p, n_coarse, lv.mptr, s));
  lv.n_coarse = n_coarse;
  return CSRK_OK;
}

// fine sequence (device, n = g->n) from a coarse sequence (device, lv.n_coarse)
int expand_level_dev(const csrk_dgraph *g, const Level &lv, const int64_t *seq_coarse,
                     int64_t *seq_fine, std::vector<int64_t> &sizes, int *iters,
                     cudaStream_t s) {
  const int64_t n = g->n, nb = lv.n_coarse;
  DV<int64_t> bsize, off, blk, pos_a, pos_b, outside, anchor;
  DV<uint32_t> krank, tv;
  DV<uint64_t> keys, tk;
  DV<int32_t> cand, queue;
  DV<int8_t> state;
  DV<int> flag;
  CSRK_CUDA_TRY(bsize.alloc(nb, s));
  CSRK_CUDA_TRY(off.alloc(nb + 1, s));
  CSRK_CUDA_TRY(blk.alloc(n, s));
  CSRK_CUDA_TRY(pos_a.alloc(n, s));
  CSRK_CUDA_TRY(pos_b.alloc(n, s));
  CSRK_CUDA_TRY(outside.alloc(n, s));
  CSRK_CUDA_TRY(anchor.alloc(n, s));
  CSRK_CUDA_TRY(krank.alloc(n, s));
  CSRK_CUDA_TRY(tv.alloc(n, s));
  CSRK_CUDA_TRY(keys.alloc(n, s));
  CSRK_CUDA_TRY(tk.alloc(n, s));
  CSRK_CUDA_TRY(cand.alloc(n, s));
  CSRK_CUDA_TRY(queue.alloc(n, s));
  CSRK_CUDA_TRY(state.alloc(n, s));
  CSRK_CUDA_TRY(flag.alloc(1, s));
  CSRK_CUDA_TRY(cudaMemsetAsync(state.p, 0, n, s));
  // key ranks (degree, weight, index)
  DV<uint32_t> order;
  CSRK_CUDA_TRY(order.alloc(n, s));
  key_rank_keys_kernel<<<nbk(n), 256, 0, s>>>(g->ptr, g->nw, n, keys.p, order.p);
  CSRK_TRY(radix_sort_pairs(keys.p, order.p, tk.p, tv.p, n, 0, 64, s));
  scatter_rank_kernel<<<nbk(n), 256, 0, s>>>(order.p, n, krank.p);
  block_size_kernel<<<nbk(nb), 256, 0, s>>>(seq_coarse, lv.mptr, nb, bsize.p);
  CSRK_TRY(exclusive_scan_i64(bsize.p, nb, off.p, s));
  block_of_kernel<<<nbk(nb), 256, 0, s>>>(seq_coarse, lv.mptr, lv.mem, off.p, nb, blk.p,
                                          pos_a.p);
  outside_kernel<<<nbk(n), 256, 0, s>>>(g->ptr, g->idx, blk.p, n, outside.p);
  int it = 0;
  for (;; ++it) {
    order_blocks_kernel<<<nbk(nb, 128), 128, 0, s>>>(
        g->ptr, g->idx, krank.p, seq_coarse, lv.mptr, lv.mem, off.p, blk.p, outside.p, nb,
        pos_a.p, pos_b.p, anchor.p, cand.p, queue.p, state.p);
    int h = 0;
    CSRK_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
    pos_diff_kernel<<<nbk(n), 256, 0, s>>>(pos_a.p, pos_b.p, n, flag.p);
    CSRK_CUDA_TRY(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    std::swap(pos_a.p, pos_b.p);
    if (!h) break;
  }
  seq_from_pos_kernel<<<nbk(n), 256, 0, s>>>(pos_a.p, n, seq_fine);
  sizes.resize(nb);
  CSRK_CUDA_TRY(cudaMemcpyAsync(sizes.data(), bsize.p, nb * sizeof(int64_t),
                                cudaMemcpyDeviceToHost, s));
  CSRK_CUDA_TRY(cudaStreamSynchronize(s));
  if (iters) *iters = it + 1;
  return CSRK_OK;
}

}  // namespace

// CSRK_BANDK_PROFILE=1: per-phase wall time of the device Band-k
struct DevPhase {
  const char *name;
  std::chrono::steady_clock::time_point t0;
  cudaStream_t s;
  DevPhase(const char *n, cudaStream_t st) : name(n), t0(std::chrono::steady_clock::now()), s(st) {}
  ~DevPhase() {
    if (!std::getenv("CSRK_BANDK_PROFILE")) return;
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "[band_k dev] %-12s %8.3f s\n", name,
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
};

int band_k_dev(const csrk_matrix *a, int k, const double *targets, csrk_bandk_result &res,
               int64_t *fwd_dev_out, cudaStream_t s) {
  const int64_t n = a->n_rows;
  std::vector<csrk_dgraph *> graphs;
  std::vector<Level> levels;
  std::vector<int64_t *> tofree;
  auto cleanup = [&]() {
    for (auto *g : graphs) graph_free_dev(g);
    for (auto &lv : levels) {
      cudaFree(lv.mptr);
      cudaFree(lv.mem);
    }
    for (auto *p : tofree) cudaFree(p);
  };
  int rc = CSRK_OK;
  csrk_dgraph *g0 = nullptr;
  int64_t *base = nullptr, *base_inv = nullptr;
  do {
    { DevPhase ph("build", s); rc = graph_build_dev(a, &g0); }
    if (rc != CSRK_OK) break;
    if (cudaMalloc(&base, n * sizeof(int64_t)) != cudaSuccess ||
        cudaMalloc(&base_inv, n * sizeof(int64_t)) != cudaSuccess) {
      rc = CSRK_ENOMEM;
      break;
    }
    tofree.push_back(base);
    tofree.push_back(base_inv);
    { DevPhase ph("wbo-base", s); rc = graph_wbo_dev(g0, base, s); }
    if (rc != CSRK_OK) break;
    inv64_kernel<<<nbk(n), 256, 0, s>>>(base, n, base_inv);
    csrk_dgraph *g0r = nullptr;
    if ((rc = graph_relabel_dev(g0, base, base_inv, s, &g0r)) != CSRK_OK) break;
    graph_free_dev(g0);
    g0 = nullptr;
    graphs.push_back(g0r);
    for (int t = 0; t < k - 1 && rc == CSRK_OK; ++t) {
      const csrk_dgraph *fine = graphs.back();
      int32_t *f2c = nullptr;
      if (cudaMalloc(&f2c, (fine->n > 0 ? fine->n : 1) * sizeof(int32_t)) != cudaSuccess) {
        rc = CSRK_ENOMEM;
        break;
      }
      tofree.push_back(reinterpret_cast<int64_t *>(f2c));
      csrk_dgraph *coarse = nullptr;
      { DevPhase ph("coarsen", s); rc = graph_coarsen_dev(fine, targets[t], f2c, &coarse, s); }
      if (rc != CSRK_OK) break;
      const int64_t m = coarse->n;
      int64_t *ord = nullptr, *ord_inv = nullptr;
      if (cudaMalloc(&ord, (m > 0 ? m : 1) * sizeof(int64_t)) != cudaSuccess ||
          cudaMalloc(&ord_inv, (m > 0 ? m : 1) * sizeof(int64_t)) != cudaSuccess) {
        graph_free_dev(coarse);
        rc = CSRK_ENOMEM;
        break;
      }
      tofree.push_back(ord);
      tofree.push_back(ord_inv);
      if ((rc = graph_wbo_dev(coarse, ord, s)) != CSRK_OK) {
        graph_free_dev(coarse);
        break;
      }
      inv64_kernel<<<nbk(m), 256, 0, s>>>(ord, m, ord_inv);
      csrk_dgraph *coarse_r = nullptr;
      rc = graph_relabel_dev(coarse, ord, ord_inv, s, &coarse_r);
      graph_free_dev(coarse);
      if (rc != CSRK_OK) break;
      compose_f2c_kernel<<<nbk(fine->n), 256, 0, s>>>(f2c, ord, fine->n);
      Level lv;
      if ((rc = make_level(f2c, fine->n, m, lv, s)) != CSRK_OK) {
        graph_free_dev(coarse_r);
        break;
      }
      graphs.push_back(coarse_r);
      levels.push_back(lv);
    }
    if (rc != CSRK_OK) break;
    // expand top-down
    int64_t *seq = nullptr;
    const int64_t n_top = graphs.back()->n;
    if (cudaMalloc(&seq, (n_top > 0 ? n_top : 1) * sizeof(int64_t)) != cudaSuccess) {
      rc = CSRK_ENOMEM;
      break;
    }
    iota64_kernel<<<nbk(n_top), 256, 0, s>>>(seq, n_top);
    std::vector<std::vector<int64_t>> collected;
    for (int level = k - 1; level >= 1 && rc == CSRK_OK; --level) {
      const csrk_dgraph *fine = graphs[level - 1];
      int64_t *fine_seq = nullptr;
      if (cudaMalloc(&fine_seq, (fine->n > 0 ? fine->n : 1) * sizeof(int64_t)) !=
          cudaSuccess) {
        rc = CSRK_ENOMEM;
        break;
      }
      std::vector<int64_t> sizes;
      { DevPhase ph("expand", s);
        rc = expand_level_dev(fine, levels[level - 1], seq, fine_seq, sizes, nullptr, s); }
      cudaFree(seq);
      seq = fine_seq;
      collected.push_back(std::move(sizes));
    }
    if (rc != CSRK_OK) {
      cudaFree(seq);
      break;
    }
    int64_t *fwd = fwd_dev_out;
    if (!fwd) {
      if (cudaMalloc(&fwd, n * sizeof(int64_t)) != cudaSuccess) {
        cudaFree(seq);
        rc = CSRK_ENOMEM;
        break;
      }
      tofree.push_back(fwd);
    }
    final_perm_kernel<<<nbk(n), 256, 0, s>>>(seq, base_inv, n, fwd);
    cudaFree(seq);
    res.fwd.resize(n);
    if (cudaMemcpyAsync(res.fwd.data(), fwd, n * sizeof(int64_t), cudaMemcpyDeviceToHost,
                        s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      rc = CSRK_ECUDA;
      break;
    }
    res.sizes1 = collected.back();
    if (k == 3) res.sizes2 = collected.front();
  } while (false);
  if (g0) graph_free_dev(g0);
  cleanup();
  if (rc == CSRK_OK && cudaGetLastError() != cudaSuccess) rc = CSRK_ECUDA;
  return rc;
}

}  // namespace csrk

extern "C" int csrk_band_k_device(const csrk_matrix *a, int k, const double *targets,
                                  csrk_bandk_result **out) {
  if (!a || !targets || !out) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  if (k != 2 && k != 3) {
    csrk::set_error("k must be 2 or 3");
    return CSRK_EINVAL;
  }
  if (a->n_rows == 0) {
    csrk::set_error("cannot reorder an empty matrix");
    return CSRK_EINVAL;
  }
  if (a->n_rows != a->n_cols) {
    csrk::set_error("graph construction requires a square matrix");
    return CSRK_EINVAL;
  }
  for (int t = 0; t < k - 1; ++t)
    if (!(targets[t] >= 1.0)) {
      csrk::set_error("target_weight must be at least 1");
      return CSRK_EINVAL;
    }
  CSRK_CUDA_TRY(cudaSetDevice(a->device));
  auto *res = new csrk_bandk_result();
  const int rc = csrk::band_k_dev(a, k, targets, *res, nullptr, a->stream);
  cudaStreamSynchronize(a->stream);
  csrk::trim_async_pool();  // the builder's scratch goes back to the driver
  if (rc != CSRK_OK) {
    delete res;
    if (rc == CSRK_ECUDA) csrk::set_error("CUDA error in device band_k");
    return rc;
  }
  *out = res;
  return CSRK_OK;
}
