// Device weighted_bandwidth_order (reverse Cuthill-McKee with
// pseudo-peripheral starts), bit-exact with reorder.py:240-336.
//
// The sequential algorithm (per component, largest first, ties by smallest
// index): start from a pseudo-peripheral node, BFS appending each dequeued
// node's still-unvisited neighbours sorted by key = (degree, node weight,
// index), reverse the whole order at the end.  Level-synchronous form used
// here: the nodes of BFS level L+1 are exactly the
// unvisited neighbours of level L; a node is appended by the FIRST level-L
// node (in queue order) adjacent to it, so its queue position is the pair
// (min position of a level-L neighbour, key rank).  Sorting each new level by
// (component rank, parent position, key rank) reproduces the sequential queue
// exactly.  All components advance together.
//
//   krank      rank of every node by (degree, weight, index): one stable sort
//   components label propagation + pointer jumping; label = min index, which
//              is also the reference's "min(c)" and enumeration root
//   pseudo-peripheral starts: repeated multi-source BFS (reorder.py:263-278)

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace csrk {
namespace {

constexpr int32_t kNone = -1;
constexpr uint32_t kInf = 0xffffffffu;

inline unsigned nblocks(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return static_cast<unsigned>(b);
}

#define GSTRIDE(i, n)                                                      \
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < (n); \
       i += int64_t(gridDim.x) * blockDim.x)

__global__ void key_kernel(const int64_t *__restrict__ ptr, const int32_t *__restrict__ nw,
                           int64_t n, uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  GSTRIDE(v, n) {
    keys[v] = (static_cast<uint64_t>(ptr[v + 1] - ptr[v]) << 32) | static_cast<uint32_t>(nw[v]);
    vals[v] = static_cast<uint32_t>(v);
  }
}

__global__ void rank_kernel(const uint32_t *__restrict__ sorted, int64_t n,
                            uint32_t *__restrict__ krank) {
  GSTRIDE(i, n) { krank[sorted[i]] = static_cast<uint32_t>(i); }
}

__global__ void label_init_kernel(int32_t *__restrict__ label, int64_t n) {
  GSTRIDE(v, n) { label[v] = static_cast<int32_t>(v); }
}

__global__ void label_hook_kernel(const int64_t *__restrict__ ptr,
                                  const int32_t *__restrict__ idx, int64_t n,
                                  int32_t *__restrict__ label, int *__restrict__ changed) {
  GSTRIDE(v, n) {
    const int32_t old = label[v];
    int32_t m = old;
    for (int64_t p = ptr[v]; p < ptr[v + 1]; ++p) m = min(m, label[idx[p]]);
    if (m < old) {  // hook v and its old root onto the smaller label
      atomicMin(&label[v], m);
      atomicMin(&label[old], m);
      *changed = 1;
    }
  }
}

__global__ void label_jump_kernel(int32_t *__restrict__ label, int64_t n) {
  GSTRIDE(v, n) {
    int32_t l = label[v];
    while (label[l] != l) l = label[l];
    label[v] = l;
  }
}

// component sizes and per-component minimum key rank
__global__ void comp_stats_kernel(const int32_t *__restrict__ label,
                                  const uint32_t *__restrict__ krank, int64_t n,
                                  int32_t *__restrict__ size, uint32_t *__restrict__ minrank) {
  GSTRIDE(v, n) {
    atomicAdd(&size[label[v]], 1);
    atomicMin(&minrank[label[v]], krank[v]);
  }
}

// roots ordered by (-size, root): key ((n - size) << 32 | root)
__global__ void root_keys_kernel(const int32_t *__restrict__ label,
                                 const int32_t *__restrict__ size, int64_t n,
                                 uint64_t *__restrict__ keys, uint32_t *__restrict__ vals,
                                 int *__restrict__ count) {
  GSTRIDE(v, n) {
    if (label[v] == v) {
      const int slot = atomicAdd(count, 1);
      keys[slot] = (static_cast<uint64_t>(n - size[v]) << 32) | static_cast<uint32_t>(v);
      vals[slot] = static_cast<uint32_t>(v);
    }
  }
}

// ---- multi-source BFS for the pseudo-peripheral search --------------------

__global__ void bfs_seed_kernel(const int32_t *__restrict__ seeds, int64_t k,
                                int32_t *__restrict__ depth, int32_t *__restrict__ frontier) {
  GSTRIDE(i, k) {
    depth[seeds[i]] = 0;
    frontier[i] = seeds[i];
  }
}

__global__ void bfs_expand_kernel(const int64_t *__restrict__ ptr,
                                  const int32_t *__restrict__ idx,
                                  const int32_t *__restrict__ frontier, int64_t fsize, int32_t level,
                                  int32_t *__restrict__ depth, int32_t *__restrict__ next,
                                  int *__restrict__ next_count) {
  GSTRIDE(i, fsize) {
    const int32_t v = frontier[i];
    for (int64_t p = ptr[v]; p < ptr[v + 1]; ++p) {
      const int32_t u = idx[p];
      if (depth[u] == kNone && atomicCAS(&depth[u], kNone, level + 1) == kNone)
        next[atomicAdd(next_count, 1)] = u;
    }
  }
}

// eccentricity per component and min key rank on the last level
__global__ void ecc_kernel(const int32_t *__restrict__ depth, const int32_t *__restrict__ label,
                           int64_t n, int32_t *__restrict__ ecc) {
  GSTRIDE(v, n) {
    if (depth[v] != kNone) atomicMax(&ecc[label[v]], depth[v]);
  }
}

__global__ void last_level_kernel(const int32_t *__restrict__ depth,
                                  const int32_t *__restrict__ label,
                                  const int32_t *__restrict__ ecc,
                                  const uint32_t *__restrict__ krank, int64_t n,
                                  uint32_t *__restrict__ lastmin) {
  GSTRIDE(v, n) {
    const int32_t d = depth[v];
    if (d != kNone && d == ecc[label[v]]) atomicMin(&lastmin[label[v]], krank[v]);
  }
}

// ---- Cuthill-McKee levels ----------------------------------------------

__global__ void cm_claim_kernel(const int64_t *__restrict__ ptr, const int32_t *__restrict__ idx,
                                const int32_t *__restrict__ frontier, int64_t fsize,
                                const int32_t *__restrict__ pos, uint32_t *__restrict__ claim,
                                int32_t *__restrict__ inq, int32_t *__restrict__ next,
                                int *__restrict__ next_count) {
  GSTRIDE(i, fsize) {
    const int32_t v = frontier[i];
    const uint32_t pv = static_cast<uint32_t>(pos[v]);
    for (int64_t p = ptr[v]; p < ptr[v + 1]; ++p) {
      const int32_t u = idx[p];
      if (pos[u] != kNone) continue;
      atomicMin(&claim[u], pv);
      if (atomicExch(&inq[u], 1) == 0) next[atomicAdd(next_count, 1)] = u;
    }
  }
}

// single-component levels: one 64-bit key (claim << kbits | krank)
__global__ void cm_key_kernel(const int32_t *__restrict__ next, int64_t k,
                              const uint32_t *__restrict__ claim,
                              const uint32_t *__restrict__ krank, int kbits,
                              uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  GSTRIDE(i, k) {
    const int32_t u = next[i];
    keys[i] = (static_cast<uint64_t>(claim[u]) << kbits) | krank[u];
    vals[i] = static_cast<uint32_t>(u);
  }
}

__global__ void comp_key_kernel(const uint32_t *__restrict__ order, int64_t k,
                                const int32_t *__restrict__ label,
                                const int32_t *__restrict__ crank,
                                uint64_t *__restrict__ keys) {
  GSTRIDE(i, k) { keys[i] = static_cast<uint32_t>(crank[label[order[i]]]); }
}

// positions: u at sorted index i of component c gets qlen[c] + (i - first
// index of c in this level); qlen grows by the level's count of c
__global__ void cm_place_kernel(const uint32_t *__restrict__ order, int64_t k,
                                const int32_t *__restrict__ label, int32_t *__restrict__ qlen,
                                int32_t *__restrict__ pos, uint32_t *__restrict__ claim,
                                int32_t *__restrict__ inq, int32_t *__restrict__ frontier) {
  GSTRIDE(i, k) {
    const int32_t u = static_cast<int32_t>(order[i]);
    const int32_t c = label[u];
    // first index of this component's run (components are contiguous runs)
    int64_t lo = 0, hi = i;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (label[order[mid]] == c)
        hi = mid;
      else
        lo = mid + 1;
    }
    pos[u] = qlen[c] + static_cast<int32_t>(i - lo);
    claim[u] = kInf;
    inq[u] = 0;
    frontier[i] = u;
  }
}

__global__ void cm_count_kernel(const uint32_t *__restrict__ order, int64_t k,
                                const int32_t *__restrict__ label, int32_t *__restrict__ qlen) {
  GSTRIDE(i, k) { atomicAdd(&qlen[label[order[i]]], 1); }
}

__global__ void final_fwd_kernel(const int32_t *__restrict__ pos,
                                 const int32_t *__restrict__ label,
                                 const int64_t *__restrict__ coff, int64_t n,
                                 int64_t *__restrict__ fwd) {
  GSTRIDE(v, n) { fwd[v] = n - 1 - (coff[label[v]] + pos[v]); }
}


// ---- per-component state on the device ----------------------------------

// component rank of every root and the components' first queue offsets
__global__ void comp_layout_kernel(const uint32_t *__restrict__ roots, int64_t n_comp,
                                   const int32_t *__restrict__ size,
                                   const int64_t *__restrict__ size_off,
                                   int32_t *__restrict__ crank, int64_t *__restrict__ coff) {
  GSTRIDE(c, n_comp) {
    const uint32_t r = roots[c];
    crank[r] = static_cast<int32_t>(c);
    coff[r] = size_off[c];
  }
}

__global__ void comp_sizes_kernel(const uint32_t *__restrict__ roots, int64_t n_comp,
                                  const int32_t *__restrict__ size, int64_t *__restrict__ out) {
  GSTRIDE(c, n_comp) { out[c] = size[roots[c]]; }
}

// pseudo-peripheral state: start = min-key node; best_ecc = -1; active
__global__ void pp_init_kernel(const uint32_t *__restrict__ roots, int64_t n_comp,
                               const uint32_t *__restrict__ minrank,
                               const uint32_t *__restrict__ by_key,
                               int32_t *__restrict__ start, int32_t *__restrict__ best_node,
                               int32_t *__restrict__ best_ecc, int8_t *__restrict__ active) {
  GSTRIDE(c, n_comp) {
    start[c] = static_cast<int32_t>(by_key[minrank[roots[c]]]);
    best_node[c] = -1;
    best_ecc[c] = -1;
    active[c] = 1;
  }
}

// seeds of the next BFS: starts of the still-active components
__global__ void pp_seeds_kernel(const int32_t *__restrict__ start,
                                const int8_t *__restrict__ active, int64_t n_comp,
                                int32_t *__restrict__ seeds, int *__restrict__ count) {
  GSTRIDE(c, n_comp) {
    if (active[c]) seeds[atomicAdd(count, 1)] = start[c];
  }
}

// reorder.py:270-278 for every active component after its BFS
__global__ void pp_update_kernel(const uint32_t *__restrict__ roots, int64_t n_comp,
                                 const int32_t *__restrict__ ecc,
                                 const uint32_t *__restrict__ lastmin,
                                 const uint32_t *__restrict__ by_key,
                                 int32_t *__restrict__ start, int32_t *__restrict__ best_node,
                                 int32_t *__restrict__ best_ecc, int8_t *__restrict__ active,
                                 int *__restrict__ still_active) {
  GSTRIDE(c, n_comp) {
    if (!active[c]) continue;
    const uint32_t r = roots[c];
    const int32_t e = ecc[r];
    if (e <= best_ecc[c]) {
      active[c] = 0;
      continue;
    }
    best_ecc[c] = e;
    best_node[c] = start[c];
    start[c] = static_cast<int32_t>(by_key[lastmin[r]]);
    if (start[c] == best_node[c]) {
      active[c] = 0;
      continue;
    }
    atomicAdd(still_active, 1);
  }
}

// Cuthill-McKee level 0: every component's start at queue position 0
__global__ void cm_init_kernel(const uint32_t *__restrict__ roots, int64_t n_comp,
                               const int32_t *__restrict__ best_node, int32_t *__restrict__ pos,
                               int32_t *__restrict__ qlen, int32_t *__restrict__ frontier) {
  GSTRIDE(c, n_comp) {
    pos[best_node[c]] = 0;
    qlen[roots[c]] = 1;
    frontier[c] = best_node[c];
  }
}

template <typename T>
struct DBuf {
  T *p = nullptr;
  ~DBuf() { cudaFree(p); }
  cudaError_t alloc(int64_t n) { return cudaMalloc(&p, (n > 0 ? n : 1) * sizeof(T)); }
};

int bits_for(int64_t n) {
  int b = 1;
  while ((int64_t(1) << b) <= n) ++b;
  return b;
}

}  // namespace

int graph_wbo_dev(const csrk_dgraph *g, int64_t *fwd_dev, cudaStream_t s) {
  const int64_t n = g->n;
  if (n == 0) return CSRK_OK;
  DBuf<uint64_t> keys, tkeys;
  DBuf<uint32_t> vals, tvals, krank, by_key, claim, lastmin, minrank;
  DBuf<int32_t> label, size, depth, frontier, next, pos, inq, ecc, crank, qlen;
  DBuf<int32_t> start, best_node, best_ecc;
  DBuf<int8_t> active;
  DBuf<int> counter;
  DBuf<int64_t> coff, csize, csize_off;
  CSRK_CUDA_TRY(keys.alloc(n));
  CSRK_CUDA_TRY(tkeys.alloc(n));
  CSRK_CUDA_TRY(vals.alloc(n));
  CSRK_CUDA_TRY(tvals.alloc(n));
  CSRK_CUDA_TRY(krank.alloc(n));
  CSRK_CUDA_TRY(by_key.alloc(n));
  CSRK_CUDA_TRY(claim.alloc(n));
  CSRK_CUDA_TRY(lastmin.alloc(n));
  CSRK_CUDA_TRY(minrank.alloc(n));
  CSRK_CUDA_TRY(label.alloc(n));
  CSRK_CUDA_TRY(size.alloc(n));
  CSRK_CUDA_TRY(depth.alloc(n));
  CSRK_CUDA_TRY(frontier.alloc(n));
  CSRK_CUDA_TRY(next.alloc(n));
  CSRK_CUDA_TRY(pos.alloc(n));
  CSRK_CUDA_TRY(inq.alloc(n));
  CSRK_CUDA_TRY(ecc.alloc(n));
  CSRK_CUDA_TRY(crank.alloc(n));
  CSRK_CUDA_TRY(qlen.alloc(n));
  CSRK_CUDA_TRY(counter.alloc(4));
  CSRK_CUDA_TRY(coff.alloc(n + 1));

  // 1. key ranks: stable sort of (degree, weight) keeps index order on ties;
  //    by_key[rank] = node
  key_kernel<<<nblocks(n), 256, 0, s>>>(g->ptr, g->nw, n, keys.p, by_key.p);
  CSRK_TRY(radix_sort_pairs(keys.p, by_key.p, tkeys.p, tvals.p, n, 0, 64, s));
  rank_kernel<<<nblocks(n), 256, 0, s>>>(by_key.p, n, krank.p);

  // 2. components (label = minimum index), hook + jump rounds checked every 4
  label_init_kernel<<<nblocks(n), 256, 0, s>>>(label.p, n);
  for (;;) {
    int h = 0;
    for (int j = 0; j < 4; ++j) {
      if (j == 3) CSRK_CUDA_TRY(cudaMemsetAsync(counter.p, 0, sizeof(int), s));
      label_hook_kernel<<<nblocks(n), 256, 0, s>>>(g->ptr, g->idx, n, label.p, counter.p);
      label_jump_kernel<<<nblocks(n), 256, 0, s>>>(label.p, n);
    }
    CSRK_CUDA_TRY(cudaMemcpyAsync(&h, counter.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    if (!h) break;
  }
  CSRK_CUDA_TRY(cudaMemsetAsync(size.p, 0, n * sizeof(int32_t), s));
  CSRK_CUDA_TRY(cudaMemsetAsync(minrank.p, 0xff, n * sizeof(uint32_t), s));
  comp_stats_kernel<<<nblocks(n), 256, 0, s>>>(label.p, krank.p, n, size.p, minrank.p);
  CSRK_CUDA_TRY(cudaMemsetAsync(counter.p, 0, sizeof(int), s));
  root_keys_kernel<<<nblocks(n), 256, 0, s>>>(label.p, size.p, n, keys.p, vals.p, counter.p);
  int n_comp = 0;
  CSRK_CUDA_TRY(cudaMemcpyAsync(&n_comp, counter.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CSRK_CUDA_TRY(cudaStreamSynchronize(s));
  // roots in component order (-size, root); vals keeps them
  CSRK_TRY(radix_sort_pairs(keys.p, vals.p, tkeys.p, tvals.p, n_comp, 0, 64, s));
  const uint32_t *roots = vals.p;
  CSRK_CUDA_TRY(csize.alloc(n_comp));
  CSRK_CUDA_TRY(csize_off.alloc(n_comp + 1));
  CSRK_CUDA_TRY(start.alloc(n_comp));
  CSRK_CUDA_TRY(best_node.alloc(n_comp));
  CSRK_CUDA_TRY(best_ecc.alloc(n_comp));
  CSRK_CUDA_TRY(active.alloc(n_comp));
  comp_sizes_kernel<<<nblocks(n_comp), 256, 0, s>>>(roots, n_comp, size.p, csize.p);
  CSRK_TRY(exclusive_scan_i64(csize.p, n_comp, csize_off.p, s));
  comp_layout_kernel<<<nblocks(n_comp), 256, 0, s>>>(roots, n_comp, size.p, csize_off.p,
                                                     crank.p, coff.p);

  // 3. pseudo-peripheral start of every component (reorder.py:263-278),
  //    all components' BFS runs together, state stays on the device
  pp_init_kernel<<<nblocks(n_comp), 256, 0, s>>>(roots, n_comp, minrank.p, by_key.p, start.p,
                                                 best_node.p, best_ecc.p, active.p);
  int64_t n_active = n_comp;
  while (n_active > 0) {
    int k = 0;
    CSRK_CUDA_TRY(cudaMemsetAsync(counter.p, 0, sizeof(int), s));
    pp_seeds_kernel<<<nblocks(n_comp), 256, 0, s>>>(start.p, active.p, n_comp, next.p,
                                                    counter.p);
    CSRK_CUDA_TRY(cudaMemcpyAsync(&k, counter.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CSRK_CUDA_TRY(cudaMemsetAsync(depth.p, 0xff, n * sizeof(int32_t), s));
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    bfs_seed_kernel<<<nblocks(k), 256, 0, s>>>(next.p, k, depth.p, frontier.p);
    int64_t fsize = k;
    for (int32_t level = 0; fsize > 0; ++level) {
      int cnt = 0;
      CSRK_CUDA_TRY(cudaMemsetAsync(counter.p, 0, sizeof(int), s));
      bfs_expand_kernel<<<nblocks(fsize), 256, 0, s>>>(g->ptr, g->idx, frontier.p, fsize, level,
                                                       depth.p, next.p, counter.p);
      CSRK_CUDA_TRY(cudaMemcpyAsync(&cnt, counter.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      CSRK_CUDA_TRY(cudaStreamSynchronize(s));
      std::swap(frontier.p, next.p);
      fsize = cnt;
    }
    CSRK_CUDA_TRY(cudaMemsetAsync(ecc.p, 0xff, n * sizeof(int32_t), s));
    ecc_kernel<<<nblocks(n), 256, 0, s>>>(depth.p, label.p, n, ecc.p);
    CSRK_CUDA_TRY(cudaMemsetAsync(lastmin.p, 0xff, n * sizeof(uint32_t), s));
    last_level_kernel<<<nblocks(n), 256, 0, s>>>(depth.p, label.p, ecc.p, krank.p, n,
                                                 lastmin.p);
    int still = 0;
    CSRK_CUDA_TRY(cudaMemsetAsync(counter.p, 0, sizeof(int), s));
    pp_update_kernel<<<nblocks(n_comp), 256, 0, s>>>(roots, n_comp, ecc.p, lastmin.p, by_key.p,
                                                     start.p, best_node.p, best_ecc.p,
                                                     active.p, counter.p);
    CSRK_CUDA_TRY(cudaMemcpyAsync(&still, counter.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    n_active = still;
  }

  // 4. Cuthill-McKee queues, all components level by level
  CSRK_CUDA_TRY(cudaMemsetAsync(claim.p, 0xff, n * sizeof(uint32_t), s));
  CSRK_CUDA_TRY(cudaMemsetAsync(inq.p, 0, n * sizeof(int32_t), s));
  CSRK_CUDA_TRY(cudaMemsetAsync(pos.p, 0xff, n * sizeof(int32_t), s));
  CSRK_CUDA_TRY(cudaMemsetAsync(qlen.p, 0, n * sizeof(int32_t), s));
  cm_init_kernel<<<nblocks(n_comp), 256, 0, s>>>(roots, n_comp, best_node.p, pos.p, qlen.p,
                                                 frontier.p);
  // (the level sorts below reuse keys / vals; roots are not needed past here)
  const int kbits = bits_for(n);
  int64_t fsize = n_comp;
  while (fsize > 0) {
    int cnt = 0;
    CSRK_CUDA_TRY(cudaMemsetAsync(counter.p, 0, sizeof(int), s));
    cm_claim_kernel<<<nblocks(fsize), 256, 0, s>>>(g->ptr, g->idx, frontier.p, fsize, pos.p,
                                                   claim.p, inq.p, next.p, counter.p);
    CSRK_CUDA_TRY(cudaMemcpyAsync(&cnt, counter.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    if (cnt == 0) break;
    cm_key_kernel<<<nblocks(cnt), 256, 0, s>>>(next.p, cnt, claim.p, krank.p, kbits, keys.p,
                                               vals.p);
    const int key_bits = ((2 * kbits + 7) / 8) * 8;
    CSRK_TRY(radix_sort_pairs(keys.p, vals.p, tkeys.p, tvals.p, cnt, 0, key_bits, s));
    if (n_comp > 1) {
      comp_key_kernel<<<nblocks(cnt), 256, 0, s>>>(vals.p, cnt, label.p, crank.p, keys.p);
      CSRK_TRY(radix_sort_pairs(keys.p, vals.p, tkeys.p, tvals.p, cnt, 0, 32, s));
    }
    cm_place_kernel<<<nblocks(cnt), 256, 0, s>>>(vals.p, cnt, label.p, qlen.p, pos.p, claim.p,
                                                 inq.p, frontier.p);
    cm_count_kernel<<<nblocks(cnt), 256, 0, s>>>(vals.p, cnt, label.p, qlen.p);
    fsize = cnt;
  }
  if (std::getenv("CSRK_BANDK_PROFILE"))
    std::fprintf(stderr, "[band_k dev]   wbo n=%lld components=%d\n",
                 static_cast<long long>(n), n_comp);
  final_fwd_kernel<<<nblocks(n), 256, 0, s>>>(pos.p, label.p, coff.p, n, fwd_dev);
  CSRK_CUDA_TRY(cudaGetLastError());
  CSRK_CUDA_TRY(cudaStreamSynchronize(s));
  return CSRK_OK;
}

}  // namespace csrk

extern "C" int csrk_dgraph_wbo(const csrk_dgraph *g, int64_t *fwd_host) {
  if (!g || !fwd_host) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(g->device));
  int64_t *d = nullptr;
  CSRK_CUDA_TRY(cudaMalloc(&d, (g->n > 0 ? g->n : 1) * sizeof(int64_t)));
  const int rc = csrk::graph_wbo_dev(g, d, nullptr);
  if (rc == CSRK_OK)
    CSRK_CUDA_TRY(cudaMemcpy(fwd_host, d, g->n * sizeof(int64_t), cudaMemcpyDeviceToHost));
  cudaFree(d);
  return rc;
}
