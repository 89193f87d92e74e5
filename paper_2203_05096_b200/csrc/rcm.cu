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
// (min position of a level-L neighbour, key rank).  Ordering each new level
// by (component rank, parent position, key rank) reproduces the sequential
// queue exactly; the frontier is kept in that order, so each parent's
// children form one run of the next level and only need ranking among
// themselves.  All components advance together.
//
//   krank      rank of every node by (degree, weight, index): one stable sort
//   components label propagation + pointer jumping; label = min index, which
//              is also the reference's "min(c)" and enumeration root
//   pseudo-peripheral starts: repeated multi-source BFS (reorder.py:263-278)

#include <algorithm>
#include <chrono>
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

// one BFS level; the frontier size is read from the device (`sizes[0]`) and
// the next level's is counted into `sizes[1]`, so a batch of levels is
// queued without host round trips (levels past the last do nothing)
__global__ void bfs_expand_kernel(const int64_t *__restrict__ ptr,
                                  const int32_t *__restrict__ idx,
                                  const int32_t *__restrict__ frontier,
                                  const int *__restrict__ sizes, int32_t level,
                                  int32_t *__restrict__ depth, int32_t *__restrict__ next,
                                  int *__restrict__ next_count) {
  const int64_t fsize = sizes[0];
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
//
// The frontier is kept in queue order -- by (component rank, position) --
// so a frontier INDEX orders parents exactly as their positions do.  A new
// node is claimed by the smallest index of a frontier neighbour; the
// children of one parent then form one contiguous run of the next level
// (runs in parent order), ordered inside by key rank.  Per level: claim,
// count per parent, an exclusive scan, and a placement that ranks each
// parent's children by counting -- no sort of the level.

constexpr int32_t kBigDegree = 128;  // parents of larger degree: block path

__global__ void cm_claim_kernel(const int64_t *__restrict__ ptr, const int32_t *__restrict__ idx,
                                const int32_t *__restrict__ frontier, int64_t fsize,
                                const int32_t *__restrict__ pos, uint32_t *__restrict__ claim) {
  GSTRIDE(i, fsize) {
    const int32_t v = frontier[i];
    for (int64_t p = ptr[v]; p < ptr[v + 1]; ++p) {
      const int32_t u = idx[p];
      if (pos[u] == kNone && claim[u] > static_cast<uint32_t>(i))
        atomicMin(&claim[u], static_cast<uint32_t>(i));
    }
  }
}

// children won by each parent; parents of large degree go to the big list
__global__ void cm_count_kernel(const int64_t *__restrict__ ptr, const int32_t *__restrict__ idx,
                                const int32_t *__restrict__ frontier, int64_t fsize,
                                const int32_t *__restrict__ pos,
                                const uint32_t *__restrict__ claim, int64_t *__restrict__ cnt,
                                int32_t *__restrict__ big, int *__restrict__ n_big) {
  GSTRIDE(i, fsize) {
    const int32_t v = frontier[i];
    int64_t c = 0;
    for (int64_t p = ptr[v]; p < ptr[v + 1]; ++p) {
      const int32_t u = idx[p];
      c += (pos[u] == kNone && claim[u] == static_cast<uint32_t>(i));
    }
    cnt[i] = c;
    if (ptr[v + 1] - ptr[v] > kBigDegree && c > 0) big[atomicAdd(n_big, 1)] = static_cast<int32_t>(i);
  }
}

// first slot of every component's run in the next level
__global__ void cm_runs_kernel(const int32_t *__restrict__ frontier, int64_t fsize,
                               const int32_t *__restrict__ label,
                               const int64_t *__restrict__ off, int64_t *__restrict__ lvl_start) {
  GSTRIDE(i, fsize) {
    const int32_t c = label[frontier[i]];
    if (i == 0 || label[frontier[i - 1]] != c) lvl_start[c] = off[i];
  }
}

// small parents: one thread places all its children in the next level
// (rank = its children with a smaller key rank); positions are committed by
// cm_commit_kernel, so `pos == none` still marks this level's children
__global__ void cm_place_kernel(const int64_t *__restrict__ ptr, const int32_t *__restrict__ idx,
                                const int32_t *__restrict__ frontier, int64_t fsize,
                                const uint32_t *__restrict__ claim,
                                const uint32_t *__restrict__ krank,
                                const int32_t *__restrict__ pos,
                                const int64_t *__restrict__ off, int32_t *__restrict__ next) {
  GSTRIDE(i, fsize) {
    const int32_t v = frontier[i];
    const int64_t a = ptr[v], b = ptr[v + 1];
    if (b - a > kBigDegree || off[i + 1] == off[i]) continue;
    const uint32_t me = static_cast<uint32_t>(i);
    for (int64_t p = a; p < b; ++p) {
      const int32_t u = idx[p];
      if (claim[u] != me || pos[u] != kNone) continue;
      const uint32_t ku = krank[u];
      int64_t r = 0;
      for (int64_t q = a; q < b; ++q) {
        const int32_t w = idx[q];
        r += (claim[w] == me && pos[w] == kNone && krank[w] < ku);
      }
      next[off[i] + r] = u;
    }
  }
}

// big parents: one block each, one thread per adjacency entry
__global__ void cm_place_big_kernel(const int64_t *__restrict__ ptr,
                                    const int32_t *__restrict__ idx,
                                    const int32_t *__restrict__ frontier,
                                    const int32_t *__restrict__ big, const int *__restrict__ n_big,
                                    const uint32_t *__restrict__ claim,
                                    const uint32_t *__restrict__ krank,
                                    const int32_t *__restrict__ pos,
                                    const int64_t *__restrict__ off, int32_t *__restrict__ next) {
  for (int bi = blockIdx.x; bi < *n_big; bi += gridDim.x) {
    const int64_t i = big[bi];
    const int32_t v = frontier[i];
    const int64_t a = ptr[v], b = ptr[v + 1];
    const uint32_t me = static_cast<uint32_t>(i);
    for (int64_t p = a + threadIdx.x; p < b; p += blockDim.x) {
      const int32_t u = idx[p];
      if (claim[u] != me || pos[u] != kNone) continue;
      const uint32_t ku = krank[u];
      int64_t r = 0;
      for (int64_t q = a; q < b; ++q) {
        const int32_t w = idx[q];
        r += (claim[w] == me && pos[w] == kNone && krank[w] < ku);
      }
      next[off[i] + r] = u;
    }
  }
}

// queue positions of the placed level: component c's run starts at
// lvl_start[c] and continues its queue at qlen[c]
__global__ void cm_commit_kernel(const int32_t *__restrict__ next, int64_t total,
                                 const int32_t *__restrict__ label,
                                 const int32_t *__restrict__ qlen,
                                 const int64_t *__restrict__ lvl_start, int32_t *__restrict__ pos) {
  GSTRIDE(j, total) {
    const int32_t u = next[j];
    const int32_t c = label[u];
    pos[u] = qlen[c] + static_cast<int32_t>(j - lvl_start[c]);
  }
}

// queue lengths grow by each component's run in the placed level
__global__ void cm_qlen_kernel(const int32_t *__restrict__ frontier, int64_t fsize,
                               const int32_t *__restrict__ label,
                               const int64_t *__restrict__ off,
                               const int64_t *__restrict__ lvl_start, int32_t *__restrict__ qlen) {
  GSTRIDE(i, fsize) {
    const int32_t c = label[frontier[i]];
    if (i == fsize - 1 || label[frontier[i + 1]] != c)
      qlen[c] += static_cast<int32_t>(off[i + 1] - lvl_start[c]);
  }
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
struct DBuf {  // stream-ordered scratch from the kept pool (keep_async_pool)
  T *p = nullptr;
  cudaStream_t st = nullptr;
  ~DBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  cudaError_t alloc(int64_t n, cudaStream_t s) {
    keep_async_pool();
    st = s;
    return cudaMallocAsync(&p, (n > 0 ? n : 1) * sizeof(T), s);
  }
};


}  // namespace

int graph_wbo_dev(const csrk_dgraph *g, int64_t *fwd_dev, cudaStream_t s) {
  const int64_t n = g->n;
  if (n == 0) return CSRK_OK;
  // CSRK_BANDK_PROFILE=1: wall time of each phase (synchronising)
  const bool prof = std::getenv("CSRK_BANDK_PROFILE") != nullptr && n > (1 << 20);
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char *name) {
    if (!prof) return;
    cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[band_k dev]     wbo %-10s %.3f s\n", name,
                 std::chrono::duration<double>(t - t_last).count());
    t_last = t;
  };
  DBuf<uint64_t> keys, tkeys;
  DBuf<uint32_t> vals, tvals, krank, by_key, claim, lastmin, minrank;
  DBuf<int32_t> label, size, depth, frontier, next, pos, ecc, crank, qlen;
  DBuf<int32_t> start, best_node, best_ecc;
  DBuf<int8_t> active;
  DBuf<int> counter;
  DBuf<int64_t> coff, csize, csize_off;
  CSRK_CUDA_TRY(keys.alloc(n, s));
  CSRK_CUDA_TRY(tkeys.alloc(n, s));
  CSRK_CUDA_TRY(vals.alloc(n, s));
  CSRK_CUDA_TRY(tvals.alloc(n, s));
  CSRK_CUDA_TRY(krank.alloc(n, s));
  CSRK_CUDA_TRY(by_key.alloc(n, s));
  CSRK_CUDA_TRY(claim.alloc(n, s));
  CSRK_CUDA_TRY(lastmin.alloc(n, s));
  CSRK_CUDA_TRY(minrank.alloc(n, s));
  CSRK_CUDA_TRY(label.alloc(n, s));
  CSRK_CUDA_TRY(size.alloc(n, s));
  CSRK_CUDA_TRY(depth.alloc(n, s));
  CSRK_CUDA_TRY(frontier.alloc(n, s));
  CSRK_CUDA_TRY(next.alloc(n, s));
  CSRK_CUDA_TRY(pos.alloc(n, s));
  CSRK_CUDA_TRY(ecc.alloc(n, s));
  CSRK_CUDA_TRY(crank.alloc(n, s));
  CSRK_CUDA_TRY(qlen.alloc(n, s));
  CSRK_CUDA_TRY(counter.alloc(4, s));
  CSRK_CUDA_TRY(coff.alloc(n + 1, s));
  phase("alloc");

  // 1. key ranks: stable sort of (degree, weight) keeps index order on ties;
  //    by_key[rank] = node
  key_kernel<<<nblocks(n), 256, 0, s>>>(g->ptr, g->nw, n, keys.p, by_key.p);
  CSRK_TRY(radix_sort_pairs(keys.p, by_key.p, tkeys.p, tvals.p, n, 0, 64, s));
  rank_kernel<<<nblocks(n), 256, 0, s>>>(by_key.p, n, krank.p);
  phase("keys");

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
  CSRK_CUDA_TRY(csize.alloc(n_comp, s));
  CSRK_CUDA_TRY(csize_off.alloc(n_comp + 1, s));
  CSRK_CUDA_TRY(start.alloc(n_comp, s));
  CSRK_CUDA_TRY(best_node.alloc(n_comp, s));
  CSRK_CUDA_TRY(best_ecc.alloc(n_comp, s));
  CSRK_CUDA_TRY(active.alloc(n_comp, s));
  comp_sizes_kernel<<<nblocks(n_comp), 256, 0, s>>>(roots, n_comp, size.p, csize.p);
  CSRK_TRY(exclusive_scan_i64(csize.p, n_comp, csize_off.p, s));
  comp_layout_kernel<<<nblocks(n_comp), 256, 0, s>>>(roots, n_comp, size.p, csize_off.p,
                                                     crank.p, coff.p);

  phase("components");
  // 3. pseudo-peripheral start of every component (reorder.py:263-278),
  //    all components' BFS runs together, state stays on the device
  pp_init_kernel<<<nblocks(n_comp), 256, 0, s>>>(roots, n_comp, minrank.p, by_key.p, start.p,
                                                 best_node.p, best_ecc.p, active.p);
  constexpr int kBfsBatch = 8;  // even: the frontier ends each batch in `frontier`
  DBuf<int> lsize;
  CSRK_CUDA_TRY(lsize.alloc(kBfsBatch + 1, s));
  const unsigned bfs_grid = nblocks(n) < 148 * 8 ? nblocks(n) : 148 * 8;
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
    // levels in batches of kBfsBatch with one host check per batch: the
    // frontier sizes live in lsize[0..kBfsBatch] on the device
    int last = k;
    for (int32_t level = 0; last > 0;) {
      CSRK_CUDA_TRY(cudaMemsetAsync(lsize.p, 0, (kBfsBatch + 1) * sizeof(int), s));
      CSRK_CUDA_TRY(cudaMemcpyAsync(lsize.p, &last, sizeof(int), cudaMemcpyHostToDevice, s));
      for (int j = 0; j < kBfsBatch; ++j, ++level) {
        bfs_expand_kernel<<<bfs_grid, 256, 0, s>>>(g->ptr, g->idx, frontier.p, lsize.p + j,
                                                   level, depth.p, next.p, lsize.p + j + 1);
        std::swap(frontier.p, next.p);
      }
      CSRK_CUDA_TRY(cudaMemcpyAsync(&last, lsize.p + kBfsBatch, sizeof(int),
                                    cudaMemcpyDeviceToHost, s));
      CSRK_CUDA_TRY(cudaStreamSynchronize(s));
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

  phase("pseudo-per");
  // 4. Cuthill-McKee queues, all components level by level (see the CM
  //    kernels above): one host round trip per level, for its size
  CSRK_CUDA_TRY(cudaMemsetAsync(claim.p, 0xff, n * sizeof(uint32_t), s));
  CSRK_CUDA_TRY(cudaMemsetAsync(pos.p, 0xff, n * sizeof(int32_t), s));
  CSRK_CUDA_TRY(cudaMemsetAsync(qlen.p, 0, n * sizeof(int32_t), s));
  cm_init_kernel<<<nblocks(n_comp), 256, 0, s>>>(roots, n_comp, best_node.p, pos.p, qlen.p,
                                                 frontier.p);
  DBuf<int64_t> cnt, off, lvl_start;
  DBuf<int32_t> big;
  CSRK_CUDA_TRY(cnt.alloc(n, s));
  CSRK_CUDA_TRY(off.alloc(n + 1, s));
  CSRK_CUDA_TRY(lvl_start.alloc(n, s));
  CSRK_CUDA_TRY(big.alloc(n, s));
  int64_t fsize = n_comp;
  for (;;) {
    cm_claim_kernel<<<nblocks(fsize), 256, 0, s>>>(g->ptr, g->idx, frontier.p, fsize, pos.p,
                                                   claim.p);
    CSRK_CUDA_TRY(cudaMemsetAsync(counter.p, 0, sizeof(int), s));
    cm_count_kernel<<<nblocks(fsize), 256, 0, s>>>(g->ptr, g->idx, frontier.p, fsize, pos.p,
                                                   claim.p, cnt.p, big.p, counter.p);
    CSRK_TRY(exclusive_scan_i64(cnt.p, fsize, off.p, s));
    int64_t total = 0;
    CSRK_CUDA_TRY(cudaMemcpyAsync(&total, off.p + fsize, sizeof(total), cudaMemcpyDeviceToHost,
                                  s));
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    if (total == 0) break;
    cm_runs_kernel<<<nblocks(fsize), 256, 0, s>>>(frontier.p, fsize, label.p, off.p,
                                                  lvl_start.p);
    cm_place_kernel<<<nblocks(fsize), 256, 0, s>>>(g->ptr, g->idx, frontier.p, fsize, claim.p,
                                                   krank.p, pos.p, off.p, next.p);
    cm_place_big_kernel<<<148, 256, 0, s>>>(g->ptr, g->idx, frontier.p, big.p, counter.p,
                                            claim.p, krank.p, pos.p, off.p, next.p);
    cm_commit_kernel<<<nblocks(total), 256, 0, s>>>(next.p, total, label.p, qlen.p,
                                                    lvl_start.p, pos.p);
    cm_qlen_kernel<<<nblocks(fsize), 256, 0, s>>>(frontier.p, fsize, label.p, off.p,
                                                  lvl_start.p, qlen.p);
    std::swap(frontier.p, next.p);
    fsize = total;
  }
  if (std::getenv("CSRK_BANDK_PROFILE"))
    std::fprintf(stderr, "[band_k dev]   wbo n=%lld components=%d\n",
                 static_cast<long long>(n), n_comp);
  phase("cm-levels");
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
