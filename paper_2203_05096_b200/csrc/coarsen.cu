// Device heavy-edge matching and coarsening, bit-exact with reorder.py:138-237.
//
// heavy_edge_matching visits nodes in (degree, index) order; an unmatched
// node v picks its unmatched neighbour u with the smallest key
// (-edge weight, |u - v|, u), else matches itself.  Parallel form: with
// rank(v) the visit position, node u is still unmatched at v's turn iff
// rank(u) > rank(v) and u was not taken by a chooser ranked before v; v
// chooses iff it was not taken by an earlier chooser.  Each iteration
// recomputes every choice from the previous iteration's "taken by" array
// (min over choosers of (rank << 32 | node)).  A node's decision depends
// only on lower-ranked nodes, so the iteration reaches the sequential
// result and stops changing; the fixed point is unique.
//
// coarsen repeats {band-order and relabel (from round 2), match, number the
// representatives min(v, match[v]) in index order, contract} until the mean
// coarse weight reaches the target or a round shrinks by less than 5%.

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace csrk {
namespace {

inline unsigned nb(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return static_cast<unsigned>(b);
}

#define GS(i, n)                                                           \
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < (n); \
       i += int64_t(gridDim.x) * blockDim.x)

constexpr uint64_t kFree = ~0ull;

__global__ void deg_key_kernel(const int64_t *__restrict__ ptr, int64_t n,
                               uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  GS(v, n) {
    keys[v] = static_cast<uint64_t>(ptr[v + 1] - ptr[v]);
    vals[v] = static_cast<uint32_t>(v);
  }
}

__global__ void vrank_kernel(const uint32_t *__restrict__ order, int64_t n,
                             uint32_t *__restrict__ rank) {
  GS(i, n) { rank[order[i]] = static_cast<uint32_t>(i); }
}

// one Jacobi sweep: choices from `taken_prev`, new claims into `taken_next`
// (all free on entry); `reset` -- the array the next sweep claims into, read
// by nobody in this one -- is set free on the way
__global__ void match_sweep_kernel(const int64_t *__restrict__ ptr,
                                   const int32_t *__restrict__ idx,
                                   const int32_t *__restrict__ ew,
                                   const uint32_t *__restrict__ rank, int64_t n,
                                   const uint64_t *__restrict__ taken_prev,
                                   uint64_t *__restrict__ taken_next,
                                   uint64_t *__restrict__ reset,
                                   int32_t *__restrict__ choice) {
  GS(v, n) {
    reset[v] = kFree;
    const uint32_t rv = rank[v];
    int32_t best = -1;
    if ((taken_prev[v] >> 32) >= rv) {  // v is free at its turn
      int32_t bw = 0;
      int64_t bd = 0;
      for (int64_t p = ptr[v]; p < ptr[v + 1]; ++p) {
        const int32_t u = idx[p];
        if (rank[u] < rv || (taken_prev[u] >> 32) < rv) continue;  // matched by then
        const int32_t w = ew[p];
        const int64_t d = u > v ? int64_t(u) - v : int64_t(v) - u;
        if (best < 0 || w > bw || (w == bw && (d < bd || (d == bd && u < best)))) {
          best = u;
          bw = w;
          bd = d;
        }
      }
      if (best >= 0)
        atomicMin(reinterpret_cast<unsigned long long *>(&taken_next[best]),
                  (static_cast<unsigned long long>(rv) << 32) | static_cast<uint32_t>(v));
      choice[v] = best >= 0 ? best : static_cast<int32_t>(v);
    } else {
      choice[v] = -2;  // taken
    }
  }
}

// did the sweep change the "taken by" array?
__global__ void diff_kernel(const uint64_t *__restrict__ a, const uint64_t *__restrict__ b,
                            int64_t n, int *__restrict__ changed) {
  GS(i, n) {
    if (a[i] != b[i]) *changed = 1;
  }
}

__global__ void fill_u64_kernel(uint64_t *__restrict__ a, int64_t n, uint64_t v) {
  GS(i, n) { a[i] = v; }
}

__global__ void match_final_kernel(const uint64_t *__restrict__ taken,
                                   const int32_t *__restrict__ choice, int64_t n,
                                   int32_t *__restrict__ match) {
  GS(v, n) {
    match[v] = choice[v] == -2 ? static_cast<int32_t>(taken[v] & 0xffffffffu) : choice[v];
  }
}

// representatives: new id = rank of min(v, match[v]) among representatives
__global__ void rep_flag_kernel(const int32_t *__restrict__ match, int64_t n,
                                int64_t *__restrict__ flag) {
  GS(v, n) { flag[v] = match[v] >= v ? 1 : 0; }
}

__global__ void rep_id_kernel(const int32_t *__restrict__ match,
                              const int64_t *__restrict__ pos, int64_t n,
                              int32_t *__restrict__ new_id) {
  GS(v, n) {
    const int32_t r = match[v] >= v ? static_cast<int32_t>(v) : match[v];
    new_id[v] = static_cast<int32_t>(pos[r]);
  }
}

__global__ void compose_kernel(int32_t *__restrict__ f2c, const int32_t *__restrict__ map,
                               int64_t n) {
  GS(i, n) { f2c[i] = map[f2c[i]]; }
}

__global__ void compose64_kernel(int32_t *__restrict__ f2c, const int64_t *__restrict__ map,
                                 int64_t n) {
  GS(i, n) { f2c[i] = static_cast<int32_t>(map[f2c[i]]); }
}

__global__ void iota32_kernel(int32_t *__restrict__ a, int64_t n) {
  GS(i, n) { a[i] = static_cast<int32_t>(i); }
}

__global__ void inv_kernel(const int64_t *__restrict__ fwd, int64_t n,
                           int64_t *__restrict__ inv) {
  GS(i, n) { inv[fwd[i]] = i; }
}

template <typename T>
struct DB {  // stream-ordered scratch from the kept pool (keep_async_pool)
  T *p = nullptr;
  cudaStream_t st = nullptr;
  ~DB() {
    if (p) cudaFreeAsync(p, st);
  }
  cudaError_t alloc(int64_t n, cudaStream_t s) {
    keep_async_pool();
    st = s;
    return cudaMallocAsync(&p, (n > 0 ? n : 1) * sizeof(T), s);
  }
};

}  // namespace

int graph_wbo_dev(const csrk_dgraph *g, int64_t *fwd_dev, cudaStream_t s);
int graph_relabel_dev(const csrk_dgraph *g, const int64_t *fwd_dev, const int64_t *inv_dev,
                      cudaStream_t s, csrk_dgraph **out);
int graph_contract_dev(const csrk_dgraph *g, const int32_t *f2c_dev, int64_t m_coarse,
                       cudaStream_t s, csrk_dgraph **out);
void graph_free_dev(csrk_dgraph *g);

// match[n] (device) = heavy_edge_matching(g); iterations returned in *iters
int graph_match_dev(const csrk_dgraph *g, int32_t *match, int *iters, cudaStream_t s) {
  const int64_t n = g->n;
  if (n == 0) return CSRK_OK;
  DB<uint64_t> keys, tkeys, ta, tb, tc;
  DB<uint32_t> vals, tvals, rank;
  DB<int32_t> choice;
  DB<int> flag;
  CSRK_CUDA_TRY(keys.alloc(n, s));
  CSRK_CUDA_TRY(tkeys.alloc(n, s));
  CSRK_CUDA_TRY(vals.alloc(n, s));
  CSRK_CUDA_TRY(tvals.alloc(n, s));
  CSRK_CUDA_TRY(rank.alloc(n, s));
  CSRK_CUDA_TRY(ta.alloc(n, s));
  CSRK_CUDA_TRY(tb.alloc(n, s));
  CSRK_CUDA_TRY(tc.alloc(n, s));
  CSRK_CUDA_TRY(choice.alloc(n, s));
  CSRK_CUDA_TRY(flag.alloc(1, s));
  deg_key_kernel<<<nb(n), 256, 0, s>>>(g->ptr, n, keys.p, vals.p);
  CSRK_TRY(radix_sort_pairs(keys.p, vals.p, tkeys.p, tvals.p, n, 0, 32, s));
  vrank_kernel<<<nb(n), 256, 0, s>>>(vals.p, n, rank.p);
  fill_u64_kernel<<<nb(n), 256, 0, s>>>(ta.p, n, kFree);
  fill_u64_kernel<<<nb(n), 256, 0, s>>>(tb.p, n, kFree);
  fill_u64_kernel<<<nb(n), 256, 0, s>>>(tc.p, n, kFree);
  // sweeps run in batches of 8 with one host check per batch: sweeps past
  // the fixed point change nothing, and only the batch's last sweep decides.
  // Three "taken by" arrays rotate (read, claimed into, reset for the next
  // sweep), so no pass of its own resets one between sweeps.
  constexpr int kBatch = 8;
  int it = 0;
  for (;;) {
    for (int j = 0; j < kBatch; ++j, ++it) {
      match_sweep_kernel<<<nb(n), 256, 0, s>>>(g->ptr, g->idx, g->ew, rank.p, n, ta.p, tb.p,
                                               tc.p, choice.p);
      if (j == kBatch - 1) {
        CSRK_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
        diff_kernel<<<nb(n), 256, 0, s>>>(ta.p, tb.p, n, flag.p);
      }
      uint64_t *t = ta.p;  // (read, claim, reset) <- (claim, reset, read)
      ta.p = tb.p;
      tb.p = tc.p;
      tc.p = t;
    }
    int h = 0;
    CSRK_CUDA_TRY(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    if (!h) break;
  }
  match_final_kernel<<<nb(n), 256, 0, s>>>(ta.p, choice.p, n, match);
  CSRK_CUDA_TRY(cudaGetLastError());
  if (iters) *iters = it;
  return CSRK_OK;
}

// coarsen(g, target): the coarse graph (owned by *out) and f2c[g->n] (device)
int graph_coarsen_dev(const csrk_dgraph *g, double target, int32_t *f2c, csrk_dgraph **out,
                      cudaStream_t s) {
  const int64_t total = g->n;
  const bool prof = std::getenv("CSRK_BANDK_PROFILE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char *name, int64_t nn) {
    if (!prof) return;
    cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[band_k dev]     coarsen %-9s n=%-9lld %.3f s\n", name,
                 static_cast<long long>(nn), std::chrono::duration<double>(t - t_last).count());
    t_last = t;
  };
  iota32_kernel<<<nb(total), 256, 0, s>>>(f2c, total);
  csrk_dgraph *cur = nullptr;  // owned intermediate (null = g itself)
  auto cur_g = [&]() -> const csrk_dgraph * { return cur ? cur : g; };
  bool first = true;
  int rc = CSRK_OK;
  while (rc == CSRK_OK) {
    const int64_t n = cur_g()->n;
    if (n == 0 || !(static_cast<double>(total) / static_cast<double>(n) < target)) break;
    if (!first) {
      DB<int64_t> band, inv;
      if (band.alloc(n, s) != cudaSuccess || inv.alloc(n, s) != cudaSuccess) return CSRK_ENOMEM;
      rc = graph_wbo_dev(cur_g(), band.p, s);
      if (rc != CSRK_OK) break;
      inv_kernel<<<nb(n), 256, 0, s>>>(band.p, n, inv.p);
      csrk_dgraph *rel = nullptr;
      rc = graph_relabel_dev(cur_g(), band.p, inv.p, s, &rel);
      if (rc != CSRK_OK) break;
      if (cur) graph_free_dev(cur);
      cur = rel;
      compose64_kernel<<<nb(total), 256, 0, s>>>(f2c, band.p, total);
      phase("order", n);
    }
    first = false;
    DB<int32_t> match, new_id;
    DB<int64_t> flag, pos;
    if (match.alloc(n, s) != cudaSuccess || new_id.alloc(n, s) != cudaSuccess ||
        flag.alloc(n, s) != cudaSuccess || pos.alloc(n + 1, s) != cudaSuccess)
      return CSRK_ENOMEM;
    int sweeps = 0;
    rc = graph_match_dev(cur_g(), match.p, &sweeps, s);
    phase("matching", n);
    if (std::getenv("CSRK_BANDK_PROFILE"))
      std::fprintf(stderr, "[band_k dev]   matching n=%lld sweeps=%d\n",
                   static_cast<long long>(n), sweeps);
    if (rc != CSRK_OK) break;
    rep_flag_kernel<<<nb(n), 256, 0, s>>>(match.p, n, flag.p);
    rc = exclusive_scan_i64(flag.p, n, pos.p, s);
    if (rc != CSRK_OK) break;
    int64_t m = 0;
    CSRK_CUDA_TRY(cudaMemcpyAsync(&m, pos.p + n, sizeof(m), cudaMemcpyDeviceToHost, s));
    rep_id_kernel<<<nb(n), 256, 0, s>>>(match.p, pos.p, n, new_id.p);
    compose_kernel<<<nb(total), 256, 0, s>>>(f2c, new_id.p, total);
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    csrk_dgraph *con = nullptr;
    rc = graph_contract_dev(cur_g(), new_id.p, m, s, &con);
    if (rc != CSRK_OK) break;
    phase("contract", n);
    if (cur) graph_free_dev(cur);
    cur = con;
    if (static_cast<double>(n - m) < 0.05 * static_cast<double>(n)) break;
  }
  if (rc != CSRK_OK) {
    if (cur) graph_free_dev(cur);
    return rc;
  }
  if (!cur) {
    // no round ran: the coarse graph is a copy of g (identity map)
    int64_t *fwd = nullptr, *inv = nullptr;
    CSRK_CUDA_TRY(cudaMalloc(&fwd, (g->n > 0 ? g->n : 1) * sizeof(int64_t)));
    CSRK_CUDA_TRY(cudaMalloc(&inv, (g->n > 0 ? g->n : 1) * sizeof(int64_t)));
    std::vector<int64_t> id(g->n);
    for (int64_t i = 0; i < g->n; ++i) id[i] = i;
    cudaMemcpy(fwd, id.data(), g->n * sizeof(int64_t), cudaMemcpyHostToDevice);
    cudaMemcpy(inv, id.data(), g->n * sizeof(int64_t), cudaMemcpyHostToDevice);
    rc = graph_relabel_dev(g, fwd, inv, s, &cur);
    cudaFree(fwd);
    cudaFree(inv);
    if (rc != CSRK_OK) return rc;
  }
  CSRK_CUDA_TRY(cudaStreamSynchronize(s));
  *out = cur;
  return CSRK_OK;
}

}  // namespace csrk

using namespace csrk;

extern "C" {

int csrk_dgraph_match(const csrk_dgraph *g, int64_t *match_host, int *iters) {
  if (!g || !match_host) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(g->device));
  int32_t *d = nullptr;
  CSRK_CUDA_TRY(cudaMalloc(&d, (g->n > 0 ? g->n : 1) * sizeof(int32_t)));
  int rc = graph_match_dev(g, d, iters, nullptr);
  if (rc == CSRK_OK) {
    std::vector<int32_t> h(g->n);
    cudaError_t e = cudaMemcpy(h.data(), d, g->n * sizeof(int32_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = CSRK_ECUDA;
    for (int64_t i = 0; i < g->n; ++i) match_host[i] = h[i];
  }
  cudaFree(d);
  return rc;
}

int csrk_dgraph_coarsen(const csrk_dgraph *g, double target, int64_t *f2c_host,
                        csrk_dgraph **out) {
  if (!g || !f2c_host || !out) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (!(target >= 1.0)) {
    set_error("target_weight must be at least 1");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(g->device));
  int32_t *d = nullptr;
  CSRK_CUDA_TRY(cudaMalloc(&d, (g->n > 0 ? g->n : 1) * sizeof(int32_t)));
  *out = nullptr;
  int rc = graph_coarsen_dev(g, target, d, out, nullptr);
  if (rc == CSRK_OK) {
    std::vector<int32_t> h(g->n);
    if (cudaMemcpy(h.data(), d, g->n * sizeof(int32_t), cudaMemcpyDeviceToHost) !=
        cudaSuccess)
      rc = CSRK_ECUDA;
    for (int64_t i = 0; i < g->n; ++i) f2c_host[i] = h[i];
  }
  cudaFree(d);
  return rc;
}

}  // extern "C"
