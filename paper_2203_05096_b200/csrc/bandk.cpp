// Native Band-k reordering: a bit-exact restatement of the reference's
// reorder.py (pkg/src/csrk/reorder.py) in C++.
//
// Every greedy choice of the reference is reproduced with the same total
// order, so the permutation and the per-level group sizes are identical:
//   build_graph            reorder.py:115-135   pattern of A + A^T, no diagonal
//   _graph_from_edges      reorder.py:87-112    rows sorted, parallel edges summed
//   heavy_edge_matching    reorder.py:138-173   visit (deg, idx); pick min
//                                               (-w, |u-v|, u) unmatched neighbour
//   _contract              reorder.py:176-184
//   _relabel_graph         reorder.py:192-196
//   coarsen                reorder.py:199-237   stop at mean weight >= target or
//                                               shrink < MIN_MATCH_SHRINK
//   _bfs_levels /
//   _pseudo_peripheral     reorder.py:240-278
//   weighted_bandwidth_order reorder.py:281-336 components (-size, min idx),
//                                               CM BFS with (deg, weight, idx)
//                                               sorted frontiers, reversed
//   _order_members         reorder.py:339-387   seed (anchor, outside unplaced, key)
//   _expand_level          reorder.py:390-412
//   band_k                 reorder.py:415-469
//
// Internals use int32 node ids and weights (n and every weight sum are below
// 2^31 because nnz <= 2^31 - 1, format.py:35-37) and int64 adjacency offsets.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <new>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/csrk.h"

namespace csrk {
void set_error(const char *fmt, ...);
}

namespace {

using i32 = int32_t;
using i64 = int64_t;

constexpr double kMinMatchShrink = 0.05;  // reorder.py:32

// optional phase timing (CSRK_BANDK_PROFILE=1 prints to stderr)
struct PhaseClock {
  static double acc[8];
  static const char *names[8];
  int id;
  std::chrono::steady_clock::time_point t0;
  explicit PhaseClock(int i) : id(i), t0(std::chrono::steady_clock::now()) {}
  ~PhaseClock() {
    acc[id] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  static void report() {
    if (!std::getenv("CSRK_BANDK_PROFILE")) return;
    for (int i = 0; i < 6; ++i) std::fprintf(stderr, "[band_k] %-10s %8.3f s\n", names[i], acc[i]);
    for (double &a : acc) a = 0.0;
  }
};
double PhaseClock::acc[8] = {0};
const char *PhaseClock::names[8] = {"build", "wbo", "relabel", "matching", "contract",
                                    "expand", "", ""};

struct Graph {
  i32 n = 0;
  std::vector<i64> ptr;  // n + 1
  std::vector<i32> idx;  // neighbour ids, ascending per row
  std::vector<i32> ew;   // edge weights aligned with idx
  std::vector<i32> nw;   // node weights
  i64 deg(i32 v) const { return ptr[v + 1] - ptr[v]; }
};

struct InvalidArg : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Sort each row's (target, weight) pairs by target and merge equal targets
// by summing weights (the stable-sort-then-reduce of reorder.py:91-109; the
// order of an integer sum is immaterial).  `rows` holds, per row, a
// contiguous packed span [start[r], start[r] + cnt[r]) of (target << 32 |
// weight).  Produces the compacted graph arrays.
void finish_rows(i32 n, const std::vector<i64> &start,
                 const std::vector<i64> &cnt, std::vector<uint64_t> &packed,
                 bool merge_unit, Graph &g) {
  g.ptr.assign(static_cast<size_t>(n) + 1, 0);
  std::vector<i64> kept(n, 0);
#pragma omp parallel for schedule(dynamic, 4096)
  for (i32 r = 0; r < n; ++r) {
    uint64_t *b = packed.data() + start[r];
    uint64_t *e = b + cnt[r];
    std::sort(b, e);
    i64 out = 0;
    for (uint64_t *p = b; p < e;) {
      const uint64_t tgt = *p >> 32;
      uint64_t w = 0;
      uint64_t *q = p;
      for (; q < e && (*q >> 32) == tgt; ++q) w += (*q & 0xffffffffu);
      if (merge_unit) w = 1;  // build_graph: unique pairs, unit weight
      b[out++] = (tgt << 32) | (w & 0xffffffffu);
      p = q;
    }
    kept[r] = out;
  }
  for (i32 r = 0; r < n; ++r) g.ptr[r + 1] = g.ptr[r] + kept[r];
  g.idx.resize(g.ptr[n]);
  g.ew.resize(g.ptr[n]);
#pragma omp parallel for schedule(dynamic, 4096)
  for (i32 r = 0; r < n; ++r) {
    const uint64_t *b = packed.data() + start[r];
    i64 o = g.ptr[r];
    for (i64 j = 0; j < kept[r]; ++j) {
      g.idx[o + j] = static_cast<i32>(b[j] >> 32);
      g.ew[o + j] = static_cast<i32>(b[j] & 0xffffffffu);
    }
  }
  g.n = n;
}

Graph build_graph(i64 n64, const uint32_t *row_ptr, const uint32_t *col_idx) {
  PhaseClock pc(0);
  const i32 n = static_cast<i32>(n64);
  // counts and fills run in parallel; slot order inside a row is irrelevant
  // because finish_rows sorts every row
  std::vector<i64> cnt(n, 0);
#pragma omp parallel for schedule(dynamic, 4096)
  for (i32 r = 0; r < n; ++r)
    for (i64 p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
      const i32 c = static_cast<i32>(col_idx[p]);
      if (c != r) {
#pragma omp atomic
        ++cnt[r];
#pragma omp atomic
        ++cnt[c];
      }
    }
  std::vector<i64> start(static_cast<size_t>(n) + 1, 0);
  for (i32 r = 0; r < n; ++r) start[r + 1] = start[r] + cnt[r];
  std::vector<uint64_t> packed(start[n]);
  std::vector<i64> fill(start.begin(), start.end() - 1);
#pragma omp parallel for schedule(dynamic, 4096)
  for (i32 r = 0; r < n; ++r)
    for (i64 p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
      const i32 c = static_cast<i32>(col_idx[p]);
      if (c != r) {
        i64 a, b;
#pragma omp atomic capture
        a = fill[r]++;
#pragma omp atomic capture
        b = fill[c]++;
        packed[a] = (static_cast<uint64_t>(c) << 32) | 1u;
        packed[b] = (static_cast<uint64_t>(r) << 32) | 1u;
      }
    }
  Graph g;
  finish_rows(n, start, cnt, packed, /*merge_unit=*/true, g);
  g.nw.assign(n, 1);
  return g;
}

// node v becomes fwd[v]  (reorder.py:192-196)
Graph relabel(const Graph &g, const std::vector<i32> &fwd,
              const std::vector<i32> &inv) {
  PhaseClock pc(2);
  Graph out;
  const i32 n = g.n;
  std::vector<i64> start(static_cast<size_t>(n) + 1, 0), cnt(n);
  for (i32 i = 0; i < n; ++i) {
    cnt[i] = g.deg(inv[i]);
    start[i + 1] = start[i] + cnt[i];
  }
  std::vector<uint64_t> packed(start[n]);
#pragma omp parallel for schedule(dynamic, 4096)
  for (i32 i = 0; i < n; ++i) {
    const i32 v = inv[i];
    i64 o = start[i];
    for (i64 p = g.ptr[v]; p < g.ptr[v + 1]; ++p)
      packed[o++] = (static_cast<uint64_t>(fwd[g.idx[p]]) << 32) |
                    static_cast<uint32_t>(g.ew[p]);
  }
  finish_rows(n, start, cnt, packed, false, out);
  out.nw.resize(n);
#pragma omp parallel for
  for (i32 i = 0; i < n; ++i) out.nw[i] = g.nw[inv[i]];
  return out;
}

// collapse nodes by f2c into m coarse nodes (reorder.py:176-184)
Graph contract(const Graph &g, const std::vector<i32> &f2c, i32 m) {
  PhaseClock pc(4);
  const i32 n = g.n;
  std::vector<i64> cnt(m, 0);
#pragma omp parallel for schedule(dynamic, 4096)
  for (i32 v = 0; v < n; ++v) {
    const i32 cv = f2c[v];
    i64 c = 0;
    for (i64 p = g.ptr[v]; p < g.ptr[v + 1]; ++p) c += f2c[g.idx[p]] != cv;
#pragma omp atomic
    cnt[cv] += c;
  }
  std::vector<i64> start(static_cast<size_t>(m) + 1, 0);
  for (i32 c = 0; c < m; ++c) start[c + 1] = start[c] + cnt[c];
  std::vector<uint64_t> packed(start[m]);
  std::vector<i64> fill(start.begin(), start.end() - 1);
#pragma omp parallel for schedule(dynamic, 4096)
  for (i32 v = 0; v < n; ++v) {
    const i32 cv = f2c[v];
    for (i64 p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
      const i32 cu = f2c[g.idx[p]];
      if (cu != cv) {
        i64 slot;
#pragma omp atomic capture
        slot = fill[cv]++;
        packed[slot] = (static_cast<uint64_t>(cu) << 32) | static_cast<uint32_t>(g.ew[p]);
      }
    }
  }
  Graph out;
  finish_rows(m, start, cnt, packed, false, out);
  out.nw.assign(m, 0);
  for (i32 v = 0; v < n; ++v) out.nw[f2c[v]] += g.nw[v];
  return out;
}

// visit order: ascending degree, ties by index (reorder.py:151) -- a
// counting sort by degree is exactly that stable order
std::vector<i32> degree_order(const Graph &g) {
  i64 maxd = 0;
  for (i32 v = 0; v < g.n; ++v) maxd = std::max(maxd, g.deg(v));
  std::vector<i64> bucket(static_cast<size_t>(maxd) + 2, 0);
  for (i32 v = 0; v < g.n; ++v) ++bucket[g.deg(v) + 1];
  for (i64 d = 0; d <= maxd; ++d) bucket[d + 1] += bucket[d];
  std::vector<i32> order(g.n);
  for (i32 v = 0; v < g.n; ++v) order[bucket[g.deg(v)]++] = v;
  return order;
}

std::vector<i32> heavy_edge_matching(const Graph &g) {
  PhaseClock pc(3);
  const i32 n = g.n;
  std::vector<i32> match(n, -1);
  for (i32 v : degree_order(g)) {
    if (match[v] >= 0) continue;
    i32 best = -1;
    i32 best_w = 0;
    i64 best_d = 0;
    for (i64 p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
      const i32 u = g.idx[p];
      if (match[u] >= 0) continue;
      const i32 w = g.ew[p];
      const i64 d = u > v ? static_cast<i64>(u) - v : static_cast<i64>(v) - u;
      // key (-w, |u - v|, u), smaller wins
      if (best < 0 || w > best_w || (w == best_w && (d < best_d ||
                                                      (d == best_d && u < best)))) {
        best = u;
        best_w = w;
        best_d = d;
      }
    }
    if (best >= 0) {
      match[v] = best;
      match[best] = v;
    } else {
      match[v] = v;
    }
  }
  return match;
}

// key (degree, node weight, index) of reorder.py:292
struct KeyLess {
  const Graph *g;
  bool operator()(i32 a, i32 b) const {
    const i64 da = g->deg(a), db = g->deg(b);
    if (da != db) return da < db;
    if (g->nw[a] != g->nw[b]) return g->nw[a] < g->nw[b];
    return a < b;
  }
};

struct Permutation32 {
  std::vector<i32> fwd, inv;
};

// BFS level structure from `start` restricted to its component: returns the
// eccentricity and the min-key node of the last level (reorder.py:240-278)
struct BfsScratch {
  std::vector<i64> stamp;
  std::vector<i32> frontier, next;
  i64 cur = 0;
};

void bfs_last_level(const Graph &g, i32 start, BfsScratch &s, i64 &ecc,
                    i32 &best_last) {
  KeyLess less{&g};
  const i64 mark = ++s.cur;
  s.stamp[start] = mark;
  s.frontier.assign(1, start);
  ecc = 0;
  while (true) {
    s.next.clear();
    for (i32 v : s.frontier)
      for (i64 p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
        const i32 u = g.idx[p];
        if (s.stamp[u] != mark) {
          s.stamp[u] = mark;
          s.next.push_back(u);
        }
      }
    if (s.next.empty()) break;
    s.frontier.swap(s.next);
    ++ecc;
  }
  best_last = s.frontier[0];
  for (i32 v : s.frontier)
    if (less(v, best_last)) best_last = v;
}

i32 pseudo_peripheral(const Graph &g, const std::vector<i32> &comp,
                      BfsScratch &s) {
  KeyLess less{&g};
  i32 start = comp[0];
  for (i32 v : comp)
    if (less(v, start)) start = v;
  i32 best_node = start;
  i64 best_ecc = -1;
  while (true) {
    i64 ecc;
    i32 cand;
    bfs_last_level(g, start, s, ecc, cand);
    if (ecc <= best_ecc) return best_node;
    best_ecc = ecc;
    best_node = start;
    start = cand;
    if (start == best_node) return best_node;
  }
}

Permutation32 weighted_bandwidth_order(const Graph &g) {
  PhaseClock pc(1);
  const i32 n = g.n;
  KeyLess less{&g};
  // connected components in root-index order; a component's first node is
  // its minimum index, so the sort key (-size, min) is (-size, root)
  std::vector<char> seen(n, 0);
  std::vector<i32> comp_nodes;
  comp_nodes.reserve(n);
  std::vector<i64> comp_start;
  for (i32 root = 0; root < n; ++root) {
    if (seen[root]) continue;
    comp_start.push_back(static_cast<i64>(comp_nodes.size()));
    size_t head = comp_nodes.size();
    comp_nodes.push_back(root);
    seen[root] = 1;
    while (head < comp_nodes.size()) {
      const i32 v = comp_nodes[head++];
      for (i64 p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
        const i32 u = g.idx[p];
        if (!seen[u]) {
          seen[u] = 1;
          comp_nodes.push_back(u);
        }
      }
    }
  }
  const size_t nc = comp_start.size();
  comp_start.push_back(static_cast<i64>(comp_nodes.size()));
  std::vector<size_t> corder(nc);
  std::iota(corder.begin(), corder.end(), 0);
  std::sort(corder.begin(), corder.end(), [&](size_t a, size_t b) {
    const i64 sa = comp_start[a + 1] - comp_start[a];
    const i64 sb = comp_start[b + 1] - comp_start[b];
    if (sa != sb) return sa > sb;
    return comp_nodes[comp_start[a]] < comp_nodes[comp_start[b]];
  });

  BfsScratch scratch;
  scratch.stamp.assign(n, 0);
  std::vector<i32> order;
  order.reserve(n);
  std::vector<char> visited(n, 0);
  std::vector<i32> fresh, comp;
  for (size_t ci : corder) {
    comp.assign(comp_nodes.begin() + comp_start[ci],
                comp_nodes.begin() + comp_start[ci + 1]);
    const i32 start = pseudo_peripheral(g, comp, scratch);
    visited[start] = 1;
    size_t head = order.size();
    order.push_back(start);
    while (head < order.size()) {
      const i32 v = order[head++];
      fresh.clear();
      for (i64 p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
        const i32 u = g.idx[p];
        if (!visited[u]) {
          visited[u] = 1;
          fresh.push_back(u);
        }
      }
      std::sort(fresh.begin(), fresh.end(), less);
      order.insert(order.end(), fresh.begin(), fresh.end());
    }
  }
  std::reverse(order.begin(), order.end());
  Permutation32 perm;
  perm.fwd.resize(n);
  perm.inv = order;
  for (i32 i = 0; i < n; ++i) perm.fwd[order[i]] = i;
  return perm;
}

struct Coarsening {
  Graph coarse;
  std::vector<i32> f2c;
};

Coarsening coarsen(const Graph &g, double target) {
  if (!(target >= 1.0)) throw InvalidArg("target_weight must be at least 1");
  const i64 total = g.n;
  Graph cur = g;
  std::vector<i32> f2c(g.n);
  std::iota(f2c.begin(), f2c.end(), 0);
  bool first = true;
  while (cur.n > 0 &&
         static_cast<double>(total) / static_cast<double>(cur.n) < target) {
    if (!first) {
      Permutation32 band = weighted_bandwidth_order(cur);
      cur = relabel(cur, band.fwd, band.inv);
      for (auto &c : f2c) c = band.fwd[c];
    }
    first = false;
    const i32 before = cur.n;
    std::vector<i32> match = heavy_edge_matching(cur);
    // reps = min(v, match[v]); np.unique ranks the representatives
    std::vector<i32> new_ids(before);
    i32 m = 0;
    for (i32 v = 0; v < before; ++v)
      if (match[v] >= v) new_ids[v] = m++;
    for (i32 v = 0; v < before; ++v)
      if (match[v] < v) new_ids[v] = new_ids[match[v]];
    for (auto &c : f2c) c = new_ids[c];
    cur = contract(cur, new_ids, m);
    if (static_cast<double>(before - m) <
        kMinMatchShrink * static_cast<double>(before))
      break;
  }
  return {std::move(cur), std::move(f2c)};
}

// members of each coarse node, ascending fine index (stable argsort)
void members_of(const std::vector<i32> &f2c, i32 m, std::vector<i64> &mptr,
                std::vector<i32> &mem) {
  mptr.assign(static_cast<size_t>(m) + 1, 0);
  for (i32 c : f2c) ++mptr[c + 1];
  for (i32 c = 0; c < m; ++c) mptr[c + 1] += mptr[c];
  mem.resize(f2c.size());
  std::vector<i64> fill(mptr.begin(), mptr.end() - 1);
  for (i32 v = 0; v < static_cast<i32>(f2c.size()); ++v) mem[fill[f2c[v]]++] = v;
}

struct Level {  // a coarsening map after band ordering of the coarse level
  std::vector<i64> mptr;  // members of coarse node c: mem[mptr[c]..mptr[c+1])
  std::vector<i32> mem;
};

// _expand_level + _order_members (reorder.py:339-412)
void expand_level(const Graph &g, const Level &lv, const std::vector<i32> &seq,
                  std::vector<i32> &fine_seq, std::vector<i64> &sizes) {
  PhaseClock pc(5);
  const i32 n = g.n;
  KeyLess less{&g};
  std::vector<i64> placed(n, -1);
  std::vector<char> in_block(n, 0), remaining(n, 0), vis(n, 0);
  fine_seq.clear();
  fine_seq.reserve(n);
  sizes.clear();
  sizes.reserve(seq.size());
  struct Cand {
    i64 anchor;
    i64 outside;
    i32 v;
  };
  std::vector<Cand> cands;
  std::vector<i32> queue, fresh;
  const i64 kInf = std::numeric_limits<i64>::max();
  for (i32 c : seq) {
    const i32 *mb = lv.mem.data() + lv.mptr[c];
    const i64 cnt = lv.mptr[c + 1] - lv.mptr[c];
    sizes.push_back(cnt);
    for (i64 j = 0; j < cnt; ++j) {
      in_block[mb[j]] = 1;
      remaining[mb[j]] = 1;
    }
    // seed keys never change while the block is being ordered: members'
    // placed positions are only written after the whole block is done
    cands.clear();
    for (i64 j = 0; j < cnt; ++j) {
      const i32 v = mb[j];
      i64 anchor = kInf, outside = 0;
      for (i64 p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
        const i32 u = g.idx[p];
        if (in_block[u]) continue;
        const i64 pos = placed[u];
        if (pos >= 0) {
          if (pos < anchor) anchor = pos;
        } else {
          ++outside;
        }
      }
      cands.push_back({anchor, outside, v});
    }
    auto cand_less = [&](const Cand &a, const Cand &b) {
      if (a.anchor != b.anchor) return a.anchor < b.anchor;
      if (a.outside != b.outside) return a.outside < b.outside;
      return less(a.v, b.v);
    };
    std::sort(cands.begin(), cands.end(), cand_less);
    size_t next_seed = 0;
    i64 left = cnt;
    while (left > 0) {
      while (!remaining[cands[next_seed].v]) ++next_seed;
      const i32 seed = cands[next_seed].v;
      queue.clear();
      queue.push_back(seed);
      vis[seed] = 1;
      for (size_t head = 0; head < queue.size(); ++head) {
        const i32 v = queue[head];
        fresh.clear();
        for (i64 p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
          const i32 u = g.idx[p];
          if (in_block[u] && remaining[u] && !vis[u]) {
            vis[u] = 1;
            fresh.push_back(u);
          }
        }
        std::sort(fresh.begin(), fresh.end(), less);
        queue.insert(queue.end(), fresh.begin(), fresh.end());
      }
      for (i32 v : queue) {
        remaining[v] = 0;
        vis[v] = 0;
        placed[v] = static_cast<i64>(fine_seq.size());
        fine_seq.push_back(v);
      }
      left -= static_cast<i64>(queue.size());
    }
    for (i64 j = 0; j < cnt; ++j) in_block[mb[j]] = 0;
  }
}

}  // namespace

struct csrk_bandk_result {
  std::vector<int64_t> fwd;
  std::vector<int64_t> sizes1, sizes2;
};

namespace {

void band_k(i64 n64, const uint32_t *row_ptr, const uint32_t *col_idx, int k,
            const double *targets, csrk_bandk_result &res) {
  if (k != 2 && k != 3) throw InvalidArg("k must be 2 or 3");
  if (n64 == 0) throw InvalidArg("cannot reorder an empty matrix");
  if (n64 > std::numeric_limits<i32>::max())
    throw InvalidArg("band_k supports at most 2^31 - 1 rows");
  Graph g0 = build_graph(n64, row_ptr, col_idx);
  Permutation32 base = weighted_bandwidth_order(g0);
  g0 = relabel(g0, base.fwd, base.inv);
  std::vector<Graph> graphs;
  graphs.push_back(std::move(g0));
  std::vector<Level> levels;
  for (int t = 0; t < k - 1; ++t) {
    Coarsening cz = coarsen(graphs.back(), targets[t]);
    Permutation32 order = weighted_bandwidth_order(cz.coarse);
    Graph coarse = relabel(cz.coarse, order.fwd, order.inv);
    // relabelled map: f2c' = order.fwd[f2c]; members of c' = members of inv[c']
    for (auto &c : cz.f2c) c = order.fwd[c];
    Level lv;
    members_of(cz.f2c, coarse.n, lv.mptr, lv.mem);
    graphs.push_back(std::move(coarse));
    levels.push_back(std::move(lv));
  }
  std::vector<i32> seq(graphs.back().n);
  std::iota(seq.begin(), seq.end(), 0);
  std::vector<std::vector<i64>> collected;
  std::vector<i32> fine;
  for (int level = k - 1; level >= 1; --level) {
    std::vector<i64> sizes;
    expand_level(graphs[level - 1], levels[level - 1], seq, fine, sizes);
    seq.swap(fine);
    collected.push_back(std::move(sizes));
  }
  res.fwd.assign(n64, 0);
  for (i64 i = 0; i < n64; ++i) res.fwd[base.inv[seq[i]]] = i;
  PhaseClock::report();
  res.sizes1 = collected.back();
  if (k == 3) res.sizes2 = collected.front();
}

Graph graph_from_arrays(i64 n, const int64_t *adj_ptr, const int64_t *adj_idx,
                        const int64_t *edge_weight, const int64_t *node_weight) {
  if (n < 0 || n > std::numeric_limits<i32>::max())
    throw InvalidArg("graph size out of range");
  Graph g;
  g.n = static_cast<i32>(n);
  g.ptr.assign(adj_ptr, adj_ptr + n + 1);
  const i64 m = g.ptr[n];
  g.idx.resize(m);
  g.ew.assign(m, 1);
  g.nw.assign(n, 1);
  for (i64 p = 0; p < m; ++p) g.idx[p] = static_cast<i32>(adj_idx[p]);
  if (edge_weight)
    for (i64 p = 0; p < m; ++p) g.ew[p] = static_cast<i32>(edge_weight[p]);
  if (node_weight)
    for (i64 v = 0; v < n; ++v) g.nw[v] = static_cast<i32>(node_weight[v]);
  return g;
}

template <typename F>
int guarded(F &&f) {
  try {
    f();
    return CSRK_OK;
  } catch (const InvalidArg &e) {
    csrk::set_error("%s", e.what());
    return CSRK_EINVAL;
  } catch (const std::bad_alloc &) {
    csrk::set_error("out of host memory in band_k");
    return CSRK_ENOMEM;
  } catch (const std::exception &e) {
    csrk::set_error("%s", e.what());
    return CSRK_EINVAL;
  }
}

}  // namespace

struct csrk_graph {
  Graph g;
  std::vector<int32_t> f2c;
};

extern "C" {

int csrk_band_k(int64_t n, const uint32_t *row_ptr, const uint32_t *col_idx,
                int k, const double *targets, csrk_bandk_result **out) {
  if (!out) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  *out = nullptr;
  auto *res = new (std::nothrow) csrk_bandk_result();
  if (!res) {
    csrk::set_error("out of host memory");
    return CSRK_ENOMEM;
  }
  int rc = guarded([&] { band_k(n, row_ptr, col_idx, k, targets, *res); });
  if (rc != CSRK_OK) {
    delete res;
    return rc;
  }
  *out = res;
  return CSRK_OK;
}

int csrk_bandk_result_sizes(const csrk_bandk_result *r, int64_t out[3]) {
  if (!r || !out) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  out[0] = static_cast<int64_t>(r->fwd.size());
  out[1] = static_cast<int64_t>(r->sizes1.size());
  out[2] = static_cast<int64_t>(r->sizes2.size());
  return CSRK_OK;
}

int csrk_bandk_result_get(const csrk_bandk_result *r, int64_t *fwd,
                          int64_t *sizes1, int64_t *sizes2) {
  if (!r) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  if (fwd) std::memcpy(fwd, r->fwd.data(), r->fwd.size() * sizeof(int64_t));
  if (sizes1)
    std::memcpy(sizes1, r->sizes1.data(), r->sizes1.size() * sizeof(int64_t));
  if (sizes2)
    std::memcpy(sizes2, r->sizes2.data(), r->sizes2.size() * sizeof(int64_t));
  return CSRK_OK;
}

int csrk_bandk_result_free(csrk_bandk_result *r) {
  delete r;
  return CSRK_OK;
}

int csrk_heavy_edge_matching(int64_t n, const int64_t *adj_ptr,
                             const int64_t *adj_idx,
                             const int64_t *edge_weight, int64_t *match) {
  return guarded([&] {
    Graph g = graph_from_arrays(n, adj_ptr, adj_idx, edge_weight, nullptr);
    std::vector<i32> m = heavy_edge_matching(g);
    for (i64 v = 0; v < n; ++v) match[v] = m[v];
  });
}

int csrk_weighted_bandwidth_order(int64_t n, const int64_t *adj_ptr,
                                  const int64_t *adj_idx,
                                  const int64_t *node_weight, int64_t *fwd) {
  return guarded([&] {
    Graph g = graph_from_arrays(n, adj_ptr, adj_idx, nullptr, node_weight);
    Permutation32 p = weighted_bandwidth_order(g);
    for (i64 v = 0; v < n; ++v) fwd[v] = p.fwd[v];
  });
}

int csrk_build_graph(int64_t n, const uint32_t *row_ptr,
                     const uint32_t *col_idx, csrk_graph **out) {
  if (!out) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  *out = nullptr;
  auto *r = new (std::nothrow) csrk_graph();
  if (!r) {
    csrk::set_error("out of host memory");
    return CSRK_ENOMEM;
  }
  int rc = guarded([&] {
    if (n > std::numeric_limits<i32>::max())
      throw InvalidArg("graph size out of range");
    r->g = build_graph(n, row_ptr, col_idx);
  });
  if (rc != CSRK_OK) {
    delete r;
    return rc;
  }
  *out = r;
  return CSRK_OK;
}

int csrk_coarsen(int64_t n, const int64_t *adj_ptr, const int64_t *adj_idx,
                 const int64_t *edge_weight, const int64_t *node_weight,
                 double target, csrk_graph **out) {
  if (!out) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  *out = nullptr;
  auto *r = new (std::nothrow) csrk_graph();
  if (!r) {
    csrk::set_error("out of host memory");
    return CSRK_ENOMEM;
  }
  int rc = guarded([&] {
    Graph g = graph_from_arrays(n, adj_ptr, adj_idx, edge_weight, node_weight);
    Coarsening cz = coarsen(g, target);
    r->g = std::move(cz.coarse);
    r->f2c = std::move(cz.f2c);
  });
  if (rc != CSRK_OK) {
    delete r;
    return rc;
  }
  *out = r;
  return CSRK_OK;
}

int csrk_graph_sizes(const csrk_graph *r, int64_t out[3]) {
  if (!r || !out) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  out[0] = r->g.n;
  out[1] = r->g.n ? r->g.ptr[r->g.n] : 0;
  out[2] = static_cast<int64_t>(r->f2c.size());
  return CSRK_OK;
}

int csrk_graph_get(const csrk_graph *r, int64_t *adj_ptr, int64_t *adj_idx,
                   int64_t *edge_weight, int64_t *node_weight, int64_t *f2c) {
  if (!r) {
    csrk::set_error("null argument");
    return CSRK_EINVAL;
  }
  const Graph &g = r->g;
  const i64 m = g.n ? g.ptr[g.n] : 0;
  if (adj_ptr) {
    if (g.n == 0)
      adj_ptr[0] = 0;
    else
      for (i64 i = 0; i <= g.n; ++i) adj_ptr[i] = g.ptr[i];
  }
  if (adj_idx)
    for (i64 p = 0; p < m; ++p) adj_idx[p] = g.idx[p];
  if (edge_weight)
    for (i64 p = 0; p < m; ++p) edge_weight[p] = g.ew[p];
  if (node_weight)
    for (i64 v = 0; v < g.n; ++v) node_weight[v] = g.nw[v];
  if (f2c)
    for (size_t v = 0; v < r->f2c.size(); ++v) f2c[v] = r->f2c[v];
  return CSRK_OK;
}

int csrk_graph_free(csrk_graph *r) {
  delete r;
  return CSRK_OK;
}

}  // extern "C"
