// Internal declarations shared by the translation units of libcsrk_cuda.so.
#pragma once

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/csrk.h"

namespace csrk {

void set_error(const char *fmt, ...);

// A tile plan of the streaming kernel: tile t covers rows
// [tile_row[t], tile_row[t+1]) made of whole groups.
constexpr int64_t kDefaultTileCost = 2048;  // nonzeros + rows per tile (round-1 plan)
constexpr int64_t kDeepRingTileCost = 1536; // tile of the 3-stage ring (regular rows)
constexpr int64_t kDefaultStages = 2;       // TMA ring depth per CTA (plan sweep)
constexpr int64_t kDefaultCtasPerSm = 3;    // resident streaming CTAs per SM
constexpr int kGatherAuto = 2;
constexpr int64_t kLongRow = 128;  // rows longer than this are summed a warp each

// Auto schedule (round-2 plan re-sweep on the final kernel,
// profiles/r02l_*, r02m_plan_confirm.jsonl, r02n_*; round 1:
// r01_sched_sweep.txt):
//  * regular rows (variance <= 10, the paper's class boundary) without long
//    rows: tiles of 1536 cost units and a 3-stage ring -- three stages still
//    fit three f64 CTAs (196 KB) and the deeper ring hides the TMA round
//    trip (interleaved in one process: C3 f64 0.390 -> 0.359 ms, C3 f32
//    0.271 -> 0.246 at 4 CTAs, C2 f64 0.264 -> 0.258);
//  * irregular rows or rows longer than kLongRow: tiles of 2048, 2 stages
//    and 2 CTAs per SM (~120 KB of L1 for the random x gathers; the deeper
//    plan lost 28 % on the power-law probe, where the long-row kernel also
//    needs room beside the streaming kernel);
//  * 3 CTAs per SM in f64 and 4 in f32 for regular rows (half the bytes per
//    nonzero, so more tiles in flight);
//  * the serial order over rows longer than 16 nonzeros gathers first
//    (C3 +13 %); short rows keep the inline gathers (C2 -15 % otherwise).
//  * irregular rows without long rows whose lengths spread less than their
//    mean squared (C5; the inline-gather class below): tiles of 1536, 2
//    stages, 3 CTAs -- the same shared memory and carveout as 2 x 2 x 2048,
//    one more tile in flight per SM (C5 f64 0.2066 -> 0.2037 ms, f32 0.1789
//    -> 0.1717).  Wider spreads (power-law rows capped at 64 / 128, f64
//    gather-first) keep 2048 x 2 x 2: 0.1356 vs 0.1394 ms
//    (profiles/r02_c5_plan_confirm.jsonl).
inline bool irregular_inline(double row_var, double mean_row, int64_t n_long) {
  return row_var > 10.0 && n_long == 0 && row_var <= mean_row * mean_row;
}
inline int auto_ctas(double row_var, int value_bytes, int64_t n_long = 1,
                     double mean_row = 0.0) {
  if (row_var > 10.0) return irregular_inline(row_var, mean_row, n_long) ? 3 : 2;
  return value_bytes == 4 ? 4 : 3;
}
// tile cost base of the auto plan (auto_tile_cost refines it per order)
inline bool small_tiles(double row_var, int64_t n_long, double mean_row);
#ifndef CSRK_OLD_AUTO
// regular rows without long rows: 3-stage ring at tile 1536; otherwise the
// round-1 plan (2 stages, tile 2048: auto_tile_cost below)
inline bool deep_ring(double row_var, int64_t n_long) { return row_var <= 10.0 && n_long == 0; }
#else
inline bool deep_ring(double, int64_t) { return false; }
#endif
inline int64_t auto_stages(double row_var, int64_t n_long) {
  return deep_ring(row_var, n_long) ? 3 : 2;
}
inline bool small_tiles(double row_var, int64_t n_long, double mean_row) {
  return deep_ring(row_var, n_long) || irregular_inline(row_var, mean_row, n_long);
}
// Gather first in the serial order when rows are long (C3: 27-nonzero rows)
// or their lengths spread wider than their mean (a thread per row then waits
// on the longest row of its warp; power-law rows, mean 9.8 / variance 238:
// 1.67 -> 2.36 TB/s), inline otherwise (C5: mean 10 / variance 30 loses 2 %).
// In the strided order gather first when rows are shorter than the
// sub-warp (most lanes would idle through the inline batches): C2 nx = 8
// 2.30 -> 2.86 TB/s, C5 nx = 16 1.18 -> 1.36, C1 nx = 32 0.44 -> 0.65; rows
// at least a sub-warp long keep inline gathers (C3 nx = 8 5.33 vs 4.07).
inline bool auto_gather(int variant, int nx, double mean_row, double row_var) {
  if (variant == CSRK_SERIAL) return mean_row > 16.0 || row_var > mean_row * mean_row;
  int p = 1;
  while (p < nx) p <<= 1;
  return mean_row < p;
}

// Tile cost for a launch in the STRIDED order: the 256 consumer threads
// hold 256 / P rows per pass (P = nx rounded up to a power of two), and a
// tile whose last pass is mostly empty idles that share of the threads until
// the stage is released.  When the default 2048-cost tile fills its passes
// below 85 %, shrink it to a whole number of full passes (5 % slack for the
// row-count spread of group-aligned cuts).  C3 (27-nonzero rows) with nx = 4:
// 74 rows = 1.2 passes of 64 -> 1684-cost tiles of ~61 rows, 5.1 -> 5.6 TB/s
// (profiles/r01_sched_sweep.txt).  The serial order keeps 2048: short rows
// fill 256 rows per tile, long rows gather first.
inline int64_t auto_tile_cost(double mean_row, int variant, int nx,
                              int64_t base = kDefaultTileCost) {
  if (variant != CSRK_STRIDED) return base;
  int p = 1;
  while (p < nx) p <<= 1;
  const double per_row = mean_row + 1.0;
  const double slots = 256.0 / p;
  const double rows = static_cast<double>(base) / per_row;
  const double passes = rows / slots > 1.0 ? static_cast<double>(static_cast<int64_t>(rows / slots + 0.999999)) : 1.0;
  if (rows / (passes * slots) >= 0.85) return base;
  double full = static_cast<double>(static_cast<int64_t>(rows / slots));
  if (full < 1.0) full = 1.0;
  int64_t tc = static_cast<int64_t>(full * slots * per_row * 0.95);
  if (tc > base) tc = base;
  if (tc < 512) tc = 512;
  return tc;
}

struct TilePlan {
  int64_t tile_cost = 0;  // requested nonzeros + rows per tile
  int64_t cap = 0;        // stage capacity, nonzeros
  int64_t rcap = 0;       // stage capacity, rows
  int64_t stages = 0;     // ring depth
  int64_t n_tiles = 0;
  bool group_aligned = false;    // tile cuts only on SSR / SR boundaries
  // schedule (csrk_matrix_set_schedule): requested gather mode (0 inline,
  // 1 gather-first, 2 auto) and CTAs per SM (0 = auto), plus the row
  // statistics the auto choices read (measured when the plan is built)
  int gather_first = kGatherAuto;
  int ctas_per_sm = 0;
  double mean_row = 0.0, row_var = 0.0;
  double mean_short = 0.0;  // mean length of the rows the streaming kernel sums (<= kLongRow)
  bool row_stats = false;
  bool auto_tile = true;  // tile cost follows the launch's order (auto_tile_cost)
  int cut_mode = 0;       // 0 auto, 1 rows, 2 groups (csrk_matrix_set_cut_mode)
  uint64_t gen = 0;       // bumped whenever tile_row is rebuilt
  uint32_t *tile_row = nullptr;  // device, n_tiles + 1
  uint32_t *tile_ptr = nullptr;  // device, n_tiles + 1 (same allocation): row_ptr[tile_row]
  // rows longer than kLongRow: n_long row indices in the long-row kernel's
  // work order (longest first), then n_long (start, end) nonzero ranges in
  // row order -- the holes the streaming kernel does not stage -- then the
  // n_long rows in row order
  uint32_t *long_rows = nullptr;
  uint32_t *tile_long = nullptr;  // n_tiles + 1 (tile_row's allocation): first hole per tile
  int64_t n_long = 0;
};

// the holes (uint2 pairs) follow the work order at an 8-byte boundary
inline const uint2 *long_holes(const TilePlan &pl) {
  return reinterpret_cast<const uint2 *>(pl.long_rows + ((pl.n_long + 1) & ~int64_t(1)));
}
// and the long rows in row order after the holes
inline const uint32_t *long_rows_asc(const TilePlan &pl) {
  return reinterpret_cast<const uint32_t *>(long_holes(pl) + pl.n_long);
}

}  // namespace csrk

struct csrk_matrix {
  int device = 0;
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  int k = 1;
  int64_t n_sr = 0, n_ssr = 0;
  uint32_t *row_ptr = nullptr;  // n_rows + 1, padded (padded_rows)
  uint32_t *col_idx = nullptr;  // nnz, padded to a multiple of 4 (+4)
  double *vals64 = nullptr;     // nnz, padded
  float *vals32 = nullptr;      // optional
  uint32_t *sr_ptr = nullptr;   // n_sr + 1 (k >= 2)
  uint32_t *ssr_ptr = nullptr;  // n_ssr + 1 (k == 3)
  csrk::TilePlan plan;          // current streaming plan
  int sm_count = 0;
  // host-API staging and the overlapped host pipeline (csrk_spmv_host)
  struct Pipe {
    int chunks = 0;
    std::vector<int> weights;  // chunk weights the cuts were computed for
    int64_t plan_tiles = -1;  // n_tiles the cuts were computed for
    std::vector<int64_t> tile_cut, row_cut;  // chunks + 1
    std::vector<int> x_ready;                // x chunk needed by chunk c
    std::vector<int64_t> x_cut;              // x (column) chunk bounds
    std::string xmode;                       // CSRK_PIPE_XCUT the cuts used
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev_x, ev_c;
    std::vector<cudaEvent_t> ev_x_t, ev_c_t;  // timing events (trace only)
  } pipe;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // the long-row kernel's side streams: one per caller stream (forked from /
  // joined to it), so launches on different streams -- or one being
  // captured into a CUDA graph -- never share fork / join state
  struct Side {
    cudaStream_t caller = nullptr, side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
  };
  std::vector<Side> sides;
  // Thread safety: every C-ABI entry point that plans, stages or launches on
  // a matrix holds this lock (include/csrk.h "Threading"), so concurrent
  // callers of one handle serialise instead of racing on the plan, the
  // staging buffers and the pipeline streams.
  mutable std::mutex mu;
  void *x_stage = nullptr, *y_stage = nullptr;
  size_t x_stage_bytes = 0, y_stage_bytes = 0;
};

struct csrk_dgraph {
  int device = 0;
  int64_t n = 0, m = 0;
  int64_t *ptr = nullptr;
  int32_t *idx = nullptr, *ew = nullptr, *nw = nullptr;
};

namespace csrk {

// The stream-ordered allocator's default pool returns freed memory to the
// driver at every synchronisation (release threshold 0), so a loop that
// allocates scratch with cudaMallocAsync and synchronises -- one Band-k level
// per iteration -- re-maps device memory each time (measured: the CM levels
// of C2 took 3.3 s instead of 0.4 s on some boxes).  Keep up to 32 GB cached
// in the pool of every device the library uses.
inline void keep_async_pool() {
  static std::atomic<unsigned> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  if (dev < 32 && ((done.load(std::memory_order_relaxed) >> dev) & 1u)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = 32ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  if (dev < 32) done.fetch_or(1u << dev, std::memory_order_relaxed);
}

// One-shot builders (device Band-k, pack, COO -> CSR) hand the scratch they
// cached in the pool back to the driver when they finish (after their final
// synchronisation), so cudaMalloc-based allocators -- PyTorch's caching
// allocator, NCCL -- can use it; the raised threshold above only keeps
// memory mapped across the level loops *inside* one build.
inline void trim_async_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
}

// padded element count for col_idx / vals allocations: room for the 16-byte
// aligned over-read of the TMA bulk copies at both ends of a span.
inline int64_t padded_nnz(int64_t nnz) { return ((nnz + 3) / 4) * 4 + 8; }
inline int64_t padded_rows(int64_t n_rows) { return ((n_rows + 1 + 3) / 4) * 4 + 8; }

int alloc_matrix_arrays(csrk_matrix *m, bool want64, bool want32);
int ensure_plan(csrk_matrix *m, int64_t tile_cost, int64_t cap, int64_t stages,
                cudaStream_t s, bool force = false);
// before a whole-matrix launch: re-plan for the launch's order when the plan
// is automatic (cached; rebuilds only when the tile cost changes)
int prepare_plan(const csrk_matrix *m, int value_type, int variant, int nx);
int launch_spmv(const csrk_matrix *m, int value_type, int variant, int nx,
                const void *x, void *y, cudaStream_t stream, int64_t t0 = 0,
                int64_t t1 = -1);
int launch_spmv_dot(const csrk_matrix *m, int value_type, int variant, int nx,
                    const void *x, void *y, cudaStream_t stream, double *dot_part,
                    int64_t dot_slots, bool *fused);
int chunk_max_cols(const csrk_matrix *m, const uint32_t *row_cut_dev, int chunks,
                   uint32_t *out_dev, cudaStream_t s);
int launch_listing3(const csrk_matrix *m, int dx, int dy, const double *x,
                    double *y, int64_t *trace, cudaStream_t stream);
int launch_listing4(const csrk_matrix *m, int dx, int dy, int dz,
                    const double *x, double *y, int64_t *trace,
                    cudaStream_t stream);
int launch_gather_probe(const csrk_matrix *m, int mode, const double *x, double *out,
                        cudaStream_t stream);
int launch_f64_to_f32(const double *in, float *out, int64_t n, cudaStream_t s);
int exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, cudaStream_t s);
int radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *tmp_keys,
                     uint32_t *tmp_vals, int64_t n, int begin_bit, int end_bit,
                     cudaStream_t s);

}  // namespace csrk

#define CSRK_CUDA_TRY(expr)                                                 \
  do {                                                                      \
    cudaError_t e_ = (expr);                                                \
    if (e_ != cudaSuccess) {                                                \
      csrk::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_),   \
                      __FILE__, __LINE__, cudaGetErrorString(e_));          \
      return e_ == cudaErrorMemoryAllocation ? CSRK_ENOMEM : CSRK_ECUDA;    \
    }                                                                       \
  } while (0)

// the per-matrix lock of the C-ABI entry points (csrk_matrix::mu)
#define CSRK_LOCK(m) std::lock_guard<std::mutex> csrk_lock_guard_((m)->mu)

#define CSRK_TRY(expr)            \
  do {                            \
    int rc_ = (expr);             \
    if (rc_ != CSRK_OK) return rc_; \
  } while (0)
