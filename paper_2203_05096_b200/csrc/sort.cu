// Stable LSD radix sort of (uint64 key, uint32 value) pairs on the device --
// the sorting primitive of device-side CSR-k construction (graph building,
// relabelling and contraction sort rows by composite keys).
//
// 8-bit digits, one pass per byte in [begin_bit, end_bit).  A pass is
//   1. per-tile digit histograms, stored digit-major (hist[d * tiles + t]);
//   2. an exclusive scan of the histograms (construct.cu's scan) -> global
//      offsets, so equal digits keep tile order;
//   3. a scatter in which each tile ranks its items stably: the tile's items
//      are visited in index order, 256 per round; within a round a warp
//      finds equal digits with __match_any_sync and counts lower lanes, and
//      per-warp digit counts give the offset of earlier warps.
// Stability makes the LSD passes compose into a full stable sort.

#include <cstdint>
#include <utility>

#include "internal.h"

namespace csrk {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 8;
constexpr int kSortTile = kSortThreads * kSortRounds;  // 2048 items
constexpr int kWarps = kSortThreads / 32;

__global__ void __launch_bounds__(kSortThreads)
    digit_hist_kernel(const uint64_t *__restrict__ keys, int64_t n, int shift,
                      int64_t tiles, int64_t *__restrict__ hist) {
  __shared__ unsigned int counts[256];
  counts[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = blockIdx.x * int64_t(kSortTile);
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&counts[(keys[i] >> shift) & 0xffu], 1u);
  }
  __syncthreads();
  hist[threadIdx.x * tiles + blockIdx.x] = counts[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads)
    digit_scatter_kernel(const uint64_t *__restrict__ keys_in,
                         const uint32_t *__restrict__ vals_in, int64_t n, int shift,
                         int64_t tiles, const int64_t *__restrict__ offsets,
                         uint64_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out) {
  __shared__ unsigned int warp_cnt[kWarps][256];
  __shared__ unsigned int running[256];
  __shared__ int64_t tile_off[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  running[threadIdx.x] = 0;
  tile_off[threadIdx.x] = offsets[threadIdx.x * tiles + blockIdx.x];
  const int64_t base = blockIdx.x * int64_t(kSortTile);
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int r = 0; r < kSortRounds; ++r) {
    for (int w = 0; w < kWarps; ++w) warp_cnt[w][threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = base + r * kSortThreads + threadIdx.x;
    const bool valid = i < n;
    uint64_t key = 0;
    uint32_t val = 0;
    unsigned d = 256;  // out-of-range sentinel digit for invalid lanes
    if (valid) {
      key = keys_in[i];
      val = vals_in[i];
      d = static_cast<unsigned>((key >> shift) & 0xffu);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned rank_in_warp = __popc(peers & lt_mask);
    if (valid && rank_in_warp == 0) warp_cnt[warp][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      unsigned before = running[d];
      for (int w = 0; w < warp; ++w) before += warp_cnt[w][d];
      const int64_t pos = tile_off[d] + before + rank_in_warp;
      keys_out[pos] = key;
      vals_out[pos] = val;
    }
    __syncthreads();
    unsigned add = 0;
    for (int w = 0; w < kWarps; ++w) add += warp_cnt[w][threadIdx.x];
    running[threadIdx.x] += add;
  }
}

}  // namespace


// Sort `n` pairs by key bits [begin_bit, end_bit) (multiples of 8), stable.
// keys / vals are updated in place; tmp_keys / tmp_vals are n-element
// scratch buffers.
int radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *tmp_keys,
                     uint32_t *tmp_vals, int64_t n, int begin_bit, int end_bit,
                     cudaStream_t s) {
  if (n <= 1) return CSRK_OK;
  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  int64_t *hist = nullptr, *offs = nullptr;
  keep_async_pool();

  CSRK_CUDA_TRY(cudaMallocAsync(&hist, 256 * tiles * sizeof(int64_t), s));
  keep_async_pool();

  CSRK_CUDA_TRY(cudaMallocAsync(&offs, (256 * tiles + 1) * sizeof(int64_t), s));
  uint64_t *kin = keys, *kout = tmp_keys;
  uint32_t *vin = vals, *vout = tmp_vals;
  int passes = 0;
  int rc = CSRK_OK;
  for (int shift = begin_bit; shift < end_bit && rc == CSRK_OK; shift += 8) {
    digit_hist_kernel<<<static_cast<unsigned>(tiles), kSortThreads, 0, s>>>(
        kin, n, shift, tiles, hist);
    rc = exclusive_scan_i64(hist, 256 * tiles, offs, s);
    if (rc != CSRK_OK) break;
    digit_scatter_kernel<<<static_cast<unsigned>(tiles), kSortThreads, 0, s>>>(
        kin, vin, n, shift, tiles, offs, kout, vout);
    std::swap(kin, kout);
    std::swap(vin, vout);
    ++passes;
  }
  if (rc == CSRK_OK && (passes & 1)) {
    cudaMemcpyAsync(keys, kin, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(vals, vin, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
  }
  cudaFreeAsync(hist, s);
  cudaFreeAsync(offs, s);
  if (rc == CSRK_OK) CSRK_CUDA_TRY(cudaGetLastError());
  return rc;
}

}  // namespace csrk

extern "C" int csrk_sort_pairs(int device, int64_t n, uint64_t *keys, uint32_t *vals,
                               int begin_bit, int end_bit, void *stream) {
  if ((n > 0 && (!keys || !vals)) || begin_bit < 0 || end_bit > 64 || begin_bit % 8 ||
      end_bit % 8) {
    csrk::set_error("invalid argument to csrk_sort_pairs");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint64_t *tk = nullptr;
  uint32_t *tv = nullptr;
  csrk::keep_async_pool();

  CSRK_CUDA_TRY(cudaMallocAsync(&tk, (n > 0 ? n : 1) * sizeof(uint64_t), s));
  csrk::keep_async_pool();

  CSRK_CUDA_TRY(cudaMallocAsync(&tv, (n > 0 ? n : 1) * sizeof(uint32_t), s));
  const int rc = csrk::radix_sort_pairs(keys, vals, tk, tv, n, begin_bit, end_bit, s);
  cudaFreeAsync(tk, s);
  cudaFreeAsync(tv, s);
  return rc;
}
