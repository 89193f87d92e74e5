// CSR-k SpMV kernels for sm_100a.
//
// Bitwise contract: every reference kernel sums a row
// strictly left to right with the multiply and the add rounded separately
// (reference kernels.py:117-147, 224-228), so the products and sums below use
// __dmul_rn / __dadd_rn, which the compiler never contracts into DFMA.  The
// STRIDED order reproduces emulate_gpu_spmv35 (kernels.py:284-324): nonzero p
// of a row feeds lane p mod nx, each lane sums serially from 0.0, and the
// lanes are combined by the zero-padded halving tree of _tree_reduce
// (kernels.py:268-281), here a __shfl_down_sync tree.
//
// The streaming kernel (csrk_stream_kernel) is the B200 hot path:
//   * one CTA per tile; a tile is a run of whole super-super-rows (k=3),
//     super-rows (k=2) or rows (k=1) holding about `tile_nnz` nonzeros
//     (the paper's block <-> SSR mapping, Listing 3, coarsened so a
//     CTA moves enough bytes to keep HBM3e busy);
//   * the tile's contiguous vals / col_idx span is moved HBM -> shared memory
//     by one TMA bulk copy each (cp.async.bulk + mbarrier complete_tx) with an
//     L2 evict-first policy, so the streamed matrix does not push x out of L2;
//   * rows go to threads (SERIAL) or to nx-lane sub-warps (STRIDED); x is
//     gathered through the read-only path; y is stored coalesced.
// Tiles larger than the stage are walked in row-aligned chunks; a single row
// larger than the stage is summed straight from global memory by one warp.

#include <cstdint>

#include "internal.h"

namespace csrk {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(count)
               : "memory");
  // make the initialised barrier visible to the async (TMA) proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar,
                                                      uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_addr(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n"
      "  .reg .pred done;\n"
      "WAIT_%=:\n"
      "  mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      "  @!done bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;"
               : "=l"(pol));
  return pol;
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar`.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void tma_bulk_load(void *dst, const void *src,
                                              uint32_t bytes, uint64_t *bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::"
      "cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

template <typename V>
struct Elem;
template <>
struct Elem<double> {
  static constexpr uint32_t kPerVec = 2;  // elements per 16 bytes
  __device__ static double load_x(const double *x, uint32_t c) {
    return __ldg(x + c);
  }
  __device__ static double out(double acc) { return acc; }
};
template <>
struct Elem<float> {
  static constexpr uint32_t kPerVec = 4;
  __device__ static double load_x(const float *x, uint32_t c) {
    return static_cast<double>(__ldg(x + c));
  }
  __device__ static float out(double acc) { return __double2float_rn(acc); }
};

__host__ __device__ constexpr int pow2_ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// Serial left-to-right sum of one row from (possibly shared) arrays.
// `vb` / `cb` are the element offsets of the staged spans.
template <typename V>
__device__ __forceinline__ double row_sum_serial(const V *__restrict__ sv,
                                                 const uint32_t *__restrict__ sc,
                                                 uint32_t s, uint32_t e,
                                                 const V *__restrict__ x) {
  double acc = 0.0;
  uint32_t p = s;
  // 8-wide batches: issue the x gathers of a batch before the ordered adds
  for (; p + 8 <= e; p += 8) {
    double pv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      pv[j] = __dmul_rn(static_cast<double>(sv[p + j]),
                        Elem<V>::load_x(x, sc[p + j]));
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, pv[j]);
  }
  for (; p < e; ++p)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(sv[p]),
                                   Elem<V>::load_x(x, sc[p])));
  return acc;
}

// Lane partial of the STRIDED order: lane l sums nonzeros l, l+nx, ...
template <typename V, int NX>
__device__ __forceinline__ double row_partial_strided(
    const V *__restrict__ sv, const uint32_t *__restrict__ sc, uint32_t s,
    uint32_t e, int lane, const V *__restrict__ x) {
  double acc = 0.0;
  if (lane < NX) {
    for (uint32_t p = s + lane; p < e; p += NX)
      acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(sv[p]),
                                     Elem<V>::load_x(x, sc[p])));
  }
  return acc;
}

template <int P>
__device__ __forceinline__ double subwarp_tree(double acc) {
#pragma unroll
  for (int off = P / 2; off >= 1; off >>= 1) {
    double o = __shfl_down_sync(0xffffffffu, acc, off, P);
    acc = __dadd_rn(acc, o);
  }
  return acc;
}

// A row longer than the shared stage: summed from global memory by warp 0.
template <typename V, int NX>
__device__ void long_row(const uint32_t *__restrict__ row_ptr,
                         const uint32_t *__restrict__ col_idx,
                         const V *__restrict__ vals, const V *__restrict__ x,
                         V *__restrict__ y, uint32_t r) {
  const int tid = threadIdx.x;
  if (tid >= 32) return;
  const uint32_t s = row_ptr[r], e = row_ptr[r + 1];
  if constexpr (NX == 0) {
    // products in parallel, the ordered sum broadcast through shuffles
    double acc = 0.0;
    for (uint32_t p0 = s; p0 < e; p0 += 32) {
      const uint32_t p = p0 + tid;
      double prod = 0.0;
      if (p < e)
        prod = __dmul_rn(static_cast<double>(vals[p]),
                         Elem<V>::load_x(x, col_idx[p]));
      const uint32_t cnt = (e - p0) < 32u ? (e - p0) : 32u;
      for (uint32_t j = 0; j < cnt; ++j)
        acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, prod, j));
    }
    if (tid == 0) y[r] = Elem<V>::out(acc);
  } else {
    constexpr int P = pow2_ceil(NX);
    double acc = 0.0;
    if (tid < P) acc = row_partial_strided<V, NX>(vals, col_idx, s, e, tid, x);
    acc = subwarp_tree<P>(acc);
    if (tid == 0) y[r] = Elem<V>::out(acc);
  }
}

template <typename V, int NX>
__global__ void __launch_bounds__(kThreads)
    csrk_stream_kernel(const uint32_t *__restrict__ row_ptr,
                       const uint32_t *__restrict__ col_idx,
                       const V *__restrict__ vals, const V *__restrict__ x,
                       V *__restrict__ y, const uint32_t *__restrict__ tile_row,
                       uint32_t cap) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  V *sv = reinterpret_cast<V *>(smem + 16);
  uint32_t *sc = reinterpret_cast<uint32_t *>(
      smem + 16 + ((static_cast<size_t>(cap) + 8) * sizeof(V) + 15) / 16 * 16);

  constexpr uint32_t VPV = Elem<V>::kPerVec;
  const int tid = threadIdx.x;
  const uint32_t r0 = tile_row[blockIdx.x];
  const uint32_t r1 = tile_row[blockIdx.x + 1];
  if (tid == 0) mbar_init(bar, 1);
  __syncthreads();
  const uint64_t policy = evict_first_policy();

  uint32_t phase = 0;
  uint32_t ra = r0;
  while (ra < r1) {
    const uint32_t pa = row_ptr[ra];
    uint32_t rb = r1;
    if (row_ptr[r1] - pa > cap) {
      // largest rb in [ra, r1) with row_ptr[rb] - pa <= cap
      uint32_t lo = ra, hi = r1;
      while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (row_ptr[mid] - pa <= cap)
          lo = mid;
        else
          hi = mid;
      }
      rb = lo;
    }
    if (rb == ra) {  // one row longer than the stage
      long_row<V, NX>(row_ptr, col_idx, vals, x, y, ra);
      ra += 1;
      continue;
    }
    const uint32_t pb = row_ptr[rb];
    const uint32_t va0 = pa & ~(VPV - 1), va1 = (pb + VPV - 1) & ~(VPV - 1);
    const uint32_t ca0 = pa & ~3u, ca1 = (pb + 3u) & ~3u;
    const bool staged = pb > pa;
    if (staged && tid == 0) {
      const uint32_t vbytes = (va1 - va0) * static_cast<uint32_t>(sizeof(V));
      const uint32_t cbytes = (ca1 - ca0) * 4u;
      mbar_arrive_expect_tx(bar, vbytes + cbytes);
      tma_bulk_load(sv, vals + va0, vbytes, bar, policy);
      tma_bulk_load(sc, col_idx + ca0, cbytes, bar, policy);
    }
    // shift so that sv_[p] / sc_[p] address global nonzero p
    const V *sv_ = sv - va0;
    const uint32_t *sc_ = sc - ca0;

    if constexpr (NX == 0) {
      // row pointers of this thread's first row load while the copy runs
      uint32_t r = ra + tid;
      uint32_t s = 0, e = 0;
      if (r < rb) {
        s = row_ptr[r];
        e = row_ptr[r + 1];
      }
      if (staged) mbar_wait(bar, phase);
      for (; r < rb; r += kThreads) {
        if (r != ra + tid) {
          s = row_ptr[r];
          e = row_ptr[r + 1];
        }
        y[r] = Elem<V>::out(row_sum_serial<V>(sv_, sc_, s, e, x));
      }
    } else {
      constexpr int P = pow2_ceil(NX);
      constexpr int kSubPerWarp = 32 / P;
      constexpr int kSubPerCta = kThreads / P;
      const int lane = tid % P;
      const int sub = tid / P;
      const int warp_first = (tid / 32) * kSubPerWarp;
      if (staged) mbar_wait(bar, phase);
      for (uint32_t base = ra + warp_first; base < rb; base += kSubPerCta) {
        const uint32_t r = base + (sub - warp_first);
        double acc = 0.0;
        if (r < rb)
          acc = row_partial_strided<V, NX>(sv_, sc_, row_ptr[r], row_ptr[r + 1],
                                           lane, x);
        acc = subwarp_tree<P>(acc);
        if (r < rb && lane == 0) y[r] = Elem<V>::out(acc);
      }
    }
    if (staged) phase ^= 1u;
    __syncthreads();  // stage is rewritten by the next chunk
    ra = rb;
  }
}

// tile_row[t] = first row of group t*Q (k=3: SSR, k=2: SR, k=1: row)
__global__ void build_tiles_kernel(const uint32_t *__restrict__ sr_ptr,
                                   const uint32_t *__restrict__ ssr_ptr, int k,
                                   int64_t n_groups, int64_t n_rows, int64_t q,
                                   int64_t n_tiles, uint32_t *tile_row) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t > n_tiles) return;
  const int64_t g = t * q < n_groups ? t * q : n_groups;
  uint32_t r;
  if (g == n_groups)
    r = static_cast<uint32_t>(n_rows);
  else if (k == 3)
    r = sr_ptr[ssr_ptr[g]];
  else if (k == 2)
    r = sr_ptr[g];
  else
    r = static_cast<uint32_t>(g);
  tile_row[t] = r;
}

// ---- literal paper mappings (with trace) -----------------------------------

__device__ __forceinline__ void put_trace(int64_t *trace, int64_t n, uint32_t row,
                                          int64_t block, int64_t z, int64_t y,
                                          int64_t xf, int64_t xc, int64_t depth) {
  trace[0 * n + row] = row;
  trace[1 * n + row] = block;
  trace[2 * n + row] = z;
  trace[3 * n + row] = y;
  trace[4 * n + row] = xf;
  trace[5 * n + row] = xc;
  trace[6 * n + row] = depth;
}

// PAPER Listing 3 / emulate_gpu_spmv3 (kernels.py:231-261): block = SSR,
// threadIdx.y strides super-rows, threadIdx.x strides rows, serial rows.
__global__ void listing3_kernel(const uint32_t *__restrict__ row_ptr,
                                const uint32_t *__restrict__ col_idx,
                                const double *__restrict__ vals,
                                const uint32_t *__restrict__ sr_ptr,
                                const uint32_t *__restrict__ ssr_ptr,
                                const double *__restrict__ x,
                                double *__restrict__ y, int64_t *trace,
                                int64_t n) {
  const int64_t b = blockIdx.x;
  const uint32_t s0 = ssr_ptr[b], s1 = ssr_ptr[b + 1];
  for (uint32_t sr = s0 + threadIdx.y; sr < s1; sr += blockDim.y) {
    const uint32_t q0 = sr_ptr[sr], q1 = sr_ptr[sr + 1];
    for (uint32_t row = q0 + threadIdx.x; row < q1; row += blockDim.x) {
      double acc = 0.0;
      for (uint32_t p = row_ptr[row]; p < row_ptr[row + 1]; ++p)
        acc = __dadd_rn(acc, __dmul_rn(vals[p], __ldg(x + col_idx[p])));
      y[row] = acc;
      if (trace) put_trace(trace, n, row, b, 0, threadIdx.y, threadIdx.x, 1, 0);
    }
  }
}

// PAPER Listing 4 / emulate_gpu_spmv35 (kernels.py:284-324): block = SSR,
// z strides super-rows, y strides rows, x strides the nonzeros of a row into
// temp[x]; the x lanes are combined by the halving tree in shared memory.
// Loop trip counts are made block-uniform so every __syncthreads is reached
// by all threads.
__global__ void listing4_kernel(const uint32_t *__restrict__ row_ptr,
                                const uint32_t *__restrict__ col_idx,
                                const double *__restrict__ vals,
                                const uint32_t *__restrict__ sr_ptr,
                                const uint32_t *__restrict__ ssr_ptr,
                                const double *__restrict__ x,
                                double *__restrict__ y, int64_t *trace,
                                int64_t n, int pw, int depth) {
  extern __shared__ double temp[];  // [dz][dy][pw]
  __shared__ uint32_t max_rows;
  const int dx = blockDim.x, dy = blockDim.y, dz = blockDim.z;
  const int tx = threadIdx.x, ty = threadIdx.y, tz = threadIdx.z;
  const int flat = (tz * dy + ty) * dx + tx;
  const int nthreads = dx * dy * dz;
  const int64_t b = blockIdx.x;
  const uint32_t s0 = ssr_ptr[b], s1 = ssr_ptr[b + 1];
  // zero the padding lanes [dx, pw) once; the tree never writes them
  for (int i = flat; i < dz * dy * pw; i += nthreads) temp[i] = 0.0;
  if (flat == 0) max_rows = 0;
  __syncthreads();
  uint32_t local_max = 0;
  for (uint32_t sr = s0 + flat; sr < s1; sr += nthreads) {
    const uint32_t len = sr_ptr[sr + 1] - sr_ptr[sr];
    local_max = len > local_max ? len : local_max;
  }
  atomicMax(&max_rows, local_max);
  __syncthreads();
  const uint32_t iters_z = (s1 - s0 + dz - 1) / dz;
  const uint32_t iters_y = (max_rows + dy - 1) / dy;
  double *slot = temp + (tz * dy + ty) * pw;
  for (uint32_t iz = 0; iz < iters_z; ++iz) {
    const uint32_t sr = s0 + tz + iz * dz;
    const bool vz = sr < s1;
    const uint32_t q0 = vz ? sr_ptr[sr] : 0, q1 = vz ? sr_ptr[sr + 1] : 0;
    for (uint32_t iy = 0; iy < iters_y; ++iy) {
      const uint32_t row = q0 + ty + iy * dy;
      const bool valid = vz && row < q1;
      double part = 0.0;
      if (valid) {
        const uint32_t pe = row_ptr[row + 1];
        for (uint32_t p = row_ptr[row] + tx; p < pe; p += dx)
          part = __dadd_rn(part, __dmul_rn(vals[p], __ldg(x + col_idx[p])));
      }
      slot[tx] = part;
      __syncthreads();
      for (int stride = pw / 2; stride >= 1; stride >>= 1) {
        if (tx < stride) slot[tx] = __dadd_rn(slot[tx], slot[tx + stride]);
        __syncthreads();
      }
      if (valid && tx == 0) {
        y[row] = slot[0];
        if (trace)
          put_trace(trace, n, row, b, (sr - s0) % dz, (row - q0) % dy, 0, dx,
                    depth);
      }
      __syncthreads();
    }
  }
}

__global__ void f64_to_f32_kernel(const double *__restrict__ in,
                                  float *__restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = __double2float_rn(in[i]);
}

template <typename V>
size_t stage_bytes(uint32_t cap) {
  return 16 + ((static_cast<size_t>(cap) + 8) * sizeof(V) + 15) / 16 * 16 +
         (static_cast<size_t>(cap) + 8) * 4;
}

template <typename V, int NX>
int launch_stream(const csrk_matrix *m, const V *vals, const V *x, V *y,
                  cudaStream_t stream) {
  const uint32_t cap = static_cast<uint32_t>(m->plan.cap);
  const size_t smem = stage_bytes<V>(cap);
  auto kern = csrk_stream_kernel<V, NX>;
  CSRK_CUDA_TRY(cudaFuncSetAttribute(
      kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<static_cast<unsigned>(m->plan.n_tiles), kThreads, smem, stream>>>(
      m->row_ptr, m->col_idx, vals, x, y, m->plan.tile_row, cap);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

template <typename V>
int dispatch_nx(const csrk_matrix *m, int variant, int nx, const V *vals,
                const V *x, V *y, cudaStream_t s) {
  if (variant == CSRK_SERIAL) return launch_stream<V, 0>(m, vals, x, y, s);
  switch (nx) {
#define CSRK_NX_CASE(N) \
  case N:               \
    return launch_stream<V, N>(m, vals, x, y, s);
    CSRK_NX_CASE(1)
    CSRK_NX_CASE(2)
    CSRK_NX_CASE(3)
    CSRK_NX_CASE(4)
    CSRK_NX_CASE(5)
    CSRK_NX_CASE(6)
    CSRK_NX_CASE(7)
    CSRK_NX_CASE(8)
    CSRK_NX_CASE(9)
    CSRK_NX_CASE(10)
    CSRK_NX_CASE(11)
    CSRK_NX_CASE(12)
    CSRK_NX_CASE(13)
    CSRK_NX_CASE(14)
    CSRK_NX_CASE(15)
    CSRK_NX_CASE(16)
    CSRK_NX_CASE(20)
    CSRK_NX_CASE(24)
    CSRK_NX_CASE(28)
    CSRK_NX_CASE(32)
#undef CSRK_NX_CASE
    default:
      set_error("strided SpMV supports nx in 1..16, 20, 24, 28, 32; got %d "
                "(use the listing-4 kernel for other block dimensions)",
                nx);
      return CSRK_EINVAL;
  }
}

}  // namespace

bool strided_nx_supported(int nx) {
  return (nx >= 1 && nx <= 16) || nx == 20 || nx == 24 || nx == 28 || nx == 32;
}

int ensure_plan(csrk_matrix *m, int64_t tile_nnz, int64_t cap, cudaStream_t s) {
  if (tile_nnz <= 0) tile_nnz = 2048;
  if (cap <= 0) cap = 4096;
  if (cap < 16) cap = 16;
  if (cap > 16384) cap = 16384;
  if (m->plan.tile_row && m->plan.tile_nnz == tile_nnz && m->plan.cap == cap)
    return CSRK_OK;
  int64_t n_groups = m->k == 3 ? m->n_ssr : (m->k == 2 ? m->n_sr : m->n_rows);
  int64_t q = 1;
  if (n_groups > 0 && m->nnz > 0) {
    const double per_group = static_cast<double>(m->nnz) / n_groups;
    q = static_cast<int64_t>(static_cast<double>(tile_nnz) / per_group + 0.5);
    if (q < 1) q = 1;
  }
  const int64_t n_tiles = n_groups > 0 ? (n_groups + q - 1) / q : 0;
  if (n_tiles > 0x7fffffffLL) {
    set_error("too many tiles (%lld)", static_cast<long long>(n_tiles));
    return CSRK_EINVAL;
  }
  if (m->plan.tile_row) {
    CSRK_CUDA_TRY(cudaFree(m->plan.tile_row));
    m->plan.tile_row = nullptr;
  }
  CSRK_CUDA_TRY(cudaMalloc(&m->plan.tile_row, (n_tiles + 1) * sizeof(uint32_t)));
  const int threads = 256;
  const int64_t blocks = (n_tiles + 1 + threads - 1) / threads;
  build_tiles_kernel<<<static_cast<unsigned>(blocks), threads, 0, s>>>(
      m->sr_ptr, m->ssr_ptr, m->k, n_groups, m->n_rows, q, n_tiles,
      m->plan.tile_row);
  CSRK_CUDA_TRY(cudaGetLastError());
  m->plan.tile_nnz = tile_nnz;
  m->plan.cap = cap;
  m->plan.n_tiles = n_tiles;
  return CSRK_OK;
}

int launch_spmv(const csrk_matrix *m, int value_type, int variant, int nx,
                const void *x, void *y, cudaStream_t stream) {
  if (variant != CSRK_SERIAL && variant != CSRK_STRIDED) {
    set_error("unknown SpMV variant %d", variant);
    return CSRK_EINVAL;
  }
  if (m->n_rows == 0) return CSRK_OK;
  if (!m->plan.tile_row) {
    set_error("matrix has no tile plan");
    return CSRK_EINVAL;
  }
  if (value_type == CSRK_F64) {
    if (!m->vals64) {
      set_error("matrix holds no float64 values");
      return CSRK_EINVAL;
    }
    return dispatch_nx<double>(m, variant, nx, m->vals64,
                               static_cast<const double *>(x),
                               static_cast<double *>(y), stream);
  }
  if (value_type == CSRK_F32) {
    if (!m->vals32) {
      set_error("matrix holds no float32 values");
      return CSRK_EINVAL;
    }
    return dispatch_nx<float>(m, variant, nx, m->vals32,
                              static_cast<const float *>(x),
                              static_cast<float *>(y), stream);
  }
  set_error("unknown value type %d", value_type);
  return CSRK_EINVAL;
}

int launch_listing3(const csrk_matrix *m, int dx, int dy, const double *x,
                    double *y, int64_t *trace, cudaStream_t stream) {
  if (m->n_ssr == 0) return CSRK_OK;
  dim3 block(dx, dy, 1);
  listing3_kernel<<<static_cast<unsigned>(m->n_ssr), block, 0, stream>>>(
      m->row_ptr, m->col_idx, m->vals64, m->sr_ptr, m->ssr_ptr, x, y, trace,
      m->n_rows);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

int launch_listing4(const csrk_matrix *m, int dx, int dy, int dz,
                    const double *x, double *y, int64_t *trace,
                    cudaStream_t stream) {
  if (m->n_ssr == 0) return CSRK_OK;
  int pw = 1, depth = 0;
  while (pw < dx) {
    pw <<= 1;
    ++depth;
  }
  dim3 block(dx, dy, dz);
  const size_t smem = static_cast<size_t>(dz) * dy * pw * sizeof(double);
  if (smem > 48 * 1024) {
    CSRK_CUDA_TRY(cudaFuncSetAttribute(
        listing4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>(smem)));
  }
  listing4_kernel<<<static_cast<unsigned>(m->n_ssr), block, smem, stream>>>(
      m->row_ptr, m->col_idx, m->vals64, m->sr_ptr, m->ssr_ptr, x, y, trace,
      m->n_rows, pw, depth);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

int launch_f64_to_f32(const double *in, float *out, int64_t n, cudaStream_t s) {
  if (n == 0) return CSRK_OK;
  f64_to_f32_kernel<<<148 * 8, 256, 0, s>>>(in, out, n);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

}  // namespace csrk
