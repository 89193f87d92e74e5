// Literal PAPER Listing 3 / Listing 4 kernels with the reference's lane
// trace (emulate_gpu_spmv3 / emulate_gpu_spmv35, reference kernels.py:231-324),
// plus small utility kernels.  These reproduce the paper's launch mapping
// (block = super-super-row) exactly; the B200 hot path is spmv.cu.

#include <cstdint>

#include "internal.h"

namespace csrk {
namespace {

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


// ---- x-isolation probe (diagnostic, not on the SpMV path) -----------------
//
// SURVEY.md 8(d) asks for the L2 hit rate of the x gathers alone.  ncu's
// lts / l1tex hit rates of the SpMV kernel mix the streamed matrix (always a
// miss) with the x gathers.  These two kernels walk col_idx in the streaming
// kernel's distribution (2048-entry chunks, persistent CTAs, chunk
// blockIdx.x + k * gridDim.x): MODE 0 reads col_idx only, MODE 1 reads
// col_idx and gathers x[col_idx[p]].  The difference of their sector
// counters (hits, lookups) is the x gathers' own.
template <int MODE>
__global__ void __launch_bounds__(256)
    gather_probe_kernel(const uint32_t *__restrict__ col_idx,
                        const double *__restrict__ x, int64_t nnz,
                        double *__restrict__ out) {
  constexpr int64_t kChunk = 2048;
  const int64_t chunks = (nnz + kChunk - 1) / kChunk;
  double acc = 0.0;
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int64_t p1 = (c + 1) * kChunk < nnz ? (c + 1) * kChunk : nnz;
#pragma unroll 4
    for (int64_t p = c * kChunk + threadIdx.x; p < p1; p += 256) {
      const uint32_t col = __ldcs(col_idx + p);
      if constexpr (MODE == 0)
        acc += static_cast<double>(col);
      else
        acc += __ldg(x + col);
    }
  }
  if (acc == -1.0e300) out[0] = acc;  // keeps the loads; never true
}

}  // namespace

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

int launch_gather_probe(const csrk_matrix *m, int mode, const double *x, double *out,
                        cudaStream_t stream) {
  if (m->nnz == 0) return CSRK_OK;
  const unsigned grid = 148 * 6;
  if (mode == 0)
    gather_probe_kernel<0><<<grid, 256, 0, stream>>>(m->col_idx, x, m->nnz, out);
  else
    gather_probe_kernel<1><<<grid, 256, 0, stream>>>(m->col_idx, x, m->nnz, out);
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
