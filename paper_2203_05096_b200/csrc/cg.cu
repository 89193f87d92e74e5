// Conjugate-gradient loop around the CSR-k SpMV (
// BASELINE config C4: "100 repeated SpMVs as a CG inner loop").
//
// The reference has no solver; this is a new caller of spmv_csr3.  Each CG
// iteration is five kernels on one stream and never returns to the host, so
// a whole run of iterations is captured once into a CUDA graph and replayed:
//   1. Ap = A p                      (csrk_stream_kernel, bitwise spmv_csr3)
//   2. partial p.Ap                  (block partials, fixed order)
//   3. alpha = rr / pAp; x += alpha p; r -= alpha Ap; partial r.r
//   4. beta = rr' / rr; p = r + beta p; rr = rr'   (reads the partials)
// Scalars live in device memory.  Reductions use a fixed two-level tree
// (per-block partials, then one block), so results are deterministic run to
// run.  Vectors are float64 or float32 (reductions always in float64).

#include <cstdint>
#include <type_traits>

#include "internal.h"

namespace csrk {
namespace {

constexpr int kRedThreads = 512;
constexpr int kRedBlocks = 148 * 4;  // partial-sum slots

struct CgScalars {
  double rr;       // r.r of the current residual
  double pap;      // p.Ap
  double rr_new;   // r.r after the update
  double alpha, beta;
  double pad[3];
};

template <typename T>
__device__ __forceinline__ double block_sum(double v, double *red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  }
  return s;  // valid in thread 0
}

// sum of the kRedBlocks partials in a fixed order (one warp)
__device__ __forceinline__ double fold_partials(const double *partials) {
  double s = 0.0;
  if (threadIdx.x < 32) {
    for (int i = threadIdx.x; i < kRedBlocks; i += 32) s += partials[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  }
  return s;
}

// fp32 vectors (round 2): 16-byte accesses and fp32 arithmetic.  The scalar
// kernels converted every element to fp64 (F2F.F64.F32 on both sides of a
// DFMA) and loaded 4 bytes per thread, which left the f32 CG loop short of
// the HBM roofline; here x, r, p update with fp32 FMAs (alpha / beta rounded
// to fp32 once) and each thread's 4-element batch of a reduction is summed in
// fp32 before it is folded into the fp64 accumulator (one conversion per 4
// elements; the batch error is at most 4 unit roundoffs of its sum of
// magnitudes).  fp64 vectors keep the scalar kernels bit for bit.
#ifndef CSRK_CG_VEC
#define CSRK_CG_VEC 1
#endif
#ifndef CSRK_CG_UNROLL  // direction kernel: two float4 of p and r in flight
#define CSRK_CG_UNROLL 1  // (C4 f32 270 -> 248 us, profiles/r02_c4_f32_split.txt)
#endif

__device__ __forceinline__ float sq4(float4 v) {
  return fmaf(v.w, v.w, fmaf(v.z, v.z, fmaf(v.y, v.y, v.x * v.x)));
}
__device__ __forceinline__ float dot4(float4 a, float4 b) {
  return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, a.x * b.x)));
}
__device__ __forceinline__ float4 axpy4(float a, float4 x, float4 y) {  // a x + y
  return make_float4(fmaf(a, x.x, y.x), fmaf(a, x.y, y.y), fmaf(a, x.z, y.z),
                     fmaf(a, x.w, y.w));
}

// vector part [0, n4) as float4, the last n % 4 elements by the first threads
struct VecSpan {
  int64_t n4, tid, stride;
  __device__ VecSpan(int64_t n)
      : n4(n >> 2), tid(blockIdx.x * int64_t(blockDim.x) + threadIdx.x),
        stride(int64_t(gridDim.x) * blockDim.x) {}
};

inline bool vec16(const void *a, const void *b = nullptr, const void *c = nullptr,
                  const void *d = nullptr) {
  const uintptr_t m = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                      reinterpret_cast<uintptr_t>(c) | reinterpret_cast<uintptr_t>(d);
  return CSRK_CG_VEC && (m & 15u) == 0;
}

// fp64 partial of a . b over this thread's elements (VEC: fp32 float4 batches)
template <typename T, bool VEC>
__device__ __forceinline__ double dot_thread(const T *__restrict__ a, const T *__restrict__ b,
                                             int64_t n) {
  double s = 0.0;
  if constexpr (VEC) {
    const VecSpan v(n);
    const float4 *a4 = reinterpret_cast<const float4 *>(a);
    const float4 *b4 = reinterpret_cast<const float4 *>(b);
    for (int64_t i = v.tid; i < v.n4; i += v.stride)
      s += static_cast<double>(dot4(a4[i], b4[i]));
    for (int64_t i = (v.n4 << 2) + v.tid; i < n; i += v.stride)
      s += static_cast<double>(a[i]) * static_cast<double>(b[i]);
  } else {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
      s += static_cast<double>(a[i]) * static_cast<double>(b[i]);
  }
  return s;
}

// x += alpha p; r -= alpha Ap; returns this thread's fp64 partial of r.r
template <typename T, bool VEC>
__device__ __forceinline__ double update_thread(T *__restrict__ x, T *__restrict__ r,
                                                const T *__restrict__ p,
                                                const T *__restrict__ ap, int64_t n,
                                                double alpha) {
  double s = 0.0;
  if constexpr (VEC) {
    const float af = static_cast<float>(alpha);
    const VecSpan v(n);
    float4 *x4 = reinterpret_cast<float4 *>(x);
    float4 *r4 = reinterpret_cast<float4 *>(r);
    const float4 *p4 = reinterpret_cast<const float4 *>(p);
    const float4 *a4 = reinterpret_cast<const float4 *>(ap);
    for (int64_t i = v.tid; i < v.n4; i += v.stride) {
      const float4 pv = p4[i], av = a4[i], xv = x4[i], rv = r4[i];
      x4[i] = axpy4(af, pv, xv);
      const float4 rn = axpy4(-af, av, rv);
      r4[i] = rn;
      s += static_cast<double>(sq4(rn));
    }
    for (int64_t i = (v.n4 << 2) + v.tid; i < n; i += v.stride) {
      x[i] = fmaf(af, p[i], x[i]);
      const float ri = fmaf(-af, ap[i], r[i]);
      r[i] = ri;
      s += static_cast<double>(ri) * static_cast<double>(ri);
    }
  } else {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
      x[i] = static_cast<T>(static_cast<double>(x[i]) + alpha * static_cast<double>(p[i]));
      const double ri = static_cast<double>(r[i]) - alpha * static_cast<double>(ap[i]);
      r[i] = static_cast<T>(ri);
      const double rv = static_cast<double>(static_cast<T>(ri));
      s += rv * rv;
    }
  }
  return s;
}

// p = r + beta p
template <typename T, bool VEC>
__device__ __forceinline__ void direction_thread(T *__restrict__ p, const T *__restrict__ r,
                                                 int64_t n, double beta) {
  if constexpr (VEC) {
    const float bf = static_cast<float>(beta);
    const VecSpan v(n);
    float4 *p4 = reinterpret_cast<float4 *>(p);
    const float4 *r4 = reinterpret_cast<const float4 *>(r);
#if CSRK_CG_UNROLL
    // two float4 of p and r in flight per thread before the stores
    int64_t i = v.tid;
    for (; i + v.stride < v.n4; i += 2 * v.stride) {
      const float4 pa = p4[i], ra = r4[i], pb = p4[i + v.stride], rb = r4[i + v.stride];
      p4[i] = axpy4(bf, pa, ra);
      p4[i + v.stride] = axpy4(bf, pb, rb);
    }
    if (i < v.n4) p4[i] = axpy4(bf, p4[i], r4[i]);
#else
    for (int64_t i = v.tid; i < v.n4; i += v.stride) p4[i] = axpy4(bf, p4[i], r4[i]);
#endif
    for (int64_t i = (v.n4 << 2) + v.tid; i < n; i += v.stride) p[i] = fmaf(bf, p[i], r[i]);
  } else {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
      p[i] = static_cast<T>(static_cast<double>(r[i]) + beta * static_cast<double>(p[i]));
  }
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(kRedThreads)
    dot_partial_kernel(const T *__restrict__ a, const T *__restrict__ b, int64_t n,
                       double *__restrict__ partials) {
  __shared__ double red[32];
  const double s = dot_thread<T, VEC>(a, b, n);
  const double t = block_sum<T>(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// alpha = rr / pAp; x += alpha p; r -= alpha Ap; partial r.r
template <typename T, bool VEC>
__global__ void __launch_bounds__(kRedThreads)
    cg_update_kernel(T *__restrict__ x, T *__restrict__ r, const T *__restrict__ p,
                     const T *__restrict__ ap, int64_t n, const double *__restrict__ pap_part,
                     CgScalars *__restrict__ sc, double *__restrict__ rr_part) {
  __shared__ double red[32];
  __shared__ double s_alpha;
  if (threadIdx.x < 32) {
    const double pap = fold_partials(pap_part);
    if (threadIdx.x == 0) {
      const double alpha = pap != 0.0 ? sc->rr / pap : 0.0;
      s_alpha = alpha;
      if (blockIdx.x == 0) {
        sc->pap = pap;
        sc->alpha = alpha;
      }
    }
  }
  __syncthreads();
  const double s = update_thread<T, VEC>(x, r, p, ap, n, s_alpha);
  const double t = block_sum<T>(s, red);
  if (threadIdx.x == 0) rr_part[blockIdx.x] = t;
}

// beta = rr' / rr; p = r + beta p; rr = rr' (block 0 publishes)
template <typename T, bool VEC>
__global__ void __launch_bounds__(kRedThreads)
    cg_direction_kernel(T *__restrict__ p, const T *__restrict__ r, int64_t n,
                        const double *__restrict__ rr_part, CgScalars *__restrict__ sc) {
  __shared__ double s_beta, s_rr;
  if (threadIdx.x < 32) {
    const double rr_new = fold_partials(rr_part);
    if (threadIdx.x == 0) {
      s_beta = sc->rr != 0.0 ? rr_new / sc->rr : 0.0;
      s_rr = rr_new;
    }
  }
  __syncthreads();
  direction_thread<T, VEC>(p, r, n, s_beta);
  // every block read sc->rr above; a grid-wide order is needed before the
  // write, so the publish happens in the next kernel (set_rr_kernel)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->rr_new = s_rr;
    sc->beta = s_beta;
  }
}

__global__ void set_rr_kernel(CgScalars *sc) { sc->rr = sc->rr_new; }

// r = b - A x computed as r = b - ax; p = r; rr = r.r partials
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    cg_init_kernel(const T *__restrict__ b, const T *__restrict__ ax, T *__restrict__ r,
                   T *__restrict__ p, int64_t n, double *__restrict__ rr_part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T ri = static_cast<T>(static_cast<double>(b[i]) - static_cast<double>(ax[i]));
    r[i] = ri;
    p[i] = ri;
    s += static_cast<double>(ri) * static_cast<double>(ri);
  }
  const double t = block_sum<T>(s, red);
  if (threadIdx.x == 0) rr_part[blockIdx.x] = t;
}

__global__ void cg_init_scalar_kernel(const double *__restrict__ rr_part,
                                      CgScalars *__restrict__ sc) {
  const double rr = fold_partials(rr_part);
  if (threadIdx.x == 0) {
    sc->rr = rr;
    sc->rr_new = rr;
  }
}

// power-iteration normalisation x = y / max|y| (the repeated-SpMV loop of
// SURVEY.md §8(d)): partial max, then scale
template <typename T>
__global__ void absmax_partial_kernel(const T *__restrict__ y, int64_t n,
                                      double *__restrict__ partials) {
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    m = fmax(m, fabs(static_cast<double>(y[i])));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) partials[blockIdx.x] = m;
  }
}

template <typename T>
__global__ void scale_by_max_kernel(const T *__restrict__ y, T *__restrict__ x, int64_t n,
                                    const double *__restrict__ partials) {
  __shared__ double s_inv;
  if (threadIdx.x < 32) {
    double m = 0.0;
    for (int i = threadIdx.x; i < kRedBlocks; i += 32) m = fmax(m, partials[i]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) s_inv = m > 0.0 ? 1.0 / m : 0.0;
  }
  __syncthreads();
  const double inv = s_inv;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    x[i] = static_cast<T>(static_cast<double>(y[i]) * inv);
}

// ---- step kernels of the distributed CG (dist.DistCG) -------------------
//
// Across GPUs every dot product is a rank-local partial followed by an
// all-reduce, so the iteration is split where the all-reduces go: each
// kernel below ends its own reduction on the device (the last block to
// finish folds the per-block partials in a fixed order -- deterministic, one
// launch), and the scalars live in a caller-owned device array that the
// caller's NCCL all-reduce updates in place between the kernels:
//   dot(p, Ap) -> sc[PAP]          | all-reduce sc[PAP]
//   update     -> x, r, sc[RRNEW]  | all-reduce sc[RRNEW]
//   direction  -> p, sc[RR] = sc[RRNEW]
// Three launches + two all-reduces per iteration beside the SpMV, all on one
// stream without host synchronisation (graph-capturable).
enum { kScRR = 0, kScPAP = 1, kScRRNew = 2, kScAlpha = 3, kScBeta = 4 };

// the last block of the grid to arrive folds `partials` into *out and
// re-arms the counter
__device__ __forceinline__ void last_block_fold(const double *partials, unsigned *counter,
                                                double *out) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += 32)
      v += reinterpret_cast<const volatile double *>(partials)[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) {
      *out = v;
      *counter = 0u;
    }
  }
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(kRedThreads)
    dist_dot_kernel(const T *__restrict__ a, const T *__restrict__ b, int64_t n,
                    double *__restrict__ partials, unsigned *counter, double *out) {
  __shared__ double red[32];
  const double s = dot_thread<T, VEC>(a, b, n);
  const double t = block_sum<T>(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
  last_block_fold(partials, counter, out);
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(kRedThreads)
    dist_update_kernel(T *__restrict__ x, T *__restrict__ r, const T *__restrict__ p,
                       const T *__restrict__ ap, int64_t n, double *__restrict__ sc,
                       double *__restrict__ partials, unsigned *counter) {
  __shared__ double red[32];
  const double pap = sc[kScPAP];
  const double alpha = pap != 0.0 ? sc[kScRR] / pap : 0.0;
  const double s = update_thread<T, VEC>(x, r, p, ap, n, alpha);
  const double t = block_sum<T>(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[kScAlpha] = alpha;
  last_block_fold(partials, counter, sc + kScRRNew);
}

// p = r + beta p with beta = rr' / rr; the last block publishes rr = rr'
template <typename T, bool VEC>
__global__ void __launch_bounds__(kRedThreads)
    dist_direction_kernel(T *__restrict__ p, const T *__restrict__ r, int64_t n,
                          double *__restrict__ sc, unsigned *counter) {
  const double rr = sc[kScRR], rr_new = sc[kScRRNew];
  const double beta = rr != 0.0 ? rr_new / rr : 0.0;
  direction_thread<T, VEC>(p, r, n, beta);
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {  // every block has read sc[RR]
    sc[kScBeta] = beta;
    sc[kScRR] = rr_new;
    *counter = 0u;
  }
}

struct Scratch {
  double *pap_part = nullptr, *rr_part = nullptr;
  CgScalars *sc = nullptr;
};

template <typename T>
int cg_run(const csrk_matrix *m, int value_type, int variant, int nx, const T *b, T *x,
           T *r, T *p, T *ap, int iters, double *scalars_out, cudaStream_t s) {
  const int64_t n = m->n_rows;
  Scratch w;
  keep_async_pool();

  CSRK_CUDA_TRY(cudaMallocAsync(&w.pap_part, kRedBlocks * sizeof(double), s));
  keep_async_pool();

  CSRK_CUDA_TRY(cudaMallocAsync(&w.rr_part, kRedBlocks * sizeof(double), s));
  keep_async_pool();

  CSRK_CUDA_TRY(cudaMallocAsync(&w.sc, sizeof(CgScalars), s));
  CSRK_CUDA_TRY(cudaMemsetAsync(w.pap_part, 0, kRedBlocks * sizeof(double), s));
  CSRK_CUDA_TRY(cudaMemsetAsync(w.rr_part, 0, kRedBlocks * sizeof(double), s));
  CSRK_CUDA_TRY(cudaMemsetAsync(w.sc, 0, sizeof(CgScalars), s));
  // fp32 vectors aligned to 16 bytes take the float4 / fp32-arithmetic kernels
  const bool vec = std::is_same<T, float>::value && vec16(x, r, p, ap);
  int rc = launch_spmv(m, value_type, variant, nx, x, ap, s);  // ap = A x0
  if (rc == CSRK_OK) {
    cg_init_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(b, ap, r, p, n, w.rr_part);
    cg_init_scalar_kernel<<<1, 32, 0, s>>>(w.rr_part, w.sc);
  }
  for (int it = 0; rc == CSRK_OK && it < iters; ++it) {
    // Ap = A p with the p . Ap partials fused into the SpMV when the launch
    // allows it (serial inline order, no long rows): saves re-reading p and
    // Ap; otherwise the separate dot kernel
    bool fused = false;
    rc = launch_spmv_dot(m, value_type, variant, nx, p, ap, s, w.pap_part, kRedBlocks,
                         &fused);
    if (rc == CSRK_OK && !fused) {
      rc = launch_spmv(m, value_type, variant, nx, p, ap, s);
      if (rc == CSRK_OK) {
        if (vec)
          dot_partial_kernel<T, true><<<kRedBlocks, kRedThreads, 0, s>>>(p, ap, n, w.pap_part);
        else
          dot_partial_kernel<T, false><<<kRedBlocks, kRedThreads, 0, s>>>(p, ap, n, w.pap_part);
      }
    }
    if (rc != CSRK_OK) break;
    if (vec) {
      cg_update_kernel<T, true><<<kRedBlocks, kRedThreads, 0, s>>>(x, r, p, ap, n, w.pap_part,
                                                                  w.sc, w.rr_part);
      cg_direction_kernel<T, true><<<kRedBlocks, kRedThreads, 0, s>>>(p, r, n, w.rr_part, w.sc);
    } else {
      cg_update_kernel<T, false><<<kRedBlocks, kRedThreads, 0, s>>>(x, r, p, ap, n, w.pap_part,
                                                                   w.sc, w.rr_part);
      cg_direction_kernel<T, false><<<kRedBlocks, kRedThreads, 0, s>>>(p, r, n, w.rr_part,
                                                                      w.sc);
    }
    set_rr_kernel<<<1, 1, 0, s>>>(w.sc);
  }
  cudaError_t e = cudaGetLastError();
  if (rc == CSRK_OK && e != cudaSuccess) {
    set_error("CUDA error %s in cg: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    rc = CSRK_ECUDA;
  }
  if (rc == CSRK_OK && scalars_out) {
    CgScalars h;
    e = cudaMemcpyAsync(&h, w.sc, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      set_error("CUDA error %s in cg: %s", cudaGetErrorName(e), cudaGetErrorString(e));
      rc = CSRK_ECUDA;
    } else {
      scalars_out[0] = h.rr;
      scalars_out[1] = h.alpha;
      scalars_out[2] = h.beta;
      scalars_out[3] = h.pap;
    }
  }
  cudaFreeAsync(w.pap_part, s);
  cudaFreeAsync(w.rr_part, s);
  cudaFreeAsync(w.sc, s);
  return rc;
}

template <typename T>
int power_run(const csrk_matrix *m, int value_type, int variant, int nx, T *x, T *y,
              int iters, cudaStream_t s) {
  double *part = nullptr;
  keep_async_pool();

  CSRK_CUDA_TRY(cudaMallocAsync(&part, kRedBlocks * sizeof(double), s));
  int rc = CSRK_OK;
  for (int it = 0; it < iters && rc == CSRK_OK; ++it) {
    rc = launch_spmv(m, value_type, variant, nx, x, y, s);
    if (rc != CSRK_OK) break;
    absmax_partial_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(y, m->n_rows, part);
    scale_by_max_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(y, x, m->n_rows, part);
  }
  cudaFreeAsync(part, s);
  if (rc == CSRK_OK) CSRK_CUDA_TRY(cudaGetLastError());
  return rc;
}

}  // namespace
}  // namespace csrk

using namespace csrk;

extern "C" {

int csrk_cg(const csrk_matrix *m, int value_type, int variant, int nx, const void *b,
            void *x, void *r, void *p, void *ap, int iters, double *scalars,
            void *stream) {
  if (!m || !b || !x || !r || !p || !ap || iters < 0) {
    set_error("invalid argument to csrk_cg");
    return CSRK_EINVAL;
  }
  if (m->n_rows != m->n_cols) {
    set_error("CG requires a square matrix");
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  CSRK_TRY(prepare_plan(m, value_type, variant, nx));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (value_type == CSRK_F32)
    return cg_run<float>(m, value_type, variant, nx, static_cast<const float *>(b),
                         static_cast<float *>(x), static_cast<float *>(r),
                         static_cast<float *>(p), static_cast<float *>(ap), iters,
                         scalars, s);
  return cg_run<double>(m, value_type, variant, nx, static_cast<const double *>(b),
                        static_cast<double *>(x), static_cast<double *>(r),
                        static_cast<double *>(p), static_cast<double *>(ap), iters,
                        scalars, s);
}

int csrk_power(const csrk_matrix *m, int value_type, int variant, int nx, void *x,
               void *y, int iters, void *stream) {
  if (!m || !x || !y || iters < 0) {
    set_error("invalid argument to csrk_power");
    return CSRK_EINVAL;
  }
  if (m->n_rows != m->n_cols) {  // y becomes the next x
    set_error("power iterations require a square matrix");
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  CSRK_TRY(prepare_plan(m, value_type, variant, nx));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (value_type == CSRK_F32)
    return power_run<float>(m, value_type, variant, nx, static_cast<float *>(x),
                            static_cast<float *>(y), iters, s);
  return power_run<double>(m, value_type, variant, nx, static_cast<double *>(x),
                           static_cast<double *>(y), iters, s);
}

}  // extern "C"

namespace {
inline unsigned red_grid(int64_t n) {
  int64_t b = (n + kRedThreads - 1) / kRedThreads;
  return static_cast<unsigned>(b < 1 ? 1 : (b > kRedBlocks ? kRedBlocks : b));
}
}  // namespace

extern "C" {

int csrk_vec_dot(int value_type, int64_t n, const void *a, const void *b, double *partials,
                 unsigned *counter, double *out, void *stream) {
  if (n < 0 || (n > 0 && (!a || !b)) || !partials || !counter || !out) {
    set_error("invalid argument to csrk_vec_dot");
    return CSRK_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned g = red_grid(n);
  if (value_type == CSRK_F32 && vec16(a, b))
    dist_dot_kernel<float, true><<<g, kRedThreads, 0, s>>>(static_cast<const float *>(a),
                                                           static_cast<const float *>(b), n,
                                                           partials, counter, out);
  else if (value_type == CSRK_F32)
    dist_dot_kernel<float, false><<<g, kRedThreads, 0, s>>>(static_cast<const float *>(a),
                                                            static_cast<const float *>(b), n,
                                                            partials, counter, out);
  else
    dist_dot_kernel<double, false><<<g, kRedThreads, 0, s>>>(static_cast<const double *>(a),
                                                      static_cast<const double *>(b), n,
                                                      partials, counter, out);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

int csrk_cg_update(int value_type, int64_t n, void *x, void *r, const void *p, const void *ap,
                   double *scalars, double *partials, unsigned *counter, void *stream) {
  if (n < 0 || (n > 0 && (!x || !r || !p || !ap)) || !scalars || !partials || !counter) {
    set_error("invalid argument to csrk_cg_update");
    return CSRK_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned g = red_grid(n);
  if (value_type == CSRK_F32 && vec16(x, r, p, ap))
    dist_update_kernel<float, true><<<g, kRedThreads, 0, s>>>(
        static_cast<float *>(x), static_cast<float *>(r), static_cast<const float *>(p),
        static_cast<const float *>(ap), n, scalars, partials, counter);
  else if (value_type == CSRK_F32)
    dist_update_kernel<float, false><<<g, kRedThreads, 0, s>>>(
        static_cast<float *>(x), static_cast<float *>(r), static_cast<const float *>(p),
        static_cast<const float *>(ap), n, scalars, partials, counter);
  else
    dist_update_kernel<double, false><<<g, kRedThreads, 0, s>>>(
        static_cast<double *>(x), static_cast<double *>(r), static_cast<const double *>(p),
        static_cast<const double *>(ap), n, scalars, partials, counter);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

int csrk_cg_direction(int value_type, int64_t n, void *p, const void *r, double *scalars,
                      unsigned *counter, void *stream) {
  if (n < 0 || (n > 0 && (!p || !r)) || !scalars || !counter) {
    set_error("invalid argument to csrk_cg_direction");
    return CSRK_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned g = red_grid(n);
  if (value_type == CSRK_F32 && vec16(p, r))
    dist_direction_kernel<float, true><<<g, kRedThreads, 0, s>>>(
        static_cast<float *>(p), static_cast<const float *>(r), n, scalars, counter);
  else if (value_type == CSRK_F32)
    dist_direction_kernel<float, false><<<g, kRedThreads, 0, s>>>(
        static_cast<float *>(p), static_cast<const float *>(r), n, scalars, counter);
  else
    dist_direction_kernel<double, false><<<g, kRedThreads, 0, s>>>(
        static_cast<double *>(p), static_cast<const double *>(r), n, scalars, counter);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

}  // extern "C"
