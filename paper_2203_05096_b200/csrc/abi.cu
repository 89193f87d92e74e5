// extern "C" entry points of libcsrk_cuda.so (declared in include/csrk.h).
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"

namespace csrk {

static thread_local std::string g_last_error;

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int alloc_matrix_arrays(csrk_matrix *m, bool want64, bool want32) {
  const int64_t pn = padded_nnz(m->nnz);
  CSRK_CUDA_TRY(cudaMalloc(&m->row_ptr, padded_rows(m->n_rows) * sizeof(uint32_t)));
  CSRK_CUDA_TRY(cudaMemset(m->row_ptr, 0, padded_rows(m->n_rows) * sizeof(uint32_t)));
  CSRK_CUDA_TRY(cudaMalloc(&m->col_idx, pn * sizeof(uint32_t)));
  CSRK_CUDA_TRY(cudaMemset(m->col_idx, 0, pn * sizeof(uint32_t)));
  if (want64) {
    CSRK_CUDA_TRY(cudaMalloc(&m->vals64, pn * sizeof(double)));
    CSRK_CUDA_TRY(cudaMemset(m->vals64, 0, pn * sizeof(double)));
  }
  if (want32) {
    CSRK_CUDA_TRY(cudaMalloc(&m->vals32, pn * sizeof(float)));
    CSRK_CUDA_TRY(cudaMemset(m->vals32, 0, pn * sizeof(float)));
  }
  if (m->k >= 2)
    CSRK_CUDA_TRY(cudaMalloc(&m->sr_ptr, (m->n_sr + 1) * sizeof(uint32_t)));
  if (m->k == 3)
    CSRK_CUDA_TRY(cudaMalloc(&m->ssr_ptr, (m->n_ssr + 1) * sizeof(uint32_t)));
  CSRK_CUDA_TRY(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
  CSRK_CUDA_TRY(cudaEventCreate(&m->ev0));
  CSRK_CUDA_TRY(cudaEventCreate(&m->ev1));
  return CSRK_OK;
}

static void release(csrk_matrix *m) {
  if (!m) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(m->device);
  cudaFree(m->row_ptr);
  cudaFree(m->col_idx);
  cudaFree(m->vals64);
  cudaFree(m->vals32);
  cudaFree(m->sr_ptr);
  cudaFree(m->ssr_ptr);
  cudaFree(m->plan.tile_row);
  cudaFree(m->plan.long_rows);
  cudaFree(m->x_stage);
  cudaFree(m->y_stage);
  for (auto e : m->pipe.ev_x) cudaEventDestroy(e);
  for (auto e : m->pipe.ev_c) cudaEventDestroy(e);
  if (m->pipe.h2d) cudaStreamDestroy(m->pipe.h2d);
  if (m->pipe.comp) cudaStreamDestroy(m->pipe.comp);
  if (m->pipe.d2h) cudaStreamDestroy(m->pipe.d2h);
  for (auto &sd : m->sides) {
    cudaEventDestroy(sd.fork);
    cudaEventDestroy(sd.join);
    cudaStreamDestroy(sd.side);
  }
  if (m->ev0) cudaEventDestroy(m->ev0);
  if (m->ev1) cudaEventDestroy(m->ev1);
  if (m->stream) cudaStreamDestroy(m->stream);
  delete m;
  cudaSetDevice(cur);
}

// Validation of a packed layout, with the reference's messages
// (format.py:71-98 CsrMatrix, format.py:180-202 CsrKMatrix).
static int validate_host(int64_t n_rows, int64_t n_cols, int64_t nnz,
                         const uint32_t *row_ptr, int k, int64_t n_sr,
                         const uint32_t *sr_ptr, int64_t n_ssr,
                         const uint32_t *ssr_ptr) {
  if (n_rows < 0 || n_cols < 0) {
    set_error("matrix dimensions must be non-negative");
    return CSRK_EINVAL;
  }
  if (nnz > 2147483647LL) {
    set_error("nnz %lld exceeds the 32-bit index limit 2147483647",
              static_cast<long long>(nnz));
    return CSRK_EINVAL;
  }
  if (row_ptr[0] != 0) {
    set_error("row_ptr[0] must be 0");
    return CSRK_EINVAL;
  }
  if (static_cast<int64_t>(row_ptr[n_rows]) != nnz) {
    set_error("col_idx and vals must have length row_ptr[-1]");
    return CSRK_EINVAL;
  }
  if (k < 1 || k > 3) {
    set_error("k must be 2 or 3");
    return CSRK_EINVAL;
  }
  const uint32_t *ptrs[2] = {sr_ptr, ssr_ptr};
  const int64_t lens[2] = {n_sr, n_ssr};
  int64_t below = n_rows;
  for (int level = 1; level < k; ++level) {
    const uint32_t *p = ptrs[level - 1];
    const int64_t len = lens[level - 1];
    if (!p || len < 0 || p[0] != 0) {
      set_error("level %d pointer array must start at 0", level);
      return CSRK_EINVAL;
    }
    for (int64_t i = 0; i < len; ++i)
      if (p[i + 1] <= p[i]) {
        set_error("level %d pointer array must be strictly increasing", level);
        return CSRK_EINVAL;
      }
    if (static_cast<int64_t>(p[len]) != below) {
      set_error("level %d pointer array must end at %lld, got %lld", level,
                static_cast<long long>(below), static_cast<long long>(p[len]));
      return CSRK_EINVAL;
    }
    below = len;
  }
  return CSRK_OK;
}

}  // namespace csrk

using namespace csrk;

extern "C" {

int csrk_abi_version(void) { return CSRK_ABI_VERSION; }

const char *csrk_last_error(void) { return g_last_error.c_str(); }

int csrk_device_count(int *count) {
  CSRK_CUDA_TRY(cudaGetDeviceCount(count));
  return CSRK_OK;
}

int csrk_buffer_alloc(int device, int64_t bytes, void **out) {
  if (!out || bytes < 0) {
    set_error("invalid buffer request");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(device));
  CSRK_CUDA_TRY(cudaMalloc(out, bytes > 0 ? static_cast<size_t>(bytes) : 16));
  return CSRK_OK;
}

int csrk_buffer_free(int device, void *p) {
  if (!p) return CSRK_OK;
  CSRK_CUDA_TRY(cudaSetDevice(device));
  CSRK_CUDA_TRY(cudaFree(p));
  return CSRK_OK;
}

int csrk_memcpy(void *dst, const void *src, int64_t bytes, int kind,
                void *stream) {
  if (bytes <= 0) return CSRK_OK;
  const cudaMemcpyKind k = kind == 0   ? cudaMemcpyHostToDevice
                           : kind == 1 ? cudaMemcpyDeviceToHost
                                       : cudaMemcpyDeviceToDevice;
  if (stream) {
    CSRK_CUDA_TRY(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), k,
                                  static_cast<cudaStream_t>(stream)));
  } else {
    CSRK_CUDA_TRY(cudaMemcpy(dst, src, static_cast<size_t>(bytes), k));
  }
  return CSRK_OK;
}

int csrk_memset(void *dst, int value, int64_t bytes, void *stream) {
  if (bytes <= 0) return CSRK_OK;
  CSRK_CUDA_TRY(cudaMemsetAsync(dst, value, static_cast<size_t>(bytes),
                                static_cast<cudaStream_t>(stream)));
  if (!stream) CSRK_CUDA_TRY(cudaStreamSynchronize(nullptr));
  return CSRK_OK;
}

int csrk_stream_sync(void *stream) {
  CSRK_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return CSRK_OK;
}

int csrk_device_sync(int device) {
  CSRK_CUDA_TRY(cudaSetDevice(device));
  CSRK_CUDA_TRY(cudaDeviceSynchronize());
  return CSRK_OK;
}

int csrk_matrix_upload(int device, int64_t n_rows, int64_t n_cols, int64_t nnz,
                       const uint32_t *row_ptr, const uint32_t *col_idx,
                       const double *vals, int k, int64_t n_sr,
                       const uint32_t *sr_ptr, int64_t n_ssr,
                       const uint32_t *ssr_ptr, int value_types,
                       csrk_matrix **out) {
  if (!out || !row_ptr || (nnz > 0 && (!col_idx || !vals))) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  *out = nullptr;
  CSRK_TRY(validate_host(n_rows, n_cols, nnz, row_ptr, k, n_sr, sr_ptr, n_ssr,
                         ssr_ptr));
  if ((value_types & (CSRK_F64 | CSRK_F32)) == 0) value_types = CSRK_F64;
  // a column >= n_cols would read outside x
  for (int64_t p = 0; p < nnz; ++p)
    if (static_cast<int64_t>(col_idx[p]) >= n_cols) {
      set_error("column index out of range");
      return CSRK_EINVAL;
    }
  CSRK_CUDA_TRY(cudaSetDevice(device));
  csrk_matrix *m = new csrk_matrix();
  m->device = device;
  m->n_rows = n_rows;
  m->n_cols = n_cols;
  m->nnz = nnz;
  m->k = k;
  m->n_sr = k >= 2 ? n_sr : 0;
  m->n_ssr = k == 3 ? n_ssr : 0;
  int rc = alloc_matrix_arrays(m, true, (value_types & CSRK_F32) != 0);
  if (rc != CSRK_OK) {
    release(m);
    return rc;
  }
  auto fail = [&](cudaError_t e) {
    set_error("CUDA error %s during upload: %s", cudaGetErrorName(e),
              cudaGetErrorString(e));
    release(m);
    return CSRK_ECUDA;
  };
  cudaError_t e;
  if ((e = cudaMemcpy(m->row_ptr, row_ptr, (n_rows + 1) * sizeof(uint32_t),
                      cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(e);
  if (nnz > 0) {
    if ((e = cudaMemcpy(m->col_idx, col_idx, nnz * sizeof(uint32_t),
                        cudaMemcpyHostToDevice)) != cudaSuccess)
      return fail(e);
    if ((e = cudaMemcpy(m->vals64, vals, nnz * sizeof(double),
                        cudaMemcpyHostToDevice)) != cudaSuccess)
      return fail(e);
  }
  if (k >= 2 && (e = cudaMemcpy(m->sr_ptr, sr_ptr, (n_sr + 1) * sizeof(uint32_t),
                                cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(e);
  if (k == 3 &&
      (e = cudaMemcpy(m->ssr_ptr, ssr_ptr, (n_ssr + 1) * sizeof(uint32_t),
                      cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(e);
  if (m->vals32) {
    rc = launch_f64_to_f32(m->vals64, m->vals32, nnz, m->stream);
    if (rc != CSRK_OK) {
      release(m);
      return rc;
    }
  }
  rc = ensure_plan(m, 0, 0, 0, m->stream);
  if (rc == CSRK_OK && (e = cudaStreamSynchronize(m->stream)) != cudaSuccess)
    return fail(e);
  if (rc != CSRK_OK) {
    release(m);
    return rc;
  }
  *out = m;
  return CSRK_OK;
}

int csrk_matrix_free(csrk_matrix *m) {
  release(m);
  return CSRK_OK;
}

int csrk_matrix_shape(const csrk_matrix *m, int64_t out[7]) {
  if (!m || !out) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  out[0] = m->n_rows;
  out[1] = m->n_cols;
  out[2] = m->nnz;
  out[3] = m->k;
  out[4] = m->n_sr;
  out[5] = m->n_ssr;
  out[6] = m->device;
  return CSRK_OK;
}

int csrk_matrix_download(const csrk_matrix *m, uint32_t *row_ptr,
                         uint32_t *col_idx, double *vals, uint32_t *sr_ptr,
                         uint32_t *ssr_ptr) {
  if (!m) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  CSRK_CUDA_TRY(cudaStreamSynchronize(m->stream));
  if (row_ptr)
    CSRK_CUDA_TRY(cudaMemcpy(row_ptr, m->row_ptr,
                             (m->n_rows + 1) * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost));
  if (col_idx && m->nnz)
    CSRK_CUDA_TRY(cudaMemcpy(col_idx, m->col_idx, m->nnz * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost));
  if (vals && m->nnz)
    CSRK_CUDA_TRY(cudaMemcpy(vals, m->vals64, m->nnz * sizeof(double),
                             cudaMemcpyDeviceToHost));
  if (sr_ptr && m->k >= 2)
    CSRK_CUDA_TRY(cudaMemcpy(sr_ptr, m->sr_ptr, (m->n_sr + 1) * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost));
  if (ssr_ptr && m->k == 3)
    CSRK_CUDA_TRY(cudaMemcpy(ssr_ptr, m->ssr_ptr,
                             (m->n_ssr + 1) * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost));
  return CSRK_OK;
}

int csrk_matrix_add_f32(csrk_matrix *m) {
  if (!m) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (m->vals32) return CSRK_OK;
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  const int64_t pn = padded_nnz(m->nnz);
  CSRK_CUDA_TRY(cudaMalloc(&m->vals32, pn * sizeof(float)));
  CSRK_CUDA_TRY(cudaMemsetAsync(m->vals32, 0, pn * sizeof(float), m->stream));
  CSRK_TRY(launch_f64_to_f32(m->vals64, m->vals32, m->nnz, m->stream));
  CSRK_CUDA_TRY(cudaStreamSynchronize(m->stream));
  return CSRK_OK;
}

int csrk_matrix_set_plan(csrk_matrix *m, int64_t tile_cost, int64_t cap,
                         int64_t stages) {
  if (!m) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  CSRK_TRY(ensure_plan(m, tile_cost, cap, stages, m->stream));
  m->plan.auto_tile = tile_cost <= 0;
  CSRK_CUDA_TRY(cudaStreamSynchronize(m->stream));
  return CSRK_OK;
}

int csrk_spmv(const csrk_matrix *m, int value_type, int variant, int nx,
              const void *x, void *y, void *stream) {
  if (!m || (m->n_rows > 0 && (!x || !y))) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  CSRK_TRY(prepare_plan(m, value_type, variant, nx));
  return launch_spmv(m, value_type, variant, nx, x, y,
                     static_cast<cudaStream_t>(stream));
}

int csrk_spmv_tiles(const csrk_matrix *m, int value_type, int variant, int nx,
                    const void *x, void *y, int64_t t0, int64_t t1, void *stream) {
  if (!m || (m->n_rows > 0 && (!x || !y))) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (t0 < 0 || t1 < t0 || t1 > m->plan.n_tiles) {
    set_error("tile range [%lld, %lld) outside 0..%lld", static_cast<long long>(t0),
              static_cast<long long>(t1), static_cast<long long>(m->plan.n_tiles));
    return CSRK_EINVAL;
  }
  if (t1 == t0) return CSRK_OK;
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  return launch_spmv(m, value_type, variant, nx, x, y, static_cast<cudaStream_t>(stream),
                     t0, t1);
}

int csrk_matrix_tile_rows(const csrk_matrix *m, uint32_t *out) {
  if (!m || !out) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (!m->plan.tile_row) {
    set_error("matrix has no tile plan");
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  CSRK_CUDA_TRY(cudaMemcpy(out, m->plan.tile_row, (m->plan.n_tiles + 1) * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost));
  return CSRK_OK;
}

// Host-buffer SpMV.  With pinned host x / y and a square matrix the copies
// and the kernel overlap: x goes up in row-aligned chunks on one stream, the
// rows of chunk c are computed on a second stream as soon as the x chunks
// covering their column footprint have landed (Band-k keeps footprints
// banded), and y chunk c goes down on a third stream -- both PCIe directions
// busy at once.  Pageable buffers take the plain H2D -> kernel -> D2H path.
// Chunk weights of the host pipeline (CSRK_PIPE_SHAPE): "uN" = N equal
// chunks; "rM" (default r12) = ramps 1, 2, 4 | M chunks of 8 | 4, 2, 1.  Small
// chunks at both ends shorten the fill (the first y chunk can go down while
// most of x is still going up) and the drain (the last kernel + D2H).
static std::vector<int> pipe_weights() {
  const char *env = std::getenv("CSRK_PIPE_SHAPE");
  std::string shape = env && *env ? env : "r12";
  int v = std::atoi(shape.c_str() + 1);
  std::vector<int> w;
  if (shape[0] == 'u' && v >= 1 && v <= 256) {
    w.assign(v, 1);
  } else {
    if (shape[0] != 'r' || v < 1 || v > 256) v = 12;
    w = {1, 2, 4};
    for (int i = 0; i < v; ++i) w.push_back(8);
    w.insert(w.end(), {4, 2, 1});
  }
  return w;
}

static int ensure_pipe(csrk_matrix *m, const std::vector<int> &weights) {
  auto &pp = m->pipe;
  const int chunks = static_cast<int>(weights.size());
  const char *xc_env = std::getenv("CSRK_PIPE_XCUT");
  const std::string xmode = xc_env ? xc_env : "";
  if (pp.weights == weights && pp.plan_tiles == m->plan.n_tiles && pp.xmode == xmode)
    return CSRK_OK;
  pp.xmode = xmode;
  const int64_t nt = m->plan.n_tiles;
  int64_t wsum = 0;
  for (int w : weights) wsum += w;
  pp.tile_cut.assign(chunks + 1, 0);
  pp.row_cut.assign(chunks + 1, 0);
  std::vector<uint32_t> rc(chunks + 1);
  int64_t wacc = 0;
  for (int c = 0; c <= chunks; ++c) {
    pp.tile_cut[c] = nt * wacc / wsum;
    if (c < chunks) wacc += weights[c];
    uint32_t r = 0;
    CSRK_CUDA_TRY(cudaMemcpy(&r, m->plan.tile_row + pp.tile_cut[c], sizeof(r),
                             cudaMemcpyDeviceToHost));
    rc[c] = r;
    pp.row_cut[c] = r;
  }
  uint32_t *d_cut = nullptr, *d_max = nullptr;
  CSRK_CUDA_TRY(cudaMalloc(&d_cut, (chunks + 1) * sizeof(uint32_t)));
  CSRK_CUDA_TRY(cudaMalloc(&d_max, chunks * sizeof(uint32_t)));
  std::vector<uint32_t> mx(chunks);
  cudaError_t e = cudaMemcpy(d_cut, rc.data(), (chunks + 1) * sizeof(uint32_t),
                             cudaMemcpyHostToDevice);
  int rc2 = e == cudaSuccess ? chunk_max_cols(m, d_cut, chunks, d_max, nullptr)
                             : CSRK_ECUDA;
  if (rc2 == CSRK_OK)
    e = cudaMemcpy(mx.data(), d_max, chunks * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  cudaFree(d_cut);
  cudaFree(d_max);
  if (rc2 != CSRK_OK) return rc2;
  CSRK_CUDA_TRY(e);
  // x chunk c ends at the column footprint of row chunk c, so kernel c
  // waits for exactly x chunks 0..c (x cut on the row cuts instead made
  // kernel c wait one or two chunks longer -- the band reaches past the cut)
  const char *xc = std::getenv("CSRK_PIPE_XCUT");
  const bool by_rows = xc && std::strcmp(xc, "rows") == 0;
  pp.x_cut.assign(chunks + 1, 0);
  pp.x_ready.assign(chunks, 0);
  for (int c = 0; c < chunks; ++c) {
    if (by_rows) {
      pp.x_cut[c + 1] = pp.row_cut[c + 1];
      int j = 0;
      while (j + 1 < chunks && pp.row_cut[j + 1] <= static_cast<int64_t>(mx[c])) ++j;
      pp.x_ready[c] = j;
    } else {
      int64_t e = std::max<int64_t>(pp.x_cut[c], static_cast<int64_t>(mx[c]) + 1);
      pp.x_cut[c + 1] = std::min<int64_t>(e, m->n_cols);
      pp.x_ready[c] = c;
    }
  }
  pp.x_cut[chunks] = m->n_cols;
  if (!pp.h2d) {
    CSRK_CUDA_TRY(cudaStreamCreateWithFlags(&pp.h2d, cudaStreamNonBlocking));
    CSRK_CUDA_TRY(cudaStreamCreateWithFlags(&pp.comp, cudaStreamNonBlocking));
    CSRK_CUDA_TRY(cudaStreamCreateWithFlags(&pp.d2h, cudaStreamNonBlocking));
  }
  for (auto ev : pp.ev_x) cudaEventDestroy(ev);
  for (auto ev : pp.ev_c) cudaEventDestroy(ev);
  pp.ev_x.assign(chunks, nullptr);
  pp.ev_c.assign(chunks, nullptr);
  for (int c = 0; c < chunks; ++c) {
    CSRK_CUDA_TRY(cudaEventCreateWithFlags(&pp.ev_x[c], cudaEventDisableTiming));
    CSRK_CUDA_TRY(cudaEventCreateWithFlags(&pp.ev_c[c], cudaEventDisableTiming));
  }
  pp.chunks = chunks;
  pp.weights = weights;
  pp.plan_tiles = nt;
  return CSRK_OK;
}

static bool is_pinned(const void *p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}


int csrk_spmv_host(csrk_matrix *m, int value_type, int variant, int nx,
                   const void *x_host, void *y_host) {
  if (!m || (m->n_rows > 0 && (!x_host || !y_host))) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  const size_t es = value_type == CSRK_F32 ? sizeof(float) : sizeof(double);
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  CSRK_TRY(prepare_plan(m, value_type, variant, nx));
  const size_t xb = static_cast<size_t>(m->n_cols) * es + 16;
  const size_t yb = static_cast<size_t>(m->n_rows) * es + 16;
  if (m->x_stage_bytes < xb) {
    cudaFree(m->x_stage);
    m->x_stage = nullptr;
    CSRK_CUDA_TRY(cudaMalloc(&m->x_stage, xb));
    m->x_stage_bytes = xb;
  }
  if (m->y_stage_bytes < yb) {
    cudaFree(m->y_stage);
    m->y_stage = nullptr;
    CSRK_CUDA_TRY(cudaMalloc(&m->y_stage, yb));
    m->y_stage_bytes = yb;
  }
  // each chunk adds a launch and three stream operations: keep the count low
  // and put the small chunks where the pipeline fills and drains
  const std::vector<int> weights = pipe_weights();
  int64_t wsum = 0;
  for (int w : weights) wsum += w;
  const int chunks = static_cast<int>(weights.size());
  const bool pipelined = m->n_rows == m->n_cols && m->n_rows >= (1 << 20) &&
                         m->plan.n_tiles >= 4 * wsum && is_pinned(x_host) &&
                         is_pinned(y_host);
  if (pipelined) {
    CSRK_TRY(ensure_pipe(m, weights));
    auto &pp = m->pipe;
    const bool trace = std::getenv("CSRK_PIPE_TRACE") != nullptr;
    std::vector<cudaEvent_t> tr;
    cudaEvent_t tr0 = nullptr;
    if (trace) {
      tr.resize(3 * chunks);
      for (auto &e : tr) cudaEventCreate(&e);
      cudaEventCreate(&tr0);
      cudaEventRecord(tr0, pp.h2d);
      pp.ev_x_t.assign(chunks, nullptr);
      pp.ev_c_t.assign(chunks, nullptr);
      for (int c = 0; c < chunks; ++c) {
        pp.ev_x_t[c] = tr[3 * c];
        pp.ev_c_t[c] = tr[3 * c + 1];
      }
    }
    char *xs = static_cast<char *>(m->x_stage);
    char *ys = static_cast<char *>(m->y_stage);
    const char *xh = static_cast<const char *>(x_host);
    char *yh = static_cast<char *>(y_host);
    // D2H ordering (CSRK_PIPE_D2H): "host" (default) enqueues y chunk c once
    // the host has seen kernel c finish; "event" makes the D2H stream wait on
    // the kernel's event.  A copy queued behind a cross-stream wait restarts
    // the copy engine late (measured: 16 ordered chunks 3.36 ms vs 3.00 ms
    // host-ordered, tools/pcie_probe.py).
    const char *d2h_mode = std::getenv("CSRK_PIPE_D2H");
    const bool host_ordered = !(d2h_mode && std::strcmp(d2h_mode, "event") == 0);
    for (int c = 0; c < chunks; ++c) {
      const size_t off = pp.x_cut[c] * es, len = (pp.x_cut[c + 1] - pp.x_cut[c]) * es;
      if (len)
        CSRK_CUDA_TRY(cudaMemcpyAsync(xs + off, xh + off, len, cudaMemcpyHostToDevice,
                                      pp.h2d));
      CSRK_CUDA_TRY(cudaEventRecord(pp.ev_x[c], pp.h2d));
      if (trace) CSRK_CUDA_TRY(cudaEventRecord(pp.ev_x_t[c], pp.h2d));
    }
    CSRK_CUDA_TRY(cudaEventRecord(m->ev0, pp.comp));
    for (int c = 0; c < chunks; ++c) {
      CSRK_CUDA_TRY(cudaStreamWaitEvent(pp.comp, pp.ev_x[pp.x_ready[c]], 0));
      CSRK_TRY(launch_spmv(m, value_type, variant, nx, m->x_stage, ys, pp.comp,
                           pp.tile_cut[c], pp.tile_cut[c + 1]));
      CSRK_CUDA_TRY(cudaEventRecord(pp.ev_c[c], pp.comp));
      if (trace) CSRK_CUDA_TRY(cudaEventRecord(pp.ev_c_t[c], pp.comp));
      if (host_ordered) continue;
      const size_t off = pp.row_cut[c] * es, len = (pp.row_cut[c + 1] - pp.row_cut[c]) * es;
      CSRK_CUDA_TRY(cudaStreamWaitEvent(pp.d2h, pp.ev_c[c], 0));
      if (len)
        CSRK_CUDA_TRY(cudaMemcpyAsync(yh + off, ys + off, len, cudaMemcpyDeviceToHost,
                                      pp.d2h));
    }
    if (host_ordered) {
      for (int c = 0; c < chunks; ++c) {
        const size_t off = pp.row_cut[c] * es,
                     len = (pp.row_cut[c + 1] - pp.row_cut[c]) * es;
        CSRK_CUDA_TRY(cudaEventSynchronize(pp.ev_c[c]));
        if (len)
          CSRK_CUDA_TRY(cudaMemcpyAsync(yh + off, ys + off, len, cudaMemcpyDeviceToHost,
                                        pp.d2h));
      }
    }
    CSRK_CUDA_TRY(cudaEventRecord(m->ev1, pp.comp));
    if (trace) {
      for (int c = 0; c < chunks; ++c) {
        CSRK_CUDA_TRY(cudaEventRecord(tr[3 * c + 2], pp.d2h));
      }
    }
    CSRK_CUDA_TRY(cudaStreamSynchronize(pp.d2h));
    CSRK_CUDA_TRY(cudaStreamSynchronize(pp.comp));
    if (trace) {
      // CSRK_PIPE_TRACE=1: per-chunk completion times (ms after the first
      // H2D was enqueued) of H2D / kernel, and the D2H stream's end
      float t_end = 0.f;
      cudaEventElapsedTime(&t_end, tr0, tr[3 * (chunks - 1) + 2]);
      for (int c = 0; c < chunks; ++c) {
        float th = 0.f, tk = 0.f;
        cudaEventElapsedTime(&th, tr0, pp.ev_x_t[c]);
        cudaEventElapsedTime(&tk, tr0, pp.ev_c_t[c]);
        std::fprintf(stderr,
                     "[pipe] chunk %2d rows %9lld x %9lld x_ready %2d  h2d %.3f  kernel %.3f\n",
                     c, static_cast<long long>(pp.row_cut[c + 1] - pp.row_cut[c]),
                     static_cast<long long>(pp.x_cut[c + 1] - pp.x_cut[c]), pp.x_ready[c],
                     th, tk);
      }
      std::fprintf(stderr, "[pipe] d2h (%s-ordered) done %.3f ms\n",
                   host_ordered ? "host" : "event", t_end);
      for (auto e : tr) cudaEventDestroy(e);
      cudaEventDestroy(tr0);
    }
    return CSRK_OK;
  }
  if (m->n_cols)
    CSRK_CUDA_TRY(cudaMemcpyAsync(m->x_stage, x_host, m->n_cols * es,
                                  cudaMemcpyHostToDevice, m->stream));
  CSRK_CUDA_TRY(cudaEventRecord(m->ev0, m->stream));
  CSRK_TRY(launch_spmv(m, value_type, variant, nx, m->x_stage, m->y_stage,
                       m->stream));
  CSRK_CUDA_TRY(cudaEventRecord(m->ev1, m->stream));
  if (m->n_rows)
    CSRK_CUDA_TRY(cudaMemcpyAsync(y_host, m->y_stage, m->n_rows * es,
                                  cudaMemcpyDeviceToHost, m->stream));
  CSRK_CUDA_TRY(cudaStreamSynchronize(m->stream));
  return CSRK_OK;
}

int csrk_matrix_plan(const csrk_matrix *m, int64_t out[10]) {
  if (!m || !out) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  out[0] = m->plan.tile_cost;
  out[1] = m->plan.cap;
  out[2] = m->plan.rcap;
  out[3] = m->plan.stages;
  out[4] = m->plan.n_tiles;
  out[5] = m->plan.group_aligned ? 1 : 0;
  out[6] = m->plan.gather_first;
  out[7] = m->plan.ctas_per_sm ? m->plan.ctas_per_sm : auto_ctas(m->plan.row_var, 8, m->plan.n_long, m->plan.mean_short);
  out[8] = m->plan.cut_mode;
  out[9] = m->plan.n_long;
  return CSRK_OK;
}

int csrk_matrix_plan_ctas(const csrk_matrix *m, int value_type, int64_t *ctas) {
  if (!m || !ctas || (value_type != CSRK_F64 && value_type != CSRK_F32)) {
    set_error("invalid argument to csrk_matrix_plan_ctas");
    return CSRK_EINVAL;
  }
  *ctas = m->plan.ctas_per_sm ? m->plan.ctas_per_sm
                              : auto_ctas(m->plan.row_var, value_type == CSRK_F32 ? 4 : 8,
                                          m->plan.n_long, m->plan.mean_short);
  return CSRK_OK;
}

int csrk_matrix_set_cut_mode(csrk_matrix *m, int mode) {
  if (!m) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (mode < 0 || mode > 2) {
    set_error("cut mode must be 0 (auto), 1 (rows) or 2 (groups), got %d", mode);
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  if (mode == m->plan.cut_mode) return CSRK_OK;
  m->plan.cut_mode = mode;
  if (m->n_rows == 0) return CSRK_OK;
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  // rebuild the current plan with the new cuts
  const bool keep = m->plan.auto_tile;
  CSRK_TRY(ensure_plan(m, m->plan.tile_cost, m->plan.cap, m->plan.stages, m->stream, true));
  m->plan.auto_tile = keep;
  CSRK_CUDA_TRY(cudaStreamSynchronize(m->stream));
  return CSRK_OK;
}

int csrk_matrix_prepare(csrk_matrix *m, int value_type, int variant, int nx) {
  if (!m) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (variant != CSRK_SERIAL && variant != CSRK_STRIDED) {
    set_error("unknown SpMV variant %d", variant);
    return CSRK_EINVAL;
  }
  if (value_type != CSRK_F64 && value_type != CSRK_F32) {
    set_error("unknown value type %d", value_type);
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  CSRK_TRY(prepare_plan(m, value_type, variant, nx));
  CSRK_CUDA_TRY(cudaStreamSynchronize(m->stream));
  return CSRK_OK;
}

int csrk_matrix_set_schedule(csrk_matrix *m, int gather, int ctas_per_sm) {
  if (!m) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (gather < 0 || gather > 2) {
    set_error("gather mode must be 0 (inline), 1 (gather-first) or 2 (auto), got %d",
              gather);
    return CSRK_EINVAL;
  }
  if (ctas_per_sm < 0 || ctas_per_sm > 8) {
    set_error("ctas_per_sm must be in 0..8, got %d", ctas_per_sm);
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  m->plan.gather_first = gather;
  m->plan.ctas_per_sm = ctas_per_sm;
  return CSRK_OK;
}

int csrk_last_kernel_ms(const csrk_matrix *m, float *ms) {
  if (!m || !ms) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  CSRK_CUDA_TRY(cudaEventElapsedTime(ms, m->ev0, m->ev1));
  return CSRK_OK;
}

int csrk_spmv_listing3(const csrk_matrix *m, int dx, int dy, const double *x,
                       double *y, int64_t *trace, void *stream) {
  if (!m) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (m->k != 3) {
    set_error("emulate_gpu_spmv3 requires k = 3");
    return CSRK_EINVAL;
  }
  if (dx < 1 || dy < 1 || dx * dy > 1024) {
    set_error("block holds %d threads, limit is 1024", dx * dy);
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  return launch_listing3(m, dx, dy, x, y, trace,
                         static_cast<cudaStream_t>(stream));
}

int csrk_spmv_listing4(const csrk_matrix *m, int dx, int dy, int dz,
                       const double *x, double *y, int64_t *trace,
                       void *stream) {
  if (!m) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (m->k != 3) {
    set_error("emulate_gpu_spmv35 requires k = 3");
    return CSRK_EINVAL;
  }
  if (dx < 1 || dy < 1 || dz < 1 || dx * dy * dz > 1024) {
    set_error("block holds %d threads, limit is 1024", dx * dy * dz);
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  return launch_listing4(m, dx, dy, dz, x, y, trace,
                         static_cast<cudaStream_t>(stream));
}

int csrk_probe_gather(const csrk_matrix *m, int mode, const double *x, double *out,
                      void *stream) {
  if (!m || !out || (mode != 0 && !x)) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (mode != 0 && mode != 1) {
    set_error("probe mode must be 0 (col_idx only) or 1 (col_idx + x gathers)");
    return CSRK_EINVAL;
  }
  CSRK_LOCK(m);
  CSRK_CUDA_TRY(cudaSetDevice(m->device));
  return launch_gather_probe(m, mode, x, out, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
