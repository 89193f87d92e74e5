// Multi-GPU row-block CSR-k SpMV behind the C-ABI (SURVEY.md §8(b)
// "csrk_mg_create / csrk_mg_spmv", §8(e)).  One process per GPU; rank g
// owns the rows [cuts[g], cuts[g+1]) of the packed matrix -- whole
// super-super-rows balanced by nonzeros, the reference's static chunks
// (kernels.py:150-155) with nonzero weights -- as a csrk_matrix whose
// columns are local to its footprint window x_local = x[x0, x1).
//
// One csrk_mg_spmv:
//   comm stream: wait for the caller's stream, then the halo exchange --
//     ncclSend / ncclRecv of exactly the windows each rank's rows read from
//     each peer (halo) or the literal north-star all-gather of every owned
//     slice (padded to the largest) followed by window copies;
//   caller stream: the interior tiles (rows that read owned columns only)
//     while the exchange is in flight, then -- after the comm stream's
//     event -- the boundary tiles before and after them.
// y_own is bitwise the single-GPU y: rows are summed whole by the same
// kernel in the same order, only the launch is split.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": torch's bundled copy
// when the process already has it, else the system library), so the library
// itself has no link-time NCCL dependency and the single-GPU entry points
// work without it.  The host planning functions (partition, footprints,
// transfer plan) need no GPU and are tested against dist.py on CPU.

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"

namespace csrk {
namespace {

struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
  std::string why;
};

const Nccl &nccl() {
  static const Nccl lib = [] {
    Nccl n;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char *e = dlerror();
      n.why = e ? e : "libnccl.so.2 not found";
      return n;
    }
#define CSRK_NCCL_SYM(field, name)                                  \
  n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name));    \
  if (!n.field) {                                                   \
    n.why = std::string("libnccl lacks ") + name;                   \
    return n;                                                       \
  }
    CSRK_NCCL_SYM(get_unique_id, "ncclGetUniqueId")
    CSRK_NCCL_SYM(comm_init_rank, "ncclCommInitRank")
    CSRK_NCCL_SYM(comm_destroy, "ncclCommDestroy")
    CSRK_NCCL_SYM(send, "ncclSend")
    CSRK_NCCL_SYM(recv, "ncclRecv")
    CSRK_NCCL_SYM(all_gather, "ncclAllGather")
    CSRK_NCCL_SYM(group_start, "ncclGroupStart")
    CSRK_NCCL_SYM(group_end, "ncclGroupEnd")
    CSRK_NCCL_SYM(error_string, "ncclGetErrorString")
#undef CSRK_NCCL_SYM
    n.ok = true;
    return n;
  }();
  return lib;
}

#define CSRK_NCCL_TRY(expr)                                                       \
  do {                                                                            \
    ncclResult_t r_ = (expr);                                                     \
    if (r_ != ncclSuccess) {                                                      \
      csrk::set_error("NCCL error %d at %s:%d: %s", static_cast<int>(r_), __FILE__, \
                      __LINE__, csrk::nccl().error_string(r_));                   \
      return CSRK_ENCCL;                                                          \
    }                                                                             \
  } while (0)

// largest row r with a nonzero whose first column < own0, and smallest row
// with last column >= own1 (rows are column-sorted, so first / last entries
// are the extremes): interior rows are (lo_bad, hi_bad)
__global__ void boundary_rows_kernel(const uint32_t *__restrict__ row_ptr,
                                     const uint32_t *__restrict__ col_idx, int64_t n_rows,
                                     uint32_t own0, uint32_t own1,
                                     unsigned long long *lo_bad,   // max r + 1, 0 = none
                                     unsigned long long *hi_bad) {  // min r, n = none
  unsigned long long lo = 0, hi = static_cast<unsigned long long>(n_rows);
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = row_ptr[r], e = row_ptr[r + 1];
    if (e == s) continue;
    if (col_idx[s] < own0) lo = static_cast<unsigned long long>(r) + 1;
    if (col_idx[e - 1] >= own1 && static_cast<unsigned long long>(r) < hi)
      hi = static_cast<unsigned long long>(r);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = max(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = min(hi, __shfl_down_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(lo_bad, lo);
    atomicMin(hi_bad, hi);
  }
}

struct Transfer {
  int peer;
  int64_t lo, hi;  // global columns
};

}  // namespace
}  // namespace csrk

struct csrk_mg {
  int rank = 0, world = 1, device = 0, mode = CSRK_MG_HALO;
  csrk_matrix *block = nullptr;  // borrowed
  ncclComm_t comm = nullptr;
  std::vector<int64_t> cuts;     // world + 1 global row cuts
  int64_t x0 = 0, n_local_cols = 0;
  std::vector<csrk::Transfer> sends, recvs;
  int64_t interior_a = 0, interior_b = 0;  // local rows
  int64_t t_lo = 0, t_hi = 0, n_tiles = -1;
  uint64_t plan_gen = ~0ull;
  int64_t maxlen = 0;           // largest owned slice (all-gather padding)
  void *mine = nullptr, *every = nullptr;  // all-gather buffers
  size_t ag_elem = 0;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_go = nullptr, ev_done = nullptr;
  std::mutex mu;
};

namespace csrk {
namespace {

// interior tile range of the block's current plan: tiles whose rows all lie
// in [a, b) (dist.interior_tiles)
int refresh_tiles(csrk_mg *h) {
  csrk_matrix *m = h->block;
  if (!m || m->n_rows == 0) {
    h->t_lo = h->t_hi = h->n_tiles = 0;
    return CSRK_OK;
  }
  if (h->n_tiles == m->plan.n_tiles && h->plan_gen == m->plan.gen) return CSRK_OK;
  const int64_t nt = m->plan.n_tiles;
  std::vector<uint32_t> tr(static_cast<size_t>(nt + 1));
  CSRK_CUDA_TRY(cudaMemcpy(tr.data(), m->plan.tile_row, (nt + 1) * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost));
  const int64_t a = h->interior_a, b = h->interior_b;
  const int64_t t_lo = std::lower_bound(tr.begin(), tr.end(), static_cast<uint32_t>(a)) - tr.begin();
  const int64_t t_hi = (std::upper_bound(tr.begin(), tr.end(), static_cast<uint32_t>(b)) - tr.begin()) - 1;
  h->t_lo = t_lo;
  h->t_hi = std::max(t_lo, t_hi);
  h->n_tiles = nt;
  h->plan_gen = m->plan.gen;
  return CSRK_OK;
}

ncclDataType_t nccl_type(int value_type) {
  return value_type == CSRK_F32 ? ncclFloat32 : ncclFloat64;
}

}  // namespace
}  // namespace csrk

using namespace csrk;

extern "C" {

int csrk_mg_partition(const uint32_t *row_ptr, const uint32_t *sr_ptr, const uint32_t *ssr_ptr,
                      int64_t n_ssr, int parts, int64_t *cuts) {
  if (!row_ptr || !sr_ptr || !ssr_ptr || !cuts || n_ssr < 0) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (parts < 1) {
    set_error("parts must be >= 1, got %d", parts);
    return CSRK_EINVAL;
  }
  // nonzero offset at every SSR start (and the end), like dist.partition_by_nnz
  auto ssr_row = [&](int64_t s) { return static_cast<int64_t>(sr_ptr[ssr_ptr[s]]); };
  auto nnz_at = [&](int64_t s) { return static_cast<int64_t>(row_ptr[ssr_row(s)]); };
  const int64_t total = static_cast<int64_t>(row_ptr[ssr_row(n_ssr)]);
  cuts[0] = 0;
  for (int g = 1; g < parts; ++g) {
    const int64_t target = (total * g + parts - 1) / parts;
    int64_t lo = 0, hi = n_ssr + 1;  // first s with nnz_at(s) >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (nnz_at(mid) >= target)
        hi = mid;
      else
        lo = mid + 1;
    }
    cuts[g] = ssr_row(std::min(lo, n_ssr));
  }
  cuts[parts] = ssr_row(n_ssr);
  for (int g = 1; g <= parts; ++g) cuts[g] = std::max(cuts[g], cuts[g - 1]);
  return CSRK_OK;
}

int csrk_mg_footprints(const uint32_t *row_ptr, const uint32_t *col_idx, const int64_t *cuts,
                       int parts, int64_t *fps) {
  if (!row_ptr || !cuts || !fps || (parts > 0 && !col_idx && row_ptr[cuts[parts]] > 0)) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  for (int g = 0; g < parts; ++g) {
    const int64_t a = row_ptr[cuts[g]], b = row_ptr[cuts[g + 1]];
    if (b > a) {
      uint32_t lo = col_idx[a], hi = col_idx[a];
      for (int64_t p = a; p < b; ++p) {
        lo = std::min(lo, col_idx[p]);
        hi = std::max(hi, col_idx[p]);
      }
      fps[2 * g] = lo;
      fps[2 * g + 1] = static_cast<int64_t>(hi) + 1;
    } else {
      fps[2 * g] = fps[2 * g + 1] = cuts[g];
    }
  }
  return CSRK_OK;
}

int csrk_mg_plan(int world, const int64_t *cuts, const int64_t *fps, int64_t *out,
                 int64_t cap, int64_t *count) {
  if (!cuts || !fps || !count || (cap > 0 && !out)) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  int64_t n = 0;
  for (int dst = 0; dst < world; ++dst) {
    const int64_t lo = fps[2 * dst], hi = fps[2 * dst + 1];
    for (int src = 0; src < world; ++src) {
      if (src == dst) continue;
      const int64_t a = std::max(lo, cuts[src]), b = std::min(hi, cuts[src + 1]);
      if (b > a) {
        if (n < cap) {
          out[4 * n] = src;
          out[4 * n + 1] = dst;
          out[4 * n + 2] = a;
          out[4 * n + 3] = b;
        }
        ++n;
      }
    }
  }
  *count = n;
  return CSRK_OK;
}

int csrk_mg_unique_id(unsigned char *id) {
  if (!id) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  const Nccl &n = nccl();
  if (!n.ok) {
    set_error("NCCL unavailable: %s", n.why.c_str());
    return CSRK_ENCCL;
  }
  ncclUniqueId u;
  CSRK_NCCL_TRY(n.get_unique_id(&u));
  static_assert(sizeof(u) == CSRK_MG_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id, &u, sizeof(u));
  return CSRK_OK;
}

int csrk_mg_create(int rank, int world, const unsigned char *id, const int64_t *cuts,
                   const int64_t *fps, csrk_matrix *block, int64_t x0, int mode,
                   csrk_mg **out) {
  if (!cuts || !fps || !out) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (world < 1 || rank < 0 || rank >= world) {
    set_error("rank %d outside world %d", rank, world);
    return CSRK_EINVAL;
  }
  if (mode != CSRK_MG_HALO && mode != CSRK_MG_ALLGATHER) {
    set_error("unknown exchange mode %d", mode);
    return CSRK_EINVAL;
  }
  const int64_t r0 = cuts[rank], r1 = cuts[rank + 1];
  if (block && block->n_rows != r1 - r0) {
    set_error("block holds %lld rows, the cuts give rank %d %lld",
              static_cast<long long>(block->n_rows), rank, static_cast<long long>(r1 - r0));
    return CSRK_EINVAL;
  }
  if (!block && r1 > r0) {
    set_error("rank %d owns rows but has no block", rank);
    return CSRK_EINVAL;
  }
  const Nccl &n = nccl();
  if (id && !n.ok) {
    set_error("NCCL unavailable: %s", n.why.c_str());
    return CSRK_ENCCL;
  }
  int dev = 0;
  CSRK_CUDA_TRY(cudaGetDevice(&dev));
  if (block) {
    dev = block->device;
    CSRK_CUDA_TRY(cudaSetDevice(dev));
  }
  auto h = new csrk_mg();
  h->rank = rank;
  h->world = world;
  h->device = dev;
  h->mode = mode;
  h->block = block;
  h->cuts.assign(cuts, cuts + world + 1);
  h->x0 = x0;
  h->n_local_cols = block ? block->n_cols : 0;
  for (int g = 0; g < world; ++g) h->maxlen = std::max(h->maxlen, cuts[g + 1] - cuts[g]);
  // the transfer plan (dist.halo_plan): dst needs x[lo, hi) owned by src
  for (int dst = 0; dst < world; ++dst) {
    const int64_t lo = fps[2 * dst], hi = fps[2 * dst + 1];
    for (int src = 0; src < world; ++src) {
      if (src == dst) continue;
      const int64_t a = std::max(lo, cuts[src]), b = std::min(hi, cuts[src + 1]);
      if (b <= a) continue;
      if (src == rank) h->sends.push_back({dst, a, b});
      if (dst == rank) h->recvs.push_back({src, a, b});
    }
  }
  for (const auto &t : h->recvs)
    if (t.lo < x0 || t.hi > x0 + h->n_local_cols) {
      set_error("halo window [%lld, %lld) outside the block's x window [%lld, %lld)",
                static_cast<long long>(t.lo), static_cast<long long>(t.hi),
                static_cast<long long>(x0), static_cast<long long>(x0 + h->n_local_cols));
      delete h;
      return CSRK_EINVAL;
    }
  int rc = CSRK_OK;
  do {
    if (block && block->n_rows > 0) {
      // interior rows: read owned columns only
      unsigned long long *d = nullptr;
      unsigned long long hv[2] = {0, static_cast<unsigned long long>(block->n_rows)};
      if (cudaMalloc(&d, 2 * sizeof(unsigned long long)) != cudaSuccess) {
        set_error("cudaMalloc failed");
        rc = CSRK_ENOMEM;
        break;
      }
      cudaMemcpy(d, hv, sizeof(hv), cudaMemcpyHostToDevice);
      const int64_t own0 = r0 - x0, own1 = r1 - x0;
      boundary_rows_kernel<<<148 * 4, 256>>>(block->row_ptr, block->col_idx, block->n_rows,
                                             static_cast<uint32_t>(std::max<int64_t>(own0, 0)),
                                             static_cast<uint32_t>(std::max<int64_t>(own1, 0)),
                                             d, d + 1);
      const cudaError_t e = cudaMemcpy(hv, d, sizeof(hv), cudaMemcpyDeviceToHost);
      cudaFree(d);
      if (e != cudaSuccess) {
        set_error("CUDA error %s in the boundary-row scan", cudaGetErrorName(e));
        rc = CSRK_ECUDA;
        break;
      }
      h->interior_a = static_cast<int64_t>(hv[0]);
      h->interior_b = std::max(h->interior_a, static_cast<int64_t>(hv[1]));
    }
    if (cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_go, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming) != cudaSuccess) {
      set_error("stream / event creation failed");
      rc = CSRK_ECUDA;
      break;
    }
    if (!id) break;  // no communicator: the caller exchanges the halo itself
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    const ncclResult_t r = n.comm_init_rank(&h->comm, world, u, rank);
    if (r != ncclSuccess) {
      set_error("NCCL error %d in ncclCommInitRank: %s", static_cast<int>(r), n.error_string(r));
      rc = CSRK_ENCCL;
      break;
    }
  } while (false);
  if (rc != CSRK_OK) {
    csrk_mg_destroy(h);
    return rc;
  }
  *out = h;
  return CSRK_OK;
}

int csrk_mg_spmv(csrk_mg *h, int value_type, int variant, int nx, void *x_local,
                 void *y_own, void *stream) {
  if (!h || (h->block && h->block->n_rows > 0 && (!x_local || !y_own))) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  if (value_type != CSRK_F64 && value_type != CSRK_F32) {
    set_error("unknown value type %d", value_type);
    return CSRK_EINVAL;
  }
  std::lock_guard<std::mutex> lk(h->mu);
  CSRK_CUDA_TRY(cudaSetDevice(h->device));
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Nccl &n = nccl();
  const size_t es = value_type == CSRK_F32 ? 4 : 8;
  csrk_matrix *m = h->block;
  if (m && m->n_rows > 0) {
    std::lock_guard<std::mutex> ml(m->mu);
    CSRK_TRY(prepare_plan(m, value_type, variant, nx));
    CSRK_TRY(refresh_tiles(h));
  }
  unsigned char *xl = static_cast<unsigned char *>(x_local);
  // 1. the exchange on the comm stream, after the caller's writes of x
  const bool exchange = h->comm && h->world > 1 && (!h->sends.empty() || !h->recvs.empty() ||
                                         h->mode == CSRK_MG_ALLGATHER);
  if (exchange) {
    CSRK_CUDA_TRY(cudaEventRecord(h->ev_go, s));
    CSRK_CUDA_TRY(cudaStreamWaitEvent(h->comm_stream, h->ev_go, 0));
    if (h->mode == CSRK_MG_HALO) {
      CSRK_NCCL_TRY(n.group_start());
      for (const auto &t : h->sends)
        CSRK_NCCL_TRY(n.send(xl + (t.lo - h->x0) * es, static_cast<size_t>(t.hi - t.lo),
                             nccl_type(value_type), t.peer, h->comm, h->comm_stream));
      for (const auto &t : h->recvs)
        CSRK_NCCL_TRY(n.recv(xl + (t.lo - h->x0) * es, static_cast<size_t>(t.hi - t.lo),
                             nccl_type(value_type), t.peer, h->comm, h->comm_stream));
      CSRK_NCCL_TRY(n.group_end());
    } else {
      if (h->ag_elem != es) {
        if (h->mine) cudaFree(h->mine);
        if (h->every) cudaFree(h->every);
        h->mine = h->every = nullptr;
        CSRK_CUDA_TRY(cudaMalloc(&h->mine, std::max<int64_t>(h->maxlen, 1) * es));
        CSRK_CUDA_TRY(cudaMalloc(&h->every, std::max<int64_t>(h->maxlen, 1) * es * h->world));
        CSRK_CUDA_TRY(cudaMemsetAsync(h->mine, 0, std::max<int64_t>(h->maxlen, 1) * es,
                                      h->comm_stream));
        h->ag_elem = es;
      }
      const int64_t lo = h->cuts[h->rank], hi = h->cuts[h->rank + 1];
      if (hi > lo)
        CSRK_CUDA_TRY(cudaMemcpyAsync(h->mine, xl + (lo - h->x0) * es, (hi - lo) * es,
                                      cudaMemcpyDeviceToDevice, h->comm_stream));
      CSRK_NCCL_TRY(n.all_gather(h->mine, h->every, static_cast<size_t>(h->maxlen),
                                 nccl_type(value_type), h->comm, h->comm_stream));
      for (const auto &t : h->recvs) {
        const int64_t off = t.peer * h->maxlen + (t.lo - h->cuts[t.peer]);
        CSRK_CUDA_TRY(cudaMemcpyAsync(xl + (t.lo - h->x0) * es,
                                      static_cast<unsigned char *>(h->every) + off * es,
                                      (t.hi - t.lo) * es, cudaMemcpyDeviceToDevice,
                                      h->comm_stream));
      }
    }
    CSRK_CUDA_TRY(cudaEventRecord(h->ev_done, h->comm_stream));
  }
  if (!m || m->n_rows == 0) {
    if (exchange) CSRK_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_done, 0));
    return CSRK_OK;
  }
  std::lock_guard<std::mutex> ml(m->mu);
  // 2. interior tiles while the halo is in flight
  if (h->t_hi > h->t_lo)
    CSRK_TRY(launch_spmv(m, value_type, variant, nx, x_local, y_own, s, h->t_lo, h->t_hi));
  // 3. boundary tiles after it
  if (exchange) CSRK_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_done, 0));
  if (h->t_lo > 0)
    CSRK_TRY(launch_spmv(m, value_type, variant, nx, x_local, y_own, s, 0, h->t_lo));
  if (h->t_hi < h->n_tiles)
    CSRK_TRY(launch_spmv(m, value_type, variant, nx, x_local, y_own, s, h->t_hi, h->n_tiles));
  return CSRK_OK;
}

int csrk_mg_info(const csrk_mg *h, int64_t *out) {
  if (!h || !out) {
    set_error("null argument");
    return CSRK_EINVAL;
  }
  int64_t sent = 0, recv = 0;
  for (const auto &t : h->sends) sent += t.hi - t.lo;
  for (const auto &t : h->recvs) recv += t.hi - t.lo;
  if (h->mode == CSRK_MG_ALLGATHER && h->world > 1) {
    sent = h->maxlen;
    recv = (h->world - 1) * h->maxlen;
  }
  out[0] = h->interior_a;
  out[1] = h->interior_b;
  out[2] = h->t_lo;
  out[3] = h->t_hi;
  out[4] = h->n_tiles;
  out[5] = sent;
  out[6] = recv;
  out[7] = static_cast<int64_t>(h->sends.size());
  out[8] = static_cast<int64_t>(h->recvs.size());
  return CSRK_OK;
}

int csrk_mg_destroy(csrk_mg *h) {
  if (!h) return CSRK_OK;
  cudaSetDevice(h->device);
  if (h->comm_stream) cudaStreamSynchronize(h->comm_stream);
  if (h->comm && nccl().ok) nccl().comm_destroy(h->comm);
  if (h->mine) cudaFree(h->mine);
  if (h->every) cudaFree(h->every);
  if (h->ev_go) cudaEventDestroy(h->ev_go);
  if (h->ev_done) cudaEventDestroy(h->ev_done);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  delete h;
  return CSRK_OK;
}

}  // extern "C"
