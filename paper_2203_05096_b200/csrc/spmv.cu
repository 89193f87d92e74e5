// CSR-k streaming SpMV for sm_100a -- the hot path.
//
// Bitwise contract: every reference kernel sums a row
// strictly left to right with the multiply and the add rounded separately
// (reference kernels.py:117-147, 224-228), so products and sums use
// __dmul_rn / __dadd_rn, which are never contracted into DFMA.  The STRIDED
// order reproduces emulate_gpu_spmv35 (kernels.py:284-324): nonzero p of a
// row feeds lane p mod nx, each lane sums serially from 0.0, and the lanes
// are combined by the zero-padded halving tree of _tree_reduce
// (kernels.py:268-281), here a __shfl_down_sync tree.
//
// Design (B200):
//   * tiles: contiguous row ranges balanced by cost = nonzeros + rows (merge
//     path).  When every group (super-super-row for k=3, super-row for k=2)
//     is small against the tile, tile cuts fall only on group boundaries, so
//     a CTA always owns whole super-super-rows (the paper's block <-> SSR
//     mapping, Listing 3, coarsened to a B200-sized unit of work);
//   * persistent, warp-specialised CTAs: warp 0 is the producer and moves
//     each tile's vals / col_idx / row_ptr spans HBM -> shared memory with
//     TMA bulk copies (cp.async.bulk + mbarrier complete_tx, L2 evict-first
//     so the streamed matrix does not push x out of L2) into an S-stage ring;
//     warps 1..8 consume: rows to threads (SERIAL) or to nx-lane sub-warps
//     (STRIDED), x gathered through the read-only path, y stored coalesced,
//     and release the stage through an `empty` mbarrier;
//   * a tile that does not fit a stage (a very long row) is computed from
//     global memory by the consumers ("direct" mode).

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace csrk {
namespace {

#ifndef CSRK_PRED_LDS
#define CSRK_PRED_LDS 1
#endif
constexpr bool kPredLds = CSRK_PRED_LDS != 0;
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kThreads = kConsumers + 32;
constexpr uint32_t kStaged = 0, kDirect = 1;

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  // make initialised barriers visible to the async (TMA) proxy
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

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar))
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

__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// bulk prefetch of [src, src + bytes) into L2 (src, bytes 16-byte aligned)
__device__ __forceinline__ void l2_prefetch_bulk(const void *src, uint32_t bytes,
                                                 uint64_t policy) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src),
               "r"(bytes), "l"(policy)
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

// x[c] through the read-only path with a 32-bit index: one IMAD.WIDE.U32
// for the address (the plain x + c of a predicated-loaded index compiled to
// a zeroed 64-bit pair, LEA and LEA.HI.X per gather)
#ifndef CSRK_LDG_ASM
#define CSRK_LDG_ASM 1
#endif
__device__ __forceinline__ double ldg_x(const double *x, uint32_t c) {
  if (!CSRK_LDG_ASM) return __ldg(x + c);
  double v;
  asm("{\n\t.reg .u64 a;\n\tmul.wide.u32 a, %1, 8;\n\tadd.u64 a, a, %2;\n\t"
      "ld.global.nc.f64 %0, [a];\n\t}"
      : "=d"(v)
      : "r"(c), "l"(x));
  return v;
}
__device__ __forceinline__ float ldg_x(const float *x, uint32_t c) {
  if (!CSRK_LDG_ASM) return __ldg(x + c);
  float v;
  asm("{\n\t.reg .u64 a;\n\tmul.wide.u32 a, %1, 4;\n\tadd.u64 a, a, %2;\n\t"
      "ld.global.nc.f32 %0, [a];\n\t}"
      : "=f"(v)
      : "r"(c), "l"(x));
  return v;
}

// x gathers of one batch: slot j loads x[c[j]] when j < cnt (the lanes past
// the row end issue no load -- each cost an extra 128-byte line of the
// L1TEX data pipe, x[0], per load instruction: ~9 % of C5's gather
// wavefronts).  One asm block per batch, so all of its loads are issued
// back to back, each into its own register (predicating them in C++ let
// ptxas split the batch and serialise the loads).  Batches of other sizes
// use the per-slot form.
#ifndef CSRK_PRED_LDG
#define CSRK_PRED_LDG 1
#endif
template <int B, typename V>
__device__ __forceinline__ void gather_batch(const V *x, const uint32_t (&c)[B], uint32_t cnt,
                                             V (&xv)[B]) {
#pragma unroll
  for (int j = 0; j < B; ++j) xv[j] = ldg_x(x, static_cast<uint32_t>(j) < cnt ? c[j] : 0u);
}
template <>
__device__ __forceinline__ void gather_batch<8, double>(
    const double *x, const uint32_t (&c)[8], uint32_t cnt, double (&xv)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) xv[j] = 0.0;
  asm("{\n\t.reg .pred q<8>;\n\t.reg .u64 a<8>;\n\t"
      "setp.gt.u32 q0, %17, 0;\n\t"
      "setp.gt.u32 q1, %17, 1;\n\t"
      "setp.gt.u32 q2, %17, 2;\n\t"
      "setp.gt.u32 q3, %17, 3;\n\t"
      "setp.gt.u32 q4, %17, 4;\n\t"
      "setp.gt.u32 q5, %17, 5;\n\t"
      "setp.gt.u32 q6, %17, 6;\n\t"
      "setp.gt.u32 q7, %17, 7;\n\t"
      "mul.wide.u32 a0, %8, 8;\n\tadd.u64 a0, a0, %16;\n\t"
      "mul.wide.u32 a1, %9, 8;\n\tadd.u64 a1, a1, %16;\n\t"
      "mul.wide.u32 a2, %10, 8;\n\tadd.u64 a2, a2, %16;\n\t"
      "mul.wide.u32 a3, %11, 8;\n\tadd.u64 a3, a3, %16;\n\t"
      "mul.wide.u32 a4, %12, 8;\n\tadd.u64 a4, a4, %16;\n\t"
      "mul.wide.u32 a5, %13, 8;\n\tadd.u64 a5, a5, %16;\n\t"
      "mul.wide.u32 a6, %14, 8;\n\tadd.u64 a6, a6, %16;\n\t"
      "mul.wide.u32 a7, %15, 8;\n\tadd.u64 a7, a7, %16;\n\t"
      "@q0 ld.global.nc.f64 %0, [a0];\n\t"
      "@q1 ld.global.nc.f64 %1, [a1];\n\t"
      "@q2 ld.global.nc.f64 %2, [a2];\n\t"
      "@q3 ld.global.nc.f64 %3, [a3];\n\t"
      "@q4 ld.global.nc.f64 %4, [a4];\n\t"
      "@q5 ld.global.nc.f64 %5, [a5];\n\t"
      "@q6 ld.global.nc.f64 %6, [a6];\n\t"
      "@q7 ld.global.nc.f64 %7, [a7];\n\t"
      "}"
      : "+d"(xv[0]), "+d"(xv[1]), "+d"(xv[2]), "+d"(xv[3]), "+d"(xv[4]), "+d"(xv[5]),
        "+d"(xv[6]), "+d"(xv[7])
      : "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(c[5]), "r"(c[6]), "r"(c[7]),
        "l"(x), "r"(cnt));
}
template <>
__device__ __forceinline__ void gather_batch<8, float>(
    const float *x, const uint32_t (&c)[8], uint32_t cnt, float (&xv)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) xv[j] = 0.0f;
  asm("{\n\t.reg .pred q<8>;\n\t.reg .u64 a<8>;\n\t"
      "setp.gt.u32 q0, %17, 0;\n\t"
      "setp.gt.u32 q1, %17, 1;\n\t"
      "setp.gt.u32 q2, %17, 2;\n\t"
      "setp.gt.u32 q3, %17, 3;\n\t"
      "setp.gt.u32 q4, %17, 4;\n\t"
      "setp.gt.u32 q5, %17, 5;\n\t"
      "setp.gt.u32 q6, %17, 6;\n\t"
      "setp.gt.u32 q7, %17, 7;\n\t"
      "mul.wide.u32 a0, %8, 4;\n\tadd.u64 a0, a0, %16;\n\t"
      "mul.wide.u32 a1, %9, 4;\n\tadd.u64 a1, a1, %16;\n\t"
      "mul.wide.u32 a2, %10, 4;\n\tadd.u64 a2, a2, %16;\n\t"
      "mul.wide.u32 a3, %11, 4;\n\tadd.u64 a3, a3, %16;\n\t"
      "mul.wide.u32 a4, %12, 4;\n\tadd.u64 a4, a4, %16;\n\t"
      "mul.wide.u32 a5, %13, 4;\n\tadd.u64 a5, a5, %16;\n\t"
      "mul.wide.u32 a6, %14, 4;\n\tadd.u64 a6, a6, %16;\n\t"
      "mul.wide.u32 a7, %15, 4;\n\tadd.u64 a7, a7, %16;\n\t"
      "@q0 ld.global.nc.f32 %0, [a0];\n\t"
      "@q1 ld.global.nc.f32 %1, [a1];\n\t"
      "@q2 ld.global.nc.f32 %2, [a2];\n\t"
      "@q3 ld.global.nc.f32 %3, [a3];\n\t"
      "@q4 ld.global.nc.f32 %4, [a4];\n\t"
      "@q5 ld.global.nc.f32 %5, [a5];\n\t"
      "@q6 ld.global.nc.f32 %6, [a6];\n\t"
      "@q7 ld.global.nc.f32 %7, [a7];\n\t"
      "}"
      : "+f"(xv[0]), "+f"(xv[1]), "+f"(xv[2]), "+f"(xv[3]), "+f"(xv[4]), "+f"(xv[5]),
        "+f"(xv[6]), "+f"(xv[7])
      : "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(c[5]), "r"(c[6]), "r"(c[7]),
        "l"(x), "r"(cnt));
}
template <>
__device__ __forceinline__ void gather_batch<4, double>(
    const double *x, const uint32_t (&c)[4], uint32_t cnt, double (&xv)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) xv[j] = 0.0;
  asm("{\n\t.reg .pred q<4>;\n\t.reg .u64 a<4>;\n\t"
      "setp.gt.u32 q0, %9, 0;\n\t"
      "setp.gt.u32 q1, %9, 1;\n\t"
      "setp.gt.u32 q2, %9, 2;\n\t"
      "setp.gt.u32 q3, %9, 3;\n\t"
      "mul.wide.u32 a0, %4, 8;\n\tadd.u64 a0, a0, %8;\n\t"
      "mul.wide.u32 a1, %5, 8;\n\tadd.u64 a1, a1, %8;\n\t"
      "mul.wide.u32 a2, %6, 8;\n\tadd.u64 a2, a2, %8;\n\t"
      "mul.wide.u32 a3, %7, 8;\n\tadd.u64 a3, a3, %8;\n\t"
      "@q0 ld.global.nc.f64 %0, [a0];\n\t"
      "@q1 ld.global.nc.f64 %1, [a1];\n\t"
      "@q2 ld.global.nc.f64 %2, [a2];\n\t"
      "@q3 ld.global.nc.f64 %3, [a3];\n\t"
      "}"
      : "+d"(xv[0]), "+d"(xv[1]), "+d"(xv[2]), "+d"(xv[3])
      : "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "l"(x), "r"(cnt));
}
template <>
__device__ __forceinline__ void gather_batch<4, float>(
    const float *x, const uint32_t (&c)[4], uint32_t cnt, float (&xv)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) xv[j] = 0.0f;
  asm("{\n\t.reg .pred q<4>;\n\t.reg .u64 a<4>;\n\t"
      "setp.gt.u32 q0, %9, 0;\n\t"
      "setp.gt.u32 q1, %9, 1;\n\t"
      "setp.gt.u32 q2, %9, 2;\n\t"
      "setp.gt.u32 q3, %9, 3;\n\t"
      "mul.wide.u32 a0, %4, 4;\n\tadd.u64 a0, a0, %8;\n\t"
      "mul.wide.u32 a1, %5, 4;\n\tadd.u64 a1, a1, %8;\n\t"
      "mul.wide.u32 a2, %6, 4;\n\tadd.u64 a2, a2, %8;\n\t"
      "mul.wide.u32 a3, %7, 4;\n\tadd.u64 a3, a3, %8;\n\t"
      "@q0 ld.global.nc.f32 %0, [a0];\n\t"
      "@q1 ld.global.nc.f32 %1, [a1];\n\t"
      "@q2 ld.global.nc.f32 %2, [a2];\n\t"
      "@q3 ld.global.nc.f32 %3, [a3];\n\t"
      "}"
      : "+f"(xv[0]), "+f"(xv[1]), "+f"(xv[2]), "+f"(xv[3])
      : "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "l"(x), "r"(cnt));
}

template <typename V>
struct Elem;
template <>
struct Elem<double> {
  static constexpr uint32_t kPerVec = 2;  // elements per 16 bytes
  __device__ static double load_x(const double *x, uint32_t c) {
    return ldg_x(x, c);
  }
  __device__ static double out(double acc) { return acc; }
};
template <>
struct Elem<float> {
  static constexpr uint32_t kPerVec = 4;
  __device__ static double load_x(const float *x, uint32_t c) {
    return static_cast<double>(ldg_x(x, c));
  }
  __device__ static float out(double acc) { return __double2float_rn(acc); }
};

__host__ __device__ constexpr int pow2_ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

__host__ __device__ constexpr uint32_t round_up(uint32_t v, uint32_t a) {
  return (v + a - 1) / a * a;
}

// Shared-memory geometry of one pipeline stage (host and device agree).
struct Geometry {
  uint32_t cap, rcap, stages;
  uint32_t v_elems, c_elems, r_elems, s_elems;  // allocated elements per stage
  uint32_t v_off, c_off, r_off, s_off, stage_bytes, header_bytes;

  // CSR stages: vals / col_idx spans (cap) and row pointers (rcap + 1).
  __host__ __device__ Geometry(uint32_t cap_, uint32_t rcap_, uint32_t stages_,
                               uint32_t vsize)
      : cap(cap_), rcap(rcap_), stages(stages_) {
    v_elems = cap + 8;       // alignment slack at both ends
    c_elems = cap + 8;
    r_elems = rcap + 1 + 8;  // rows + 1 pointers
    s_elems = 0;
    v_off = 0;
    c_off = round_up(v_elems * vsize, 128);
    r_off = c_off + round_up(c_elems * 4, 128);
    s_off = r_off + round_up(r_elems * 4, 128);
    stage_bytes = s_off + round_up(s_elems * 4, 128);
    header_bytes = round_up(stages * (8 + 8 + 32), 128);
  }
  __host__ __device__ uint32_t total_bytes() const {
    return header_bytes + stages * stage_bytes;
  }
};

struct StageMeta {
  uint32_t r0, r1;  // row range of the tile
  uint32_t va0;     // first staged vals element (16-byte aligned)
  uint32_t ca0;     // first staged col_idx element
  uint32_t ra0;     // first staged row_ptr element
  uint32_t mode;    // kStaged or kDirect
  uint32_t h0, h1;  // the tile's long rows: holes[h0 .. h1) (not staged)
};

// ---- per-row arithmetic ---------------------------------------------------

// fp32 values (a device-only extension; the reference is f64): a batch of
// up to B products is summed left to right in fp32 with fused multiply-adds
// and the batch sum is added to the row's fp64 accumulator, so the error is
// at most B unit roundoffs of the batch's |A||x| (B <= 8: 4.8e-7 of the row's
// |A||x|, inside north_star's 1e-5 for any row length) at one conversion and
// one fp64 add per batch instead of two conversions, a DMUL and a DADD per
// nonzero (the f32 kernels were issue-bound on F2F.F64.F32: C2 f32 ncu r02).
template <int B>
__device__ __forceinline__ float chunk_f32(const float (&v)[B], const float (&xv)[B],
                                           uint32_t count) {
  float part = 0.0f;
#pragma unroll
  for (int j = 0; j < B; ++j)
    if (static_cast<uint32_t>(j) < count) part = __fmaf_rn(v[j], xv[j], part);
  return part;
}
template <int B>
__device__ __forceinline__ float chunk_f32(const double (&)[B], const double (&)[B],
                                           uint32_t) {
  return 0.0f;  // (f64 instantiations never call it)
}

// Serial left-to-right row sum.  Every batch issues all of its x gathers
// before the ordered adds: lanes past the row end load x[0] (their result is
// discarded), so the loads are unconditional and independent -- predicating
// them lets the compiler serialise the gathers through one register pair,
// which left one load in flight per thread.  Pointing every spare lane at the
// same line costs an L1 wavefront at most once per load instruction, where
// clamping to each row's last element cost one per lane (random gathers are
// bound by L1TEX at one 128-byte line per cycle per SM).
template <int B, typename V>
__device__ __forceinline__ double row_serial(const V *__restrict__ sv,
                                             const uint32_t *__restrict__ sc,
                                             uint32_t s, uint32_t e,
                                             const V *__restrict__ x) {
  double acc = 0.0;
  if (s == e) return acc;
  const uint32_t last = e - 1;
  for (uint32_t p = s; p < e; p += B) {
    uint32_t c[B];
    V v[B], xv[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      if (kPredLds) {
        // lanes past the row end issue no shared loads (their bank traffic
        // was a third of C5's shared wavefronts: rows of 1..19 in batches of 8)
        const bool in = p + j <= last;
        c[j] = in ? sc[p + j] : 0u;
        v[j] = in ? sv[p + j] : V(0);
      } else {
        const uint32_t q = min(p + j, last);
        c[j] = p + j <= last ? sc[q] : 0u;
        v[j] = sv[q];
      }
    }
    if (CSRK_PRED_LDG) {
      gather_batch<B, V>(x, c, e - p, xv);
    } else {
#pragma unroll
      for (int j = 0; j < B; ++j) xv[j] = ldg_x(x, c[j]);
    }
    if constexpr (sizeof(V) == 8) {
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (p + j < e) acc = __dadd_rn(acc, __dmul_rn(v[j], xv[j]));
    } else {
      acc = __dadd_rn(acc, static_cast<double>(chunk_f32<B>(v, xv, e - p)));
    }
  }
  return acc;
}

// Lane partial of the STRIDED order: lane l sums nonzeros l, l+nx, ... in
// order; batches of B strided elements load before they are added.
template <int NX, int B, typename V>
__device__ __forceinline__ double lane_partial(const V *__restrict__ sv,
                                               const uint32_t *__restrict__ sc,
                                               uint32_t s, uint32_t e, int lane,
                                               const V *__restrict__ x) {
  double acc = 0.0;
  if (lane >= NX || s + lane >= e) return acc;
  const uint32_t first = s + lane;
  const uint32_t count = (e - first + NX - 1) / NX;  // this lane's elements
  const uint32_t last = first + (count - 1) * NX;
  for (uint32_t p = first; p < e; p += B * NX) {
    uint32_t c[B];
    V v[B], xv[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      if (kPredLds) {
        const bool in = p + j * NX <= last;
        c[j] = in ? sc[p + j * NX] : 0u;
        v[j] = in ? sv[p + j * NX] : V(0);
      } else {
        const uint32_t q = min(p + j * NX, last);
        c[j] = p + j * NX <= last ? sc[q] : 0u;
        v[j] = sv[q];
      }
    }
    if (CSRK_PRED_LDG) {
      gather_batch<B, V>(x, c, (e - p + NX - 1) / NX, xv);
    } else {
#pragma unroll
      for (int j = 0; j < B; ++j) xv[j] = ldg_x(x, c[j]);
    }
    if constexpr (sizeof(V) == 8) {
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (p + j * NX < e) acc = __dadd_rn(acc, __dmul_rn(v[j], xv[j]));
    } else {
      acc = __dadd_rn(acc, static_cast<double>(chunk_f32<B>(v, xv, (e - p + NX - 1) / NX)));
    }
  }
  return acc;
}

// GATHER-FIRST tiles: the consumers first replace every staged value by its
// product vals[p] * x[col[p]] (__dmul_rn, the same rounding the inline path
// applies), issuing the whole tile's x gathers at once -- balanced over the
// 256 consumer threads and independent of the row structure -- and then sum
// the products from shared memory in the row's exact order.  Bitwise equal
// to the inline path; it decouples gather memory-level parallelism from row
// lengths, which is what bounds irregular matrices (C5).
template <typename V>
__device__ __forceinline__ void gather_products(V *__restrict__ sv,
                                                const uint32_t *__restrict__ sc,
                                                uint32_t q0, uint32_t q1,
                                                const V *__restrict__ x, int ct) {
  constexpr int U = 8;
  if (q0 >= q1) return;
  const uint32_t last = q1 - 1;
  for (uint32_t p = q0 + ct; p < q1; p += kConsumers * U) {
    uint32_t c[U];
    double xv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) c[j] = sc[min(p + j * kConsumers, last)];
#pragma unroll
    for (int j = 0; j < U; ++j) xv[j] = Elem<V>::load_x(x, c[j]);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint32_t q = p + j * kConsumers;
      if (q < q1) sv[q] = __dmul_rn(static_cast<double>(sv[q]), xv[j]);
    }
  }
}

// gather_products for a tile with long rows: their nonzeros (the holes,
// ascending [start, end) pairs) were not staged and are not touched
template <typename V>
__device__ __forceinline__ void gather_products_holes(V *__restrict__ sv,
                                                      const uint32_t *__restrict__ sc,
                                                      uint32_t q0, uint32_t q1,
                                                      const V *__restrict__ x, int ct,
                                                      const uint2 *__restrict__ holes,
                                                      uint32_t h, uint32_t h1) {
  constexpr int U = 8;
  uint2 hb = h < h1 ? holes[h] : make_uint2(0xffffffffu, 0xffffffffu);
  for (uint32_t p = q0 + ct; p < q1; p += kConsumers * U) {
    uint32_t c[U];
    bool ok[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint32_t q = p + j * kConsumers;
      while (q >= hb.y) {
        ++h;
        hb = h < h1 ? holes[h] : make_uint2(0xffffffffu, 0xffffffffu);
      }
      ok[j] = q < q1 && q < hb.x;
      c[j] = ok[j] ? sc[q] : 0u;
    }
    double xv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) xv[j] = Elem<V>::load_x(x, c[j]);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint32_t q = p + j * kConsumers;
      if (ok[j]) sv[q] = __dmul_rn(static_cast<double>(sv[q]), xv[j]);
    }
  }
}

template <typename V>
__device__ __forceinline__ double row_products(const V *__restrict__ prod,
                                               uint32_t s, uint32_t e) {
  double acc = 0.0;
  for (uint32_t p = s; p < e; ++p) acc = __dadd_rn(acc, static_cast<double>(prod[p]));
  return acc;
}

template <int NX, typename V>
__device__ __forceinline__ double lane_products(const V *__restrict__ prod,
                                                uint32_t s, uint32_t e, int lane) {
  double acc = 0.0;
  if (lane >= NX) return acc;
  for (uint32_t p = s + lane; p < e; p += NX)
    acc = __dadd_rn(acc, static_cast<double>(prod[p]));
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

// rows [r0, r1) with staged (or global) arrays; `srp(r)` yields row_ptr[r]
// Rows longer than `long_len` nonzeros are skipped: the long-row kernel
// (below) sums them with a whole warp each.
template <typename V, int NX, bool PROD = false, int LB = 4, bool DOT = false,
          typename RowPtr>
__device__ __forceinline__ void compute_rows(uint32_t r0, uint32_t r1,
                                             const V *__restrict__ sv,
                                             const uint32_t *__restrict__ sc,
                                             RowPtr srp, const V *__restrict__ x,
                                             V *__restrict__ y, int ct,
                                             uint32_t long_len = 0xffffffffu,
                                             double *dot = nullptr) {
  if constexpr (NX == 0) {
    for (uint32_t r = r0 + ct; r < r1; r += kConsumers) {
      const uint32_t s = srp(r), e = srp(r + 1);
      if (e - s > long_len) continue;
      V yr;
      if constexpr (PROD)
        yr = Elem<V>::out(row_products<V>(sv, s, e));
      else
        yr = Elem<V>::out(row_serial<LB == 2 ? 4 : (LB == 7 ? 7 : 8), V>(sv, sc, s, e, x));
      y[r] = yr;
      // fused x . y partial (the CG's p . Ap): x[r] * (stored y[r]) in f64
      if constexpr (DOT)
        *dot = __dadd_rn(*dot, __dmul_rn(static_cast<double>(ldg_x(x, r)),
                                          static_cast<double>(yr)));
    }
  } else {
    constexpr int P = pow2_ceil(NX);
    constexpr int kSubPerWarp = 32 / P;
    constexpr int kSubs = kConsumers / P;
    const int lane = ct % P;
    const int sub = ct / P;
    const int warp_first = (ct / 32) * kSubPerWarp;
    for (uint32_t base = r0 + warp_first; base < r1; base += kSubs) {
      const uint32_t r = base + (sub - warp_first);
      double acc = 0.0;
      bool mine = r < r1;
      if (mine) {
        const uint32_t s = srp(r), e = srp(r + 1);
        mine = e - s <= long_len;
        if (mine) {
          if constexpr (PROD)
            acc = lane_products<NX, V>(sv, s, e, lane);
          else
            acc = lane_partial<NX, LB, V>(sv, sc, s, e, lane, x);
        }
      }
      acc = subwarp_tree<P>(acc);
      if (mine && lane == 0) y[r] = Elem<V>::out(acc);
    }
  }
}

// a tile whose rows do not fit a stage: SERIAL rows are summed by whole
// warps (products in parallel, ordered adds through shuffles)
template <typename V, int NX, bool DOT = false>
__device__ void compute_direct(uint32_t r0, uint32_t r1,
                               const uint32_t *__restrict__ row_ptr,
                               const uint32_t *__restrict__ col_idx,
                               const V *__restrict__ vals,
                               const V *__restrict__ x, V *__restrict__ y,
                               int ct, uint32_t long_len = 0xffffffffu,
                               double *dot = nullptr) {
  if constexpr (NX == 0) {
    const int lane = ct & 31, warp = ct >> 5;
    for (uint32_t r = r0 + warp; r < r1; r += kConsumerWarps) {
      const uint32_t s = row_ptr[r], e = row_ptr[r + 1];
      if (e - s > long_len) continue;
      double acc = 0.0;
      for (uint32_t p0 = s; p0 < e; p0 += 32) {
        const uint32_t p = p0 + lane;
        double prod = 0.0;
        if (p < e)
          prod = __dmul_rn(static_cast<double>(vals[p]),
                           Elem<V>::load_x(x, col_idx[p]));
        const uint32_t cnt = (e - p0) < 32u ? (e - p0) : 32u;
        for (uint32_t j = 0; j < cnt; ++j)
          acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, prod, j));
      }
      if (lane == 0) {
        const V yr = Elem<V>::out(acc);
        y[r] = yr;
        if constexpr (DOT)
          *dot = __dadd_rn(*dot, __dmul_rn(static_cast<double>(ldg_x(x, r)),
                                            static_cast<double>(yr)));
      }
    }
  } else {
    compute_rows<V, NX>(r0, r1, vals, col_idx,
                        [&](uint32_t r) { return row_ptr[r]; }, x, y, ct, long_len);
  }
}

// Per-CTA event timeline of the streaming kernel (diagnostic build only:
// tools/build_variant.sh tl -DCSRK_TIMELINE=1, read by tools/timeline_probe.py
// through csrk_debug_timeline).  Slot 0: %globaltimer at entry (aligns the
// SMs); slots 1-5: SM clock cycles after entry at the producer's first TMA
// issue, the consumers' first full stage, their last stage released, the
// producer's exit, and the CTA's tile count.
#ifndef CSRK_TIMELINE
#define CSRK_TIMELINE 0
#endif
#if CSRK_TIMELINE
constexpr int kTlSlots = 6, kTlCtas = 4096;
__device__ unsigned long long g_timeline[kTlCtas * kTlSlots];
__device__ __forceinline__ unsigned long long tl_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL_ENTRY()                                                             \
  const long long tl_c0 = clock64();                                           \
  if (threadIdx.x == 0 && blockIdx.x < kTlCtas)                                \
    g_timeline[blockIdx.x * kTlSlots] = tl_gtimer()
#define TL_MARK(slot)                                                          \
  if (blockIdx.x < kTlCtas)                                                    \
  g_timeline[blockIdx.x * kTlSlots + (slot)] =                                 \
      static_cast<unsigned long long>(clock64() - tl_c0)
#define TL_SET(slot, v) \
  if (blockIdx.x < kTlCtas) g_timeline[blockIdx.x * kTlSlots + (slot)] = (v)
#else
#define TL_ENTRY()
#define TL_MARK(slot)
#define TL_SET(slot, v)
#endif

// The tiles a CTA of the persistent grid takes: [first, end) in steps of
// `step`.  Round-robin (tile b, b + grid, ...) by default; CSRK_CONTIG_TILES=1
// gives each CTA one contiguous run of tiles instead (successive tiles of
// a CTA then gather from nearly the same window of x: the A/B of
// DESIGN.md §4 "tile order").
#ifndef CSRK_CONTIG_TILES
#define CSRK_CONTIG_TILES 0
#endif
struct TileRun {
  uint32_t first, end, step;
};
__device__ __forceinline__ TileRun tile_run(uint32_t n_tiles) {
#if CSRK_CONTIG_TILES
  const uint32_t g = gridDim.x, b = blockIdx.x;
  const uint32_t q = n_tiles / g, r = n_tiles % g;
  const uint32_t first = b * q + (b < r ? b : r);
  return {first, first + q + (b < r ? 1u : 0u), 1u};
#else
  return {blockIdx.x, n_tiles, gridDim.x};
#endif
}

template <typename V, int NX, bool GF, int LB = 4, bool DOT = false>
__global__ void __launch_bounds__(kThreads, 2)
    csrk_stream_kernel(const uint32_t *__restrict__ row_ptr,
                       const uint32_t *__restrict__ col_idx,
                       const V *__restrict__ vals, const V *__restrict__ x,
                       V *__restrict__ y, const uint32_t *__restrict__ tile_row,
                       const uint32_t *__restrict__ tile_ptr, uint32_t n_tiles,
                       uint32_t cap, uint32_t rcap, uint32_t stages, uint32_t long_len,
                       const uint32_t *__restrict__ tile_long,
                       const uint2 *__restrict__ holes, uint64_t x_bytes,
                       uint32_t pf_chunk, double *__restrict__ dot_part) {
  extern __shared__ __align__(128) unsigned char smem[];
  const Geometry geo(cap, rcap, stages, sizeof(V));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem);
  uint64_t *empty = full + stages;
  StageMeta *meta = reinterpret_cast<StageMeta *>(empty + stages);
  unsigned char *stage0 = smem + geo.header_bytes;

  const int tid = threadIdx.x;
  TL_ENTRY();
  if (tid == 0) {
    for (uint32_t s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (tid < 32) {
    // ---------------- producer warp ----------------
    if (tid != 0) return;
    constexpr uint32_t VPV = Elem<V>::kPerVec;
    const uint64_t policy = evict_first_policy();
    // x prefetch (small x only, see launch_stream): CTA b pulls slice b of x
    // into L2 with evict_last, so the tiles' gathers hit L2 instead of
    // waiting out HBM latency on first touch, and the evict_first matrix
    // stream does not displace it
    if (pf_chunk) {
      const uint64_t off = static_cast<uint64_t>(blockIdx.x) * pf_chunk;
      if (off < x_bytes) {
        const uint64_t left = x_bytes - off;
        const uint32_t b = static_cast<uint32_t>(left < pf_chunk ? left : pf_chunk) & ~15u;
        if (b) l2_prefetch_bulk(reinterpret_cast<const unsigned char *>(x) + off, b,
                                evict_last_policy());
      }
    }
    // the next tile's bounds (rows and their nonzero offsets, precomputed in
    // the plan) load while this tile waits for its stage: the producer never
    // spends a dependent global round trip between two TMA issues
    const TileRun run = tile_run(n_tiles);
    uint32_t nr0 = 0, nr1 = 0, np0 = 0, np1 = 0, nh0 = 0, nh1 = 0;
    if (run.first < run.end) {
      nr0 = tile_row[run.first];
      nr1 = tile_row[run.first + 1];
      np0 = tile_ptr[run.first];
      np1 = tile_ptr[run.first + 1];
      if (tile_long) {
        nh0 = tile_long[run.first];
        nh1 = tile_long[run.first + 1];
      }
    }
    // ring position: stage s and the parity of its fill (no integer
    // division per tile: it cost ~25 instructions per tile and warp)
    uint32_t i = 0, s = 0, ph = 0;
    for (uint32_t t = run.first; t < run.end;
         t += run.step, ++i, s = (s + 1 == stages) ? 0 : s + 1, ph ^= (s == 0)) {
      const uint32_t r0 = nr0, r1 = nr1, p0 = np0, p1 = np1, h0 = nh0, h1 = nh1;
      const uint32_t tn = t + run.step;
      if (tn < run.end) {
        nr0 = tile_row[tn];
        nr1 = tile_row[tn + 1];
        np0 = tile_ptr[tn];
        np1 = tile_ptr[tn + 1];
        if (tile_long) {
          nh0 = tile_long[tn];
          nh1 = tile_long[tn + 1];
        }
      }
      if (i >= stages) mbar_wait(&empty[s], ph ^ 1u);
      StageMeta &md = meta[s];
      md.r0 = r0;
      md.r1 = r1;
      md.h0 = h0;
      md.h1 = h1;
      if (p1 - p0 <= cap && r1 - r0 <= rcap && !(r1 - r0 == 1 && h1 > h0)) {
        unsigned char *st = stage0 + s * geo.stage_bytes;
        const uint32_t va0 = p0 & ~(VPV - 1);
        const uint32_t ca0 = p0 & ~3u;
        const uint32_t ra0 = r0 & ~3u, ra1 = round_up(r1 + 1, 4);
        const uint32_t rb = (ra1 - ra0) * 4u;
        md.va0 = va0;
        md.ca0 = ca0;
        md.ra0 = ra0;
        md.mode = kStaged;
        // the tile's nonzeros minus its long rows (holes longer than 128
        // entries, so the 16-byte-rounded segments never overlap); one
        // segment [p0, p1) without long rows
        uint32_t tx = rb;
        for (uint32_t pass = 0; pass < 2; ++pass) {
          uint32_t a = p0;
          for (uint32_t h = h0; h <= h1; ++h) {
            const uint2 hb = h < h1 ? holes[h] : make_uint2(p1, p1);
            if (hb.x > a) {
              const uint32_t v0 = a & ~(VPV - 1), v1 = round_up(hb.x, VPV);
              const uint32_t c0 = a & ~3u, c1 = round_up(hb.x, 4);
              const uint32_t vb = (v1 - v0) * static_cast<uint32_t>(sizeof(V));
              const uint32_t cb = (c1 - c0) * 4u;
              if (pass == 0) {
                tx += vb + cb;
              } else {
                tma_bulk_load(st + geo.v_off + (v0 - va0) * sizeof(V), vals + v0, vb,
                              &full[s], policy);
                tma_bulk_load(st + geo.c_off + (c0 - ca0) * 4u, col_idx + c0, cb, &full[s],
                              policy);
              }
            }
            a = hb.y;
          }
          if (pass == 0) mbar_arrive_expect_tx(&full[s], tx);
        }
        tma_bulk_load(st + geo.r_off, row_ptr + ra0, rb, &full[s], policy);
      } else {
        md.mode = kDirect;
        mbar_arrive(&full[s]);
      }
      if (i == 0) TL_MARK(1);
    }
    TL_MARK(4);
    TL_SET(5, i);
    // every TMA of this CTA is issued: the next kernel on the stream (a
    // repeated SpMV) may start its own prologue and matrix stream on the SMs
    // this grid frees (programmatic dependent launch, launch_stream)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }

  // ---------------- consumer warps ----------------
  // Under programmatic dependent launch the producer streams the matrix
  // (read-only for the handle's lifetime) while the previous kernel on the
  // stream is still running; x is read and y written only after that kernel
  // has completed and its writes are visible.  A no-op without the launch
  // attribute.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int ct = tid - 32;
  double dot = 0.0;  // DOT: this thread's x . y partial over its rows
  uint32_t s = 0, ph = 0;
  const TileRun run = tile_run(n_tiles);
  for (uint32_t t = run.first; t < run.end;
       t += run.step, s = (s + 1 == stages) ? 0 : s + 1, ph ^= (s == 0)) {
    mbar_wait(&full[s], ph);
    if (CSRK_TIMELINE && ct == 0 && t == run.first) TL_MARK(2);
    const StageMeta md = meta[s];
    if (md.mode == kStaged) {
      const unsigned char *st = stage0 + s * geo.stage_bytes;
      const V *sv = reinterpret_cast<const V *>(st + geo.v_off) - md.va0;
      const uint32_t *sc = reinterpret_cast<const uint32_t *>(st + geo.c_off) - md.ca0;
      const uint32_t *sr = reinterpret_cast<const uint32_t *>(st + geo.r_off) - md.ra0;
      if constexpr (GF) {
        V *svw = const_cast<V *>(sv);
        if (md.h1 > md.h0)
          gather_products_holes<V>(svw, sc, sr[md.r0], sr[md.r1], x, ct, holes, md.h0, md.h1);
        else
          gather_products<V>(svw, sc, sr[md.r0], sr[md.r1], x, ct);
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
        compute_rows<V, NX, true>(md.r0, md.r1, sv, sc,
                                  [&](uint32_t r) { return sr[r]; }, x, y, ct, long_len);
        // generic-proxy writes to the stage precede the next TMA fill of it
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      } else {
        compute_rows<V, NX, false, LB, DOT>(md.r0, md.r1, sv, sc,
                                            [&](uint32_t r) { return sr[r]; }, x, y, ct,
                                            long_len, &dot);
      }
    } else {
      compute_direct<V, NX, DOT>(md.r0, md.r1, row_ptr, col_idx, vals, x, y, ct, long_len,
                                 &dot);
    }
    __syncwarp();
    if ((ct & 31) == 0) mbar_arrive(&empty[s]);
  }
  if (CSRK_TIMELINE && ct == 0) TL_MARK(3);
  if constexpr (DOT) {
    // the CTA's partial in a fixed order: warp trees, then warps 0..7
    __shared__ double red[kConsumerWarps];
    for (int o = 16; o > 0; o >>= 1) dot = __dadd_rn(dot, __shfl_down_sync(0xffffffffu, dot, o));
    if ((ct & 31) == 0) red[ct >> 5] = dot;
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
    if (ct == 0) {
      double v = 0.0;
      for (int w = 0; w < kConsumerWarps; ++w) v = __dadd_rn(v, red[w]);
      dot_part[blockIdx.x] = v;
    }
  }
}

// ---- long rows -------------------------------------------------------------
//
// Power-law matrices (the paper's failure mode) put rows of
// thousands of nonzeros into single tiles: a tile then occupies one thread
// (serial order) or one sub-warp (strided order) of its CTA for the whole
// row while the rest of the CTA -- and the tiles queued behind it -- wait.
// Rows longer than kLongRow are listed when the plan is built, skipped by the
// streaming kernel, and summed here with a whole warp each, spread over the
// GPU: the serial order gathers 128 products per step in parallel and lane 0
// adds them left to right (the reference's chain, bit for bit); the strided
// order runs its nx lane chains and the halving tree as the streaming kernel
// does.  Rows outside [rows_lo, rows_hi) (a tile-range launch) are skipped.

template <typename V, int NX>
__global__ void __launch_bounds__(256)
    long_rows_kernel(const uint32_t *__restrict__ row_ptr, const uint32_t *__restrict__ col_idx,
                     const V *__restrict__ vals, const V *__restrict__ x, V *__restrict__ y,
                     const uint32_t *__restrict__ long_rows, int64_t n_long,
                     const uint32_t *__restrict__ rows_lo, const uint32_t *__restrict__ rows_hi) {
  constexpr int kChunk = 128;
  __shared__ double buf[8][kChunk];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lo = *rows_lo, hi = *rows_hi;
  const int64_t warps = int64_t(gridDim.x) * 8;
  for (int64_t i = blockIdx.x * int64_t(8) + w; i < n_long; i += warps) {
    const uint32_t r = long_rows[i];
    if (r < lo || r >= hi) continue;
    const uint32_t s = row_ptr[r], e = row_ptr[r + 1];
    // every lane gathers the products of a 128-entry chunk (the next chunk's
    // gathers issued before the current one is walked, so their latency
    // hides behind the ordered adds); the chains then walk the chunk from
    // shared memory: lane 0 alone in the serial order, lanes 0..nx-1 their
    // strided subsequences (position mod nx) in the strided order.  (A
    // register walk by shuffles measured slower: 64-bit shuffles are two
    // instructions each -- serial 517 -> 788 us on the 20 k power-law case.)
    constexpr int K = kChunk / 32;
    constexpr int L = NX == 0 ? 1 : NX;
    // D chunks in flight: the longest row's chain is the kernel's critical
    // path, and with one chunk of look-ahead each step waited out most of a
    // load latency (power-law 20 k, serial: 349 us for 474 MB)
    constexpr int D = 3;
    double v[D][K], xv[D][K];
    auto load = [&](double(&vv)[K], double(&xx)[K], uint32_t c0) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t p = c0 + k * 32 + lane;
        const uint32_t q = p < e ? p : e - 1;
        vv[k] = static_cast<double>(vals[q]);
        xx[k] = Elem<V>::load_x(x, col_idx[q]);
      }
    };
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (s + d * kChunk < e) load(v[d], xv[d], s + d * kChunk);
    double acc = 0.0;
    for (uint32_t base = s; base < e; base += D * kChunk)
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const uint32_t p0 = base + d * kChunk;
      if (p0 >= e) break;
      double prod[K];
#pragma unroll
      for (int k = 0; k < K; ++k) prod[k] = __dmul_rn(v[d][k], xv[d][k]);
      if (p0 + D * kChunk < e) load(v[d], xv[d], p0 + D * kChunk);
#pragma unroll
      for (int k = 0; k < K; ++k) buf[w][k * 32 + lane] = prod[k];
      __syncwarp();
      if (lane < L) {
        const uint32_t cnt = e - p0 < uint32_t(kChunk) ? e - p0 : uint32_t(kChunk);
        if (kChunk % L == 0 && cnt == uint32_t(kChunk)) {
          // full chunk (entry 0 at position 0 mod nx): the loads of a group
          // are independent of the chain, so they issue ahead of its adds
          constexpr int kPer = kChunk / L, kGroup = kPer < 16 ? kPer : 16;
#pragma unroll
          for (int g = 0; g < kPer; g += kGroup) {
            double t[kGroup];
#pragma unroll
            for (int q = 0; q < kGroup; ++q) t[q] = buf[w][(g + q) * L + lane];
#pragma unroll
            for (int q = 0; q < kGroup; ++q) acc = __dadd_rn(acc, t[q]);
          }
        } else {
          const uint32_t off = (p0 - s) % L;  // position of chunk entry 0 modulo nx
          for (uint32_t j = (lane + L - off) % L; j < cnt; j += L)
            acc = __dadd_rn(acc, buf[w][j]);
        }
      }
      __syncwarp();
    }
    if constexpr (NX == 0) {
      if (lane == 0) y[r] = Elem<V>::out(acc);
    } else {
      constexpr int P = pow2_ceil(NX);
      acc = subwarp_tree<P>(lane < NX ? acc : 0.0);
      if (lane == 0) y[r] = Elem<V>::out(acc);
    }
  }
}

__global__ void long_rows_list_kernel(const uint32_t *__restrict__ row_ptr, int64_t n_rows,
                                      uint32_t min_len, uint32_t *__restrict__ out,
                                      unsigned long long *__restrict__ count) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x)
    if (row_ptr[r + 1] - row_ptr[r] > min_len) {
      const unsigned long long k = atomicAdd(count, 1ull);
      if (out) out[k] = static_cast<uint32_t>(r);
    }
}

// keys of the long-row list: row order (the holes) or longest first, ties by
// row (the long-row kernel's work order: the longest chains start first)
__global__ void long_keys_kernel(const uint32_t *__restrict__ row_ptr,
                                 const uint32_t *__restrict__ rows, int64_t n, int by_len,
                                 uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = rows[k];
    const uint32_t len = row_ptr[r + 1] - row_ptr[r];
    keys[k] = by_len ? (uint64_t(0xffffffffu - len) << 32) | r : uint64_t(r);
    vals[k] = r;
  }
}

__global__ void holes_kernel(const uint32_t *__restrict__ row_ptr,
                             const uint32_t *__restrict__ rows, int64_t n,
                             uint2 *__restrict__ holes) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = rows[k];
    holes[k] = make_uint2(row_ptr[r], row_ptr[r + 1]);
  }
}

__global__ void hole_sum_kernel(const uint2 *__restrict__ holes, int64_t n,
                                unsigned long long *__restrict__ sum) {
  unsigned long long acc = 0;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x)
    acc += holes[k].y - holes[k].x;
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(sum, acc);
}

// first hole at or past each tile's first nonzero
__global__ void tile_long_kernel(const uint32_t *__restrict__ tile_ptr, int64_t n_tiles,
                                 const uint2 *__restrict__ holes, int64_t n_long,
                                 uint32_t *__restrict__ tile_long) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t > n_tiles) return;
  const uint32_t p = tile_ptr[t];
  int64_t lo = 0, hi = n_long;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (holes[mid].x >= p)
      hi = mid;
    else
      lo = mid + 1;
  }
  tile_long[t] = static_cast<uint32_t>(lo);
}

// blocks of 8 warps per SM beside the streaming kernel's CTAs
// (CSRK_LONG_BLOCKS overrides, for sweeps)
int64_t long_blocks_per_sm() {
  static const int64_t v = [] {
    const char *e = std::getenv("CSRK_LONG_BLOCKS");
    return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(8);
  }();
  return v;
}

template <typename V, int NX>
int launch_long_rows(const csrk_matrix *m, const V *vals, const V *x, V *y, cudaStream_t stream,
                     int64_t t0, int64_t t1) {
  const TilePlan &pl = m->plan;
  if (t1 < 0 || t1 > pl.n_tiles) t1 = pl.n_tiles;
  if (t0 < 0) t0 = 0;
  int64_t blocks = (pl.n_long + 7) / 8;
  if (blocks > int64_t(m->sm_count) * long_blocks_per_sm())
    blocks = int64_t(m->sm_count) * long_blocks_per_sm();
  if (blocks < 1) return CSRK_OK;
  long_rows_kernel<V, NX><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
      m->row_ptr, m->col_idx, vals, x, y, pl.long_rows, pl.n_long, pl.tile_row + t0,
      pl.tile_row + t1);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

// ---- tile plan -------------------------------------------------------------

__device__ __forceinline__ uint32_t group_start(const uint32_t *sr_ptr,
                                                const uint32_t *ssr_ptr, int k,
                                                int64_t g, int64_t n_groups,
                                                int64_t n_rows) {
  if (g >= n_groups) return static_cast<uint32_t>(n_rows);
  if (k == 3) return sr_ptr[ssr_ptr[g]];
  if (k == 2) return sr_ptr[g];
  return static_cast<uint32_t>(g);
}

// largest group cost (nonzeros + rows)
__global__ void max_group_cost_kernel(const uint32_t *__restrict__ row_ptr,
                                      const uint32_t *__restrict__ sr_ptr,
                                      const uint32_t *__restrict__ ssr_ptr,
                                      int k, int64_t n_groups, int64_t n_rows,
                                      unsigned long long *out) {
  unsigned long long mx = 0;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n_groups;
       g += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t a = group_start(sr_ptr, ssr_ptr, k, g, n_groups, n_rows);
    const uint32_t b = group_start(sr_ptr, ssr_ptr, k, g + 1, n_groups, n_rows);
    const unsigned long long c =
        static_cast<unsigned long long>(row_ptr[b] - row_ptr[a]) + (b - a);
    mx = c > mx ? c : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_down_sync(0xffffffffu, mx, o);
    mx = v > mx ? v : mx;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// sum over rows of (row length)^2, for the schedule's variance test
__global__ void row_sq_kernel(const uint32_t *__restrict__ row_ptr, int64_t n_rows,
                              unsigned long long *out) {
  unsigned long long acc = 0;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long l = row_ptr[r + 1] - row_ptr[r];
    acc += l * l;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

// tile_row[t] = first cut point (group start, or row when cut_k == 1) whose
// cost row_ptr[r] + r reaches t * tile_cost
__global__ void tile_bounds_kernel(const uint32_t *__restrict__ row_ptr,
                                   const uint32_t *__restrict__ sr_ptr,
                                   const uint32_t *__restrict__ ssr_ptr,
                                   int cut_k, int64_t n_groups, int64_t n_rows,
                                   int64_t tile_cost, int64_t n_tiles,
                                   uint32_t *__restrict__ tile_row) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t > n_tiles) return;
  if (t == n_tiles) {
    tile_row[t] = static_cast<uint32_t>(n_rows);
    return;
  }
  const int64_t target = t * tile_cost;
  int64_t lo = 0, hi = n_groups;  // answer in [0, n_groups]
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    const uint32_t r = group_start(sr_ptr, ssr_ptr, cut_k, mid, n_groups, n_rows);
    if (static_cast<int64_t>(row_ptr[r]) + r >= target)
      hi = mid;
    else
      lo = mid + 1;
  }
  tile_row[t] = group_start(sr_ptr, ssr_ptr, cut_k, lo, n_groups, n_rows);
}

// tile_ptr[t] = row_ptr[tile_row[t]]: the first nonzero of every tile
__global__ void tile_ptr_kernel(const uint32_t *__restrict__ row_ptr,
                                const uint32_t *__restrict__ tile_row, int64_t n_tiles,
                                uint32_t *__restrict__ tile_ptr) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t <= n_tiles) tile_ptr[t] = row_ptr[tile_row[t]];
}

// max column read by the rows of each chunk [row_cut[c], row_cut[c+1])
__global__ void chunk_max_col_kernel(const uint32_t *__restrict__ row_ptr,
                                     const uint32_t *__restrict__ col_idx,
                                     const uint32_t *__restrict__ row_cut,
                                     uint32_t *__restrict__ out) {
  const uint32_t c = blockIdx.x;
  const uint32_t a = row_ptr[row_cut[c]], b = row_ptr[row_cut[c + 1]];
  uint32_t mx = 0;
  for (uint32_t p = a + threadIdx.x; p < b; p += blockDim.x)
    mx = col_idx[p] > mx ? col_idx[p] : mx;
  for (int o = 16; o > 0; o >>= 1) {
    const uint32_t v = __shfl_down_sync(0xffffffffu, mx, o);
    mx = v > mx ? v : mx;
  }
  __shared__ uint32_t red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      mx = red[w] > mx ? red[w] : mx;
    out[c] = mx;
  }
}

// Whether the long-row kernel runs beside the streaming kernel (see
// dispatch_nx): always with long rows, unless CSRK_LONG_SERIAL=1.
bool long_beside(const csrk_matrix *m, int variant, int nx) {
  static const bool serial_long = [] {
    const char *e = std::getenv("CSRK_LONG_SERIAL");
    return e && e[0] == '1';
  }();
  static const int max_nx = [] {  // sweep knob: widest strided order beside
    const char *e = std::getenv("CSRK_LONG_BESIDE_NX");
    return e ? std::atoi(e) : 32;
  }();
  return m->plan.n_long > 0 && !serial_long && (variant == CSRK_SERIAL || nx <= max_nx);
}
// shared memory the streaming kernel's carveout leaves for long-row blocks
// beside it (their 8 KB buffers; without the room they could not co-reside
// and took SMs the persistent CTAs then waited for -- 2.1 -> 1.1 TB/s at
// some tile sizes on the power-law case)
constexpr int kBesideBlocks = 2;
constexpr size_t kLongBlockSmem = 8 * 128 * sizeof(double) + 1024;

// x vectors up to this size are prefetched into L2 by the streaming kernel
// (CSRK_X_PREFETCH=<MB> overrides; 0 disables)
uint64_t x_prefetch_limit() {
  static const uint64_t lim = [] {
    const char *e = std::getenv("CSRK_X_PREFETCH");
    return e ? static_cast<uint64_t>(std::atoll(e)) << 20 : (48ull << 20);
  }();
  return lim;
}

template <typename V, int NX, bool GF, int LB = 4, bool DOT = false>
int launch_stream(const csrk_matrix *m, const V *vals, const V *x, V *y,
                  cudaStream_t stream, int64_t t0, int64_t t1,
                  double *dot_part = nullptr, int64_t dot_slots = 0) {
  const TilePlan &pl = m->plan;
  const Geometry geo(static_cast<uint32_t>(pl.cap), static_cast<uint32_t>(pl.rcap),
                     static_cast<uint32_t>(pl.stages), sizeof(V));
  const size_t smem = geo.total_bytes();
  auto kern = csrk_stream_kernel<V, NX, GF, LB, DOT>;
  // attribute + occupancy queries cost host time per launch; cache them per
  // instantiation and shared-memory size (the chunked host pipeline launches
  // the kernel many times per SpMV)
  static thread_local size_t cached_smem = 0, cached_extra = 0;
  static thread_local int cached_per_sm = 0, cached_ctas = 0;
  static thread_local int cached_device = -1;
  int cur_dev = 0;
  CSRK_CUDA_TRY(cudaGetDevice(&cur_dev));
  const int ctas = pl.ctas_per_sm > 0 ? pl.ctas_per_sm
                                      : auto_ctas(pl.row_var, static_cast<int>(sizeof(V)),
                                                  pl.n_long, pl.mean_short);
  const size_t extra =
      long_beside(m, NX == 0 ? CSRK_SERIAL : CSRK_STRIDED, NX) ? kBesideBlocks * kLongBlockSmem : 0;
  int per_sm = 0;
  if (cached_smem == smem && cached_device == cur_dev && cached_ctas == ctas &&
      cached_extra == extra) {
    per_sm = cached_per_sm;
  } else {
    CSRK_CUDA_TRY(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    // Carveout = exactly what `ctas` CTAs need (+1 KB reserved each); the
    // rest of the SM's 256 KB stays L1, where the x gathers hit.  Left to
    // the driver, the carveout jumped with the stage size (a 2 KB larger
    // stage moved C5 from the 200 KB to the 228 KB carveout and cost it a
    // third of its bandwidth).
    int smem_sm = 0;
    CSRK_CUDA_TRY(cudaDeviceGetAttribute(&smem_sm,
                                         cudaDevAttrMaxSharedMemoryPerMultiprocessor,
                                         cur_dev));
    const double need = static_cast<double>(ctas) * (smem + 1024) + static_cast<double>(extra);
    int pct = static_cast<int>(need * 100.0 / smem_sm + 0.999);
    pct = pct < 1 ? 1 : (pct > 100 ? 100 : pct);
    CSRK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       pct));
    CSRK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads,
                                                                smem));
    if (per_sm > ctas) per_sm = ctas;
    cached_extra = extra;
    cached_smem = smem;
    cached_per_sm = per_sm;
    cached_ctas = ctas;
    cached_device = cur_dev;
  }
  if (per_sm < 1) {
    set_error("stream kernel does not fit on an SM (%zu bytes of shared memory)", smem);
    return CSRK_EINVAL;
  }
  if (t1 < 0 || t1 > pl.n_tiles) t1 = pl.n_tiles;
  if (t0 < 0) t0 = 0;
  const int64_t count = t1 - t0;
  int64_t grid = static_cast<int64_t>(per_sm) * m->sm_count;
  if (grid > count) grid = count;
  if (grid < 1) return CSRK_OK;
  if (DOT && grid > dot_slots) {
    set_error("fused dot needs %lld partial slots, has %lld", static_cast<long long>(grid),
              static_cast<long long>(dot_slots));
    return CSRK_EINVAL;
  }
  // x prefetch into L2 for whole-matrix launches whose x is small against
  // the 126 MB L2 (x_prefetch_bytes(), CSRK_X_PREFETCH), from a 16-byte
  // aligned x; slices of at least 4 KB
  const uint64_t x_bytes = static_cast<uint64_t>(m->n_cols) * sizeof(V);
  uint32_t pf_chunk = 0;
  if (t0 == 0 && t1 == pl.n_tiles && (reinterpret_cast<uintptr_t>(x) & 15u) == 0 &&
      x_bytes <= x_prefetch_limit()) {
    uint64_t c = (x_bytes + grid - 1) / grid;
    c = (c + 4095) / 4096 * 4096;
    pf_chunk = static_cast<uint32_t>(c);
  }
  // Programmatic dependent launch (CSRK_PDL=0 disables): back-to-back
  // SpMVs overlap the next launch's prologue and first TMA fills with the
  // previous grid's last tiles (the kernel's griddepcontrol.wait orders
  // every x read and y write after the previous kernel).  Only the matrix
  // and plan arrays are read early; they are written before the handle's
  // first launch and synchronised (upload, ensure_plan, prepare_plan).
  static const bool pdl = [] {
    const char *e = std::getenv("CSRK_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  CSRK_CUDA_TRY(cudaLaunchKernelEx(
      &cfg, kern, m->row_ptr, m->col_idx, vals, x, y, pl.tile_row + t0, pl.tile_ptr + t0,
      static_cast<uint32_t>(count), geo.cap, geo.rcap, geo.stages,
      m->plan.n_long > 0 ? static_cast<uint32_t>(kLongRow) : 0xffffffffu,
      m->plan.n_long > 0 ? static_cast<const uint32_t *>(pl.tile_long + t0) : nullptr,
      long_holes(pl), x_bytes, pf_chunk, dot_part));
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

template <typename V, bool GF>
int dispatch_main(const csrk_matrix *m, int variant, int nx, const V *vals,
                  const V *x, V *y, cudaStream_t s, int64_t t0, int64_t t1);

template <typename V>
int dispatch_long(const csrk_matrix *m, int variant, int nx, const V *vals, const V *x, V *y,
                  cudaStream_t s, int64_t t0, int64_t t1) {
  if (m->plan.n_long == 0) return CSRK_OK;
  if (variant == CSRK_SERIAL) return launch_long_rows<V, 0>(m, vals, x, y, s, t0, t1);
  switch (nx) {
#define CSRK_LONG_CASE(N) \
  case N:                 \
    return launch_long_rows<V, N>(m, vals, x, y, s, t0, t1);
    CSRK_LONG_CASE(1)
    CSRK_LONG_CASE(2)
    CSRK_LONG_CASE(3)
    CSRK_LONG_CASE(4)
    CSRK_LONG_CASE(5)
    CSRK_LONG_CASE(6)
    CSRK_LONG_CASE(7)
    CSRK_LONG_CASE(8)
    CSRK_LONG_CASE(9)
    CSRK_LONG_CASE(10)
    CSRK_LONG_CASE(11)
    CSRK_LONG_CASE(12)
    CSRK_LONG_CASE(13)
    CSRK_LONG_CASE(14)
    CSRK_LONG_CASE(15)
    CSRK_LONG_CASE(16)
    CSRK_LONG_CASE(20)
    CSRK_LONG_CASE(24)
    CSRK_LONG_CASE(28)
    CSRK_LONG_CASE(32)
#undef CSRK_LONG_CASE
    default:
      return CSRK_OK;  // (the main dispatch reports the unsupported nx)
  }
}

// The long-row kernel runs beside the streaming kernel: forked onto a side
// stream after the streaming kernel is queued (the persistent CTAs are
// resident first; their carveout leaves room for two long-row blocks per SM,
// launch_stream) and joined back before the caller's stream continues.
// Power-law, 2 M rows, max row 20 k, queued -> beside: serial 503 -> 397 us,
// nx = 4 447 -> 335, nx = 32 654 -> 560 (profiles/r01_powerlaw_probe.txt).
// CSRK_LONG_SERIAL=1 queues it behind the streaming kernel instead.
constexpr size_t kMaxSides = 8;

template <typename V, bool GF>
int dispatch_nx(const csrk_matrix *m, int variant, int nx, const V *vals,
                const V *x, V *y, cudaStream_t s, int64_t t0, int64_t t1) {
  if (!long_beside(m, variant, nx)) {
    const int rc = dispatch_main<V, GF>(m, variant, nx, vals, x, y, s, t0, t1);
    if (rc != CSRK_OK) return rc;
    return dispatch_long<V>(m, variant, nx, vals, x, y, s, t0, t1);
  }
  // the caller stream's own side stream (created on first use; the caller
  // holds the matrix lock); past kMaxSides distinct caller streams the
  // long-row kernel queues on the caller's stream instead
  csrk_matrix *mm = const_cast<csrk_matrix *>(m);
  csrk_matrix::Side *sd = nullptr;
  for (auto &c : mm->sides)
    if (c.caller == s) sd = &c;
  if (!sd && mm->sides.size() < kMaxSides) {
    csrk_matrix::Side c;
    c.caller = s;
    CSRK_CUDA_TRY(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
    CSRK_CUDA_TRY(cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming));
    CSRK_CUDA_TRY(cudaEventCreateWithFlags(&c.join, cudaEventDisableTiming));
    mm->sides.push_back(c);
    sd = &mm->sides.back();
  }
  if (!sd) {
    const int rc = dispatch_main<V, GF>(m, variant, nx, vals, x, y, s, t0, t1);
    if (rc != CSRK_OK) return rc;
    return dispatch_long<V>(m, variant, nx, vals, x, y, s, t0, t1);
  }
  CSRK_CUDA_TRY(cudaEventRecord(sd->fork, s));
  CSRK_CUDA_TRY(cudaStreamWaitEvent(sd->side, sd->fork, 0));
  int rc = dispatch_main<V, GF>(m, variant, nx, vals, x, y, s, t0, t1);
  if (rc == CSRK_OK)
    rc = dispatch_long<V>(m, variant, nx, vals, x, y, sd->side, t0, t1);
  CSRK_CUDA_TRY(cudaEventRecord(sd->join, sd->side));
  CSRK_CUDA_TRY(cudaStreamWaitEvent(s, sd->join, 0));
  return rc;
}

template <typename V, bool GF>
int dispatch_main(const csrk_matrix *m, int variant, int nx, const V *vals,
                  const V *x, V *y, cudaStream_t s, int64_t t0, int64_t t1) {
  if (variant == CSRK_SERIAL) {
    // serial batch: 8 gathers per batch (the default), or 4 for
    // CSRK_SERIAL_BATCH=4 (template LB = 2; sweep knob for irregular short
    // rows, where batches of 8 leave ~40 % of the slots past the row end)
    static const int sb = [] {
      const char *e = std::getenv("CSRK_SERIAL_BATCH");
      return e ? std::atoi(e) : 8;
    }();
    if (sb == 4) return launch_stream<V, 0, GF, 2>(m, vals, x, y, s, t0, t1);
    if (sb == 7) return launch_stream<V, 0, GF, 7>(m, vals, x, y, s, t0, t1);
    return launch_stream<V, 0, GF>(m, vals, x, y, s, t0, t1);
  }
  // Lanes gather LB of their strided elements per batch: 8 when a lane holds
  // >= 5 of its row's nonzeros on average (27-point rows with nx = 4: C3
  // 5.81 -> 6.06 TB/s), 4 for short rows (C2 / C5 lose with 8: registers)
  int p = 1;
  while (p < nx) p <<= 1;
  const bool wide = m->plan.mean_short / p >= 5.0;
  switch (nx) {
#define CSRK_NX_CASE(N)                                          \
  case N:                                                        \
    return wide ? launch_stream<V, N, GF, 8>(m, vals, x, y, s, t0, t1) \
                : launch_stream<V, N, GF, 4>(m, vals, x, y, s, t0, t1);
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

namespace {

// Long rows and the cuts.  A row longer than the pitch pulls every cut that
// falls inside it onto the row after it: those tiles are empty (power-law,
// 2 M rows, max row 20 k: 17 k of 27 k tiles), and each still cost the
// producer a stage round trip.  A tile whose nonzeros (long rows included)
// exceed the stage ran in direct mode, its short rows read from global
// memory a thread each.  So, with long rows present: empty tiles are dropped,
// and a tile too big for its stage is cut around its long rows -- the
// pieces between them fit (their cost is at most the tile's), and a tile of
// one long row is left to the long-row kernel.  Host work on n_tiles and
// n_long sized arrays, once per plan.
int recut_long(csrk_matrix *m, int64_t tile_cost, int64_t cap, int64_t rcap,
               int64_t *n_tiles_io, bool *split, cudaStream_t s) {
  const int64_t n_tiles = *n_tiles_io, n_long = m->plan.n_long;
  std::vector<uint32_t> hr(n_tiles + 1), hp(n_tiles + 1), lr(n_long);
  std::vector<uint2> holes(n_long);
  CSRK_CUDA_TRY(cudaMemcpyAsync(hr.data(), m->plan.tile_row, hr.size() * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, s));
  CSRK_CUDA_TRY(cudaMemcpyAsync(hp.data(), m->plan.tile_ptr, hp.size() * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, s));
  CSRK_CUDA_TRY(cudaMemcpyAsync(lr.data(), long_rows_asc(m->plan), n_long * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, s));
  CSRK_CUDA_TRY(cudaMemcpyAsync(holes.data(), long_holes(m->plan), n_long * sizeof(uint2),
                                cudaMemcpyDeviceToHost, s));
  CSRK_CUDA_TRY(cudaStreamSynchronize(s));
  // 1. pieces: the base tiles minus empty ones, those too big for a stage
  //    cut around their long rows; pc = first nonzero of each cut
  std::vector<uint32_t> cut, pc;
  cut.reserve(n_tiles + 1);
  pc.reserve(n_tiles + 1);
  int64_t k = 0;
  for (int64_t t = 0; t < n_tiles; ++t) {
    const uint32_t a = hr[t], b = hr[t + 1];
    if (a == b) continue;
    cut.push_back(a);
    pc.push_back(hp[t]);
    if (static_cast<int64_t>(hp[t + 1] - hp[t]) <= cap) continue;
    uint32_t last = a;
    while (k < n_long && lr[k] < a) ++k;
    for (; k < n_long && lr[k] < b; ++k) {
      const uint32_t r = lr[k];
      if (r != last) cut.push_back(last = r), pc.push_back(holes[k].x);
      if (r + 1 < b) cut.push_back(last = r + 1), pc.push_back(holes[k].y);
    }
  }
  cut.push_back(static_cast<uint32_t>(m->n_rows));
  pc.push_back(hp[n_tiles]);
  // 2. greedy merge of consecutive pieces while the tile still fits a stage
  //    (nonzeros incl. long rows <= cap, rows <= rcap) and its staged cost
  //    (nonzeros excl. long rows + rows) stays within the tile cost: the
  //    pieces between long rows join up again instead of each costing the
  //    producer a stage round trip (power-law 20 k: 35 k -> fewer tiles)
  std::vector<uint32_t> out;
  out.reserve(cut.size());
  const size_t np = cut.size() - 1;
  size_t h = 0;  // holes cursor (row order)
  auto long_nnz = [&](uint32_t a, uint32_t b) {  // nonzeros of long rows in [a, b)
    int64_t sum = 0;
    while (h < static_cast<size_t>(n_long) && lr[h] < a) ++h;
    for (size_t q = h; q < static_cast<size_t>(n_long) && lr[q] < b; ++q)
      sum += holes[q].y - holes[q].x;
    return sum;
  };
  size_t st = 0;
  int64_t lsum = long_nnz(cut[0], cut[1]);
  out.push_back(cut[0]);
  for (size_t j = 1; j < np; ++j) {
    const int64_t lj = long_nnz(cut[j], cut[j + 1]);
    const int64_t span = static_cast<int64_t>(pc[j + 1]) - pc[st];
    const int64_t rows = static_cast<int64_t>(cut[j + 1]) - cut[st];
    if (span <= cap && rows <= rcap && span - lsum - lj + rows <= tile_cost) {
      lsum += lj;  // piece j joins the current tile
      continue;
    }
    out.push_back(cut[j]);
    st = j;
    lsum = lj;
  }
  out.push_back(static_cast<uint32_t>(m->n_rows));
  if (out.size() == hr.size() && std::equal(out.begin(), out.end(), hr.begin()))
    return CSRK_OK;  // nothing to change
  *split = true;
  const int64_t nt = static_cast<int64_t>(out.size()) - 1;
  cudaFree(m->plan.tile_row);
  m->plan.tile_row = m->plan.tile_ptr = m->plan.tile_long = nullptr;
  CSRK_CUDA_TRY(cudaMalloc(&m->plan.tile_row, 3 * (nt + 1) * sizeof(uint32_t)));
  m->plan.tile_ptr = m->plan.tile_row + (nt + 1);
  m->plan.tile_long = m->plan.tile_ptr + (nt + 1);
  CSRK_CUDA_TRY(cudaMemcpyAsync(m->plan.tile_row, out.data(), out.size() * sizeof(uint32_t),
                                cudaMemcpyHostToDevice, s));
  tile_ptr_kernel<<<static_cast<unsigned>((nt + 1 + 255) / 256), 256, 0, s>>>(
      m->row_ptr, m->plan.tile_row, nt, m->plan.tile_ptr);
  CSRK_CUDA_TRY(cudaGetLastError());
  CSRK_CUDA_TRY(cudaStreamSynchronize(s));  // `out` is pageable host memory
  *n_tiles_io = nt;
  return CSRK_OK;
}

}  // namespace

int ensure_plan(csrk_matrix *m, int64_t tile_cost, int64_t cap, int64_t stages,
                cudaStream_t s, bool force) {
  if (tile_cost <= 0) tile_cost = kDefaultTileCost;
  if (tile_cost < 32) tile_cost = 32;
  if (tile_cost > 65536) tile_cost = 65536;
  if (cap <= 0) cap = tile_cost + 256;
  if (cap < 16) cap = 16;
  if (stages <= 0) stages = kDefaultStages;
  if (stages > 8) stages = 8;
  // Row room per stage: a tile holds at most `cap` rows (cost = nonzeros +
  // rows), but only tiles of near-empty rows get close; half the room keeps
  // the stage -- and so the shared-memory carveout -- small enough to leave
  // L1 for the x gathers, and a tile with more rows runs in direct mode.
  // CSRK_RCAP_DIV overrides the divisor (plan sweeps).
  int64_t rdiv = 2;
  if (const char *e = std::getenv("CSRK_RCAP_DIV")) rdiv = std::max(1, std::atoi(e));
  const int64_t rcap = std::max<int64_t>(16, cap / rdiv);
  const Geometry geo(static_cast<uint32_t>(cap), static_cast<uint32_t>(rcap),
                     static_cast<uint32_t>(stages), sizeof(double));
  if (geo.total_bytes() > 227 * 1024) {
    set_error("tile plan needs %u bytes of shared memory (> 227 KB)",
              geo.total_bytes());
    return CSRK_EINVAL;
  }
  if (!force && m->plan.tile_row && m->plan.tile_cost == tile_cost && m->plan.cap == cap &&
      m->plan.rcap == rcap && m->plan.stages == stages)
    return CSRK_OK;
  if (m->sm_count == 0) {
    int dev = 0;
    CSRK_CUDA_TRY(cudaGetDevice(&dev));
    CSRK_CUDA_TRY(cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount,
                                         dev));
  }
  if (m->n_rows > 0 && !m->plan.row_stats) {
    unsigned long long *d = nullptr, h = 0;
    keep_async_pool();

    CSRK_CUDA_TRY(cudaMallocAsync(&d, sizeof(h), s));
    CSRK_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(h), s));
    row_sq_kernel<<<148 * 8, 256, 0, s>>>(m->row_ptr, m->n_rows, d);
    CSRK_CUDA_TRY(cudaGetLastError());
    CSRK_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFreeAsync(d, s);
    const double mean = static_cast<double>(m->nnz) / static_cast<double>(m->n_rows);
    m->plan.mean_row = mean;
    m->plan.mean_short = mean;
    m->plan.row_var = static_cast<double>(h) / static_cast<double>(m->n_rows) - mean * mean;
    m->plan.row_stats = true;
    // rows longer than kLongRow: listed once for the long-row kernel
    unsigned long long *dn = nullptr, hn = 0;
    CSRK_CUDA_TRY(cudaMallocAsync(&dn, sizeof(hn), s));
    CSRK_CUDA_TRY(cudaMemsetAsync(dn, 0, sizeof(hn), s));
    long_rows_list_kernel<<<148 * 8, 256, 0, s>>>(m->row_ptr, m->n_rows,
                                                   static_cast<uint32_t>(kLongRow), nullptr, dn);
    CSRK_CUDA_TRY(cudaGetLastError());
    CSRK_CUDA_TRY(cudaMemcpyAsync(&hn, dn, sizeof(hn), cudaMemcpyDeviceToHost, s));
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    if (hn > 0) {
      const int64_t n = static_cast<int64_t>(hn);
      CSRK_CUDA_TRY(cudaMalloc(&m->plan.long_rows, (4 * n + 1) * sizeof(uint32_t)));
      m->plan.n_long = n;
      CSRK_CUDA_TRY(cudaMemsetAsync(dn, 0, sizeof(hn), s));
      long_rows_list_kernel<<<148 * 8, 256, 0, s>>>(m->row_ptr, m->n_rows,
                                                     static_cast<uint32_t>(kLongRow),
                                                     m->plan.long_rows, dn);
      CSRK_CUDA_TRY(cudaGetLastError());
      // holes in row order, then the work order
      uint64_t *keys = nullptr, *tk = nullptr;
      uint32_t *vals = nullptr, *tv = nullptr;
      keep_async_pool();
      CSRK_CUDA_TRY(cudaMallocAsync(&keys, 2 * n * sizeof(uint64_t), s));
      CSRK_CUDA_TRY(cudaMallocAsync(&vals, 2 * n * sizeof(uint32_t), s));
      tk = keys + n;
      tv = vals + n;
      const unsigned gb = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 8));
      int rc = CSRK_OK;
      for (int by_len = 0; by_len < 2 && rc == CSRK_OK; ++by_len) {
        long_keys_kernel<<<gb, 256, 0, s>>>(m->row_ptr, m->plan.long_rows, n, by_len, keys,
                                            vals);
        rc = radix_sort_pairs(keys, vals, tk, tv, n, 0, by_len ? 64 : 32, s);
        if (rc == CSRK_OK && !by_len) {
          holes_kernel<<<gb, 256, 0, s>>>(m->row_ptr, vals, n,
                                          const_cast<uint2 *>(long_holes(m->plan)));
          CSRK_CUDA_TRY(cudaMemcpyAsync(const_cast<uint32_t *>(long_rows_asc(m->plan)), vals,
                                        n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        }
      }
      if (rc == CSRK_OK)
        CSRK_CUDA_TRY(cudaMemcpyAsync(m->plan.long_rows, vals, n * sizeof(uint32_t),
                                      cudaMemcpyDeviceToDevice, s));
      unsigned long long hl = 0;
      if (rc == CSRK_OK) {  // the short rows' mean length (strided schedule choices)
        CSRK_CUDA_TRY(cudaMemsetAsync(dn, 0, sizeof(hn), s));
        hole_sum_kernel<<<gb, 256, 0, s>>>(long_holes(m->plan), n, dn);
        CSRK_CUDA_TRY(cudaMemcpyAsync(&hl, dn, sizeof(hl), cudaMemcpyDeviceToHost, s));
      }
      cudaFreeAsync(keys, s);
      cudaFreeAsync(vals, s);
      CSRK_TRY(rc);
      CSRK_CUDA_TRY(cudaGetLastError());
      CSRK_CUDA_TRY(cudaStreamSynchronize(s));
      if (m->n_rows > n)
        m->plan.mean_short = static_cast<double>(m->nnz - static_cast<int64_t>(hl)) /
                             static_cast<double>(m->n_rows - n);
    }
    cudaFreeAsync(dn, s);
    m->plan.n_long = static_cast<int64_t>(hn);
  }
  const int64_t n_groups = m->k == 3 ? m->n_ssr : (m->k == 2 ? m->n_sr : m->n_rows);
  // cut on group boundaries when every group is small against a tile
  int cut_k = 1;
  int64_t n_cuts = m->n_rows;
  int64_t max_group = 0;
  if (m->k >= 2 && n_groups > 0) {
    unsigned long long *d = nullptr, h = 0;
    keep_async_pool();

    CSRK_CUDA_TRY(cudaMallocAsync(&d, sizeof(h), s));
    CSRK_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(h), s));
    int64_t blocks = (n_groups + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    max_group_cost_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
        m->row_ptr, m->sr_ptr, m->ssr_ptr, m->k, n_groups, m->n_rows, d);
    CSRK_CUDA_TRY(cudaGetLastError());
    CSRK_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
    CSRK_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFreeAsync(d, s);
    // Group-aligned cuts (the paper's block <-> SSR mapping) shrink the
    // pitch by the largest group so every tile fits its stage; beyond an
    // eighth of a tile that costs more than the alignment is worth
    // (natural-order 7-point 256^3 with 64-row SSRs: 6.27 TB/s aligned,
    // 6.71 TB/s cut on rows, profiles/r01_sched_sweep.txt), so large groups
    // are cut on rows -- results do not depend on the cuts.
    const int mode = m->plan.cut_mode;
    if (mode == 2 || (mode == 0 && static_cast<int64_t>(h) * 8 <= tile_cost)) {
      cut_k = m->k;
      n_cuts = n_groups;
      max_group = static_cast<int64_t>(h);
    }
  }
  // A tile runs from the first cut at or past t * pitch to the first cut at
  // or past (t + 1) * pitch, so it costs less than pitch + (largest group).
  // Group cuts use pitch = tile_cost - largest group: every tile then fits
  // the stage.  Row cuts keep pitch = tile_cost; the stage's slack
  // (cap - tile_cost) covers the row that crosses a boundary.
  // (a group larger than the tile: one group per tile, direct mode when it
  // exceeds the stage -- reachable only with cut mode 2)
  // (a group of more than 3/4 of a tile cannot share a stage with its
  // neighbours: such tiles run direct, and the pitch stays at least one
  // tile so the tile count does not explode -- a pitch of 1 made C3's
  // 200-row SSRs 196 M mostly empty tiles)
  int64_t pitch = tile_cost;
  if (cut_k != 1)
    pitch = tile_cost - max_group >= tile_cost / 4 ? tile_cost - max_group
                                                   : std::max(tile_cost, max_group);
  const int64_t total_cost = m->nnz + m->n_rows;
  int64_t n_tiles = (total_cost + pitch - 1) / pitch;
  if (n_tiles > 0x7fffffffLL) {
    set_error("too many tiles (%lld)", static_cast<long long>(n_tiles));
    return CSRK_EINVAL;
  }
  if (m->plan.tile_row) {
    CSRK_CUDA_TRY(cudaFree(m->plan.tile_row));
    m->plan.tile_row = nullptr;
    m->plan.tile_ptr = m->plan.tile_long = nullptr;
  }
  // one allocation: tile_row, tile_ptr, tile_long (n_tiles + 1 each)
  CSRK_CUDA_TRY(cudaMalloc(&m->plan.tile_row, 3 * (n_tiles + 1) * sizeof(uint32_t)));
  m->plan.tile_ptr = m->plan.tile_row + (n_tiles + 1);
  m->plan.tile_long = m->plan.tile_ptr + (n_tiles + 1);
  int64_t blocks = (n_tiles + 1 + 255) / 256;
  tile_bounds_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
      m->row_ptr, m->sr_ptr, m->ssr_ptr, cut_k, n_cuts, m->n_rows, pitch,
      n_tiles, m->plan.tile_row);
  tile_ptr_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
      m->row_ptr, m->plan.tile_row, n_tiles, m->plan.tile_ptr);
  CSRK_CUDA_TRY(cudaGetLastError());
  bool split = false;
  if (m->plan.n_long > 0) {
    CSRK_TRY(recut_long(m, tile_cost, cap, rcap, &n_tiles, &split, s));
    blocks = (n_tiles + 1 + 255) / 256;
  }
  if (m->plan.n_long > 0)
    tile_long_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
        m->plan.tile_ptr, n_tiles, long_holes(m->plan),
        m->plan.n_long, m->plan.tile_long);
  CSRK_CUDA_TRY(cudaGetLastError());
  m->pipe.plan_tiles = -1;  // host-pipeline cuts index the old tiles
  ++m->plan.gen;
  m->plan.tile_cost = tile_cost;
  m->plan.cap = cap;
  m->plan.rcap = rcap;
  m->plan.stages = stages;
  m->plan.n_tiles = n_tiles;
  m->plan.group_aligned = (cut_k != 1 || m->k == 1) && !split;
  return CSRK_OK;
}

int prepare_plan(const csrk_matrix *cm, int value_type, int variant, int nx) {
  csrk_matrix *m = const_cast<csrk_matrix *>(cm);  // the plan is a cache
  if (m->n_rows == 0) return CSRK_OK;
  if (!m->plan.row_stats) CSRK_TRY(ensure_plan(m, 0, 0, 0, m->stream));
  if (!m->plan.auto_tile) return CSRK_OK;
  const bool deep = small_tiles(m->plan.row_var, m->plan.n_long, m->plan.mean_short);
  const int64_t tc = auto_tile_cost(m->plan.mean_short, variant, nx,
                                    deep ? kDeepRingTileCost : kDefaultTileCost);
  const int64_t st = auto_stages(m->plan.row_var, m->plan.n_long);
  if (tc != m->plan.tile_cost || st != m->plan.stages) {
    const bool keep = m->plan.auto_tile;
    CSRK_TRY(ensure_plan(m, tc, 0, st, m->stream));
    m->plan.auto_tile = keep;
    CSRK_CUDA_TRY(cudaStreamSynchronize(m->stream));
  }
  return CSRK_OK;
}

int chunk_max_cols(const csrk_matrix *m, const uint32_t *row_cut_dev, int chunks,
                   uint32_t *out_dev, cudaStream_t s) {
  chunk_max_col_kernel<<<chunks, 256, 0, s>>>(m->row_ptr, m->col_idx, row_cut_dev,
                                             out_dev);
  CSRK_CUDA_TRY(cudaGetLastError());
  return CSRK_OK;
}

// y = A x with the CTA partials of x . y written to dot_part[0, grid) (the
// CG's p . Ap): fused into the streaming kernel for whole
// launches in the serial order with inline gathers and no long rows -- the
// dot kernel then need not re-read x and y (2 n values per iteration).
// *fused = false (and nothing launched) otherwise; the caller runs the
// plain SpMV and its own dot.
int launch_spmv_dot(const csrk_matrix *m, int value_type, int variant, int nx,
                    const void *x, void *y, cudaStream_t stream, double *dot_part,
                    int64_t dot_slots, bool *fused) {
  *fused = false;
  if (variant != CSRK_SERIAL || m->n_rows == 0 || !m->plan.tile_row || m->plan.n_long > 0 ||
      std::getenv("CSRK_NO_FUSED_DOT"))
    return CSRK_OK;
  if (value_type == CSRK_F64) {
    if (!m->vals64) return CSRK_OK;
    const int g = m->plan.gather_first;
    if (g == 1 || (g == kGatherAuto && auto_gather(variant, nx, m->plan.mean_row, m->plan.row_var)))
      return CSRK_OK;
    *fused = true;
    return launch_stream<double, 0, false, 4, true>(
        m, m->vals64, static_cast<const double *>(x), static_cast<double *>(y), stream, 0,
        m->plan.n_tiles, dot_part, dot_slots);
  }
  // fp32: the separate dot kernel.  The fused epilogue's per-row fp64 work
  // (two F2F.F64.F32, a DMUL, a DADD and the x[r] load) slows the fp32
  // streaming kernel by more than the dot kernel's re-read of p and Ap
  // costs: C4 512^3 SpMV 1425.5 us + dot 165.6 us vs 1643.6 us fused (ncu),
  // 2.458 vs 2.497 ms per CG iteration (profiles/r02_c4_f32_split.txt).
  // CSRK_FUSED_DOT_F32=1 keeps the fused launch for fp32.
  if (value_type == CSRK_F32) {
    const char *f = std::getenv("CSRK_FUSED_DOT_F32");
    if (!m->vals32 || !(f && f[0] == '1')) return CSRK_OK;
    *fused = true;
    return launch_stream<float, 0, false, 4, true>(
        m, m->vals32, static_cast<const float *>(x), static_cast<float *>(y), stream, 0,
        m->plan.n_tiles, dot_part, dot_slots);
  }
  return CSRK_OK;
}

int launch_spmv(const csrk_matrix *m, int value_type, int variant, int nx,
                const void *x, void *y, cudaStream_t stream, int64_t t0,
                int64_t t1) {
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
    const int g = m->plan.gather_first;
    if (g == 1 || (g == kGatherAuto && auto_gather(variant, nx, m->plan.mean_row, m->plan.row_var)))
      return dispatch_nx<double, true>(m, variant, nx, m->vals64,
                                       static_cast<const double *>(x),
                                       static_cast<double *>(y), stream, t0, t1);
    return dispatch_nx<double, false>(m, variant, nx, m->vals64,
                               static_cast<const double *>(x),
                               static_cast<double *>(y), stream, t0, t1);
  }
  if (value_type == CSRK_F32) {
    if (!m->vals32) {
      set_error("matrix holds no float32 values");
      return CSRK_EINVAL;
    }
    return dispatch_nx<float, false>(m, variant, nx, m->vals32,
                              static_cast<const float *>(x),
                              static_cast<float *>(y), stream, t0, t1);
  }
  set_error("unknown value type %d", value_type);
  return CSRK_EINVAL;
}

}  // namespace csrk

#if CSRK_TIMELINE
extern "C" int csrk_debug_timeline(unsigned long long *out, int n_ctas) {
  if (!out || n_ctas < 0) return CSRK_EINVAL;
  if (n_ctas > csrk::kTlCtas) n_ctas = csrk::kTlCtas;
  return cudaMemcpyFromSymbol(out, csrk::g_timeline,
                              sizeof(unsigned long long) * csrk::kTlSlots * n_ctas) ==
                 cudaSuccess
             ? CSRK_OK
             : CSRK_ECUDA;
}
#endif
