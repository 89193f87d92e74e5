// Probe: random 8-byte gathers from a 40 MB vector, LDG vs TMA tile::gather4
// (sm_100a).  Each gather4 fetches four 32-byte rows (x viewed as n/4 rows of
// 4 doubles, one L2 sector each) into 128 bytes of shared memory.  Prints gathers/s and lines per SM-cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather_probe tma_gather_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void ldg_kernel(const double *__restrict__ x, const uint32_t *__restrict__ idx,
                           int64_t m, double *__restrict__ out) {
  double acc = 0.0;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i + 7 * st < m; i += 8 * st) {
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = idx[i + j * st];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += __ldg(x + c[j]);
  }
  for (; i < m; i += st) acc += __ldg(x + idx[i]);
  if (acc == 12345.678) out[0] = acc;
}

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kChunk = 1024;          // gathers per stage
constexpr int kStages = 2;
constexpr int kCons = 4;              // consumer warps

__global__ void __launch_bounds__(32 * (1 + kCons))
tma_kernel(const __grid_constant__ CUtensorMap tmap, const uint32_t *__restrict__ idx,
           int64_t m, double *__restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = (uint64_t *)smem;
  uint64_t *empty = full + kStages;
  double *buf = (double *)(smem + 128);  // kStages * kChunk * 4 doubles (32-byte rows)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(kCons));
    }
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  const int64_t n_chunks = (m + kChunk - 1) / kChunk;
  if (warp == 0) {
    int it = 0;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x, ++it) {
      const int s = it % kStages;
      if (it >= kStages) {
        const uint32_t ph = ((it / kStages) + 1) & 1;
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sa(&empty[s])), "r"(ph));
      }
      const int64_t base = c * kChunk;
      const int cnt = (int)((m - base) < kChunk ? (m - base) : kChunk);
      const int groups = (cnt + 3) / 4;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(groups * 128));
      __syncwarp();
      constexpr int kPer = kChunk / 4 / 32;  // gather4s per lane per chunk
      int r[kPer][4];
#pragma unroll
      for (int k = 0; k < kPer; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t q = base + 4 * (lane + 32 * k) + j;
          r[k][j] = (int)(idx[q < m ? q : base] >> 2);  // all index loads in flight at once
        }
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int g = lane + 32 * k;
        if (g >= groups) break;
        double *dst = buf + ((size_t)s * kChunk + 4 * g) * 4;  // 128-byte aligned
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     :: "r"(sa(dst)), "l"(&tmap), "r"(0), "r"(r[k][0]), "r"(r[k][1]), "r"(r[k][2]), "r"(r[k][3]), "r"(sa(&full[s])) : "memory");
      }
    }
    return;
  }
  double acc = 0.0;
  int it = 0;
  const int ct = tid - 32;
  for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x, ++it) {
    const int s = it % kStages;
    const uint32_t ph = (it / kStages) & 1;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sa(&full[s])), "r"(ph));
    const int64_t base = c * kChunk;
    const int cnt = (int)((m - base) < kChunk ? (m - base) : kChunk);
    for (int p = ct; p < cnt; p += 32 * kCons) {
      const uint32_t col = idx[base + p];
      acc += buf[((size_t)s * kChunk + p) * 4 + (col & 3)];
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])));
  }
  if (acc == 12345.678) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
  const int64_t n = 5000000;            // x: 40 MB of doubles
  const int64_t m = 50000000;           // gathers
  const int window = argc > 1 ? atoi(argv[1]) : 65536;  // +- window around a moving centre (0 = uniform)
  std::vector<uint32_t> h(m);
  std::mt19937_64 rng(1);
  for (int64_t i = 0; i < m; ++i) {
    if (window == 0) { h[i] = rng() % n; continue; }
    int64_t centre = i / 10;  // ~10 gathers per row, rows in order
    int64_t c = centre + (int64_t)(rng() % (2 * window + 1)) - window;
    h[i] = (uint32_t)(c < 0 ? 0 : (c >= n ? n - 1 : c));
  }
  double *x, *out; uint32_t *idx;
  CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&idx, m * 4));
  CK(cudaMemset(x, 0, n * 8));
  CK(cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int blocksPerSm : {4, 8, 16}) {
    for (int r = 0; r < 2; ++r) ldg_kernel<<<sms * blocksPerSm, 256>>>(x, idx, m, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) ldg_kernel<<<sms * blocksPerSm, 256>>>(x, idx, m, out);
    cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("LDG   window %d blocks/SM %2d: %.1f us  %.2f Ggathers/s  %.2f gathers/SM-cycle\n", window, blocksPerSm,
           ms * 1e3, m / (ms * 1e-3) / 1e9, m / (ms * 1e-3) / (sms * clk * 1e3));
  }
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q));
  CUtensorMap tmap;
  cuuint64_t dims[2] = {4, (cuuint64_t)(n / 4)};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {4, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
  const size_t smem = 128 + (size_t)kStages * kChunk * 32;
  CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int blocksPerSm : {1, 2, 3, 4}) {
    for (int r = 0; r < 2; ++r) tma_kernel<<<sms * blocksPerSm, 32 * (1 + kCons), smem>>>(tmap, idx, m, out);
    CK(cudaGetLastError());
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) tma_kernel<<<sms * blocksPerSm, 32 * (1 + kCons), smem>>>(tmap, idx, m, out);
    cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("TMA4  window %d blocks/SM %2d: %.1f us  %.2f Ggathers/s  %.2f gathers/SM-cycle\n", window, blocksPerSm,
           ms * 1e3, m / (ms * 1e-3) / 1e9, m / (ms * 1e-3) / (sms * clk * 1e3));
  }
  return 0;
}
