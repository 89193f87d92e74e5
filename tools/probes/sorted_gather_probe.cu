// Probe: do column-sorted gathers beat the L1TEX line rate on a C5-like
// matrix?  x = 5 M doubles (40 MB, L2-resident); 50 M gathers, row i
// reading ~10 columns i + U[-65536, 65536] (the C5 generator's reach), in
// CSR order (what the streaming kernel issues) or sorted by column within
// panels of R consecutive rows (a per-panel gather order precomputed once
// per matrix).  Same LDG kernel for all: 8 independent __ldg per thread in
// flight, consecutive lanes on consecutive list entries.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sorted_gather_probe sorted_gather_probe.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <bool NA>
__global__ void ldg_kernel(const double *__restrict__ x, const uint32_t *__restrict__ idx,
                           int64_t m, double *__restrict__ out) {
  double acc = 0.0;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i + 7 * st < m; i += 8 * st) {
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = __ldcs(idx + i + j * st);
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (NA) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[j]) : "l"(x + c[j]));
      else v[j] = __ldg(x + c[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j];
  }
  for (; i < m; i += st) acc += __ldg(x + idx[i]);
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const int64_t n = 5000000;
  std::vector<uint32_t> rp(n + 1), ci;
  ci.reserve(55000000);
  uint64_t s = 88172645463325252ull;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
  for (int64_t r = 0; r < n; ++r) {
    rp[r] = (uint32_t)ci.size();
    const int len = 1 + (int)(rnd() % 19);
    for (int k = 0; k < len; ++k) {
      int64_t c = k == 0 ? r : r + (int64_t)(rnd() % 131073) - 65536;
      c = c < 0 ? 0 : (c >= n ? n - 1 : c);
      ci.push_back((uint32_t)c);
    }
  }
  rp[n] = (uint32_t)ci.size();
  const int64_t m = (int64_t)ci.size();
  double *x; uint32_t *idx; double *out;
  CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&idx, m * 4)); CK(cudaMalloc(&out, 8));
  CK(cudaMemset(x, 0, n * 8));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int panels[] = {1, 200, 1000, 2000, 4000, 8000, 32000};
  for (int R : panels) {
    std::vector<uint32_t> v(ci);
    if (R > 1)
      for (int64_t r0 = 0; r0 < n; r0 += R) {
        const int64_t r1 = std::min<int64_t>(n, r0 + R);
        std::sort(v.begin() + rp[r0], v.begin() + rp[r1]);
      }
    CK(cudaMemcpy(idx, v.data(), m * 4, cudaMemcpyHostToDevice));
    for (int na = 0; na < 2; ++na)
      for (int bps : {4, 8}) {
        const int grid = sms * bps;
        for (int w = 0; w < 3; ++w) {
          if (na) ldg_kernel<true><<<grid, 256>>>(x, idx, m, out);
          else ldg_kernel<false><<<grid, 256>>>(x, idx, m, out);
        }
        CK(cudaEventRecord(e0));
        const int reps = 20;
        for (int w = 0; w < reps; ++w) {
          if (na) ldg_kernel<true><<<grid, 256>>>(x, idx, m, out);
          else ldg_kernel<false><<<grid, 256>>>(x, idx, m, out);
        }
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= reps;
        printf("panel %6d rows %s blocks/SM %d: %7.1f us  %6.1f Ggathers/s  %.2f gathers/SM-cycle\n", R,
               na ? "no_allocate" : "ldg        ", bps, ms * 1e3, m / (ms * 1e-3) / 1e9,
               m / (ms * 1e-3) / (sms * (clk * 1e3)));
      }
  }
  return 0;
}
