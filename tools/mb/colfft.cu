// Microbenchmark (diagnostics, not product): the four-step column pass (load a column tile
// of a complex [L1][L2] fp32 array, 2048-point column FFTs, store) under different
// schedules: lockstep 2 x 256-thread CTAs per SM (the grid tier today) vs one 512-thread CTA
// with two tile buffers whose loads run under the previous tile's FFT.
#include <cstdio>
#include <cstdint>
#include "../../paper_1509_03979_b200/csrc/cs_common.cuh"
#include "../../paper_1509_03979_b200/csrc/fft_cta.cuh"
using namespace cs;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
constexpr int L1 = 2048, L2 = 4096, LOG2L1 = 11;
__device__ __forceinline__ void cpa8(void* s, const void* g) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cpcommit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cpwaitn() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int CT, int LOG2NT, bool DB, bool DOFFT>
__global__ void __launch_bounds__(1 << LOG2NT) k_col(const float2* __restrict__ in, float2* __restrict__ out) {
  constexpr int LCT = CT == 2 ? 1 : CT == 4 ? 2 : 3;
  constexpr int tile = L1 * CT, ntiles = L2 / CT;
  constexpr int NT = 1 << LOG2NT;
  float2* tlo = reinterpret_cast<float2*>(cs_smem_base);
  float2* thi = tlo + 64;
  float2* sb0 = thi + L1 / 64;
  for (int i = threadIdx.x; i < 64 + L1 / 64; i += NT) {
    const int m = i < 64 ? i : (i - 64) * 64;
    double s, c;
    sincospi(-2.0 * m / L1, &s, &c);
    (i < 64 ? tlo[i] : thi[i - 64]) = make_float2((float)c, (float)s);
  }
  const TwTable<float> tw{tlo, thi};
  auto issue = [&](int t, float2* sb) {
    const int c0 = t * CT;
    for (int e = threadIdx.x; e < tile; e += NT)
      cpa8(&sb[swz<float>(e)], &in[(size_t)(e >> LCT) * L2 + c0 + (e & (CT - 1))]);
  };
  int buf = 0;
  if (DB && blockIdx.x < ntiles) issue(blockIdx.x, sb0);
  cpcommit();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    float2* sb = sb0 + (DB ? buf * tile : 0);
    if (DB) {
      const int tn = t + gridDim.x;
      if (tn < ntiles) issue(tn, sb0 + (buf ^ 1) * tile);
      cpcommit();
      cpwaitn<1>();
    } else {
      issue(t, sb);
      cpcommit();
      cpwaitn<0>();
    }
    __syncthreads();
    if (DOFFT) fft_cta_t<float, LOG2L1, fft_log2e(LOG2L1, LCT, LOG2NT), LCT, false>(sb, tw);
    const int c0 = t * CT;
    for (int p = threadIdx.x; p < tile / 2; p += NT) {
      const int e = 2 * p;
      float2 a = sb[swz<float>(e)], b = sb[swz<float>(e + 1)];
      *reinterpret_cast<float4*>(&out[(size_t)(e >> LCT) * L2 + c0 + (e & (CT - 1))]) = make_float4(a.x, a.y, b.x, b.y);
    }
    __syncthreads();
    buf ^= 1;
  }
}
template <class F> float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  const int R = 20;
  for (int i = 0; i < R; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / R;
}
int main() {
  const size_t n = (size_t)L1 * L2;
  float2 *in, *out;
  CK(cudaMalloc(&in, n * 8)); CK(cudaMalloc(&out, n * 8));
  CK(cudaMemset(in, 0, n * 8));
  const double bytes = 2.0 * n * 8;
  auto rep = [&](const char* name, float us) { printf("%-52s %8.1f us  %7.0f GB/s\n", name, us, bytes / us / 1e3); };
  const int tb = (64 + L1 / 64) * 8;
#define RUN(NAME, KER, GRID, NT, SMEM) \
  CK(cudaFuncSetAttribute(KER, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM)); \
  rep(NAME, timeit([&] { KER<<<GRID, NT, SMEM>>>(in, out); })); CK(cudaGetLastError());
  RUN("copy only: CT4 lockstep 296x256", (k_col<4, 8, false, false>), 296, 256, 64 * 1024 + tb);
  RUN("FFT: CT4 lockstep 296x256 (grid tier today)", (k_col<4, 8, false, true>), 296, 256, 64 * 1024 + tb);
  RUN("FFT: CT4 lockstep 148x512", (k_col<4, 9, false, true>), 148, 512, 64 * 1024 + tb);
  RUN("FFT: CT4 lockstep 296x512", (k_col<4, 9, false, true>), 296, 512, 64 * 1024 + tb);
  RUN("copy only: CT4 dbuf 148x512", (k_col<4, 9, true, false>), 148, 512, 128 * 1024 + tb);
  RUN("FFT: CT4 dbuf 148x512", (k_col<4, 9, true, true>), 148, 512, 128 * 1024 + tb);
  RUN("FFT: CT4 dbuf 148x256", (k_col<4, 8, true, true>), 148, 256, 128 * 1024 + tb);
  RUN("FFT: CT8 lockstep 148x512", (k_col<8, 9, false, true>), 148, 512, 128 * 1024 + tb);
  RUN("FFT: CT2 dbuf 296x256", (k_col<2, 8, true, true>), 296, 256, 64 * 1024 + tb);
  RUN("FFT: CT2 lockstep 592x256", (k_col<2, 8, false, true>), 592, 256, 32 * 1024 + tb);
  return 0;
}
