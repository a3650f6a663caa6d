// Microbenchmark (diagnostics, not product): moving column tiles of a complex [L1][L2]
// fp32 array (the four-step's pass A / C memory pattern) under different tilings.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
constexpr int L1 = 2048, L2 = 4096;
extern __shared__ __align__(16) unsigned char smem[];
__device__ __forceinline__ int swz(int a) { return a ^ (((a >> 4) ^ (a >> 5)) & 15); }
__device__ __forceinline__ void cpa8(void* s, const void* g) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa16(void* s, const void* g) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cpwait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cpcommit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cpwaitn() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// V1: current pattern. CT columns, 8-byte cp.async into swizzled smem, lockstep
template <int CT, bool B16>
__global__ void k_tile(const float2* __restrict__ in, float2* __restrict__ out) {
  float2* sb = reinterpret_cast<float2*>(smem);
  constexpr int LCT = CT == 2 ? 1 : CT == 4 ? 2 : CT == 8 ? 3 : 4;
  constexpr int tile = L1 * CT, ntiles = L2 / CT;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int c0 = t * CT;
    if (B16) {
      for (int p = threadIdx.x; p < tile / 2; p += blockDim.x) {
        const int e = 2 * p;
        cpa16(&sb[e], &in[(size_t)(e >> LCT) * L2 + c0 + (e & (CT - 1))]);
      }
    } else {
      for (int e = threadIdx.x; e < tile; e += blockDim.x)
        cpa8(&sb[swz(e)], &in[(size_t)(e >> LCT) * L2 + c0 + (e & (CT - 1))]);
    }
    cpwait();
    __syncthreads();
    for (int p = threadIdx.x; p < tile / 2; p += blockDim.x) {
      const int e = 2 * p;
      float2 a = B16 ? sb[e] : sb[swz(e)], b = B16 ? sb[e + 1] : sb[swz(e + 1)];
      *reinterpret_cast<float4*>(&out[(size_t)(e >> LCT) * L2 + c0 + (e & (CT - 1))]) = make_float4(a.x, a.y, b.x, b.y);
    }
    __syncthreads();
  }
}
// V4: double-buffered (two tiles in smem): loads of tile t+grid in flight while tile t is stored
template <int CT>
__global__ void k_tile_db(const float2* __restrict__ in, float2* __restrict__ out) {
  float2* sb0 = reinterpret_cast<float2*>(smem);
  constexpr int LCT = CT == 2 ? 1 : CT == 4 ? 2 : CT == 8 ? 3 : 4;
  constexpr int tile = L1 * CT, ntiles = L2 / CT;
  auto issue = [&](int t, float2* sb) {
    const int c0 = t * CT;
    for (int p = threadIdx.x; p < tile / 2; p += blockDim.x) {
      const int e = 2 * p;
      cpa16(&sb[e], &in[(size_t)(e >> LCT) * L2 + c0 + (e & (CT - 1))]);
    }
  };
  int t = blockIdx.x, buf = 0;
  if (t < ntiles) issue(t, sb0);
  cpcommit();
  for (; t < ntiles; t += gridDim.x) {
    const int tn = t + gridDim.x;
    float2* sb = sb0 + buf * tile;
    if (tn < ntiles) issue(tn, sb0 + (buf ^ 1) * tile);
    cpcommit();
    cpwaitn<1>();
    __syncthreads();
    const int c0 = t * CT;
    for (int p = threadIdx.x; p < tile / 2; p += blockDim.x) {
      const int e = 2 * p;
      float2 a = sb[e], b = sb[e + 1];
      *reinterpret_cast<float4*>(&out[(size_t)(e >> LCT) * L2 + c0 + (e & (CT - 1))]) = make_float4(a.x, a.y, b.x, b.y);
    }
    __syncthreads();
    buf ^= 1;
  }
}
// V6: plain stream copy
__global__ void k_copy(const float4* __restrict__ in, float4* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
}
// V7: row-pair copy (pass B pattern): items i < L1/2: rows i and L1-i, contiguous 32 KB each
__global__ void k_rows(const float2* __restrict__ in, float2* __restrict__ out) {
  float2* sb = reinterpret_cast<float2*>(smem);
  for (int it = blockIdx.x; it <= L1 / 2; it += gridDim.x) {
    const int ka = it, kb = (L1 - it) & (L1 - 1);
    for (int p = threadIdx.x; p < L2; p += blockDim.x) {  // 2 rows x L2/2 pairs
      const int r = p >= L2 / 2, q = p - r * (L2 / 2);
      cpa16(&sb[2 * p], &in[(size_t)(r ? kb : ka) * L2 + 2 * q]);
    }
    cpwait();
    __syncthreads();
    for (int p = threadIdx.x; p < L2; p += blockDim.x) {
      const int r = p >= L2 / 2, q = p - r * (L2 / 2);
      *reinterpret_cast<float4*>(&out[(size_t)(r ? kb : ka) * L2 + 2 * q]) = *reinterpret_cast<float4*>(&sb[2 * p]);
    }
    __syncthreads();
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
  auto rep = [&](const char* name, float us) { printf("%-44s %8.1f us  %7.0f GB/s\n", name, us, bytes / us / 1e3); };
  rep("stream copy float4 (1184 x 256)", timeit([&] { k_copy<<<148 * 8, 256>>>((const float4*)in, (float4*)out, n / 2); }));
#define RUN(NAME, KER, GRID, NT, SMEM) \
  CK(cudaFuncSetAttribute(KER, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM)); \
  rep(NAME, timeit([&] { KER<<<GRID, NT, SMEM>>>(in, out); })); CK(cudaGetLastError());
  RUN("CT4 8B swz 296x256 (current)", (k_tile<4, false>), 296, 256, 64 * 1024 + 16);
  RUN("CT4 16B 296x256", (k_tile<4, true>), 296, 256, 64 * 1024 + 16);
  RUN("CT4 16B 296x512", (k_tile<4, true>), 296, 512, 64 * 1024 + 16);
  RUN("CT8 16B 148x512", (k_tile<8, true>), 148, 512, 128 * 1024 + 16);
  RUN("CT8 16B 148x1024", (k_tile<8, true>), 148, 1024, 128 * 1024 + 16);
  RUN("CT2 16B 592x256", (k_tile<2, true>), 592, 256, 32 * 1024 + 16);
  RUN("CT2 16B 888x256 (6/SM)", (k_tile<2, true>), 888, 256, 32 * 1024 + 16);
  RUN("CT4 16B dbuf 148x512", (k_tile_db<4>), 148, 512, 128 * 1024 + 16);
  RUN("CT4 16B dbuf 148x1024", (k_tile_db<4>), 148, 1024, 128 * 1024 + 16);
  RUN("CT2 16B dbuf 296x512", (k_tile_db<2>), 296, 512, 64 * 1024 + 16);
  RUN("CT2 16B dbuf 444x256", (k_tile_db<2>), 444, 256, 64 * 1024 + 16);
  RUN("rows 16B 296x256", k_rows, 296, 256, 64 * 1024 + 16);
  RUN("rows 16B 296x512", k_rows, 296, 512, 64 * 1024 + 16);
  return 0;
}
