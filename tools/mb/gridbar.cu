// Microbenchmark (diagnostics, not product): grid-barrier variants on a cooperative grid of
// 2 x 256-thread blocks per SM (the grid tier's launch shape).
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

// (a) the grid tier's barrier: acq_rel atomic with return, target from the returned count
__device__ __forceinline__ void bar_atom(unsigned long long* cnt, unsigned nblk) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(cnt) : "memory");
    const unsigned long long target = old - old % nblk + nblk;
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
      if (v >= target) break;
    }
  }
  __syncthreads();
}
// (b) fire-and-forget release reduction, target from a block-local epoch
__device__ __forceinline__ void bar_red(unsigned long long* cnt, unsigned nblk, unsigned long long& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");
    const unsigned long long target = (++epoch) * nblk;
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
      if (v >= target) break;
    }
  }
  __syncthreads();
}
// (c) as (b), relaxed polls and one acquire fence after
__device__ __forceinline__ void bar_red_relaxed(unsigned long long* cnt, unsigned nblk, unsigned long long& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");
    const unsigned long long target = (++epoch) * nblk;
    while (true) {
      unsigned long long v;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
      if (v >= target) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
// (d) two-level: 8 blocks share a sub-counter; the last arriver of a group forwards to the top
__device__ __forceinline__ void bar_tree(unsigned long long* cnt, unsigned nblk, unsigned long long& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = blockIdx.x >> 3, ng = (nblk + 7) >> 3;
    const unsigned gsz = (g == ng - 1) ? nblk - 8 * g : 8;
    unsigned long long* sub = cnt + 16 + 16 * g;   // own 128-byte lines
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(sub) : "memory");
    ++epoch;
    if (old + 1 == epoch * gsz) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");
    const unsigned long long target = epoch * ng;
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
      if (v >= target) break;
    }
  }
  __syncthreads();
}
__global__ void k_bench(unsigned long long* cnt, int iters, int variant, unsigned long long* out, float* scratch) {
  unsigned long long epoch = 0;
  const unsigned nblk = gridDim.x;
  // some memory traffic before each barrier, as after a pass
  auto work = [&](int i) { scratch[(blockIdx.x * 256 + threadIdx.x) * 4 + (i & 3)] += 1.f; };
  bar_atom(cnt + 1024, nblk);
  long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int i = 0; i < iters; ++i) {
    work(i);
    if (variant == 0) bar_atom(cnt, nblk);
    else if (variant == 1) bar_red(cnt, nblk, epoch);
    else if (variant == 2) bar_red_relaxed(cnt, nblk, epoch);
    else bar_tree(cnt, nblk, epoch);
  }
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = g1 - g0;
  (void)t0;
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *cnt, *out; float* scratch;
  CK(cudaMalloc(&cnt, 1 << 20)); CK(cudaMalloc(&out, 64)); CK(cudaMalloc(&scratch, 64 << 20));
  const char* names[] = {"atom acq_rel + acquire poll (grid tier)", "red.release + epoch, acquire poll",
                         "red.release + epoch, relaxed poll + fence", "two-level (8 per group)"};
  for (int grid : {2 * nsm, nsm, 64}) {
    for (int v = 0; v < 4; ++v) {
      CK(cudaMemset(cnt, 0, 1 << 20));
      int iters = 20000;
      void* args[] = {&cnt, &iters, &v, &out, &scratch};
      CK(cudaLaunchCooperativeKernel((const void*)k_bench, dim3(grid), dim3(256), args, 0, 0));
      CK(cudaDeviceSynchronize());
      unsigned long long h; CK(cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost));
      printf("grid %4d  %-44s %.3f us/barrier\n", grid, names[v], h / 1e3 / iters);
    }
  }
  return 0;
}
