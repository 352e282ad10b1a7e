// Probe: cost of grid-barrier variants for the persistent kernel (592 / 444 co-resident CTAs).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
struct Bar { unsigned cnt; unsigned pad[31]; unsigned gen; unsigned pad2[31]; unsigned long long cnt64; unsigned pad3[30]; unsigned flags[64][32]; };
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) { unsigned o; asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o; }
__device__ __forceinline__ void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

template <int V>
__global__ void __launch_bounds__(256) k(Bar* b, int iters, int sleep) {
  __shared__ unsigned s;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (V == 0) {  // current: gen + count, fence.sc, nanosleep polling
        unsigned gen = ld_relaxed(&b->gen);
        __threadfence();
        unsigned a = atomicAdd(&b->cnt, 1u);
        if (a == gridDim.x - 1) { atomicExch(&b->cnt, 0u); st_release(&b->gen, gen + 1); }
        else while (ld_relaxed(&b->gen) == gen) { if (sleep) __nanosleep(sleep); }
        __threadfence();
      } else if (V == 1) {  // same with acq_rel fences
        unsigned gen = ld_relaxed(&b->gen);
        fence_acqrel();
        unsigned a = atomicAdd(&b->cnt, 1u);
        if (a == gridDim.x - 1) { atomicExch(&b->cnt, 0u); st_release(&b->gen, gen + 1); }
        else while (ld_relaxed(&b->gen) == gen) { if (sleep) __nanosleep(sleep); }
        fence_acqrel();
      } else if (V == 2) {  // monotone counter: atom.add.acq_rel, spin until count >= target
        unsigned target = (unsigned)(it + 1) * gridDim.x;
        atom_add_acqrel(&b->cnt, 1u);
        while ((int)(ld_acquire(&b->cnt) - target) < 0) { if (sleep) __nanosleep(sleep); }
      } else if (V == 3) {  // two-level: groups of 16 CTAs, group leaders to the top; flip broadcast per group
        const unsigned g = blockIdx.x / 16, ng = (gridDim.x + 15) / 16;
        const unsigned gsize = min(16u, gridDim.x - g * 16);
        unsigned gen = ld_relaxed(&b->flags[g][0]);
        fence_acqrel();
        unsigned a = atomicAdd(&b->flags[g][1], 1u);
        if (a == gsize - 1) {
          b->flags[g][1] = 0;
          unsigned t = atomicAdd(&b->cnt, 1u);
          if (t == ng - 1) { b->cnt = 0; fence_acqrel(); for (unsigned q = 0; q < ng; ++q) st_release(&b->flags[q][0], gen + 1); }
          else while (ld_relaxed(&b->flags[g][0]) == gen) { if (sleep) __nanosleep(sleep); }
        } else while (ld_relaxed(&b->flags[g][0]) == gen) { if (sleep) __nanosleep(sleep); }
        fence_acqrel();
      }
      s = it;
    }
    __syncthreads();
  }
}
template <int V>
float run(int grid, int iters, int sleep) {
  Bar* b; cudaMalloc(&b, sizeof(Bar)); cudaMemset(b, 0, sizeof(Bar));
  void* args[] = {&b, &iters, &sleep};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchCooperativeKernel((void*)k<V>, grid, 256, args, 0, 0);
  cudaMemset(b, 0, sizeof(Bar));
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((void*)k<V>, grid, 256, args, 0, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  cudaFree(b);
  if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1000.f / iters;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {4, 3}) for (int sleep : {0, 32, 64, 200}) {
    int grid = sms * per, it = 5000;
    printf("grid %d sleep %3d: v0 %.2f us  v1 %.2f us  v2 %.2f us  v3 %.2f us\n", grid, sleep, run<0>(grid, it, sleep),
           run<1>(grid, it, sleep), run<2>(grid, it, sleep), run<3>(grid, it, sleep));
  }
}
