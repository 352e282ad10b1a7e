// Probe: are P cooperative kernels launched from one process on P streams of the same
// device co-resident (each spins until all others have arrived)?  Used to decide how the
// one-GPU emulation of the multi-GPU path runs its P "ranks".
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 4) k(unsigned* flags, int me, int P, unsigned long long timeout, int* res) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) atomicAdd(&flags[me], 1u);
    unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    ok = 1;
    for (int q = 0; q < P; ++q) {
      for (;;) {
        unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + q));
        if (v) break;
        unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout) { ok = 0; break; }
      }
    }
    if (!ok) atomicExch(res + me, 1);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0);
  printf("sms %d per_sm %d\n", sms, per);
  for (int P = 2; P <= 8; P *= 2) {
    unsigned* flags; int* res; cudaMalloc(&flags, 64); cudaMalloc(&res, 64);
    cudaMemset(flags, 0, 64); cudaMemset(res, 0, 64);
    cudaStream_t s[8];
    for (int i = 0; i < P; ++i) cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
    cudaDeviceSynchronize();
    int grid = sms * per / P;
    unsigned long long to = 2000000000ull;
    for (int i = 0; i < P; ++i) {
      int me = i;
      void* args[] = {&flags, &me, &P, &to, &res};
      cudaError_t e = cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, s[i]);
      if (e) printf("launch %d: %s\n", i, cudaGetErrorString(e));
    }
    cudaError_t e = cudaDeviceSynchronize();
    int h[16]; cudaMemcpy(h, res, 64, cudaMemcpyDeviceToHost);
    int bad = 0; for (int i = 0; i < P; ++i) bad += h[i];
    printf("P=%d grid/rank=%d sync=%s timeouts=%d\n", P, grid, cudaGetErrorString(e), bad);
  }
  return 0;
}
