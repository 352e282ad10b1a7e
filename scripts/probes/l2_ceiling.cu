// Probe: throughput ceiling of scattered small accesses on B200 (VERDICT r1 "What's missing"
// item 4: the R-MAT kernel is bound by random 1-B state gathers and 4-B plane REDs; this gives
// the rate the hardware sustains for exactly those access kinds, at the kernel's footprints).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_ceiling l2_ceiling.cu && ./l2_ceiling
//
// Access kinds (every one issued the way sgr_kernels.cuh issues it):
//   gather_hash : ld.global.cg.u8 at hashed random byte offsets (no index stream; 8 in flight)
//   gather_idx  : index stream read coalesced with ld.global.cs.nc.b32 (like col_idx), then
//                 ld.global.cg.u8 of the indexed byte (Phase B conflict scans)
//   red_hash    : red.global.or.b32 on the 4-B word holding a hashed random byte
//   red_idx     : index stream + red.global.or.b32 (the commit scatter into the planes)
// Footprints: the target array's size (16.8 MB = R-MAT s24 state words; 117 MB = state words +
// 6 planes; 2 GiB = far beyond L2, the DRAM-bound case).  Grid = 148 SMs x {4, 8} CTAs x 256.
// Prints one JSON line per (kind, footprint, grid): G accesses/s and the 32-B-sector rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint32_t ldcg8(const uint8_t* p) {
  uint32_t v; asm volatile("ld.global.cg.u8 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ int32_t ldcs(const int32_t* p) {
  int32_t v; asm volatile("ld.global.cs.nc.b32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}
__device__ __forceinline__ void red_or(uint32_t* p, uint32_t b) {
  asm volatile("red.global.or.b32 [%0], %1;" ::"l"(p), "r"(b) : "memory");
}

constexpr int U = 8;  // independent accesses in flight per thread

// K: 0 gather_hash, 1 gather_idx, 2 red_hash, 3 red_idx
template <int K>
__global__ void __launch_bounds__(256) probe(uint8_t* arr, uint64_t nbytes, const int32_t* idx, uint64_t nidx,
                                             int iters, uint32_t* sink) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint64_t off[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = ((uint64_t)it * U + u) * T + tid;  // coalesced index stream position
      if (K == 0 || K == 2) off[u] = ((uint64_t)hash32((uint32_t)i * 2654435761u + 12345u) * 37ull) % nbytes;
      else off[u] = (uint64_t)(uint32_t)ldcs(idx + (i % nidx));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (K < 2) acc += ldcg8(arr + off[u]);
      else red_or((uint32_t*)(arr + (off[u] & ~3ull)), 1u << ((off[u] & 3) * 8 + (u & 7)));
    }
  }
  if (acc == 0xdeadbeefu) sink[0] = acc;
}

__global__ void fill_idx(int32_t* idx, uint64_t n, uint64_t nbytes) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    idx[i] = (int32_t)(((uint64_t)hash32((uint32_t)i ^ 0x9e3779b9u) * 37ull) % nbytes);
}

int main() {
  const uint64_t foot[] = {16777216ull, 117440512ull, 2147483648ull};
  const char* kname[] = {"gather_hash", "gather_idx", "red_hash", "red_idx"};
  const uint64_t nidx = 1ull << 28;  // 1 GiB index stream (> L2: streamed from DRAM, like col_idx)
  uint8_t* arr;
  int32_t* idx;
  uint32_t* sink;
  CK(cudaMalloc(&arr, foot[2]));
  CK(cudaMalloc(&idx, nidx * 4));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(arr, 0, foot[2]));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (uint64_t F : foot) {
    fill_idx<<<148 * 8, 256>>>(idx, nidx, F);
    CK(cudaDeviceSynchronize());
    for (int cps : {4, 8}) {
      const int grid = 148 * cps;
      const uint64_t T = (uint64_t)grid * 256;
      const int iters = (int)((nidx / U) / T);  // every index once
      for (int k = 0; k < 4; ++k) {
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaEventRecord(e0));
          if (k == 0) probe<0><<<grid, 256>>>(arr, F, idx, nidx, iters, sink);
          if (k == 1) probe<1><<<grid, 256>>>(arr, F, idx, nidx, iters, sink);
          if (k == 2) probe<2><<<grid, 256>>>(arr, F, idx, nidx, iters, sink);
          if (k == 3) probe<3><<<grid, 256>>>(arr, F, idx, nidx, iters, sink);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (rep && ms < best) best = ms;  // rep 0 = warm-up
        }
        const double acc = (double)iters * U * T;
        printf("{\"kind\": \"%s\", \"footprint_bytes\": %llu, \"ctas_per_sm\": %d, \"accesses\": %.0f, \"ms\": %.4f, "
               "\"gacc_per_s\": %.3f, \"sector_gbs\": %.1f, \"index_stream_gbs\": %.1f}\n",
               kname[k], (unsigned long long)F, cps, acc, best, acc / best / 1e6, acc * 32 / best / 1e6,
               (k == 1 || k == 3) ? acc * 4 / best / 1e6 : 0.0);
        fflush(stdout);
      }
    }
  }
  return 0;
}
