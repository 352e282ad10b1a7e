// workloads/gen_gpu.cu — the W1 R-MAT recipe on the GPU.
//
// Test/bench INPUT infrastructure, like gen.c: it holds none of the colouring method's
// arithmetic.  It emits the directed arcs of R-MAT samples whose (relabelled) source lies in a
// vertex range, as 64-bit keys ((source - range start) << 32 | target); the Python side
// (workloads.rmat_range_gpu) sorts and deduplicates them into CSR rows.  The sample recipe is
// the same as gen.c's rmat_sample, with the same double arithmetic (the comparison of
// (splitmix64(.) >> 11) * 2^-53 against a, a+b, a+b+c is exact in both), and the relabelling
// permutation pi comes from gen.c (gen_rmat_perm), so the graph is bit-identical to gen.c's
// (tests/test_workloads.py checks it).  Used where the CPU generator is too slow: scale 27
// (2^31 samples) on the test box, and every rank's own range in the multi-GPU bench.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void emit(bool want, long long key, unsigned long long* count, long long* keys,
                                     long long cap) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(count, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (want && keys) {
    const unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
    if ((long long)pos < cap) keys[pos] = key;
  }
}

__global__ void __launch_bounds__(256) k_rmat_emit(int scale, long long ns, double a, double ab, double abc,
                                                   unsigned long long base, const int32_t* __restrict__ pi,
                                                   long long cb, long long ce, unsigned long long* count,
                                                   long long* keys, long long cap) {
  const long long T = (long long)gridDim.x * blockDim.x;
  // every lane of a warp runs the same number of iterations (ballots inside)
  const long long iters = (ns + T - 1) / T;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long it = 0; it < iters; ++it, i += T) {
    long long pu = -1, pv = -1;
    if (i < ns) {
      unsigned long long u = 0, v = 0;
      for (int l = 0; l < scale; ++l) {
        const double r = (double)(splitmix64(base + 64ULL * (unsigned long long)i + (unsigned long long)l) >> 11) *
                         0x1.0p-53;
        unsigned long long bu, bv;
        if (r < a) { bu = 0; bv = 0; }
        else if (r < ab) { bu = 0; bv = 1; }
        else if (r < abc) { bu = 1; bv = 0; }
        else { bu = 1; bv = 1; }
        u = (u << 1) | bu;
        v = (v << 1) | bv;
      }
      pu = __ldg(pi + u);
      pv = __ldg(pi + v);
      if (pu == pv) pu = pv = -1;  // self loops dropped
    }
    emit(pu >= cb && pu < ce, ((pu - cb) << 32) | pv, count, keys, cap);
    emit(pv >= cb && pv < ce, ((pv - cb) << 32) | pu, count, keys, cap);
  }
}

}  // namespace

extern "C" {

// Arcs of samples [0, ns) whose source lies in [cb, ce): with keys == NULL only *count is
// produced (a counting pass); else up to cap keys are written.  Asynchronous on `stream`;
// *count (device) must be zeroed by the caller.  Returns a cudaError_t.
int gen_rmat_emit_gpu(int scale, long long ns, double a, double ab, double abc, unsigned long long seed,
                      const int32_t* pi, long long cb, long long ce, unsigned long long* count, long long* keys,
                      long long cap, void* stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_rmat_emit<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(scale, ns, a, ab, abc, seed << 40, pi, cb, ce, count, keys,
                                                         cap);
  return (int)cudaGetLastError();
}

}  // extern "C"
