// sgr_device.cuh — device side of the round-synchronous SGR colouring path (sm_100a).
//
// Paper mapping (arXiv 1606.06025, /root/reference/PAPER.md):
//   Phase A  = FirstFit (Alg. 4) with the bitset + find-first-set refinement
//              (§3.2 "Bitset Operation");
//   Phase B  = ConflictResolve (Alg. 5) fused with the W_out push and prefix /
//              aggregated atomics (§3.1 "Atomic Operation Reduction");
//   rounds   = Data-GC (Alg. 7) with double-buffered worklists in
//              ONE persistent kernel with a device-wide barrier (§3.3 "Kernel Fusion",
//              P:653-667) — no host involvement per round;
//   binning  = thread / warp / CTA per vertex by degree (§3.3 "Load Balancing");
//   CSR read through the read-only path (§3.3 "Read-only Data Caching").
//
// B200-first differences from the paper's K40c design:
//   * Jacobi rounds (north star): Phase A uses only colours committed before the round,
//     Phase B uses the round's tentative colours; the result is schedule independent.
//   * One 32-bit state word per vertex: bit31 = committed, bits 0..30 = colour (tentative
//     while bit31 = 0).  Phase A only USES committed words and only writes pending ones;
//     Phase B only reads colour bits and only sets bit31 — so neither phase ever uses a
//     bit that is being written in the same phase (aligned 32-bit words are single-copy
//     atomic), and no locks are needed.
//   * Incremental forbidden-colour mask (default): committed colours never change, so a
//     vertex's forbidden set only grows.  A committing vertex ORs its colour bit
//     (colours 1..32) into fm[w] of every neighbour (one RED per directed edge over the
//     whole run).  Phase A is then O(1): tent = ffs(~fm[v]); only when colours 1..32 are
//     all forbidden does it fall back to the exact windowed neighbour scan from colour 33.
//     GC_FLAG_PULL_FIRSTFIT selects the paper's full rescan instead (same result).
//   * Round 1 needs no Phase A: nothing is committed, so every tentative colour is 1.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gcdev {

constexpr uint32_t COMMIT = 0x80000000u;
constexpr uint32_t CMASK = 0x7fffffffu;
constexpr int NBIN = 3;            // 0 = thread, 1 = warp, 2 = CTA per vertex
constexpr int BLOCK = 256;
constexpr int WARPS = BLOCK / 32;
constexpr unsigned FULL = 0xffffffffu;

enum Policy { HIGHER_ID = 0, LOWER_ID = 1, DEGREE = 2 };
enum Status { ST_OK = 0, ST_NO_CONVERGENCE = 3, ST_WATCHDOG = 5 };
enum WorkIdx { W_A_VERT = 0, W_A_EDGE, W_B_VERT, W_B_EDGE, W_B_GATHER, W_SCATTER, W_PUSH, W_N };

// Device-side run state.  Zeroed by the host before launch.
struct DevInfo {
  uint32_t status;
  uint32_t rounds;
  uint32_t num_colors;
  uint32_t pad0;
  uint32_t binsize[NBIN];
  uint32_t cursor[NBIN];
  uint32_t cnt[3][NBIN];        // |W| per bin, triple-buffered by round (r % 3)
  uint32_t pad1[13];
  unsigned long long work[W_N];
  unsigned long long bad;       // validation / verify: first offending index + 1 (min)
  uint32_t err_code;            // validation error kind
  uint32_t pad2[31];
  uint32_t bar_count;           // grid barrier (own 128-B lines)
  uint32_t pad3[31];
  uint32_t bar_gen;
  uint32_t pad4[31];
};

struct Params {
  int32_t n;
  const int64_t* __restrict__ rp;
  const int32_t* __restrict__ ci;
  uint32_t* st;                 // state word per vertex
  uint32_t* fm;                 // forbidden colours 1..32 per vertex (incremental mode)
  int32_t* wl0;                 // worklist buffers, n entries each, bin segments
  int32_t* wl1;
  DevInfo* info;
  uint32_t* trace;
  uint32_t trace_cap;
  uint32_t* colors_out;
  uint32_t max_rounds;
  uint32_t tb;                  // thread-bin max degree
  uint32_t wb;                  // warp-bin max degree
  unsigned long long timeout_ns;
};

struct Work {
  unsigned long long v[W_N];
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < W_N; ++i) v[i] = 0;
  }
};

// ---------------------------------------------------------------- memory helpers

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// CSR is read-only for the whole kernel: non-coherent read-only path.
__device__ __forceinline__ int32_t ldc(const int32_t* __restrict__ p, int64_t i) { return __ldg(p + i); }
__device__ __forceinline__ int64_t ldr(const int64_t* __restrict__ p, int64_t i) { return __ldg(p + i); }
// Colour of a state word.
__device__ __forceinline__ uint32_t color_of(uint32_t s) { return s & CMASK; }

// ---------------------------------------------------------------- grid barrier
// Sense (generation) barrier over all co-resident CTAs of the cooperative launch, with a
// globaltimer watchdog so that a bug can never hang the GPU: on timeout the status becomes
// ST_WATCHDOG and every CTA leaves at its next barrier.  Returns false when the run must
// stop.  Release/acquire at gpu scope order every write of the phase before every read of
// the next phase (and invalidate stale L1 lines).
__device__ __forceinline__ bool grid_sync(const Params& p) {
  __syncthreads();
  if (threadIdx.x == 0) {
    DevInfo* I = p.info;
    const uint32_t gen = ld_acquire(&I->bar_gen);
    __threadfence();
    const uint32_t arrived = atomicAdd(&I->bar_count, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(&I->bar_count, 0u);
      __threadfence();
      st_release(&I->bar_gen, gen + 1);
    } else {
      const unsigned long long t0 = globaltimer();
      while (ld_acquire(&I->bar_gen) == gen) {
        __nanosleep(32);
        if (globaltimer() - t0 > p.timeout_ns) {
          atomicExch(&I->status, (uint32_t)ST_WATCHDOG);
          break;
        }
      }
    }
  }
  __syncthreads();
  return ld_relaxed(&p.info->status) != ST_WATCHDOG;
}

// ---------------------------------------------------------------- bins

__device__ __forceinline__ int bin_of(const Params& p, int64_t deg) {
  return deg <= (int64_t)p.tb ? 0 : (deg <= (int64_t)p.wb ? 1 : 2);
}

struct Bins {
  uint32_t off[NBIN];
  __device__ void load(const Params& p) {
    uint32_t b0 = ld_relaxed(&p.info->binsize[0]), b1 = ld_relaxed(&p.info->binsize[1]);
    off[0] = 0;
    off[1] = b0;
    off[2] = b0 + b1;
  }
};

// ---------------------------------------------------------------- First-Fit (Phase A)

// Exact windowed First-Fit over committed neighbours, one thread (reading C7):
// smallest colour >= base absent from the committed neighbour colours.
template <bool CW>
__device__ uint32_t firstfit_thread(const Params& p, int32_t v, uint32_t base, Work& wk) {
  const int64_t beg = ldr(p.rp, v), end = ldr(p.rp, v + 1);
  for (;;) {
    unsigned long long mask = 0;
    int64_t e = beg;
    for (; e + 4 <= end; e += 4) {
      const int32_t w0 = ldc(p.ci, e), w1 = ldc(p.ci, e + 1), w2 = ldc(p.ci, e + 2), w3 = ldc(p.ci, e + 3);
      const uint32_t s0 = p.st[w0], s1 = p.st[w1], s2 = p.st[w2], s3 = p.st[w3];
      const uint32_t d0 = color_of(s0) - base, d1 = color_of(s1) - base;
      const uint32_t d2 = color_of(s2) - base, d3 = color_of(s3) - base;
      if ((s0 & COMMIT) && d0 < 64) mask |= 1ull << d0;
      if ((s1 & COMMIT) && d1 < 64) mask |= 1ull << d1;
      if ((s2 & COMMIT) && d2 < 64) mask |= 1ull << d2;
      if ((s3 & COMMIT) && d3 < 64) mask |= 1ull << d3;
    }
    for (; e < end; ++e) {
      const uint32_t s = p.st[ldc(p.ci, e)];
      const uint32_t d = color_of(s) - base;
      if ((s & COMMIT) && d < 64) mask |= 1ull << d;
    }
    if (CW) wk.v[W_A_EDGE] += (unsigned long long)(end - beg);
    if (~mask) return base + (uint32_t)__ffsll((long long)~mask) - 1;
    base += 64;
  }
}

// Same, one warp per vertex; lanes stride over the row (coalesced 128-B col_idx reads),
// per-lane window bits combined with __reduce_or_sync, smallest free bit with __ffs.
template <bool CW>
__device__ uint32_t firstfit_warp(const Params& p, int32_t v, uint32_t base, Work& wk, int lane) {
  const int64_t beg = ldr(p.rp, v), end = ldr(p.rp, v + 1);
  for (;;) {
    uint32_t lo = 0, hi = 0;
    for (int64_t e = beg + lane; e < end; e += 32) {
      const uint32_t s = p.st[ldc(p.ci, e)];
      const uint32_t d = color_of(s) - base;
      if (s & COMMIT) {
        if (d < 32) lo |= 1u << d;
        else if (d < 64) hi |= 1u << (d - 32);
      }
    }
    lo = __reduce_or_sync(FULL, lo);
    hi = __reduce_or_sync(FULL, hi);
    if (CW && lane == 0) wk.v[W_A_EDGE] += (unsigned long long)(end - beg);
    if (~lo) return base + (uint32_t)__ffs(~lo) - 1;
    if (~hi) return base + 32 + (uint32_t)__ffs(~hi) - 1;
    base += 64;
  }
}

// Same, one CTA per vertex; window bits in shared memory.
template <bool CW>
__device__ uint32_t firstfit_cta(const Params& p, int32_t v, uint32_t base, Work& wk, uint32_t* s_win) {
  const int64_t beg = ldr(p.rp, v), end = ldr(p.rp, v + 1);
  for (;;) {
    if (threadIdx.x < 2) s_win[threadIdx.x] = 0;
    __syncthreads();
    uint32_t lo = 0, hi = 0;
    for (int64_t e = beg + threadIdx.x; e < end; e += BLOCK) {
      const uint32_t s = p.st[ldc(p.ci, e)];
      const uint32_t d = color_of(s) - base;
      if (s & COMMIT) {
        if (d < 32) lo |= 1u << d;
        else if (d < 64) hi |= 1u << (d - 32);
      }
    }
    lo = __reduce_or_sync(FULL, lo);
    hi = __reduce_or_sync(FULL, hi);
    if ((threadIdx.x & 31) == 0) {
      if (lo) atomicOr(&s_win[0], lo);
      if (hi) atomicOr(&s_win[1], hi);
    }
    __syncthreads();
    lo = s_win[0];
    hi = s_win[1];
    __syncthreads();
    if (CW && threadIdx.x == 0) wk.v[W_A_EDGE] += (unsigned long long)(end - beg);
    if (~lo) return base + (uint32_t)__ffs(~lo) - 1;
    if (~hi) return base + 32 + (uint32_t)__ffs(~hi) - 1;
    base += 64;
  }
}

// ---------------------------------------------------------------- conflict predicate

// Does v recolour because of neighbour w with the same tentative colour?  (C1, C8)
template <int POL>
__device__ __forceinline__ bool recolors(const Params& p, int32_t v, int32_t w, int64_t dv) {
  if (POL == HIGHER_ID) return v > w;
  if (POL == LOWER_ID) return v < w;
  const int64_t dw = ldr(p.rp, w + 1) - ldr(p.rp, w);
  return dv < dw || (dv == dw && v > w);
}

// ---------------------------------------------------------------- Phase B scans
// Each returns true when v must recolour (is pushed to W_out).  HIGHER_ID only needs the
// lower-id prefix of the (sorted) row and stops at the first w > v or the first hit;
// LOWER_ID scans the upper suffix from the end; DEGREE scans the whole row.

template <int POL, bool CW>
__device__ bool conflict_thread(const Params& p, int32_t v, uint32_t tent, int64_t beg, int64_t end, Work& wk) {
  if (POL == HIGHER_ID) {
    int64_t e = beg;
    for (; e + 4 <= end; e += 4) {
      const int32_t w0 = ldc(p.ci, e), w1 = ldc(p.ci, e + 1), w2 = ldc(p.ci, e + 2), w3 = ldc(p.ci, e + 3);
      // speculative gathers of the lower-id candidates (rows are sorted: w0<w1<w2<w3)
      const uint32_t c0 = w0 < v ? color_of(p.st[w0]) : 0u;
      const uint32_t c1 = w1 < v ? color_of(p.st[w1]) : 0u;
      const uint32_t c2 = w2 < v ? color_of(p.st[w2]) : 0u;
      const uint32_t c3 = w3 < v ? color_of(p.st[w3]) : 0u;
      if (w0 > v) { if (CW) { wk.v[W_B_EDGE] += e - beg + 1; wk.v[W_B_GATHER] += e - beg; } return false; }
      if (c0 == tent) { if (CW) { wk.v[W_B_EDGE] += e - beg + 1; wk.v[W_B_GATHER] += e - beg + 1; } return true; }
      if (w1 > v) { if (CW) { wk.v[W_B_EDGE] += e - beg + 2; wk.v[W_B_GATHER] += e - beg + 1; } return false; }
      if (c1 == tent) { if (CW) { wk.v[W_B_EDGE] += e - beg + 2; wk.v[W_B_GATHER] += e - beg + 2; } return true; }
      if (w2 > v) { if (CW) { wk.v[W_B_EDGE] += e - beg + 3; wk.v[W_B_GATHER] += e - beg + 2; } return false; }
      if (c2 == tent) { if (CW) { wk.v[W_B_EDGE] += e - beg + 3; wk.v[W_B_GATHER] += e - beg + 3; } return true; }
      if (w3 > v) { if (CW) { wk.v[W_B_EDGE] += e - beg + 4; wk.v[W_B_GATHER] += e - beg + 3; } return false; }
      if (c3 == tent) { if (CW) { wk.v[W_B_EDGE] += e - beg + 4; wk.v[W_B_GATHER] += e - beg + 4; } return true; }
    }
    for (; e < end; ++e) {
      const int32_t w = ldc(p.ci, e);
      if (CW) wk.v[W_B_EDGE] += 1;
      if (w > v) return false;
      if (CW) wk.v[W_B_GATHER] += 1;
      if (color_of(p.st[w]) == tent) return true;
    }
    return false;
  } else if (POL == LOWER_ID) {
    for (int64_t e = end - 1; e >= beg; --e) {
      const int32_t w = ldc(p.ci, e);
      if (CW) wk.v[W_B_EDGE] += 1;
      if (w < v) return false;
      if (CW) wk.v[W_B_GATHER] += 1;
      if (color_of(p.st[w]) == tent) return true;
    }
    return false;
  } else {
    const int64_t dv = end - beg;
    for (int64_t e = beg; e < end; ++e) {
      const int32_t w = ldc(p.ci, e);
      if (CW) { wk.v[W_B_EDGE] += 1; wk.v[W_B_GATHER] += 1; }
      if (color_of(p.st[w]) == tent && recolors<DEGREE>(p, v, w, dv)) return true;
    }
    return false;
  }
}

// Warp scan: 32 row entries per step; the step stops the scan if any lane hits or (for the
// id policies) reaches the other side of v.  Work counters follow the sequential scan.
template <int POL, bool CW>
__device__ bool conflict_warp(const Params& p, int32_t v, uint32_t tent, int64_t beg, int64_t end, Work& wk, int lane) {
  const int64_t dv = end - beg;
  const int64_t len = end - beg;
  for (int64_t k = 0; k < len; k += 32) {
    const int64_t j = k + lane;
    const bool valid = j < len;
    const int64_t e = (POL == LOWER_ID) ? end - 1 - j : beg + j;
    const int32_t w = valid ? ldc(p.ci, e) : v;
    bool side, hit = false;
    if (POL == HIGHER_ID) side = valid && w < v;
    else if (POL == LOWER_ID) side = valid && w > v;
    else side = valid;
    if (side) hit = color_of(p.st[w]) == tent && recolors<POL>(p, v, w, dv);
    const unsigned stop = __ballot_sync(FULL, hit || !side);
    if (CW) {
      // sequential-scan counters: entries / gathers up to and including the stop lane
      const int kk = stop ? __ffs(stop) - 1 : 31;
      const unsigned ev = __ballot_sync(FULL, valid && lane <= kk);
      const unsigned g = __ballot_sync(FULL, side && lane <= kk);
      if (lane == 0) { wk.v[W_B_EDGE] += __popc(ev); wk.v[W_B_GATHER] += __popc(g); }
    }
    if (__any_sync(FULL, hit)) return true;
    if (stop) return false;
  }
  return false;
}

template <int POL, bool CW>
__device__ bool conflict_cta(const Params& p, int32_t v, uint32_t tent, int64_t beg, int64_t end, Work& wk) {
  const int64_t dv = end - beg;
  const int64_t len = end - beg;
  for (int64_t k = 0; k < len; k += BLOCK) {
    const int64_t j = k + threadIdx.x;
    const bool valid = j < len;
    const int64_t e = (POL == LOWER_ID) ? end - 1 - j : beg + j;
    const int32_t w = valid ? ldc(p.ci, e) : v;
    bool side, hit = false;
    if (POL == HIGHER_ID) side = valid && w < v;
    else if (POL == LOWER_ID) side = valid && w > v;
    else side = valid;
    if (side) hit = color_of(p.st[w]) == tent && recolors<POL>(p, v, w, dv);
    if (CW) {
      // sequential-scan counters: entries up to the first stopping position
      __shared__ int s_first;
      if (threadIdx.x == 0) s_first = BLOCK;
      __syncthreads();
      if (hit || !side) atomicMin(&s_first, (int)threadIdx.x);
      __syncthreads();
      const int kk = s_first < BLOCK ? s_first : BLOCK - 1;
      const bool counted_edge = valid && (int)threadIdx.x <= kk;
      const bool counted_gather = side && (int)threadIdx.x <= kk;
      const int ne = __syncthreads_count(counted_edge);
      const int ng = __syncthreads_count(counted_gather);
      if (threadIdx.x == 0) { wk.v[W_B_EDGE] += ne; wk.v[W_B_GATHER] += ng; }
    }
    if (__syncthreads_or(hit)) return true;
    if (__syncthreads_or(!side)) return false;
  }
  return false;
}

// ---------------------------------------------------------------- commit scatter
// A winner ORs its colour bit into every neighbour's forbidden mask (incremental mode).
__device__ __forceinline__ void scatter_thread(const Params& p, uint32_t bit, int64_t beg, int64_t end) {
  for (int64_t e = beg; e < end; ++e) atomicOr(&p.fm[ldc(p.ci, e)], bit);
}

}  // namespace gcdev
