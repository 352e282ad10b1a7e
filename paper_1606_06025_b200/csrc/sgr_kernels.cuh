// sgr_kernels.cuh — phases and kernels of the SGR colouring path (sm_100a).
// Phase functions are shared by the persistent cooperative kernel (default) and by the
// one-launch-per-phase host-driven ablation (GC_FLAG_HOST_ROUNDS).
#pragma once
#include "sgr_device.cuh"

namespace gcdev {

// ---------------------------------------------------------------- a1: ingest + bins
// P0: degrees -> bin sizes; st[v] = 1 (round-1 tentative colour: nothing is committed yet,
// so First-Fit gives 1 to every vertex), fm[v] = 0.
template <bool PUSH>
__device__ void prologue_count(const Params& p) {
  __shared__ uint32_t s_cnt[NBIN];
  if (threadIdx.x < NBIN) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * BLOCK;
  for (int64_t base = (int64_t)blockIdx.x * BLOCK + (threadIdx.x & ~31); base < p.n; base += stride) {
    const int64_t v = base + lane;
    const bool act = v < p.n;
    int b = -1;
    if (act) {
      b = bin_of(p, ldr(p.rp, v + 1) - ldr(p.rp, v));
      p.st[v] = 1u;
      if (PUSH) p.fm[v] = 0u;
    }
#pragma unroll
    for (int k = 0; k < NBIN; ++k) {
      const unsigned m = __ballot_sync(FULL, b == k);
      if (m && lane == 0) atomicAdd(&s_cnt[k], (uint32_t)__popc(m));
    }
  }
  __syncthreads();
  if (threadIdx.x < NBIN && s_cnt[threadIdx.x]) atomicAdd(&p.info->binsize[threadIdx.x], s_cnt[threadIdx.x]);
}

// P1: W_1 = V, split into bin segments of wl0 (warp-aggregated cursors; order within a
// bin is free, reading C12).
__device__ void prologue_scatter(const Params& p, const Bins& bins) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * BLOCK;
  for (int64_t base = (int64_t)blockIdx.x * BLOCK + (threadIdx.x & ~31); base < p.n; base += stride) {
    const int64_t v = base + lane;
    const bool act = v < p.n;
    const int b = act ? bin_of(p, ldr(p.rp, v + 1) - ldr(p.rp, v)) : -1;
#pragma unroll
    for (int k = 0; k < NBIN; ++k) {
      const unsigned m = __ballot_sync(FULL, b == k);
      if (!m) continue;
      const int leader = __ffs(m) - 1;
      uint32_t pos = 0;
      if (lane == leader) pos = atomicAdd(&p.info->cursor[k], (uint32_t)__popc(m));
      pos = __shfl_sync(FULL, pos, leader);
      if (b == k) p.wl0[bins.off[k] + pos + __popc(m & lanemask_lt())] = (int32_t)v;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < NBIN) p.info->cnt[1][threadIdx.x] = p.info->binsize[threadIdx.x];
}

// ---------------------------------------------------------------- a2: Phase A
template <bool PUSH, bool CW>
__device__ void phase_a(const Params& p, uint32_t r, const Bins& bins, const int32_t* W, Work& wk) {
  __shared__ uint32_t s_win[2];
  const uint32_t cur = r % 3;
  const uint32_t nT = ld_relaxed(&p.info->cnt[cur][0]);
  const uint32_t nW = ld_relaxed(&p.info->cnt[cur][1]);
  const uint32_t nC = ld_relaxed(&p.info->cnt[cur][2]);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // reset the counters round r+1 will push into (last read in round r-2)
  if (blockIdx.x == 0 && threadIdx.x < NBIN) p.info->cnt[(r + 1) % 3][threadIdx.x] = 0;
  if (CW && threadIdx.x == 0 && blockIdx.x == 0) wk.v[W_A_VERT] += (unsigned long long)nT + nW + nC;

  // thread bin
  {
    const int32_t* Wb = W + bins.off[0];
    for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < nT; i += gridDim.x * BLOCK) {
      const int32_t v = Wb[i];
      uint32_t tent;
      if (PUSH) {
        const uint32_t f = p.fm[v];
        tent = (f != FULL) ? (uint32_t)__ffs(~f) : firstfit_thread<CW>(p, v, 33u, wk);
      } else {
        tent = firstfit_thread<CW>(p, v, 1u, wk);
      }
      p.st[v] = tent;
    }
  }
  // warp bin
  {
    const int32_t* Wb = W + bins.off[1];
    const uint32_t gw = blockIdx.x * WARPS + warp, nw = gridDim.x * WARPS;
    for (uint32_t i = gw; i < nW; i += nw) {
      const int32_t v = Wb[i];
      uint32_t tent;
      if (PUSH) {
        const uint32_t f = p.fm[v];
        tent = (f != FULL) ? (uint32_t)__ffs(~f) : firstfit_warp<CW>(p, v, 33u, wk, lane);
      } else {
        tent = firstfit_warp<CW>(p, v, 1u, wk, lane);
      }
      if (lane == 0) p.st[v] = tent;
    }
  }
  // CTA bin
  {
    const int32_t* Wb = W + bins.off[2];
    for (uint32_t i = blockIdx.x; i < nC; i += gridDim.x) {
      const int32_t v = Wb[i];
      uint32_t tent;
      if (PUSH) {
        const uint32_t f = p.fm[v];
        tent = (f != FULL) ? (uint32_t)__ffs(~f) : firstfit_cta<CW>(p, v, 33u, wk, s_win);
      } else {
        tent = firstfit_cta<CW>(p, v, 1u, wk, s_win);
      }
      if (threadIdx.x == 0) p.st[v] = tent;
    }
  }
}

// ---------------------------------------------------------------- a3: Phase B + push
template <int POL, bool PUSH, bool CW>
__device__ void phase_b(const Params& p, uint32_t r, const Bins& bins, const int32_t* W, int32_t* Wout, Work& wk) {
  const uint32_t cur = r % 3, nxt = (r + 1) % 3;
  const uint32_t nT = ld_relaxed(&p.info->cnt[cur][0]);
  const uint32_t nW = ld_relaxed(&p.info->cnt[cur][1]);
  const uint32_t nC = ld_relaxed(&p.info->cnt[cur][2]);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (p.trace && r <= p.trace_cap) p.trace[r - 1] = nT + nW + nC;
    if (CW) wk.v[W_B_VERT] += (unsigned long long)nT + nW + nC;
  }
  uint32_t* cnt_next = &p.info->cnt[nxt][0];

  // thread bin: one vertex per lane; losers pushed with one atomic per warp
  {
    const int32_t* Wb = W + bins.off[0];
    int32_t* Ob = Wout + bins.off[0];
    const uint32_t stride = gridDim.x * BLOCK;
    for (uint32_t base = blockIdx.x * BLOCK + warp * 32; base < nT; base += stride) {
      const uint32_t i = base + lane;
      bool lose = false;
      int32_t v = 0;
      if (i < nT) {
        v = Wb[i];
        const uint32_t tent = color_of(p.st[v]);
        const int64_t beg = ldr(p.rp, v), end = ldr(p.rp, v + 1);
        lose = conflict_thread<POL, CW>(p, v, tent, beg, end, wk);
        if (!lose) {
          p.st[v] = tent | COMMIT;
          if (PUSH && tent <= 32) {
            scatter_thread(p, 1u << (tent - 1), beg, end);
            if (CW) wk.v[W_SCATTER] += (unsigned long long)(end - beg);
          }
        }
      }
      const unsigned m = __ballot_sync(FULL, lose);
      if (m) {
        const int leader = __ffs(m) - 1;
        uint32_t pos = 0;
        if (lane == leader) pos = atomicAdd(&cnt_next[0], (uint32_t)__popc(m));
        pos = __shfl_sync(FULL, pos, leader);
        if (lose) Ob[pos + __popc(m & lanemask_lt())] = v;
        if (CW && lane == leader) wk.v[W_PUSH] += __popc(m);
      }
    }
  }
  // warp bin
  {
    const int32_t* Wb = W + bins.off[1];
    int32_t* Ob = Wout + bins.off[1];
    const uint32_t gw = blockIdx.x * WARPS + warp, nw = gridDim.x * WARPS;
    for (uint32_t i = gw; i < nW; i += nw) {
      const int32_t v = Wb[i];
      const uint32_t tent = color_of(p.st[v]);
      const int64_t beg = ldr(p.rp, v), end = ldr(p.rp, v + 1);
      const bool lose = conflict_warp<POL, CW>(p, v, tent, beg, end, wk, lane);
      if (lose) {
        if (lane == 0) {
          Ob[atomicAdd(&cnt_next[1], 1u)] = v;
          if (CW) wk.v[W_PUSH] += 1;
        }
      } else {
        if (lane == 0) p.st[v] = tent | COMMIT;
        if (PUSH && tent <= 32) {
          const uint32_t bit = 1u << (tent - 1);
          for (int64_t e = beg + lane; e < end; e += 32) atomicOr(&p.fm[ldc(p.ci, e)], bit);
          if (CW && lane == 0) wk.v[W_SCATTER] += (unsigned long long)(end - beg);
        }
      }
    }
  }
  // CTA bin
  {
    const int32_t* Wb = W + bins.off[2];
    int32_t* Ob = Wout + bins.off[2];
    for (uint32_t i = blockIdx.x; i < nC; i += gridDim.x) {
      const int32_t v = Wb[i];
      const uint32_t tent = color_of(p.st[v]);
      const int64_t beg = ldr(p.rp, v), end = ldr(p.rp, v + 1);
      const bool lose = conflict_cta<POL, CW>(p, v, tent, beg, end, wk);
      if (lose) {
        if (threadIdx.x == 0) {
          Ob[atomicAdd(&cnt_next[2], 1u)] = v;
          if (CW) wk.v[W_PUSH] += 1;
        }
      } else {
        if (threadIdx.x == 0) p.st[v] = tent | COMMIT;
        if (PUSH && tent <= 32) {
          const uint32_t bit = 1u << (tent - 1);
          for (int64_t e = beg + threadIdx.x; e < end; e += BLOCK) atomicOr(&p.fm[ldc(p.ci, e)], bit);
          if (CW && threadIdx.x == 0) wk.v[W_SCATTER] += (unsigned long long)(end - beg);
        }
      }
      __syncthreads();
    }
  }
}

// |W_{r+1}| summed over bins (read after the barrier that ends Phase B of round r).
__device__ __forceinline__ uint32_t next_total(const Params& p, uint32_t r) {
  const uint32_t nxt = (r + 1) % 3;
  return ld_relaxed(&p.info->cnt[nxt][0]) + ld_relaxed(&p.info->cnt[nxt][1]) + ld_relaxed(&p.info->cnt[nxt][2]);
}

// ---------------------------------------------------------------- a5: finalize
__device__ void epilogue(const Params& p) {
  uint32_t mx = 0;
  const int64_t stride = (int64_t)gridDim.x * BLOCK;
  for (int64_t v = (int64_t)blockIdx.x * BLOCK + threadIdx.x; v < p.n; v += stride) {
    const uint32_t c = color_of(p.st[v]);
    p.colors_out[v] = c;
    mx = c > mx ? c : mx;
  }
  mx = __reduce_max_sync(FULL, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(&p.info->num_colors, mx);
}

template <bool CW>
__device__ void flush_work(const Params& p, Work& wk) {
  if (!CW) return;
#pragma unroll
  for (int k = 0; k < W_N; ++k) {
    unsigned long long x = wk.v[k];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(&p.info->work[k], x);
  }
}

// ---------------------------------------------------------------- a4: persistent driver
// One cooperative launch runs ingest, every round and finalize.  Per round: Phase A,
// barrier, Phase B (+push), barrier; every CTA reads |W_{r+1}| and leaves together.
template <int POL, bool PUSH, bool CW>
__global__ void __launch_bounds__(BLOCK) sgr_persistent(Params p) {
  Work wk;
  wk.zero();
  prologue_count<PUSH>(p);
  if (!grid_sync(p)) return;
  Bins bins;
  bins.load(p);
  prologue_scatter(p, bins);
  if (!grid_sync(p)) return;

  int32_t* Win = p.wl0;
  int32_t* Wout = p.wl1;
  uint32_t r = 1;
  for (;;) {
    if (r > 1) {
      phase_a<PUSH, CW>(p, r, bins, Win, wk);
      if (!grid_sync(p)) return;
    }
    phase_b<POL, PUSH, CW>(p, r, bins, Win, Wout, wk);
    if (!grid_sync(p)) return;
    const uint32_t left = next_total(p, r);
    if (left == 0) break;
    if (r >= p.max_rounds) {
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(&p.info->status, (uint32_t)ST_NO_CONVERGENCE);
      flush_work<CW>(p, wk);
      return;
    }
    ++r;
    int32_t* t = Win;
    Win = Wout;
    Wout = t;
  }
  epilogue(p);
  flush_work<CW>(p, wk);
  if (blockIdx.x == 0 && threadIdx.x == 0) p.info->rounds = r;
}

// ---------------------------------------------------------------- host-driven ablation
// GC_FLAG_HOST_ROUNDS: the same phases, one (non-cooperative) launch each, the host
// reading |W_{r+1}| after every round (the paper's "CPU ... controlling the progress").
template <bool PUSH>
__global__ void __launch_bounds__(BLOCK) k_prologue_count(Params p) { prologue_count<PUSH>(p); }
__global__ void __launch_bounds__(BLOCK) k_prologue_scatter(Params p) {
  Bins b;
  b.load(p);
  prologue_scatter(p, b);
}
template <bool PUSH, bool CW>
__global__ void __launch_bounds__(BLOCK) k_phase_a(Params p, uint32_t r, int32_t* W) {
  Work wk;
  wk.zero();
  Bins b;
  b.load(p);
  phase_a<PUSH, CW>(p, r, b, W, wk);
  flush_work<CW>(p, wk);
}
template <int POL, bool PUSH, bool CW>
__global__ void __launch_bounds__(BLOCK) k_phase_b(Params p, uint32_t r, int32_t* W, int32_t* Wout) {
  Work wk;
  wk.zero();
  Bins b;
  b.load(p);
  phase_b<POL, PUSH, CW>(p, r, b, W, Wout, wk);
  flush_work<CW>(p, wk);
}
__global__ void __launch_bounds__(BLOCK) k_epilogue(Params p, uint32_t r) {
  epilogue(p);
  if (blockIdx.x == 0 && threadIdx.x == 0) p.info->rounds = r;
}

// ---------------------------------------------------------------- validation (C9)
// One warp per vertex: row_ptr monotone, 0 <= w < n, w != v, strictly increasing rows;
// optionally symmetry by binary search of v in adj(w).  Records the smallest bad vertex.
enum ValErr { VE_NONE = 0, VE_ROWPTR = 1, VE_RANGE = 2, VE_SELF = 3, VE_ORDER = 4, VE_ASYM = 5 };

__device__ __forceinline__ void report_bad(DevInfo* I, int64_t v, uint32_t code) {
  const unsigned long long key = ((unsigned long long)v << 3) | code;  // smallest vertex wins
  atomicMin(&I->bad, key + 1);
}

__global__ void __launch_bounds__(BLOCK) k_validate(int32_t n, const int64_t* __restrict__ rp,
                                                    const int32_t* __restrict__ ci, int symmetry, DevInfo* I) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * BLOCK) >> 5;
  if (gw == 0 && lane == 0 && __ldg(rp) != 0) report_bad(I, 0, VE_ROWPTR);
  for (int64_t v = gw; v < n; v += nw) {
    const int64_t beg = __ldg(rp + v), end = __ldg(rp + v + 1);
    if (end < beg) { if (lane == 0) report_bad(I, v, VE_ROWPTR); continue; }
    for (int64_t e = beg + lane; e < end; e += 32) {
      const int32_t w = __ldg(ci + e);
      if (w < 0 || w >= n) { report_bad(I, v, VE_RANGE); continue; }
      if (w == v) report_bad(I, v, VE_SELF);
      if (e > beg && __ldg(ci + e - 1) >= w) report_bad(I, v, VE_ORDER);
      if (symmetry) {
        int64_t lo = __ldg(rp + w), hi = __ldg(rp + w + 1) - 1;
        bool found = false;
        while (lo <= hi) {
          const int64_t mid = (lo + hi) >> 1;
          const int32_t x = __ldg(ci + mid);
          if (x == v) { found = true; break; }
          if (x < v) lo = mid + 1; else hi = mid - 1;
        }
        if (!found) report_bad(I, v, VE_ASYM);
      }
    }
  }
}

// ---------------------------------------------------------------- device verifier
// complete + proper + First-Fit fixpoint (pin P9), one warp per vertex.
__global__ void __launch_bounds__(BLOCK) k_verify(int32_t n, const int64_t* __restrict__ rp,
                                                  const int32_t* __restrict__ ci,
                                                  const uint32_t* __restrict__ col, DevInfo* I) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * BLOCK) >> 5;
  for (int64_t v = gw; v < n; v += nw) {
    const uint32_t c = __ldg(col + v);
    const int64_t beg = __ldg(rp + v), end = __ldg(rp + v + 1);
    if (c == 0 || (int64_t)c > end - beg + 1) { if (lane == 0) report_bad(I, v, 1); continue; }
    bool bad = false;
    for (uint32_t base = 1; base < c && !bad; base += 64) {
      uint32_t lo = 0, hi = 0;
      for (int64_t e = beg + lane; e < end; e += 32) {
        const uint32_t d = __ldg(col + __ldg(ci + e)) - base;
        if (d < 32) lo |= 1u << d;
        else if (d < 64) hi |= 1u << (d - 32);
      }
      lo = __reduce_or_sync(FULL, lo);
      hi = __reduce_or_sync(FULL, hi);
      // every colour in [base, min(c, base+64)) must be present
      const uint32_t need = c - base;  // colours base..c-1
      const unsigned long long have = ((unsigned long long)hi << 32) | lo;
      const unsigned long long want = need >= 64 ? ~0ull : ((1ull << need) - 1);
      if ((have & want) != want) bad = true;
    }
    for (int64_t e = beg + lane; e < end && !bad; e += 32)
      if (__ldg(col + __ldg(ci + e)) == c) bad = true;
    bad = __any_sync(FULL, bad);
    if (bad && lane == 0) report_bad(I, v, 2);
  }
}

}  // namespace gcdev
