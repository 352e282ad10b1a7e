// sgr_kernels.cuh — phases and kernels of the SGR colouring path (sm_100a).
// Phase functions are shared by the persistent cooperative kernel (default) and by the
// one-launch-per-phase host-driven ablation (GC_FLAG_HOST_ROUNDS).
// Template parameters: S = state word (uint8_t / uint16_t / uint32_t), POL = conflict policy,
// PUSH = incremental forbidden masks (else full rescans), CW = exact work counters.
#pragma once
#include "sgr_device.cuh"

namespace gcdev {

// ---------------------------------------------------------------- a1: ingest + bins
// P0: degrees -> bin sizes; st[v] = 1 (round-1 tentative colour: nothing is committed yet,
// so First-Fit gives 1 to every vertex), plane-0 mask byte = 0.  With 8- or 16-bit state
// words a vertex of degree > NARROW_MAX_DEG makes the run restart with 32-bit words
// (ST_NEED32); 8-bit words restart with 16-bit ones when a colour > 127 appears (Phase A).
// Dense start (p.dense_div): also the split of every vertex (ksplit, one dependent level for
// rows <= 8, else binary search) and the static list of the heavy vertices (bin 1).
template <class S, int POL, bool PUSH>
__device__ __forceinline__ void prologue_count(const Params& p, bool dense) {
  __shared__ uint32_t s_cnt[NBIN];
  if (threadIdx.x < NBIN) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  S* st = (S*)p.st;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)nblk(p) * BLOCK;
  bool wide = false;
  uint32_t maxdeg = 0;
  // the row offsets of the next iteration's vertex are loaded one iteration ahead, so that
  // their latency overlaps this vertex's split search
  const int64_t first = (int64_t)blk(p) * BLOCK + (threadIdx.x & ~31) + lane;
  int64_t nbeg = first < p.n ? ldr(p.rp, first) : 0, nend = first < p.n ? ldr(p.rp, first + 1) : 0;
  for (int64_t base = (int64_t)blk(p) * BLOCK + (threadIdx.x & ~31); base < p.n; base += stride) {
    const int64_t v = base + lane;
    const bool act = v < p.n;
    int b = -1;
    WE e;
    const int64_t cbeg = nbeg, cend_ = nend;
    if (v + stride < p.n) {
      nbeg = ldr(p.rp, v + stride);
      nend = ldr(p.rp, v + stride + 1);
    }
    if (act) {
      e.v = (int32_t)(p.v_base + v);
      e.beg = cbeg;
      const int64_t end = cend_;
      const int64_t deg = end - e.beg;
      if (sizeof(S) < 4 && deg > NARROW_MAX_DEG) wide = true;
      maxdeg = max(maxdeg, (uint32_t)min(deg, (int64_t)0xffffffff));
      b = bin_of(p, deg);
      sts(st + p.v_base + v, 1u);
      if (PUSH) sts(p.fmp + p.v_base + v, 0u);  // planes are indexed by global id
      if (p.dirty) sts(p.dirty + e.v, 0u);
      e.k = 0;
      if (dense && POL != DEGREE) {
        e.k = b == 0 ? split_fast(p, e.v, e.beg, end) : row_split(p, e.v, e.beg, end);
        p.ksplit[e.v] = e.k;
      } else if (dense) {
        p.ksplit[e.v] = (int32_t)deg;  // DEGREE: the array holds the degrees (one load per compare)
        if (dist(p)) {  // ... and the ranks holding v as a ghost need its degree
          for (uint32_t m = lds(p.bmask + e.v); m; m &= m - 1) p.peer[__ffs(m) - 1].ksplit[e.v] = (int32_t)deg;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < NBIN; ++k) {
      const unsigned m = __ballot_sync(FULL, b == k);
      if (m && lane == 0) atomicAdd(&s_cnt[k], (uint32_t)__popc(m));
    }
    if (dense) {
      const unsigned m = __ballot_sync(FULL, b == 1);
      if (m) {
        const int leader = __ffs(m) - 1;
        uint32_t pos = 0;
        if (lane == leader) pos = atomicAdd(&p.info->cursor[1], (uint32_t)__popc(m));
        pos = __shfl_sync(FULL, pos, leader);
        if (b == 1) stw(p.heavy + pos + __popc(m & lanemask_lt()), e);
      }
    }
  }
  // padding [n, pitch) of the state words, plane 0 and the marks (read, never used, by the
  // 16-vertex vectors of the dense sweeps); the multi-GPU pre-pass fills whole replicas
  if (!dist(p)) {
    for (int64_t v = (int64_t)p.n + (int64_t)blk(p) * BLOCK + threadIdx.x; v < p.plane; v += stride) {
      sts(st + v, SW<S>::COMMIT);
      if (PUSH) sts(p.fmp + v, 0u);
      if (p.dirty) sts(p.dirty + v, 0u);
    }
  }
  if (wide) set_status(p, ST_NEED32);
  maxdeg = __reduce_max_sync(FULL, maxdeg);
  if (lane == 0 && maxdeg) {  // multi-GPU: the global max (decides the dirty-set rounds everywhere)
    if (dist(p)) for (int q = 0; q < p.nranks; ++q) atomicMax(&p.peer[q].info->maxdeg, maxdeg);
    else atomicMax(&p.info->maxdeg, maxdeg);
  }
  if (blk(p) == 0 && threadIdx.x == 0) {
    p.info->wlp[0] = (unsigned long long)p.wl0;
    p.info->wlp[1] = (unsigned long long)p.wl1;
  }
  __syncthreads();
  if (threadIdx.x < NBIN && s_cnt[threadIdx.x]) atomicAdd(&p.info->binsize[threadIdx.x], s_cnt[threadIdx.x]);
}

// Multi-GPU pre-pass (before the ingest): every replica word starts pending with tentative
// colour 1 (round 1), and bmask[v] of every local vertex v = the set of other ranks owning a
// neighbour of v — exactly the ranks that read v's state word (the graph is symmetric), so the
// only ones its tentative colours and commit are sent to.  One warp per local vertex.
__device__ __forceinline__ void prologue_dist(const Params& p) {
  const int64_t T = (int64_t)nblk(p) * BLOCK;
  const int lane = threadIdx.x & 31;
  const int64_t nw = T >> 5;
  for (int64_t u = ((int64_t)blk(p) * BLOCK + threadIdx.x) >> 5; u < p.n; u += nw) {
    const int64_t beg = ldr(p.rp, u), end = ldr(p.rp, u + 1);
    uint32_t m = 0;
    for (int64_t e = beg + lane; e < end; e += 32) {
      const int32_t w = ldc(p.ci, e);
      if (w < p.v_base || w >= p.v_base + p.n) m |= 1u << owner(p, w);
    }
    m = __reduce_or_sync(FULL, m);
    if (lane == 0) sts(p.bmask + p.v_base + u, m);
  }
  if (blk(p) == 0 && threadIdx.x == 0) p.info->gtot[1] = (uint32_t)p.n_global;
}
// (the whole pitch: the 16-vertex vectors of the dense sweeps also read the ghost and padding
// entries of plane 0 and of the marks, whose values they never use)
template <class S>
__device__ __forceinline__ void fill_replica(const Params& p) {
  S* st = (S*)p.st;
  for (int64_t v = (int64_t)blk(p) * BLOCK + threadIdx.x; v < p.plane; v += (int64_t)nblk(p) * BLOCK) {
    sts(st + v, 1u);
    sts(p.fmp + v, 0u);
    if (p.dirty) sts(p.dirty + v, 0u);
  }
}

// P1: W_1 = V, split into bin segments of wl0 (warp-aggregated cursors; order within a
// bin is free, reading C12).
__device__ __forceinline__ void prologue_scatter(const Params& p, const Bins& bins) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)nblk(p) * BLOCK;
  for (int64_t base = (int64_t)blk(p) * BLOCK + (threadIdx.x & ~31); base < p.n; base += stride) {
    const int64_t v = base + lane;
    const bool act = v < p.n;
    int b = -1;
    WE e;
    if (act) {
      e.v = (int32_t)(p.v_base + v);
      e.k = -1;  // split computed by the first Phase B visit
      e.beg = ldr(p.rp, v);
      b = bin_of(p, ldr(p.rp, v + 1) - e.beg);
    }
#pragma unroll
    for (int k = 0; k < NBIN; ++k) {
      const unsigned m = __ballot_sync(FULL, b == k);
      if (!m) continue;
      const int leader = __ffs(m) - 1;
      uint32_t pos = 0;
      if (lane == leader) pos = atomicAdd(&p.info->cursor[k], (uint32_t)__popc(m));
      pos = __shfl_sync(FULL, pos, leader);
      if (b == k) stw(p.wl0 + bins.off[k] + pos + __popc(m & lanemask_lt()), e);
    }
  }
  if (blk(p) == 0 && threadIdx.x < NBIN) p.info->cnt[1][threadIdx.x] = p.info->binsize[threadIdx.x];
}

// ---- warp-flattened segment loops
// Each lane of a warp holds a segment of W_i items (a vertex's next stretch of its conflict
// scan, or a winner's row for the commit scatter).  The warp walks the concatenation of all
// segments 32 x FLAT_U items per step, so short and long segments share the lanes evenly
// instead of one lane (or one vertex at a time) doing all of a segment's work.  Item f
// belongs to the lane `owner` with E[owner-1] <= f < E[owner] (E = inclusive prefix sum of
// W over the lanes, found by a 5-step binary search over shuffles).
#ifndef GC_FLAT_U
#define GC_FLAT_U 2
#endif
constexpr int FLAT_U = GC_FLAT_U;
#ifndef GC_CAPMUL
#define GC_CAPMUL 4           // growth of the conflict-scan pass length after the first two passes
#endif  // items per lane per step (independent loads in flight)

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  return x;
}
__device__ __forceinline__ int flat_owner(uint32_t E, uint32_t f) {
  int o = 0;
#pragma unroll
  for (int b = 16; b; b >>= 1)
    if (__shfl_sync(FULL, E, o + b - 1) <= f) o += b;
  return o;
}

// Phase shared memory (one object per CTA, whichever phase function uses it).
#ifndef GC_VPL
#define GC_VPL 2
#endif
#ifndef GC_LOCAL_PASS1
#define GC_LOCAL_PASS1 1
#endif
#ifndef GC_LOCAL_SCATTER
#define GC_LOCAL_SCATTER 8        // sparse batches: rows up to this length scattered lane-locally
#endif
#ifndef GC_LOCAL_MARK
#define GC_LOCAL_MARK 16          // dense Phase A: successor ranges up to this length marked lane-locally
#endif
constexpr int VPL = GC_VPL;     // dense batches: consecutive vertices per lane
constexpr int WB = 32 * VPL;    // vertices per warp batch
struct WideSeg {                // per-warp segment table of one dense batch (slot = vertex - base)
  int64_t sbase[WB];            // row position of scan step 0
  uint32_t E[WB];               // inclusive prefix over the slots of the items of this pass
  uint32_t pos[WB];             // scan steps done
  int32_t k[WB];                // split (row start = sbase - k + 1 / sbase - k / sbase by policy)
  uint32_t deg[WB];
  int first[WB];                // work counters: first hit
  uint32_t tent[WB];
  uint32_t lost[VPL];
};
struct BSmem {
  WE pbuf[WARPS][PBUF];   // per-warp push staging (Pusher, bin 0)
  union {
    WideSeg seg[WARPS];     // dense Phase-B batches
    int32_t clist[WARPS][512];  // dense Phase A: a warp's changed vertices (N1 marks)
  };
  int first;              // conflict_cta
  int32_t k;              // cta_vertex split broadcast
  int cwfirst[WARPS][32]; // work counters: first hit per lane's vertex
};
__device__ __forceinline__ BSmem& bsmem() {
  __shared__ BSmem s;
  return s;
}

// ---------------------------------------------------------------- a2: Phase A
// Incremental-mask mode: every pending vertex is O(1) in the number of neighbours: its own
// thread reads its plane bytes two planes at a time (independent loads) until a non-full one
// gives the colour — in round r at most ceil((r-1)/8) planes can be non-empty (pin P11).
// Beyond the last plane the whole warp runs the exact windowed First-Fit (reading C7).
// 8-bit state words cannot hold colours > 127: the run restarts with 16-bit words
// (ST_NEED16).
template <class S>
__device__ __forceinline__ void store_tent(const Params& p, S* st, int32_t v, uint32_t t) {
  if (sizeof(S) == 1 && t > SW<S>::CMASK) {
    set_status(p, ST_NEED16);
  } else {
    sts(st + v, t);
    bcast_word<S>(p, v, t);
  }
}

// First free colour from the planes in Phase A of round r, 0 when all np planes are full.
// Colours committed before round r are <= r - 1 (a colour c is committed in round >= c, pin
// P11), so only planes 0..K-1, K = (r - 2) / 8 + 1, can hold any; when they are full the answer
// is 8K + 1 without reading plane K (which may not even be zeroed yet: plane k is zeroed in
// Phase A of round 8k, concurrently with this lookup).
__device__ __forceinline__ uint32_t plane_firstfit(const Params& p, int32_t v, uint32_t r) {
  const uint8_t* f = p.fmp + v;
  const uint32_t K = min(p.np, r >= 2 ? (r - 2) / 8 + 1 : 1u);
  for (uint32_t k = 0; k < K; k += 2) {
    const uint32_t b0 = lds(f + (int64_t)k * p.plane);
    const uint32_t b1 = k + 1 < K ? lds(f + (int64_t)(k + 1) * p.plane) : 0xffu;
    if (b0 != 0xffu) return 8u * k + (uint32_t)__ffs(b0 ^ 0xffu);
    if (b1 != 0xffu) return 8u * (k + 1) + (uint32_t)__ffs(b1 ^ 0xffu);
  }
  return K < p.np ? 8u * K + 1u : 0u;
}

// ---- dirty-set rounds (reading of the data-driven rationale P:453-462)
// The Phase-B outcome of a pending vertex v depends only on tent(v) and on tent(w) of its
// predecessors w (the neighbours that can make it recolour: lower ids for HIGHER_ID, higher
// ids for LOWER_ID, all for DEGREE).  A vertex still pending lost last round; if neither its
// tentative colour nor any predecessor's changed since, it loses again.  (A predecessor that
// committed with colour c either was not v's conflict — no effect — or had c = tent(v), and
// then c entered v's mask and tent(v) changed.)  So when Phase A changes tent(v) it marks v
// and its successors dirty, and Phase B of a marking round examines only dirty vertices; the
// others are losers as they stand.  Marks are set in Phase A and cleared by the Phase-B lane
// that reads them; a round that does not mark examines every pending vertex.
template <int POL, bool CW>
__device__ __forceinline__ void mark_dirty(const Params& p, int32_t v, int64_t beg, int64_t end, int32_t k, Work& wk) {
  const int64_t lo = POL == HIGHER_ID ? beg + k : beg;
  const int64_t hi = POL == LOWER_ID ? beg + k : end;
  sts(p.dirty + v, 1u);
  for (int64_t e = lo; e < hi; e += 4) {
    int32_t w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = e + u < hi ? ldc(p.ci, e + u) : -1;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (w[u] >= 0) sts(dirty_of(p, w[u]) + w[u], 1u);
  }
  if (CW) wk.v[W_MARK] += (unsigned long long)(hi - lo + 1);
}

// New tentative colour t of pending vertex v whose previous one is t_old: store it and, when
// it changed and this round marks, mark v and its successors.
template <class S, int POL, bool CW>
__device__ __forceinline__ void tent_update(const Params& p, S* st, int32_t v, uint32_t t, uint32_t t_old, bool mark,
                                            int64_t beg, int64_t end, int32_t k, uint32_t& nchg, Work& wk) {
  if (t == t_old) return;
  store_tent<S>(p, st, v, t);
  ++nchg;
  if (mark) {
    if (beg < 0) {
      beg = RP(p, v);
      end = RP(p, v + 1);
    }
    if (end < 0) end = RP(p, v + 1);
    if (k < 0 && POL != DEGREE) k = ldks(p.ksplit + v);
    mark_dirty<POL, CW>(p, v, beg, end, k, wk);
  }
}

__device__ __forceinline__ void flush_chg(const Params& p, uint32_t r, uint32_t nchg, Work& wk, bool cw) {
#ifndef GC_FLUSH_CHG
#define GC_FLUSH_CHG 0
#endif
  if (!GC_FLUSH_CHG && !cw && !p.n1chg) return;  // only the N1_CHG rule and the work counters read it
  nchg = __reduce_add_sync(FULL, nchg);
  if ((threadIdx.x & 31) == 0 && nchg) {
    atomicAdd(&p.info->chg[r % 3], nchg);
    if (cw) wk.v[W_TCHG] += nchg;
  }
}

template <class S, int POL, bool CW>
__device__ __forceinline__ void phase_a_mask(const Params& p, uint32_t r, const Bins& bins, const WE* W,
                                             const uint32_t* nb, bool mark, Work& wk) {
  S* st = (S*)p.st;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = blk(p) * WARPS + (threadIdx.x >> 5), nw = nblk(p) * WARPS;
  uint32_t nchg = 0;
#pragma unroll
  for (int b = 0; b < NBIN; ++b) {
    const WE* Wb = W + bins.off[b];
    const uint32_t cnt = nb[b];
    for (uint32_t base = gw * 32; base < cnt; base += nw * 32) {
      const uint32_t i = base + lane;
      WE e;
      e.v = 0;
      e.k = -1;
      e.beg = -1;
      uint32_t t_old = 0;
      bool fb = false;
      if (i < cnt) {
        e = ldw(Wb + i);
        t_old = lds(st + e.v) & SW<S>::CMASK;
        if (CW) wk.v[W_WDEG] += (unsigned long long)(RP(p, e.v + 1) - e.beg);
        const uint32_t t = plane_firstfit(p, e.v, r);
        if (t) tent_update<S, POL, CW>(p, st, e.v, t, t_old, mark, e.beg, -1, e.k, nchg, wk);
        else fb = true;
      }
      unsigned m = __ballot_sync(FULL, fb);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int32_t u = __shfl_sync(FULL, e.v, src);
        const uint32_t to = __shfl_sync(FULL, t_old, src);
        uint32_t t = 8u * p.np + 1u;  // > 127 when np = MAX_PLANES: 8-bit words restart
        if (sizeof(S) > 1 || t <= SW<S>::CMASK) t = firstfit_warp<S, CW>(p, u, t, wk, lane);
        if (lane == 0) tent_update<S, POL, CW>(p, st, u, t, to, mark, -1, -1, -1, nchg, wk);
      }
    }
  }
  flush_chg(p, r, nchg, wk, CW);
}

// Plane k (colours 8k+1..8k+8) is zeroed in Phase A of round 8k, before any colour it holds
// can be committed (round >= 8k+1) or looked up (Phase A of round >= 8k+1).
__device__ __forceinline__ void zero_plane(const Params& p, uint32_t r) {
  if (r % 8 != 0 || r / 8 >= p.np) return;
  uint4* q = (uint4*)(p.fmp + (int64_t)(r / 8) * p.plane);
  const int64_t nq = p.plane / 16;
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int64_t i = (int64_t)blk(p) * BLOCK + threadIdx.x; i < nq; i += (int64_t)nblk(p) * BLOCK) q[i] = z;
}

// Pull mode (GC_FLAG_PULL_FIRSTFIT, the paper's FirstFit): full neighbour scan per round;
// bin 0: degree <= 32 by the vertex's own thread, larger by the whole warp; bin 1: one CTA.
template <class S, bool CW>
__device__ __forceinline__ void phase_a_pull(const Params& p, const Bins& bins, const WE* W, const uint32_t* nb,
                                             Work& wk, uint32_t* s_win) {
  S* st = (S*)p.st;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = blk(p) * WARPS + (threadIdx.x >> 5), nw = nblk(p) * WARPS;
  {
    const WE* Wb = W + bins.off[0];
    for (uint32_t base = gw * 32; base < nb[0]; base += nw * 32) {
      const uint32_t i = base + lane;
      bool big = false;
      WE e;
      if (i < nb[0]) {
        e = ldw(Wb + i);
        const int64_t deg = RP(p, e.v + 1) - e.beg;
        if (deg <= 32) store_tent<S>(p, st, e.v, firstfit_thread<S, CW>(p, e.v, 1u, wk));
        else big = true;
      }
      unsigned m = __ballot_sync(FULL, big);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int32_t u = __shfl_sync(FULL, e.v, src);
        const uint32_t t = firstfit_warp<S, CW>(p, u, 1u, wk, lane);
        if (lane == 0) store_tent<S>(p, st, u, t);
      }
    }
  }
  {
    const WE* Wb = W + bins.off[1];
    for (uint32_t i = blk(p); i < nb[1]; i += nblk(p)) {
      const int32_t v = ldw_v(Wb + i);
      const uint32_t t = firstfit_cta<S, CW>(p, v, 1u, wk, s_win);
      if (threadIdx.x == 0) store_tent<S>(p, st, v, t);
    }
  }
}

// reset the counters round r+1 will push into and the work queues it will pop from
// (last used in round r-2)
__device__ __forceinline__ void reset_next(const Params& p, uint32_t r) {
  if (blk(p) == 0 && threadIdx.x < NBIN) {
    p.info->cnt[(r + 1) % 3][threadIdx.x] = 0;
    p.info->qctr[(r + 1) % 3][threadIdx.x][0] = 0;
    if (threadIdx.x == 0) {
      // multi-GPU: the other ranks add into this copy only at the end of Phase B of round r
      p.info->gtot[(r + 1) % 3] = 0;
      p.info->chg[(r + 1) % 3] = 0;
      p.info->wl_cnt[(r + 1) % 3] = 0;
      p.info->dl_cnt[(r + 1) % 3] = 0;
    }
  }
}

template <class S, int POL, bool PUSH, bool CW>
__device__ __forceinline__ void phase_a(const Params& p, uint32_t r, const Bins& bins, const WE* W, bool mark,
                                        Work& wk) {
  __shared__ uint32_t s_win[2];
  const uint32_t cur = r % 3;
  uint32_t nb[NBIN];
#pragma unroll
  for (int b = 0; b < NBIN; ++b) nb[b] = head().cnt[cur][b];
  reset_next(p, r);
  if (CW && threadIdx.x == 0 && blk(p) == 0) {
    wk.v[W_A_VERT] += (unsigned long long)nb[0] + nb[1];
    wk.v[W_SA_ENT] += (unsigned long long)nb[0] + nb[1];
  }
  if (PUSH) {
    zero_plane(p, r);
    phase_a_mask<S, POL, CW>(p, r, bins, W, nb, mark, wk);
  } else {
    phase_a_pull<S, CW>(p, bins, W, nb, wk, s_win);
  }
}

// Dense rounds (large |W|): W_r is implicit — every vertex whose state word is not committed —
// and Phase A walks all n state words in id order: 16 consecutive vertices per thread, their
// state words and plane-0 mask bytes read and the state words written back as 16-byte vectors
// (no other thread touches these words during Phase A; committed words are written back
// unchanged).  A vertex whose plane 0 is full reads its other planes one by one.
__device__ __forceinline__ uint4 ldv(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void stv(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <class S, int POL, bool CW>
__device__ __forceinline__ void phase_a_dense(const Params& p, uint32_t r, bool mark, Work& wk) {
  S* st = (S*)p.st;
  reset_next(p, r);
  if (CW && threadIdx.x == 0 && blk(p) == 0) {
    const uint32_t cur = r % 3;
    wk.v[W_A_VERT] += (unsigned long long)head().cnt[cur][0] + head().cnt[cur][1];
    wk.v[W_DA_SWEEP] += (unsigned long long)p.n;
  }
  zero_plane(p, r);
  const int lane = threadIdx.x & 31;
  const int64_t nthreads = (int64_t)nblk(p) * BLOCK;
  // groups of 16 global ids aligned to 16 covering this rank's range [vlo, vend)
  const int64_t vlo = p.v_base, vend = (int64_t)p.v_base + p.n, lo16 = vlo & ~(int64_t)15;
  const int64_t ngroups = (vend - lo16 + 15) / 16;
  const int64_t g0 = (int64_t)blk(p) * BLOCK + (threadIdx.x & ~31);
  uint32_t nchg = 0;
  int32_t* clist = bsmem().clist[threadIdx.x >> 5];
  for (int64_t gb = g0; gb < ngroups; gb += nthreads) {
    const int64_t g = gb + lane;
    const int64_t v0 = lo16 + g * 16;
    uint32_t fb = 0, chgm = 0;
    if (g < ngroups) {
      constexpr int NW = 4 * (int)sizeof(S);          // 32-bit words holding 16 state words
      constexpr int PER = 4 / (int)sizeof(S);          // state words per 32-bit word
      constexpr uint32_t SMASK = sizeof(S) == 4 ? 0xffffffffu : ((1u << (8 * sizeof(S))) - 1u);
      uint32_t w[NW];
#pragma unroll
      for (int i = 0; i < (int)sizeof(S); ++i) {
        const uint4 q = ldv(st + v0 + i * (16 / sizeof(S)));
        w[4 * i] = q.x;
        w[4 * i + 1] = q.y;
        w[4 * i + 2] = q.z;
        w[4 * i + 3] = q.w;
      }
      const uint4 pl = ldv(p.fmp + v0);
      const uint32_t pw[4] = {pl.x, pl.y, pl.z, pl.w};
      // plane 1 as a vector too once colours 9.. can be committed (round >= 10)
      uint4 pl1 = make_uint4(0, 0, 0, 0);
      if (r >= 10 && p.np > 1) pl1 = ldv(p.fmp + p.plane + v0);
      const uint32_t pw1[4] = {pl1.x, pl1.y, pl1.z, pl1.w};
      bool dirty = false;
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        const int wi = h / PER, sh = (h % PER) * 8 * (int)sizeof(S);
        const uint32_t sv = (w[wi] >> sh) & SMASK;
        if (v0 + h >= vlo && v0 + h < vend && !(sv & SW<S>::COMMIT)) {
          const uint32_t b0 = (pw[h >> 2] >> ((h & 3) * 8)) & 0xffu;
          const uint32_t b1 = (pw1[h >> 2] >> ((h & 3) * 8)) & 0xffu;
          const uint32_t t = b0 != 0xffu   ? (uint32_t)__ffs(b0 ^ 0xffu)
                             : b1 != 0xffu ? 8u + (uint32_t)__ffs(b1 ^ 0xffu)
                                           : plane_firstfit(p, (int32_t)(v0 + h), r);
          if (t == 0) {
            fb |= 1u << h;
          } else if (t != (sv & SW<S>::CMASK)) {
            if (sizeof(S) == 1 && t > SW<S>::CMASK) {
              set_status(p, ST_NEED16);  // the word keeps its old value: the run is widened and resumed here
            } else {
              w[wi] = (w[wi] & ~(SMASK << sh)) | ((t & SMASK) << sh);
              dirty = true;
              chgm |= 1u << h;
            }
          }
        }
      }
      if (dirty) {
        if (dist(p) && (v0 < vlo || v0 + 16 > vend)) {
          // a group straddling a rank boundary also holds ghost words that their owner may be
          // writing into this replica right now: store only this rank's changed words
#pragma unroll
          for (int h = 0; h < 16; ++h)
            if (chgm >> h & 1u) sts(st + v0 + h, (w[h / PER] >> ((h % PER) * 8 * (int)sizeof(S))) & SMASK);
        } else {
#pragma unroll
          for (int i = 0; i < (int)sizeof(S); ++i)
            stv(st + v0 + i * (16 / sizeof(S)), make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]));
        }
        if (dist(p)) {  // changed boundary vertices: the new tentative colour to their ghosts
          const uint4 bq = ldv(p.bmask + v0);
          const uint32_t bw[4] = {bq.x, bq.y, bq.z, bq.w};
#pragma unroll
          for (int h = 0; h < 16; ++h) {
            const uint32_t bm = (bw[h >> 2] >> ((h & 3) * 8)) & 0xffu;
            if ((chgm >> h & 1u) && bm)
              bcast_word<S>(p, (int32_t)(v0 + h), (w[h / PER] >> ((h % PER) * 8 * (int)sizeof(S))) & SMASK, bm);
          }
        }
      }
      nchg += __popc(chgm);
      if (CW) {  // sum of the degrees of the pending vertices (SURVEY §8(d) units)
#pragma unroll
        for (int h = 0; h < 16; ++h) {
          const int wi = h / PER, sh = (h % PER) * 8 * (int)sizeof(S);
          if (v0 + h >= vlo && v0 + h < vend && !(((w[wi] >> sh) & SMASK) & SW<S>::COMMIT))
            wk.v[W_WDEG] += (unsigned long long)(RP(p, v0 + h + 1) - RP(p, v0 + h));
        }
      }
    }
    // marks of the changed vertices and their successors: the warp's changed vertices (up to
    // 512, clustered along the colouring front) are listed in shared memory and dealt out one
    // per lane per step; the successor ranges of a step are walked as one flattened loop
    if (mark && __any_sync(FULL, chgm != 0)) {
      const uint32_t c = __popc(chgm);
      const uint32_t ci = warp_incl_scan(c, lane);
      const uint32_t tot = __shfl_sync(FULL, ci, 31);
      uint32_t at = ci - c;
      for (uint32_t cm = chgm; cm; cm &= cm - 1) clist[at++] = (int32_t)(v0 + __ffs(cm) - 1);
      __syncwarp();
      for (uint32_t i0 = 0; i0 < tot; i0 += 32) {
        int64_t lo = 0, hi = 0;
        if (i0 + lane < tot) {
          const int32_t v = clist[i0 + lane];
          const int64_t beg = RP(p, v), end = RP(p, v + 1);
          const int32_t k = POL != DEGREE ? ldks(p.ksplit + v) : 0;
          lo = POL == HIGHER_ID ? beg + k : beg;
          hi = POL == LOWER_ID ? beg + k : end;
          sts(p.dirty + v, 1u);
          if (CW) wk.v[W_MARK] += (unsigned long long)(hi - lo + 1);
        }
        const uint32_t Wn = (uint32_t)(hi - lo);
#if GC_LOCAL_SCATTER
        if (__reduce_max_sync(FULL, Wn) <= (uint32_t)GC_LOCAL_MARK) {  // short ranges: every lane its own
#pragma unroll
          for (uint32_t j0 = 0; j0 < (uint32_t)GC_LOCAL_MARK; j0 += 4) {
            if (j0 >= Wn) break;
            int32_t w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) w[u] = j0 + u < Wn ? ldc(p.ci, lo + j0 + u) : -1;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (w[u] >= 0) sts(dirty_of(p, w[u]) + w[u], 1u);
          }
          continue;
        }
#endif
        const uint32_t E = warp_incl_scan(Wn, lane);
        const uint32_t T = __shfl_sync(FULL, E, 31);
        for (uint32_t f0 = 0; f0 < T; f0 += 32 * 4) {
          int32_t w[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t f = f0 + u * 32 + lane;
            const int o = flat_owner(E, f);
            const int oc = o < 32 ? o : 31;
            const uint32_t Eo = __shfl_sync(FULL, E, oc), Wo = __shfl_sync(FULL, Wn, oc);
            const int64_t lo_o = __shfl_sync(FULL, lo, oc);
            w[u] = f < T ? ldc(p.ci, lo_o + (f - (Eo - Wo))) : -1;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (w[u] >= 0) sts(dirty_of(p, w[u]) + w[u], 1u);
        }
      }
      __syncwarp();
    }
    // colours beyond the planes: the whole warp, one vertex at a time (exact, reading C7)
    unsigned m = __ballot_sync(FULL, fb != 0);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      uint32_t f = __shfl_sync(FULL, fb, src);
      const int64_t sv0 = __shfl_sync(FULL, v0, src);
      while (f) {
        const int h = __ffs(f) - 1;
        f &= f - 1;
        const int32_t u = (int32_t)(sv0 + h);
        uint32_t t = 8u * p.np + 1u;
        if (sizeof(S) > 1 || t <= SW<S>::CMASK) t = firstfit_warp<S, CW>(p, u, t, wk, lane);
        if (lane == 0) tent_update<S, POL, CW>(p, st, u, t, lds(st + u) & SW<S>::CMASK, mark, -1, -1, -1, nchg, wk);
      }
    }
  }
  flush_chg(p, r, nchg, wk, CW);
}

// ---------------------------------------------------------------- a3: Phase B + push
// Winners commit (set the top bit of their own word) and, in mask mode, OR their colour bit
// into the forbidden mask of every neighbour; losers go to W_out through the Pusher.

// Warps pop chunks of ch items from a per-bin queue head (one atomic per chunk) so that
// costly items (long scans) do not leave the rest of the grid idle at the phase barrier.
// ch shrinks with |W| (down to one vertex per warp in the small tail rounds, where the few
// remaining vertices are the high-degree ones with long scans).
__device__ __forceinline__ uint32_t pop_chunk(uint32_t* q, uint32_t ch, int lane) {
  uint32_t b = 0;
  if (lane == 0) b = atomicAdd(q, ch);
  return __shfl_sync(FULL, b, 0);
}

// Adds the per-warp values (lane 0's v) of the whole CTA to *g with one atomic per CTA.  Every
// thread of the CTA must call it.
#ifndef GC_CTA_ADD
#define GC_CTA_ADD 1
#endif
__device__ __forceinline__ void cta_add(uint32_t* g, uint32_t v) {
  if (!GC_CTA_ADD) {
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(g, v);
    return;
  }
  __shared__ uint32_t s_sum;
  if (threadIdx.x == 0) s_sum = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_sum, v);
  __syncthreads();
  if (threadIdx.x == 0 && s_sum) atomicAdd(g, s_sum);
}

// Position of the j-th entry of a scan range in scan order.
__device__ __forceinline__ int64_t scan_pos(int64_t lo, int64_t hi, bool down, int64_t j) {
  return down ? hi - 1 - j : lo + j;
}

// ---- list rounds: winners of round r recorded for Phase A of round r+1
__device__ __forceinline__ void rec_winners(const Params& p, uint32_t r, bool win, int32_t v, int lane) {
  const unsigned m = __ballot_sync(FULL, win);
  if (!m) return;
  const int leader = __ffs(m) - 1;
  uint32_t pos = 0;
  if (lane == leader) pos = atomicAdd(&p.info->wl_cnt[r % 3], (uint32_t)__popc(m));
  pos = __shfl_sync(FULL, pos, leader);
  if (win) ((r & 1) ? p.wlw1 : p.wlw0)[pos + __popc(m & lanemask_lt())] = v;
}

// One batch of up to 32 vertices, one per lane (act).  The conflict scans of all of them
// advance together in passes over the flattened segments: pass 1 examines the first 4
// positions of every scan range (the nearest lower ids, where most conflicts are), later
// passes 12, 48, 192, ... more, so that early exit is kept for the losers while all lanes stay
// busy.  A vertex with a hit loses; a vertex whose range is exhausted wins: it commits and its
// row is scattered into the forbidden masks of its neighbours, again as one flattened loop
// over all winners of the batch.  e.k must be known (>= 0) unless POL == DEGREE; end = -1
// when not yet read.  Returns the lane's state: 0 inactive, 1 lose, 2 win.
template <class S, int POL, bool PUSH, bool CW>
__device__ __forceinline__ int batch_b(const Params& p, int lane, bool act, const WE& e, uint32_t tent, int64_t end,
                                       Work& wk, int* s_first, uint32_t rec_round = 0) {
  S* st = (S*)p.st;
  constexpr uint32_t CM = SW<S>::CMASK;
  int64_t sbase = 0, dv = 0;
  int sdir = 1;
  uint32_t len = 0, pos = 0;
  int state = 0;  // 0 inactive, 1 lose, 2 win, 3 undecided
  if (act) {
    if (POL != HIGHER_ID && end < 0) end = RP(p, e.v + 1);
    const ScanRange<POL> sr = scan_range<POL>(e.beg, e.k, end);
    sbase = sr.down ? sr.hi - 1 : sr.lo;
    sdir = sr.down ? -1 : 1;
    len = (uint32_t)(sr.hi - sr.lo);
    if (POL == DEGREE) dv = end - e.beg;
    state = len ? 3 : 2;
  }
  uint32_t cap = PROBE;
#if GC_LOCAL_PASS1
  // pass 1, lane-local: the first PROBE positions of the lane's own scan range (nearest first),
  // PROBE independent loads per lane and no owner search (the flattened passes below spend ~10
  // shuffles per item finding owners and their segment data)
  {
    int32_t w[PROBE];
#pragma unroll
    for (int u = 0; u < PROBE; ++u) w[u] = state == 3 && (uint32_t)u < len ? ldc(p.ci, sbase + sdir * u) : -1;
    int first = -1;
#pragma unroll
    for (int u = PROBE - 1; u >= 0; --u) {
      if (w[u] < 0) continue;
      const uint32_t sv = ldnb(st + w[u]);
      if ((sv & CM) == tent && recolors<POL>(p, e.v, w[u], dv)) first = u;
    }
    if (state == 3) {
      if (first >= 0) {
        state = 1;
        if (CW) { wk.v[W_B_EDGE] += first + 1; wk.v[W_B_GATHER] += first + 1; }
      } else {
        pos = len < (uint32_t)PROBE ? len : (uint32_t)PROBE;
        if (pos == len) {
          state = 2;
          if (CW) { wk.v[W_B_EDGE] += len; wk.v[W_B_GATHER] += len; }
        }
      }
    }
    cap = 3 * PROBE;
  }
#endif
  // conflict-scan passes
  for (;;) {
    const bool und = state == 3;
    if (!__any_sync(FULL, und)) break;
    const uint32_t Wn = und ? min(len - pos, cap) : 0u;
    const uint32_t E = warp_incl_scan(Wn, lane);
    const uint32_t T = __shfl_sync(FULL, E, 31);
    if (CW) s_first[lane] = 0x7fffffff;
    __syncwarp();
    uint32_t lost = 0;
    for (uint32_t f0 = 0; f0 < T; f0 += 32 * FLAT_U) {
      int32_t w[FLAT_U];
      int own[FLAT_U];
      int64_t jj[FLAT_U];
#pragma unroll
      for (int u = 0; u < FLAT_U; ++u) {
        const uint32_t f = f0 + u * 32 + lane;
        const int o = flat_owner(E, f);
        const int oc = o < 32 ? o : 31;
        const uint32_t Eo = __shfl_sync(FULL, E, oc), Wo = __shfl_sync(FULL, Wn, oc);
        const uint32_t po = __shfl_sync(FULL, pos, oc);
        const int64_t bo = __shfl_sync(FULL, sbase, oc);
        const int dro = __shfl_sync(FULL, sdir, oc);
        own[u] = f < T ? oc : -1;
        jj[u] = (int64_t)(f - (Eo - Wo) + po);
        w[u] = f < T ? ldc(p.ci, bo + dro * jj[u]) : 0;
      }
#pragma unroll
      for (int u = 0; u < FLAT_U; ++u) {
        const int oc = own[u] < 0 ? 0 : own[u];
        const uint32_t to = __shfl_sync(FULL, tent, oc);
        const int32_t vo = __shfl_sync(FULL, e.v, oc);
        const int64_t dvo = POL == DEGREE ? __shfl_sync(FULL, dv, oc) : 0;
        const uint32_t sv = own[u] >= 0 ? ldnb(st + w[u]) : 0u;
        const bool hit = own[u] >= 0 && (sv & CM) == to && recolors<POL>(p, vo, w[u], dvo);
        if (hit) {
          lost |= 1u << oc;
          if (CW) atomicMin(&s_first[oc], (int)jj[u]);
        }
      }
    }
    lost = __reduce_or_sync(FULL, lost);
    __syncwarp();
    if (und) {
      if (lost >> lane & 1u) {
        state = 1;
        if (CW) { const uint32_t ex = (uint32_t)s_first[lane] + 1; wk.v[W_B_EDGE] += ex; wk.v[W_B_GATHER] += ex; }
      } else {
        pos += Wn;
        if (pos == len) {
          state = 2;
          if (CW) { wk.v[W_B_EDGE] += len; wk.v[W_B_GATHER] += len; }
        }
      }
    }
    cap = cap < 1024 ? (cap == (uint32_t)PROBE ? 3 * PROBE : cap * GC_CAPMUL) : cap;  // 4, 12, 48, 192, 768, ...
  }
  // winners commit; the forbidden masks of their neighbours get their colour bit
  const bool win = state == 2;
  if (win) {
    sts(st + e.v, tent | SW<S>::COMMIT);
    bcast_word<S>(p, e.v, tent | SW<S>::COMMIT);
  }
  if (rec_round) rec_winners(p, rec_round, win, e.v, lane);
  if (PUSH) {
    const bool sc = win && tent <= 8u * p.np;
    if (sc && end < 0) end = RP(p, e.v + 1);
    const uint32_t Wn = sc ? (uint32_t)(end - e.beg) : 0u;
    if (CW) { wk.v[W_SCATTER] += Wn; if (!p.sfilter) wk.v[W_SCATTER_RED] += Wn; }
#if GC_LOCAL_SCATTER
    // short rows only (bounded-degree graphs): every lane scatters its own winner's row, up to
    // GC_LOCAL_SCATTER entries 4 loads at a time, without the flattened loop's owner search
    if (!p.sfilter && __reduce_max_sync(FULL, Wn) <= (uint32_t)GC_LOCAL_SCATTER) {
      if (Wn) {
        uint8_t* const pl = (dist(p) ? nullptr : p.fmp) + (int64_t)((tent - 1) >> 3) * p.plane;
        const uint32_t bit = 1u << ((tent - 1) & 7);
#pragma unroll
        for (uint32_t j0 = 0; j0 < (uint32_t)GC_LOCAL_SCATTER; j0 += 4) {
          if (j0 >= Wn) break;
          int32_t w[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t j = j0 + u;
            w[u] = j < Wn ? ldc(p.ci, e.beg + j) : -1;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (w[u] >= 0) {
              if (dist(p)) red_color<S>(p, (int64_t)((tent - 1) >> 3) * p.plane, w[u], bit);
              else red_plane<S>(pl, w[u], bit);
            }
        }
      }
      return state;
    }
#endif
    const uint32_t E = warp_incl_scan(Wn, lane);
    const uint32_t T = __shfl_sync(FULL, E, 31);
    __syncwarp();
    for (uint32_t f0 = 0; f0 < T; f0 += 32 * 4) {
      int32_t w[4];
      uint32_t wb[4];
      uint8_t* pl[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t f = f0 + u * 32 + lane;
        const int o = flat_owner(E, f);
        const int oc = o < 32 ? o : 31;
        const uint32_t Eo = __shfl_sync(FULL, E, oc), Wo = __shfl_sync(FULL, Wn, oc);
        const int64_t bo = __shfl_sync(FULL, e.beg, oc);
        const uint32_t to = __shfl_sync(FULL, tent, oc);
        wb[u] = 1u << ((to - 1) & 7);
        w[u] = f < T ? ldc(p.ci, bo + (f - (Eo - Wo))) : -1;
        pl[u] = (dist(p) && w[u] >= 0 ? fmp_of(p, w[u]) : p.fmp) + (int64_t)((to - 1) >> 3) * p.plane;
      }
      if (p.sfilter) {
        uint32_t sw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) sw[u] = w[u] >= 0 ? lds(st + w[u]) : SW<S>::COMMIT;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (!(sw[u] & SW<S>::COMMIT)) {
            red_plane<S>(pl[u], w[u], wb[u]);
            if (CW) wk.v[W_SCATTER_RED] += 1;
          }
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (w[u] >= 0) red_plane<S>(pl[u], w[u], wb[u]);
      }
    }
  }
  return state;
}

// Sparse bin 0 (degree <= t3): warps pop chunks of the worklist; one vertex per lane.
template <class S, int POL, bool PUSH, bool CW>
__device__ __forceinline__ void phase_b_coop(const Params& p, const WE* Wb, uint32_t cnt, uint32_t* q, Pusher& pu,
                                             bool mark, Work& wk, int* s_first, uint32_t rec_round) {
  S* st = (S*)p.st;
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = nblk(p) * WARPS;
  const uint32_t ch = max(1u, min(64u, cnt / (4u * nwarps)));
  for (uint32_t c0 = pop_chunk(q, ch, lane); c0 < cnt; c0 = pop_chunk(q, ch, lane)) {
    const uint32_t cend = min(c0 + ch, cnt);
    for (uint32_t bse = c0; bse < cend; bse += 32) {
      const uint32_t i = bse + lane;
      bool act = i < cend, clean = false;
      WE e;
      e.v = 0;
      e.k = 0;
      e.beg = 0;
      uint32_t tent = 0;
      int64_t end = -1;
      if (act) {
        e = ldw(Wb + i);
        if (mark) {
          if (lds(p.dirty + e.v)) sts(p.dirty + e.v, 0u);
          else clean = true;  // loses as it stands (N1)
        }
        act = !clean;
      }
      if (act) {
        tent = lds(st + e.v) & SW<S>::CMASK;
        if (e.k < 0 && POL != DEGREE) {
          end = RP(p, e.v + 1);
          e.k = row_split(p, e.v, e.beg, end);
        }
        if (CW) wk.v[W_B_EVAL] += 1;
      }
      int state = batch_b<S, POL, PUSH, CW>(p, lane, act, e, tent, end, wk, s_first, rec_round);
      if (clean) state = 1;
      pu.template push<0, CW>(state == 1, e, lane, wk.v[W_PUSH]);
    }
  }
}


// One vertex of degree > t3 by the whole CTA (bin 1).  Returns true when it loses.
template <class S, int POL, bool PUSH, bool CW>
__device__ __forceinline__ bool cta_vertex(const Params& p, WE& e, uint32_t tent, Work& wk, int* s_first,
                                           int32_t* s_k, uint32_t rec_round = 0, bool first_round = false) {
  S* st = (S*)p.st;
  const int64_t end = RP(p, e.v + 1);
  if (e.k < 0 && POL != DEGREE) {
    if (threadIdx.x == 0) *s_k = row_split(p, e.v, e.beg, end);
    __syncthreads();
    e.k = *s_k;
    __syncthreads();
  }
  const ScanRange<POL> sr = scan_range<POL>(e.beg, e.k, end);
  const bool lose = (POL != DEGREE && first_round) ? sr.hi > sr.lo  // round 1: see batch_b_wide
                                                  : conflict_cta<S, POL, CW>(p, e.v, tent, sr.lo, sr.hi, sr.down,
                                                                             end - e.beg, wk, s_first);
  if (!lose) {
    if (threadIdx.x == 0) {
      sts(st + e.v, tent | SW<S>::COMMIT);
      bcast_word<S>(p, e.v, tent | SW<S>::COMMIT);
      if (rec_round)
        (((rec_round & 1) ? p.wlw1 : p.wlw0))[atomicAdd(&p.info->wl_cnt[rec_round % 3], 1u)] = e.v;
    }
    if (PUSH && tent <= 8u * p.np) {
      scatter<S, BLOCK, CW>(p, tent, e.beg + threadIdx.x, end, wk);
      if (CW && threadIdx.x == 0) wk.v[W_SCATTER] += (unsigned long long)(end - e.beg);
    }
  }
  return lose;
}

template <class S, int POL, bool PUSH, bool CW>
__device__ __forceinline__ void phase_b(const Params& p, uint32_t r, const Bins& bins, const WE* W, WE* Wout,
                                        bool mark, Work& wk, bool rec = false) {
  const uint32_t rec_round = rec ? r : 0u;
  BSmem& sm = bsmem();
  S* st = (S*)p.st;
  const uint32_t cur = r % 3, nxt = (r + 1) % 3;
  uint32_t nb[NBIN];
#pragma unroll
  for (int b = 0; b < NBIN; ++b) nb[b] = head().cnt[cur][b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blk(p) == 0 && threadIdx.x == 0) {
    if (p.trace && r <= p.trace_cap) p.trace[r - 1] = nb[0] + nb[1];
    if (CW) {
      wk.v[W_B_VERT] += (unsigned long long)nb[0] + nb[1];
      wk.v[W_SB_ENT] += (unsigned long long)nb[0] + nb[1];
    }
  }
  uint32_t* cnt_next = &p.info->cnt[nxt][0];
  Pusher pu;
  pu.init(sm.pbuf[warp], Wout, cnt_next, bins);

  // bin 1 first (one CTA per vertex, high degrees: the longest items start early), then the
  // dynamic bin-0 queue fills the gaps.  Tail rounds (no more pending vertices than CTAs: the
  // last, high-degree vertices with long scans and scatters) give every vertex a CTA.
  const bool tail = nb[0] + nb[1] <= nblk(p);
  auto cta_loop = [&](const WE* Wb, uint32_t cnt, uint32_t* outc, WE* Ob, uint32_t first) {
    for (uint32_t i = (blk(p) + first) % nblk(p); i < cnt; i += nblk(p)) {
      WE e = ldw(Wb + i);
      if (threadIdx.x == 0) {  // one read of the state word and the dirty mark, broadcast
        uint32_t x = lds(st + e.v) & SW<S>::CMASK;
        if (mark) {
          if (lds(p.dirty + e.v)) sts(p.dirty + e.v, 0u);
          else x |= 0x40000000u;  // clean (N1)
        }
        sm.k = (int32_t)x;
      }
      __syncthreads();
      const uint32_t tx = (uint32_t)sm.k;
      __syncthreads();
      if (CW && threadIdx.x == 0 && !(tx & 0x40000000u)) wk.v[W_B_EVAL] += 1;
      if (((tx & 0x40000000u) || cta_vertex<S, POL, PUSH, CW>(p, e, tx, wk, &sm.first, &sm.k, rec_round)) &&
          threadIdx.x == 0) {
        stw(Ob + atomicAdd(outc, 1u), e);
        if (CW) wk.v[W_PUSH] += 1;
      }
      __syncthreads();
    }
  };
  cta_loop(W + bins.off[1], nb[1], &cnt_next[1], Wout + bins.off[1], 0);
  if (tail) {
    // a split still unknown (-1, first visit) is found by cta_vertex
    cta_loop(W + bins.off[0], nb[0], &cnt_next[0], Wout + bins.off[0], nb[1]);
    return;
  }
  phase_b_coop<S, POL, PUSH, CW>(p, W + bins.off[0], nb[0], &p.info->qctr[cur][0][0], pu, mark, wk, sm.cwfirst[warp],
                                 rec_round);
  pu.template flush<CW>(lane, wk.v[W_PUSH]);
}

// Dense batch: WB consecutive vertices per warp, VPL per lane (slots lane*VPL .. +VPL-1), so
// that every dependent level of the batch (state words / row offsets / splits, then col_idx,
// then the neighbours' state words, then the scatter) has VPL x more independent loads in flight
// than one vertex per lane.  The per-slot data live in a shared-memory table; the flattened item
// loop finds an item's slot by binary search over the prefix sums.  Same passes as batch_b.
__device__ __forceinline__ int seg_owner(const uint32_t* E, uint32_t f) {
  int o = 0;
#pragma unroll
  for (int b = WB / 2; b; b >>= 1)
    if (E[o + b - 1] <= f) o += b;
  return o;
}
// Writes the slots' E/W for the given per-lane W values; returns the total.
__device__ __forceinline__ uint32_t seg_prefix(WideSeg& sg, const uint32_t (&Wh)[VPL], int lane) {
  uint32_t tot = 0;
#pragma unroll
  for (int h = 0; h < VPL; ++h) tot += Wh[h];
  const uint32_t incl = warp_incl_scan(tot, lane);
  uint32_t run = incl - tot;
#pragma unroll
  for (int h = 0; h < VPL; ++h) {
    run += Wh[h];
    sg.E[lane * VPL + h] = run;
  }
  __syncwarp();
  return __shfl_sync(FULL, incl, 31);
}

template <int POL>
__device__ __forceinline__ int64_t seg_beg(const WideSeg& sg, int o) {
  return POL == HIGHER_ID ? sg.sbase[o] - sg.k[o] + 1 : (POL == LOWER_ID ? sg.sbase[o] - sg.k[o] : sg.sbase[o]);
}
template <int POL>
__device__ __forceinline__ uint32_t seg_len(const WideSeg& sg, int o) {
  return POL == HIGHER_ID ? (uint32_t)sg.k[o] : (POL == LOWER_ID ? sg.deg[o] - (uint32_t)sg.k[o] : sg.deg[o]);
}

template <class S, int POL, bool PUSH, bool CW>
__device__ __forceinline__ void batch_b_wide(const Params& p, int lane, uint32_t base, uint32_t cend, WideSeg& sg,
                                             bool push_out, bool mark, Pusher& pu, uint32_t& lost_cnt, Work& wk,
                                             uint32_t rec_round, bool first_round) {
  S* st = (S*)p.st;
  constexpr uint32_t CM = SW<S>::CMASK;
  constexpr int DIR = POL == HIGHER_ID ? -1 : 1;
  const uint32_t v0 = base + lane * VPL;
  const uint32_t vlo = (uint32_t)p.v_base;  // ids below it (first batch of a rank): not ours
  // level 1: state words, row offsets, splits of the lane's VPL vertices (independent loads)
  uint32_t states = 0;  // 8 bits per slot: 0 inactive, 1 lose, 2 win, 3 undecided
  {
    uint32_t sw[VPL];
    int64_t rpv[VPL + 1];
    int32_t kv[VPL];
#pragma unroll
    for (int h = 0; h < VPL; ++h) sw[h] = v0 + h >= vlo && v0 + h < cend ? lds(st + v0 + h) : SW<S>::COMMIT;
#pragma unroll
    for (int h = 0; h <= VPL; ++h) rpv[h] = v0 + h >= vlo && v0 + h <= cend ? RP(p, (int64_t)v0 + h) : 0;
#pragma unroll
    for (int h = 0; h < VPL; ++h)
      kv[h] = (POL != DEGREE && v0 + h >= vlo && v0 + h < cend) ? ldks(p.ksplit + v0 + h) : 0;
    uint32_t dv[VPL];
#pragma unroll
    for (int h = 0; h < VPL; ++h) dv[h] = mark && v0 + h >= vlo && v0 + h < cend ? lds(p.dirty + v0 + h) : 1u;
#pragma unroll
    for (int h = 0; h < VPL; ++h) {
      const int sl = lane * VPL + h;
      const int64_t beg = rpv[h], deg = rpv[h + 1] - rpv[h];
      const bool pend = v0 + h >= vlo && v0 + h < cend && !(sw[h] & SW<S>::COMMIT) && deg <= (int64_t)p.t3;
      const bool act = pend && dv[h];
      if (mark && pend) {
        if (dv[h]) sts(p.dirty + v0 + h, 0u);
        else states |= 1u << (8 * h);  // clean: loses as it stands (N1)
      }
      if (CW && act) wk.v[W_B_EVAL] += 1, wk.v[W_DB_EVAL] += 1;
      sg.sbase[sl] = POL == HIGHER_ID ? beg + kv[h] - 1 : (POL == LOWER_ID ? beg + kv[h] : beg);
      sg.k[sl] = kv[h];
      sg.deg[sl] = (uint32_t)deg;
      sg.tent[sl] = sw[h] & CM;
      sg.pos[sl] = 0;
      if (act) {
        const uint32_t len = POL == HIGHER_ID ? (uint32_t)kv[h] : (POL == LOWER_ID ? (uint32_t)(deg - kv[h]) : (uint32_t)deg);
        states |= (len ? 3u : 2u) << (8 * h);
      }
    }
  }
  __syncwarp();
  // round 1: every vertex is pending with tentative colour 1, so (id policies) a vertex loses
  // iff its scan range is not empty — no gathers (same result as the scan: its first position
  // conflicts)
  if (POL != DEGREE && first_round) {
#pragma unroll
    for (int h = 0; h < VPL; ++h)
      if (((states >> (8 * h)) & 0xffu) == 3u) {
        states ^= 2u << (8 * h);  // 3 -> 1
        if (CW) { wk.v[W_B_EDGE] += 1; wk.v[W_B_GATHER] += 1; }
      }
  }
  // pass 1, lane-local: the first PROBE positions of the lane's own VPL scan ranges (no owner
  // search; VPL x PROBE independent loads per lane).  Later passes are flattened.
  {
    int32_t w[VPL][PROBE];
#pragma unroll
    for (int h = 0; h < VPL; ++h) {
      const int sl = lane * VPL + h;
      const bool und = ((states >> (8 * h)) & 0xffu) == 3u;
      const uint32_t len = und ? seg_len<POL>(sg, sl) : 0u;
      const int64_t sb = sg.sbase[sl];
#pragma unroll
      for (int u = 0; u < PROBE; ++u) w[h][u] = (uint32_t)u < len ? ldc(p.ci, sb + (int64_t)DIR * u) : -1;
    }
#pragma unroll
    for (int h = 0; h < VPL; ++h) {
      const int sl = lane * VPL + h;
      if (((states >> (8 * h)) & 0xffu) != 3u) continue;
      const uint32_t t = sg.tent[sl];
      int first = -1;
#pragma unroll
      for (int u = PROBE - 1; u >= 0; --u) {
        const uint32_t sv = w[h][u] >= 0 ? ldnb(st + w[h][u]) : 0u;
        if (w[h][u] >= 0 && (sv & CM) == t && recolors<POL>(p, (int32_t)(base + sl), w[h][u], (int64_t)sg.deg[sl]))
          first = u;
      }
      const uint32_t len = seg_len<POL>(sg, sl);
      if (first >= 0) {
        states ^= 2u << (8 * h);  // 3 -> 1
        if (CW) { wk.v[W_B_EDGE] += first + 1; wk.v[W_B_GATHER] += first + 1; }
      } else {
        const uint32_t np = len < (uint32_t)PROBE ? len : (uint32_t)PROBE;
        sg.pos[sl] = np;
        if (np == len) {
          states ^= 1u << (8 * h);  // 3 -> 2
          if (CW) { wk.v[W_B_EDGE] += np; wk.v[W_B_GATHER] += np; }
        }
      }
    }
    __syncwarp();
  }
  // conflict-scan passes (levels 2-3: col_idx of the scan positions, then their state words)
  uint32_t cap = 3 * PROBE;
  for (;;) {
    const bool any = ((states | states >> 1) & 0x01010101u & (states & (states >> 1))) != 0;  // some slot == 3
    if (!__any_sync(FULL, any)) break;
    if (lane < VPL) sg.lost[lane] = 0;
    uint32_t Wh[VPL];
#pragma unroll
    for (int h = 0; h < VPL; ++h) {
      const int sl = lane * VPL + h;
      Wh[h] = ((states >> (8 * h)) & 0xffu) == 3u ? min(seg_len<POL>(sg, sl) - sg.pos[sl], cap) : 0u;
      if (CW) sg.first[sl] = 0x7fffffff;
    }
    const uint32_t T = seg_prefix(sg, Wh, lane);
    for (uint32_t f0 = 0; f0 < T; f0 += 32 * FLAT_U) {
      int32_t w[FLAT_U];
      int own[FLAT_U];
      uint32_t jj[FLAT_U];
#pragma unroll
      for (int u = 0; u < FLAT_U; ++u) {
        const uint32_t f = f0 + u * 32 + lane;
        own[u] = -1;
        w[u] = 0;
        jj[u] = 0;
        if (f < T) {
          const int o = seg_owner(sg.E, f);
          own[u] = o;
          jj[u] = f - (o ? sg.E[o - 1] : 0u) + sg.pos[o];
          w[u] = ldc(p.ci, sg.sbase[o] + (int64_t)DIR * jj[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < FLAT_U; ++u) {
        if (own[u] >= 0) {
          const int o = own[u];
          const uint32_t sv = ldnb(st + w[u]);
          const bool hit = (sv & CM) == sg.tent[o] && recolors<POL>(p, (int32_t)(base + o), w[u], (int64_t)sg.deg[o]);
          if (hit) {
            atomicOr(&sg.lost[o >> 5], 1u << (o & 31));
            if (CW) atomicMin(&sg.first[o], (int)jj[u]);
          }
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < VPL; ++h) {
      const int sl = lane * VPL + h;
      if (((states >> (8 * h)) & 0xffu) != 3u) continue;
      if (sg.lost[sl >> 5] >> (sl & 31) & 1u) {
        states ^= 2u << (8 * h);  // 3 -> 1
        if (CW) { const uint32_t ex = (uint32_t)sg.first[sl] + 1; wk.v[W_B_EDGE] += ex; wk.v[W_B_GATHER] += ex; }
      } else {
        const uint32_t np = sg.pos[sl] + Wh[h];
        sg.pos[sl] = np;
        if (np == seg_len<POL>(sg, sl)) {
          states ^= 1u << (8 * h);  // 3 -> 2
          if (CW) { wk.v[W_B_EDGE] += np; wk.v[W_B_GATHER] += np; }
        }
      }
    }
    __syncwarp();
    cap = cap < 1024 ? cap * GC_CAPMUL : cap;  // 12, 48, 192, 768, ...
  }
  // commit: winners set the top bit of their own state word
#pragma unroll
  for (int h = 0; h < VPL; ++h)
    if (((states >> (8 * h)) & 0xffu) == 2u) {
      sts(st + v0 + h, sg.tent[lane * VPL + h] | SW<S>::COMMIT);
      bcast_word<S>(p, (int32_t)(v0 + h), sg.tent[lane * VPL + h] | SW<S>::COMMIT);
    }
  if (rec_round) {
#pragma unroll
    for (int h = 0; h < VPL; ++h) rec_winners(p, rec_round, ((states >> (8 * h)) & 0xffu) == 2u, (int32_t)(v0 + h), lane);
  }
  // level 4: scatter of the winners' rows into the forbidden masks (flattened)
  if (PUSH) {
    uint32_t Wh[VPL];
#pragma unroll
    for (int h = 0; h < VPL; ++h) {
      const int sl = lane * VPL + h;
      Wh[h] = ((states >> (8 * h)) & 0xffu) == 2u && sg.tent[sl] <= 8u * p.np ? sg.deg[sl] : 0u;
      if (CW) { wk.v[W_SCATTER] += Wh[h]; if (!p.sfilter) wk.v[W_SCATTER_RED] += Wh[h]; }
    }
#if GC_LOCAL_SCATTER
    // short rows only: every lane scatters its own slots' rows (at most 4 entries each)
    uint32_t wmax = 0;
#pragma unroll
    for (int h = 0; h < VPL; ++h) wmax = Wh[h] > wmax ? Wh[h] : wmax;
    if (!p.sfilter && __reduce_max_sync(FULL, wmax) <= 4u) {
      int32_t w[VPL][4];
#pragma unroll
      for (int h = 0; h < VPL; ++h) {
        const int sl = lane * VPL + h;
#pragma unroll
        for (int u = 0; u < 4; ++u) w[h][u] = (uint32_t)u < Wh[h] ? ldc(p.ci, seg_beg<POL>(sg, sl) + u) : -1;
      }
#pragma unroll
      for (int h = 0; h < VPL; ++h) {
        const uint32_t t = sg.tent[lane * VPL + h];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (w[h][u] >= 0) red_color<S>(p, (int64_t)((t - 1) >> 3) * p.plane, w[h][u], 1u << ((t - 1) & 7));
      }
    } else
#endif
    {
    const uint32_t T = seg_prefix(sg, Wh, lane);
    for (uint32_t f0 = 0; f0 < T; f0 += 32 * 4) {
      int32_t w[4];
      int own[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t f = f0 + u * 32 + lane;
        own[u] = 0;
        w[u] = -1;
        if (f < T) {
          const int o = seg_owner(sg.E, f);
          own[u] = o;
          const uint32_t x = f - (o ? sg.E[o - 1] : 0u);
          w[u] = ldc(p.ci, seg_beg<POL>(sg, o) + x);
        }
      }
      uint32_t skip = 0;
      if (p.sfilter) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (w[u] >= 0 && (lds(st + w[u]) & SW<S>::COMMIT)) skip |= 1u << u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (w[u] < 0 || (skip >> u & 1u)) continue;
        const uint32_t t = sg.tent[own[u]];
        red_color<S>(p, (int64_t)((t - 1) >> 3) * p.plane, w[u], 1u << ((t - 1) & 7));
        if (CW && p.sfilter) wk.v[W_SCATTER_RED] += 1;
      }
    }
    }
    __syncwarp();
  }
  // losers: counted, or pushed into W_out (split known) when round r+1 runs sparse
  if (push_out) {
#pragma unroll
    for (int h = 0; h < VPL; ++h) {
      const int sl = lane * VPL + h;
      WE e;
      e.v = (int32_t)(v0 + h);
      e.k = sg.k[sl];
      e.beg = seg_beg<POL>(sg, sl);
      pu.template push<0, CW>(((states >> (8 * h)) & 0xffu) == 1u, e, lane, wk.v[W_PUSH]);
    }
  } else {
    uint32_t c = 0;
#pragma unroll
    for (int h = 0; h < VPL; ++h) c += ((states >> (8 * h)) & 0xffu) == 1u;
    lost_cnt += __reduce_add_sync(FULL, c);
  }
  __syncwarp();
}

// ---- list rounds (N1 with explicit lists; bounded-degree graphs, 8-bit state words)
// Once few vertices commit per round, the dense sweeps cost more than the work: Phase A of
// round r recomputes the tentative colour only of the neighbours of round r-1's winners (the
// only masks that changed), and Phase B of round r examines only the vertices listed dirty by
// that Phase A (the N1 rule above); every other pending vertex loses as it stands, so
// |W_{r+1}| = |W_r| - (winners of round r).  Dirty marks are set with an atomic OR on the word
// holding the mark byte, and the lane that set a mark lists the vertex (each listed once).
__device__ __forceinline__ void mark_append(const Params& p, uint32_t r, bool act, int32_t v, int lane) {
  bool nw = false;
  if (act) {
    const uint32_t sh = 8u * (uint32_t)(v & 3);
    const uint32_t old = atomicOr((uint32_t*)(p.dirty + (v & ~3)), 1u << sh);
    nw = ((old >> sh) & 0xffu) == 0u;
  }
  const unsigned m = __ballot_sync(FULL, nw);
  if (!m) return;
  const int leader = __ffs(m) - 1;
  uint32_t pos = 0;
  if (lane == leader) pos = atomicAdd(&p.info->dl_cnt[r % 3], (uint32_t)__popc(m));
  pos = __shfl_sync(FULL, pos, leader);
  if (nw) p.dl[pos + __popc(m & lanemask_lt())] = v;
}

// Marks (and lists) the cnt changed vertices of clist and their successors.
template <int POL, bool CW>
__device__ __forceinline__ void mark_flush(const Params& p, uint32_t r, const int32_t* clist, uint32_t cnt, int lane,
                                           Work& wk) {
  for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
    const bool act = i0 + lane < cnt;
    int32_t v = 0;
    int64_t lo = 0, hi = 0;
    if (act) {
      v = clist[i0 + lane];
      const int64_t beg = ldr(p.rp, v), end = ldr(p.rp, v + 1);
      const int32_t k = POL != DEGREE ? ldks(p.ksplit + v) : 0;
      lo = POL == HIGHER_ID ? beg + k : beg;
      hi = POL == LOWER_ID ? beg + k : end;
      if (CW) wk.v[W_MARK] += (unsigned long long)(hi - lo + 1);
    }
    mark_append(p, r, act, v, lane);
    const uint32_t Wn = (uint32_t)(hi - lo);
    const uint32_t E = warp_incl_scan(Wn, lane);
    const uint32_t T = __shfl_sync(FULL, E, 31);
    for (uint32_t f0 = 0; f0 < T; f0 += 32 * 2) {
      int32_t w[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t f = f0 + u * 32 + lane;
        const int o = flat_owner(E, f);
        const int oc = o < 32 ? o : 31;
        const uint32_t Eo = __shfl_sync(FULL, E, oc), Wo = __shfl_sync(FULL, Wn, oc);
        const int64_t lo_o = __shfl_sync(FULL, lo, oc);
        w[u] = f < T ? ldc(p.ci, lo_o + (f - (Eo - Wo))) : -1;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) mark_append(p, r, w[u] >= 0, w[u], lane);
    }
  }
}

template <class S, int POL, bool CW>
__device__ __forceinline__ void phase_a_list(const Params& p, uint32_t r, Work& wk) {
  S* st = (S*)p.st;
  reset_next(p, r);
  zero_plane(p, r);
  const int lane = threadIdx.x & 31;
  int32_t* clist = bsmem().clist[threadIdx.x >> 5];
  const uint32_t nwin = head().wl_cnt[(r - 1) % 3];
  const int32_t* WL = ((r - 1) & 1) ? p.wlw1 : p.wlw0;
  uint32_t* q = &p.info->qctr[r % 3][1][0];
  const uint32_t nwarps = nblk(p) * WARPS;
  const uint32_t ch = max(1u, min(32u, nwin / (4u * nwarps)));
  uint32_t nchg = 0;
  for (uint32_t c0 = pop_chunk(q, ch, lane); c0 < nwin; c0 = pop_chunk(q, ch, lane)) {
    const uint32_t cend = min(c0 + ch, nwin);
    for (uint32_t bse = c0; bse < cend; bse += 32) {
      int64_t lo = 0, hi = 0;
      if (bse + lane < cend) {
        const int32_t w = ldks(WL + bse + lane);
        lo = ldr(p.rp, w);
        hi = ldr(p.rp, w + 1);
      }
      const uint32_t Wn = (uint32_t)(hi - lo);
      const uint32_t E = warp_incl_scan(Wn, lane);
      const uint32_t T = __shfl_sync(FULL, E, 31);
      for (uint32_t f0 = 0; f0 < T; f0 += 32 * 4) {
        int32_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t f = f0 + u * 32 + lane;
          const int o = flat_owner(E, f);
          const int oc = o < 32 ? o : 31;
          const uint32_t Eo = __shfl_sync(FULL, E, oc), Wo = __shfl_sync(FULL, Wn, oc);
          const int64_t lo_o = __shfl_sync(FULL, lo, oc);
          v[u] = f < T ? ldc(p.ci, lo_o + (f - (Eo - Wo))) : -1;
        }
        uint32_t sv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) sv[u] = v[u] >= 0 ? lds(st + v[u]) : SW<S>::COMMIT;
        uint32_t chm = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (sv[u] & SW<S>::COMMIT) continue;
          const uint32_t t = plane_firstfit(p, v[u], r);  // >= 1: 8-bit words, colours <= 8 * np
          if (t != (sv[u] & SW<S>::CMASK)) {
            store_tent<S>(p, st, v[u], t);
            chm |= 1u << u;
          }
        }
        // list this step's changed vertices (<= 128) and mark them with their successors
        const uint32_t c = __popc(chm);
        nchg += c;
        const uint32_t ci = warp_incl_scan(c, lane);
        const uint32_t tot = __shfl_sync(FULL, ci, 31);
        if (tot) {
          uint32_t at = ci - c;
          for (uint32_t m = chm; m; m &= m - 1) clist[at++] = v[__ffs(m) - 1];
          __syncwarp();
          mark_flush<POL, CW>(p, r, clist, tot, lane, wk);
          __syncwarp();
        }
      }
    }
  }
  flush_chg(p, r, nchg, wk, CW);
}

template <class S, int POL, bool PUSH, bool CW>
__device__ __forceinline__ void phase_b_list(const Params& p, uint32_t r, uint32_t tot, Work& wk) {
  S* st = (S*)p.st;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blk(p) == 0 && threadIdx.x == 0) {
    if (p.trace && r <= p.trace_cap) p.trace[r - 1] = tot;
    if (CW) wk.v[W_B_VERT] += tot;
  }
  const uint32_t nd = head().dl_cnt[r % 3];
  uint32_t* q = &p.info->qctr[r % 3][0][0];
  const uint32_t nwarps = nblk(p) * WARPS;
  const uint32_t ch = max(1u, min(64u, nd / (4u * nwarps)));
  int* s_first = bsmem().cwfirst[warp];
  for (uint32_t c0 = pop_chunk(q, ch, lane); c0 < nd; c0 = pop_chunk(q, ch, lane)) {
    const uint32_t cend = min(c0 + ch, nd);
    for (uint32_t bse = c0; bse < cend; bse += 32) {
      bool act = bse + lane < cend;
      WE e;
      e.v = 0;
      e.k = 0;
      e.beg = 0;
      uint32_t tent = 0;
      if (act) {
        e.v = ldks(p.dl + bse + lane);
        sts(p.dirty + e.v, 0u);
        const uint32_t sv = lds(st + e.v);
        act = !(sv & SW<S>::COMMIT);
        tent = sv & SW<S>::CMASK;
        e.beg = ldr(p.rp, e.v);
        if (POL != DEGREE) e.k = ldks(p.ksplit + e.v);
        if (CW && act) wk.v[W_B_EVAL] += 1;
      }
      batch_b<S, POL, PUSH, CW>(p, lane, act, e, tent, -1, wk, s_first, r);
    }
  }
}

// Dense Phase B: W_r = all uncommitted vertices.  The heavy vertices (degree > t3, a static
// list built by the ingest) are taken one CTA each; the others by warps popping chunks of
// consecutive ids (coalesced state words, row offsets and splits; consecutive rows are
// contiguous in col_idx).  Losers are only counted — or, when push_out (|W_r| small enough
// that round r+1 runs sparse), pushed into W_out with the split already known.
template <class S, int POL, bool PUSH, bool CW>
__device__ __forceinline__ void phase_b_dense(const Params& p, uint32_t r, const Bins& bins, WE* Wout, bool push_out,
                                              bool mark, Work& wk, bool rec = false) {
  const uint32_t rec_round = rec ? r : 0u;
  BSmem& sm = bsmem();
  S* st = (S*)p.st;
  const uint32_t cur = r % 3, nxt = (r + 1) % 3;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blk(p) == 0 && threadIdx.x == 0) {
    const uint32_t tot = head().cnt[cur][0] + head().cnt[cur][1];
    if (p.trace && r <= p.trace_cap) p.trace[r - 1] = tot;
    if (CW) {
      wk.v[W_B_VERT] += tot;
      wk.v[W_DB_SWEEP] += (unsigned long long)p.n;
    }
  }
  uint32_t* cnt_next = &p.info->cnt[nxt][0];
  Pusher pu;
  pu.init(sm.pbuf[warp], Wout, cnt_next, bins);
  {
    const uint32_t nh = bins.size[1];
    WE* Ob = Wout + bins.off[1];
    for (uint32_t i = blk(p); i < nh; i += nblk(p)) {
      WE e = ldw(p.heavy + i);
      if (threadIdx.x == 0) {  // one read of the state word and the dirty mark, broadcast
        uint32_t x = lds(st + e.v);
        if (mark && !(x & SW<S>::COMMIT)) {
          if (lds(p.dirty + e.v)) sts(p.dirty + e.v, 0u);
          else x |= 0x40000000u;  // clean (N1)
        }
        sm.k = (int32_t)x;
      }
      __syncthreads();
      const uint32_t s = (uint32_t)sm.k;
      __syncthreads();
      if (s & SW<S>::COMMIT) continue;  // uniform over the CTA
      if (CW && threadIdx.x == 0 && !(s & 0x40000000u)) wk.v[W_B_EVAL] += 1, wk.v[W_DB_EVAL] += 1;
      if (((s & 0x40000000u) ||
           cta_vertex<S, POL, PUSH, CW>(p, e, s & SW<S>::CMASK, wk, &sm.first, &sm.k, rec_round, r == 1)) &&
          threadIdx.x == 0) {
        if (push_out) {
          stw(Ob + atomicAdd(&cnt_next[1], 1u), e);
          if (CW) wk.v[W_PUSH] += 1;
        } else {
          atomicAdd(&cnt_next[1], 1u);
        }
      }
      __syncthreads();
    }
  }
  const uint32_t nwarps = nblk(p) * WARPS;
  // chunk offsets c count from lo16 (this rank's first id rounded down to 16): vertex lo16 + c
  const uint32_t vlo = (uint32_t)p.v_base, vend = vlo + (uint32_t)p.n, lo16 = vlo & ~15u;
  const uint32_t nv = vend - lo16;
  uint32_t* q = &p.info->qctr[cur][0][0];
  uint32_t lost_cnt = 0;
  if ((mark || p.compact) && !push_out) {
    // dirty-set round: sweep the marks and state words 512 vertices per warp step (16-B
    // vectors), list the dirty pending ones in shared memory and examine only those, 32 per
    // batch (one per lane); clean pending vertices lose as they stand
    int32_t* clist = sm.clist[warp];
    int* s_first = sm.cwfirst[warp];
    constexpr uint32_t CHD = 512;
    // chunks dealt out statically, interleaved over the warps: a dynamic queue head costs one
    // same-address atomic per chunk and warp (mesh 8192^2: ~130 K per round, serialised at one
    // L2 slice), and the interleaving spreads the dirty band of the colouring front evenly
    // (with few chunks per warp the dynamic queue balances better: up to GC_DIRTY_DYN chunks per warp)
#ifndef GC_DIRTY_DYN
#define GC_DIRTY_DYN 4
#endif
    const uint32_t gw = blk(p) * WARPS + warp, nch = (nv + CHD - 1) / CHD;
    const bool dyn = nch <= GC_DIRTY_DYN * nwarps;
    for (uint32_t ck = dyn ? pop_chunk(q, 1, lane) : gw; ck < nch; ck = dyn ? pop_chunk(q, 1, lane) : ck + nwarps) {
      const uint32_t c0 = ck * CHD;
      const uint32_t v0 = lo16 + c0 + 16u * lane;
      uint32_t cand = 0, pend = 0;
      if (v0 < vend) {
        const uint4 dq = mark ? ldv(p.dirty + v0) : make_uint4(0, 0, 0, 0);
        const uint32_t dw[4] = {dq.x, dq.y, dq.z, dq.w};
        uint32_t sw[4 * sizeof(S)];
#pragma unroll
        for (int i = 0; i < (int)sizeof(S); ++i) {
          const uint4 x = ldv(st + v0 + i * (16 / sizeof(S)));
          sw[4 * i] = x.x;
          sw[4 * i + 1] = x.y;
          sw[4 * i + 2] = x.z;
          sw[4 * i + 3] = x.w;
        }
#pragma unroll
        for (int h = 0; h < 16; ++h) {
          constexpr int PER = 4 / (int)sizeof(S);
          const uint32_t sv = sw[h / PER] >> ((h % PER) * 8 * (int)sizeof(S));
          const bool pd = v0 + h >= vlo && v0 + h < vend && !(sv & SW<S>::COMMIT);
          pend |= (uint32_t)pd << h;
          cand |= (uint32_t)(pd && (!mark || ((dw[h >> 2] >> ((h & 3) * 8)) & 0xffu))) << h;
        }
      }
      const uint32_t c = __popc(cand);
      const uint32_t ci = warp_incl_scan(c, lane);
      const uint32_t tot = __shfl_sync(FULL, ci, 31);
      uint32_t at = ci - c;
      for (uint32_t m = cand; m; m &= m - 1) clist[at++] = (int32_t)(v0 + __ffs(m) - 1);
      __syncwarp();
      uint32_t won = 0;
      for (uint32_t i0 = 0; i0 < tot; i0 += 32) {
        bool act = i0 + lane < tot;
        WE e;
        e.v = 0;
        e.k = 0;
        e.beg = 0;
        uint32_t tent = 0;
        int64_t end = -1;
        if (act) {
          e.v = clist[i0 + lane];
          tent = lds(st + e.v) & SW<S>::CMASK;
          e.beg = RP(p, e.v);
          end = RP(p, e.v + 1);
          if (POL != DEGREE) e.k = ldks(p.ksplit + e.v);
          act = end - e.beg <= (int64_t)p.t3;  // heavy vertices (and their marks): the CTA loop
          if (act && mark) sts(p.dirty + e.v, 0u);
          if (CW && act) wk.v[W_B_EVAL] += 1, wk.v[W_DB_EVAL] += 1;
        }
        const int state = batch_b<S, POL, PUSH, CW>(p, lane, act, e, tent, end, wk, s_first, rec_round);
        won += __popc(__ballot_sync(FULL, state == 2));
      }
      __syncwarp();
      // heavy pending vertices are counted by the CTA loop
      uint32_t heavy_pend = 0;
      if (bins.size[1]) {
        for (uint32_t m = pend; m; m &= m - 1) {
          const int32_t v = (int32_t)(v0 + __ffs(m) - 1);
          if (RP(p, v + 1) - RP(p, v) > (int64_t)p.t3) ++heavy_pend;
        }
      }
      const uint32_t np = __reduce_add_sync(FULL, (uint32_t)__popc(pend) - heavy_pend);
      lost_cnt += np - won;
    }
    cta_add(&cnt_next[0], lane == 0 ? lost_cnt : 0u);
    return;
  }
  const uint32_t ch = max((uint32_t)WB, min(2048u, (nv / (p.dch * nwarps)) / WB * WB));
  for (uint32_t c0 = pop_chunk(q, ch, lane); c0 < nv; c0 = pop_chunk(q, ch, lane)) {
    const uint32_t cend = lo16 + min(c0 + ch, nv);
    for (uint32_t bse = lo16 + c0; bse < cend; bse += WB)
      batch_b_wide<S, POL, PUSH, CW>(p, lane, bse, cend, sm.seg[warp], push_out, mark, pu, lost_cnt, wk, rec_round,
                                     r == 1);
  }
  if (push_out) pu.template flush<CW>(lane, wk.v[W_PUSH]);
  else cta_add(&cnt_next[0], lane == 0 ? lost_cnt : 0u);
}

// |W_{r+1}| summed over bins (read after the barrier that ends Phase B of round r).
__device__ __forceinline__ uint32_t next_total(const Params& p, uint32_t r) {
  const uint32_t nxt = (r + 1) % 3;
  uint32_t t = 0;
#pragma unroll
  for (int b = 0; b < NBIN; ++b) t += head().cnt[nxt][b];
  return t;
}

// ---------------------------------------------------------------- a5: finalize
template <class S>
__device__ __forceinline__ void epilogue(const Params& p) {
  const S* st = (const S*)p.st;
  uint32_t mx = 0;
  const int64_t stride = (int64_t)nblk(p) * BLOCK;
  for (int64_t v = (int64_t)blk(p) * BLOCK + threadIdx.x; v < p.n; v += stride) {
    const uint32_t c = lds(st + p.v_base + v) & SW<S>::CMASK;
    p.colors_out[v] = c;
    mx = c > mx ? c : mx;
  }
  mx = __reduce_max_sync(FULL, mx);
  if ((threadIdx.x & 31) == 0 && mx) {
    if (dist(p)) for (int q = 0; q < p.nranks; ++q) atomicMax(&p.peer[q].info->num_colors, mx);
    else atomicMax(&p.info->num_colors, mx);
  }
}

template <bool CW>
__device__ __forceinline__ void flush_work(const Params& p, Work& wk) {
  if constexpr (CW) {
#pragma unroll
    for (int k = 0; k < W_N; ++k) {
      unsigned long long x = wk.v[k];
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
      if ((threadIdx.x & 31) == 0 && x) atomicAdd(&p.info->work[k], x);
    }
  }
}

// Diagnostics (p.phase_ns): the latest time any CTA of the grid finished the phase's work,
// before entering the barrier (slot 4r-3: Phase A, 4r-1: Phase B; 4r-2 / 4r: the barrier done).
__device__ __forceinline__ void work_stamp(const Params& p, uint32_t slot, uint32_t r) {
  if (!p.phase_ns || r > p.trace_cap) return;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&p.phase_ns[slot], globaltimer());
}

// ---------------------------------------------------------------- a4: persistent driver
// One cooperative launch runs ingest, every round and finalize.  Per round: Phase A,
// barrier, Phase B (+push), barrier; every CTA reads |W_{r+1}| and leaves together.
#ifndef GC_MINB
#define GC_MINB 4
#endif
template <class S, int POL, bool PUSH, bool CW>
__device__ __forceinline__ void sgr_body(const Params& p) {
  Work wk;
  wk.zero();
  if (threadIdx.x == 0) barriers_passed() = 0;
  __syncthreads();
  const bool dense0 = PUSH && p.dense_div != 0;
  uint32_t r = 1;
  bool dense = dense0;
  Bins bins;
  if (p.resume_r) {
    // continuation of an 8-bit run stopped by ST_NEED16 after Phase A of round resume_r: the host
    // widened the state words in place; every other array (planes, marks, worklists, counters in
    // DevInfo) is as that run left it.  Phase A of the round is redone with the wider words.
    if (threadIdx.x == 0) take_head(p);
    __syncthreads();
    bins.load(p);
    r = p.resume_r;
    dense = p.resume_dense != 0;
    goto rounds;
  }
  if (kDist && threadIdx.x == 0) {
    atomicAdd(&p.info->diag[3], 1u);  // CTAs started (watchdog report)
    p.info->stage[blk(p) & 1023] = 1;
  }
  if (dist(p)) {  // multi-GPU: replica fill + ghost masks (one cross-rank barrier)
    fill_replica<S>(p);
    if (threadIdx.x == 0) p.info->stage[blk(p) & 1023] = 2;
    prologue_dist(p);
    if (threadIdx.x == 0) p.info->stage[blk(p) & 1023] = 3;
    if (!grid_sync(p)) return;
  }
  prologue_count<S, POL, PUSH>(p, dense0);
  if (!grid_sync(p)) return;
  bins.load(p);
  if (!dense0) prologue_scatter(p, bins);
  else if (blk(p) == 0 && threadIdx.x < NBIN) p.info->cnt[1][threadIdx.x] = bins.size[threadIdx.x];
  if (!grid_sync(p)) return;
rounds:
  const bool stamp = p.phase_ns && blk(p) == 0 && threadIdx.x == 0;
  if (stamp && !p.resume_r) p.phase_ns[0] = globaltimer();

  // The worklist pointers are re-read from DevInfo every round instead of being swapped in
  // registers: with loop-carried pointer swaps, ptxas (12.9) was observed to reuse the
  // uniform register holding one of them inside the grid barrier (truncated addresses).
  // Rounds run dense (W_r implicit, id-order sweeps) while |W_r| * dense_div > n, then
  // sparse (worklists); the round whose |W_r| first falls below pushes its losers.
  bool list = false;
  uint32_t tot_list = 0;
  // list rounds: 8-bit words (colours from the planes), bounded degree, dirty marks available
  const bool can_list = sizeof(S) == 1 && PUSH && p.list_ok && p.dirty && head().maxdeg <= 64u;
  for (;;) {
    WE* Win = (WE*)head().wlp[(r + 1) & 1];
    WE* Wout = (WE*)head().wlp[r & 1];
    const uint32_t cur = r % 3;
    const uint64_t tot = list ? tot_list : (uint64_t)head().cnt[cur][0] + head().cnt[cur][1];
    // dirty-set rounds (N1) on bounded-degree graphs (max degree <= 64): measured on B200, every
    // round marks on the 27-point stencil (-22 %) and the mesh (-4 %); on R-MAT marking the
    // hub rows costs more than it saves (2.4x slower when forced), and a per-round cost model
    // based on the previous round's tentative-colour changes did no better than this rule
    bool mark = r >= 2 && (p.n1 == 2 || (p.n1 == 1 && head().maxdeg <= 64u));
    if (mark && p.n1 == 1 && p.n1chg)  // optional: only once the previous round changed few colours
      mark = r >= 3 && (uint64_t)head().chg[(r - 1) % 3] * p.n1chg < tot;
    if (r > 1) {
      if (list) phase_a_list<S, POL, CW>(p, r, wk);
      else if (dense) phase_a_dense<S, POL, CW>(p, r, mark, wk);
      else phase_a<S, POL, PUSH, CW>(p, r, bins, Win, mark, wk);
      work_stamp(p, 4 * r - 3, r);
      if (!grid_sync(p)) {
        // where a stopped run can be resumed with wider words (8-bit overflow in this Phase A)
        if (blk(p) == 0 && threadIdx.x == 0) {
          p.info->resume_r = list ? 0u : r;
          p.info->resume_mode = dense ? 1u : 0u;
        }
        return;
      }
    }
    if (stamp && r <= p.trace_cap) p.phase_ns[4 * r - 2] = globaltimer();
    // round r+1 runs as a list round when round r-1's winners x 4 (successors + 1) <= n
    // (p.list_ok == 2: from round 2 on, tests); round r then records its winners
    bool list_next = list;
    if (!list && can_list && r >= 2) {
      const uint64_t prev = (uint64_t)head().cnt[(r - 1) % 3][0] + head().cnt[(r - 1) % 3][1];
      const uint64_t won = prev > tot ? prev - tot : 0;
      list_next = p.list_ok == 2 || won * 4 * p.davg2 <= (uint64_t)p.n;
    }
    if (list) {
      phase_b_list<S, POL, PUSH, CW>(p, r, (uint32_t)tot, wk);
    } else if (dense) {
      // dirty-set rounds make the dense sweep cheap for clean vertices: stay dense longer
      const bool push_out = !list_next && tot * (mark ? p.dense_div_n1 : p.dense_div) <= (uint64_t)p.n;
      phase_b_dense<S, POL, PUSH, CW>(p, r, bins, Wout, push_out, mark, wk, list_next);
      if (push_out) dense = false;
    } else {
      phase_b<S, POL, PUSH, CW>(p, r, bins, Win, Wout, mark, wk, list_next);
    }
    // multi-GPU: |W_r| of the trace is the global one (the phase wrote the local count)
    if (dist(p) && blk(p) == 0 && threadIdx.x == 0 && p.trace && r <= p.trace_cap)
      p.trace[r - 1] = head().gtot[cur];
    work_stamp(p, 4 * r - 1, r);
    if (!grid_sync(p, dist(p) ? (int)((r + 1) % 3) : -1)) return;
    if (stamp && r <= p.trace_cap) p.phase_ns[4 * r] = globaltimer();
    uint32_t left;
    if (list) left = (uint32_t)tot - head().wl_cnt[cur];
    else if (dist(p)) left = head().gtot[(r + 1) % 3];  // global: every rank stops together
    else left = next_total(p, r);
    if (list_next) {
      list = true;
      tot_list = left;
    }
    if (left == 0) break;
    if (r >= p.max_rounds) {
      if (blk(p) == 0 && threadIdx.x == 0) atomicExch(&p.info->status, (uint32_t)ST_NO_CONVERGENCE);  // same r on every rank
      flush_work<CW>(p, wk);
      return;
    }
    ++r;
  }
  epilogue<S>(p);
  flush_work<CW>(p, wk);
  if (blk(p) == 0 && threadIdx.x == 0) p.info->rounds = r;
  if (dist(p)) grid_sync(p);  // every rank's num_colors holds the global max before the host reads it
}

template <class S, int POL, bool PUSH, bool CW>
__global__ void __launch_bounds__(BLOCK, GC_MINB) sgr_persistent(Params p) {
  sgr_body<S, POL, PUSH, CW>(p);
}
// Bounded-degree graphs with >= 8 entries per row on average (27-point stencils): 3 CTAs per SM
// with up to 80 registers (no spills; fewer CTAs in every grid barrier) measured faster there
// (stencil 128^3: 8.25 -> 7.68 ms), slower on R-MAT and the mesh.
template <int POL, bool CW>
__global__ void __launch_bounds__(BLOCK, 3) sgr_persistent_fat(Params p) {
  sgr_body<uint8_t, POL, true, CW>(p);
}

#ifdef GC_DIST_TU
// Multi-GPU entry: `ranks` ranks' parameter blocks in device memory; the launch holds G =
// gridDim.x / ranks CTAs per rank (one rank per launch on real GPUs; all emulated ranks of a
// one-GPU test group in one cooperative launch).  A CTA copies its rank's Params into shared
// memory (a run-time index into kernel parameters would put the whole block on the stack).
__device__ __forceinline__ const Params& stage_params(const Params* __restrict__ pp) {
  __shared__ __align__(16) Params sp;
  const uint32_t G = gridDim.x / (uint32_t)pp[0].nranks_in_launch;
  const Params* src = pp + blockIdx.x / G;
  for (uint32_t i = threadIdx.x; i < sizeof(Params) / 4; i += BLOCK)
    ((uint32_t*)&sp)[i] = ((const uint32_t*)src)[i];
  __syncthreads();
  return sp;
}
template <class S, int POL, bool CW>
__global__ void __launch_bounds__(BLOCK, GC_MINB) sgr_dist(const Params* __restrict__ pp) {
  sgr_body<S, POL, true, CW>(stage_params(pp));
}
template <int POL, bool CW>
__global__ void __launch_bounds__(BLOCK, 3) sgr_dist_fat(const Params* __restrict__ pp) {
  sgr_body<uint8_t, POL, true, CW>(stage_params(pp));
}
#endif

#ifndef GC_INST_TU  // the non-template kernels below live in gc_api.cu only
// ---------------------------------------------------------------- host-driven ablation
// GC_FLAG_HOST_ROUNDS: the same phases (32-bit state words), one non-cooperative launch
// each, the host reading |W_{r+1}| after every round ("CPU ... controlling the progress").
template <bool PUSH>
__global__ void __launch_bounds__(BLOCK) k_prologue_count(Params p) { prologue_count<uint32_t, HIGHER_ID, PUSH>(p, false); }
__global__ void __launch_bounds__(BLOCK) k_prologue_scatter(Params p) {
  Bins b;
  b.load(p);
  prologue_scatter(p, b);
}
template <bool PUSH, bool CW>
__global__ void __launch_bounds__(BLOCK) k_phase_a(Params p, uint32_t r, WE* W) {
  Work wk;
  wk.zero();
  Bins b;
  b.load(p);
  if (threadIdx.x == 0) take_head(p);  // the previous launch's counters
  __syncthreads();
  phase_a<uint32_t, HIGHER_ID, PUSH, CW>(p, r, b, W, false, wk);
  flush_work<CW>(p, wk);
}
template <int POL, bool PUSH, bool CW>
__global__ void __launch_bounds__(BLOCK) k_phase_b(Params p, uint32_t r, WE* W, WE* Wout) {
  Work wk;
  wk.zero();
  Bins b;
  b.load(p);
  if (threadIdx.x == 0) take_head(p);  // the previous launch's counters
  __syncthreads();
  phase_b<uint32_t, POL, PUSH, CW>(p, r, b, W, Wout, false, wk);
  flush_work<CW>(p, wk);
}
__global__ void __launch_bounds__(BLOCK) k_epilogue(Params p, uint32_t r) {
  epilogue<uint32_t>(p);
  if (blockIdx.x == 0 && threadIdx.x == 0) p.info->rounds = r;
}

// 8-bit -> 16-bit state words in place (gc_color's widening after ST_NEED16): top bit = committed,
// the rest = colour, in both widths.
__global__ void __launch_bounds__(BLOCK) k_widen8(const uint8_t* __restrict__ s8, uint16_t* __restrict__ s16,
                                                  int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < count; i += (int64_t)gridDim.x * BLOCK) {
    const uint32_t x = s8[i];
    s16[i] = (uint16_t)(((x & SW<uint8_t>::COMMIT) ? SW<uint16_t>::COMMIT : 0u) | (x & SW<uint8_t>::CMASK));
  }
}

// Grid-barrier cost probe (diagnostics only: gc__bench_grid_sync).
__global__ void __launch_bounds__(BLOCK) k_bench_sync(Params p, int iters) {
  if (threadIdx.x == 0) barriers_passed() = 0;
  for (int i = 0; i < iters; ++i)
    if (!grid_sync(p)) return;
}

// ---------------------------------------------------------------- validation (C9)
// One warp per vertex: row_ptr monotone, 0 <= w < n, w != v, strictly increasing rows;
// optionally symmetry by binary search of v in adj(w).  Records the smallest bad vertex.
enum ValErr { VE_NONE = 0, VE_ROWPTR = 1, VE_RANGE = 2, VE_SELF = 3, VE_ORDER = 4, VE_ASYM = 5 };

// I->bad starts at 0 (= nothing found); the smallest (vertex, code) key wins via atomicMax
// of its complement, decoded on the host as ~bad.
__device__ __forceinline__ void report_bad(DevInfo* I, int64_t v, uint32_t code) {
  const unsigned long long key = ((unsigned long long)v << 3) | code;
  atomicMax(&I->bad, ~key);
}

// Rows [v_base, v_base + n) of a graph on n_global vertices (one GPU: v_base = 0, n_global = n);
// the symmetry check needs every row, so it is single-GPU only.
__global__ void __launch_bounds__(BLOCK) k_validate(int32_t n, int64_t v_base, int64_t n_global,
                                                    const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                    int symmetry, DevInfo* I) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * BLOCK) >> 5;
  if (gw == 0 && lane == 0 && __ldg(rp) != 0) report_bad(I, v_base, VE_ROWPTR);
  for (int64_t u = gw; u < n; u += nw) {
    const int64_t v = v_base + u;
    const int64_t beg = __ldg(rp + u), end = __ldg(rp + u + 1);
    if (end < beg) { if (lane == 0) report_bad(I, v, VE_ROWPTR); continue; }
    for (int64_t e = beg + lane; e < end; e += 32) {
      const int32_t w = __ldg(ci + e);
      if (w < 0 || w >= n_global) { report_bad(I, v, VE_RANGE); continue; }
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
      const uint32_t need = c - base;
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

#endif  // GC_INST_TU

}  // namespace gcdev
