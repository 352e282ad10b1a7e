// dist_api.cuh — vertex-range partitioned SGR (multi-GPU path, include/gc_dist.h).
// Included at the end of gc_api.cu (same translation unit: shares its host helpers).
//
// One partition = one process/GPU holding the rows [v_begin, v_end) (row_ptr rebased to 0,
// col_idx in global ids) and a REPLICATED state word per global vertex (ghost colours).
// The round structure of the single-GPU path is kept; between the phases the caller
// exchanges packed (vertex, state word) pairs with the other partitions (NCCL all-gather over
// NVLink via torch.distributed, see paper_1606_06025_b200/dist.py):
//   round r:  [Phase A: tentative colours of the local pending vertices, pull First-Fit over
//              the replicated committed colours]  -> exchange the local pending tents
//             Phase B: conflict scan against the replicated tents, global ids decide
//              -> exchange the local winners (committed words) ; global |W| decides the end.
// Every partition therefore sees exactly the single-GPU state after each phase, so the
// colouring is bit-identical to one GPU for any cover of [0, n).
#pragma once
#include <cub/device/device_scan.cuh>

namespace gcdev {

__global__ void __launch_bounds__(BLOCK) k_fill_u32(uint32_t* p, int64_t n, uint32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) p[i] = v;
}

// (vertex, state word) of every entry of the given worklist bins; with only_committed the
// entries whose word has the commit bit (this round's winners).
__global__ void __launch_bounds__(BLOCK) k_pack(const WE* W, const uint32_t* off, const uint32_t* cnt,
                                                const uint32_t* st, int only_committed, uint32_t* out,
                                                unsigned long long* out_count, const uint8_t* boundary,
                                                int32_t v_base) {
  const int lane = threadIdx.x & 31;
  for (int b = 0; b < NBIN; ++b) {
    const uint32_t nb = cnt[b];
    const WE* Wb = W + off[b];
    for (uint32_t base = (blockIdx.x * BLOCK) + (threadIdx.x & ~31u); base < nb; base += gridDim.x * BLOCK) {
      const uint32_t i = base + lane;
      bool take = false;
      int32_t v = 0;
      uint32_t s = 0;
      if (i < nb) {
        v = ldw_v(Wb + i);
        s = lds(st + v);
        take = boundary[v - v_base] && (!only_committed || (s & SW<uint32_t>::COMMIT));
      }
      const unsigned m = __ballot_sync(FULL, take);
      if (!m) continue;
      unsigned long long pos = 0;
      if (lane == __ffs(m) - 1) pos = atomicAdd(out_count, (unsigned long long)__popc(m));
      pos = __shfl_sync(FULL, pos, __ffs(m) - 1);
      if (take) {
        const unsigned long long j = pos + __popc(m & lanemask_lt());
        out[2 * j] = (uint32_t)v;
        out[2 * j + 1] = s;
      }
    }
  }
}

__global__ void __launch_bounds__(BLOCK) k_unpack(const uint32_t* pairs, int64_t count, uint32_t* st) {
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < count; i += (int64_t)gridDim.x * BLOCK)
    st[pairs[2 * i]] = pairs[2 * i + 1];
}

// Halo adjacency (push First-Fit across partitions): for every remote vertex w, the local
// vertices adjacent to it (the symmetric half of the cut edges), as offsets hoff[w] into hadj.
// A remote winner's colour bit reaches the forbidden-colour planes of its local neighbours
// through this list when its commit pair is unpacked (the winner's own partition cannot RED
// into another GPU's planes).
// One warp per local vertex (coalesced row reads; hub rows do not serialise one thread).
__global__ void __launch_bounds__(BLOCK) k_halo_count(Params p, int64_t n_local, int64_t v_begin, int64_t v_end,
                                                      uint32_t* hcnt, uint8_t* boundary) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * BLOCK) >> 5;
  for (int64_t u = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) >> 5; u < n_local; u += nw) {
    bool b = false;
    for (int64_t e = p.rp[u] + lane; e < p.rp[u + 1]; e += 32) {
      const int32_t w = p.ci[e];
      if (w < v_begin || w >= v_end) {
        atomicAdd(&hcnt[w], 1u);
        b = true;
      }
    }
    b = __any_sync(FULL, b);
    if (lane == 0) boundary[u] = b ? 1 : 0;  // only boundary vertices' words are read remotely
  }
}
__global__ void __launch_bounds__(BLOCK) k_halo_fill(Params p, int64_t n_local, int64_t v_begin, int64_t v_end,
                                                     uint32_t* hcur, int32_t* hadj) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * BLOCK) >> 5;
  for (int64_t u = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) >> 5; u < n_local; u += nw)
    for (int64_t e = p.rp[u] + lane; e < p.rp[u + 1]; e += 32) {
      const int32_t w = p.ci[e];
      if (w < v_begin || w >= v_end) hadj[atomicAdd(&hcur[w], 1u)] = (int32_t)(v_begin + u);
    }
}
// Commit pairs of remote winners -> colour bit into the planes of their local neighbours.
__global__ void __launch_bounds__(BLOCK) k_halo_apply(const uint32_t* pairs, int64_t count, int64_t v_begin,
                                                      int64_t v_end, const uint32_t* hoff, const int32_t* hadj,
                                                      uint8_t* fmp, int64_t plane, uint32_t np) {
  const int64_t T = (int64_t)gridDim.x * BLOCK;
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < count; i += T) {
    const uint32_t w = pairs[2 * i], word = pairs[2 * i + 1];
    if (!(word & SW<uint32_t>::COMMIT) || ((int64_t)w >= v_begin && (int64_t)w < v_end)) continue;
    const uint32_t c = word & SW<uint32_t>::CMASK;
    if (c == 0 || c > 8u * np) continue;
    uint8_t* pl = fmp + (int64_t)((c - 1) >> 3) * plane;
    const uint32_t bit = 1u << ((c - 1) & 7);
    for (uint32_t j = hoff[w]; j < hoff[w + 1]; ++j) red_plane<uint32_t>(pl, hadj[j], bit);
  }
}

}  // namespace gcdev

struct gc_dist {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int grid = 0;
  int policy = 0;
  uint32_t round = 1;
  uint32_t max_rounds = 0;
  int64_t n_global = 0, v_begin = 0, v_end = 0;
  Params p;
  WE* W[2] = {nullptr, nullptr};
  int cur = 0;                       // W[cur] = W_in of the current round
  uint32_t cnt_in[NBIN] = {0, 0};    // |W_in| per bin
  uint32_t off[NBIN] = {0, 0};
  uint32_t* d_off = nullptr;         // device copies for k_pack
  uint32_t* d_cnt = nullptr;
  unsigned long long* d_count = nullptr;
  void* mem[16] = {};
  uint8_t* boundary = nullptr;       // local vertices with a remote neighbour (the only ones packed)
  uint32_t* hoff = nullptr;          // halo adjacency (push First-Fit across partitions)
  int32_t* hadj = nullptr;
  int nmem = 0;
};

namespace {

gc_status dist_fail(gc_dist* h, cudaError_t e, const char* what) {
  (void)h;
  return cuda_fail(e, what);
}

#define DK(call)                                                \
  do {                                                          \
    cudaError_t e_ = (call);                                    \
    if (e_ != cudaSuccess) return dist_fail(h, e_, #call);      \
  } while (0)

void launch_dist_b(gc_dist* h, int grid, const Params& p, uint32_t r, WE* W, WE* Wo) {
  if (h->policy == HIGHER_ID) k_phase_b<HIGHER_ID, true, false><<<grid, BLOCK, 0, h->stream>>>(p, r, W, Wo);
  else k_phase_b<LOWER_ID, true, false><<<grid, BLOCK, 0, h->stream>>>(p, r, W, Wo);
}

}  // namespace

extern "C" {

gc_status gc_dist_create(gc_dist** out, int64_t n_global, int64_t v_begin, int64_t v_end,
                         const int64_t* row_ptr_local, const int32_t* col_idx_local, const gc_opts* opts_in) {
  g_err[0] = 0;
  if (!out) {
    set_err("gc_dist_create: out is NULL");
    return GC_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  gc_opts o;
  gc_opts_default(&o);
  if (opts_in) {
    if (opts_in->struct_size != sizeof(gc_opts)) {
      set_err("gc_dist_create: bad opts->struct_size");
      return GC_ERR_INVALID_ARGUMENT;
    }
    o = *opts_in;
  }
  if (n_global < 0 || n_global > INT32_MAX || v_begin < 0 || v_end < v_begin || v_end > n_global) {
    set_err("gc_dist_create: bad range [%lld, %lld) of n=%lld", (long long)v_begin, (long long)v_end,
            (long long)n_global);
    return GC_ERR_INVALID_ARGUMENT;
  }
  if (o.policy == GC_POLICY_DEGREE) {
    set_err("gc_dist_create: GC_POLICY_DEGREE is single-GPU only (needs remote degrees)");
    return GC_ERR_UNSUPPORTED;
  }
  if (o.policy > GC_POLICY_DEGREE) {
    set_err("gc_dist_create: unknown policy %u", o.policy);
    return GC_ERR_INVALID_ARGUMENT;
  }
  const int64_t nl = v_end - v_begin;
  if (nl > 0 && (!row_ptr_local || !col_idx_local)) {
    set_err("gc_dist_create: NULL row_ptr/col_idx");
    return GC_ERR_INVALID_ARGUMENT;
  }
  if ((nl > 0 && is_device_ptr(row_ptr_local) != 1) || (nl > 0 && is_device_ptr(col_idx_local) != 1)) {
    set_err("gc_dist_create: row_ptr_local and col_idx_local must be device memory");
    return GC_ERR_INVALID_ARGUMENT;
  }
  gc_dist* h = new gc_dist();
  int prev = 0;
  cudaGetDevice(&prev);
  h->dev = o.device >= 0 ? o.device : prev;
  cudaError_t e = cudaSetDevice(h->dev);
  if (e != cudaSuccess) { delete h; return cuda_fail(e, "cudaSetDevice"); }
  DevFacts f;
  if ((e = dev_facts(h->dev, &f)) != cudaSuccess) { delete h; return cuda_fail(e, "dev_facts"); }
  if ((e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking)) != cudaSuccess) { delete h; return cuda_fail(e, "stream"); }
  h->grid = f.sms * 4;
  h->policy = (int)o.policy;
  h->n_global = n_global;
  h->v_begin = v_begin;
  h->v_end = v_end;
  h->max_rounds = o.max_rounds ? o.max_rounds : (uint32_t)(n_global + 1 > 0xffffffffLL ? 0xffffffffu : n_global + 1);
  // workspace from the per-device stream-ordered pool (cached across partitions: creating
  // and destroying a partition per colouring costs no cudaMalloc/cudaFree)
  cudaMemPool_t pool;
  if ((e = get_pool(h->dev, &pool)) != cudaSuccess) { gc_dist_destroy(h); return cuda_fail(e, "get_pool"); }
  auto alloc = [&](void** q, size_t bytes) {
    cudaError_t ee = cudaMallocFromPoolAsync(q, bytes ? bytes : 16, pool, h->stream);
    if (ee == cudaSuccess) h->mem[h->nmem++] = *q;
    return ee;
  };
  void *st, *w0, *w1, *info, *doff, *dcnt, *dcount;
  if ((e = alloc(&st, sizeof(uint32_t) * (size_t)(n_global ? n_global : 1))) != cudaSuccess ||
      (e = alloc(&w0, sizeof(WE) * (size_t)(nl ? nl : 1))) != cudaSuccess ||
      (e = alloc(&w1, sizeof(WE) * (size_t)(nl ? nl : 1))) != cudaSuccess ||
      (e = alloc(&info, sizeof(DevInfo))) != cudaSuccess || (e = alloc(&doff, 64)) != cudaSuccess ||
      (e = alloc(&dcnt, 64)) != cudaSuccess || (e = alloc(&dcount, 64)) != cudaSuccess) {
    gc_dist_destroy(h);
    return cuda_fail(e, "gc_dist_create: cudaMalloc");
  }
  // forbidden-colour planes indexed by global id (only the local bytes are ever read)
  const int64_t pitch = (n_global + 255) / 256 * 256;
  uint32_t np = (uint32_t)MAX_PLANES;
  if ((uint64_t)np * (uint64_t)pitch > (16ull << 30)) {
    const uint64_t fit = (16ull << 30) / (uint64_t)pitch;
    np = fit < 16 ? 16u : (uint32_t)fit;
  }
  void *planes, *hoff, *hcur, *bnd;
  if ((e = alloc(&planes, (size_t)pitch * np)) != cudaSuccess ||
      (e = alloc(&bnd, (size_t)(nl ? nl : 1))) != cudaSuccess ||
      (e = alloc(&hoff, sizeof(uint32_t) * (size_t)(n_global + 1))) != cudaSuccess ||
      (e = alloc(&hcur, sizeof(uint32_t) * (size_t)(n_global + 1))) != cudaSuccess) {
    gc_dist_destroy(h);
    return cuda_fail(e, "gc_dist_create: cudaMalloc");
  }
  memset(&h->p, 0, sizeof(h->p));
  Params& p = h->p;
  p.fmp = (uint8_t*)planes;
  p.plane = pitch;
  p.np = np;
  p.n = (int32_t)nl;
  p.v_base = (int32_t)v_begin;
  p.rp = row_ptr_local;
  p.ci = col_idx_local;
  p.st = st;
  p.wl0 = (WE*)w0;
  p.wl1 = (WE*)w1;
  p.info = (DevInfo*)info;
  p.max_rounds = h->max_rounds;
  p.t1 = o.thread_bin_max ? o.thread_bin_max : 16;
  p.t3 = o.warp_bin_max ? o.warp_bin_max : 1024;
  p.timeout_ns = 60ull * 1000000000ull;
  h->W[0] = (WE*)w0;
  h->W[1] = (WE*)w1;
  h->d_off = (uint32_t*)doff;
  h->d_cnt = (uint32_t*)dcnt;
  h->d_count = (unsigned long long*)dcount;
  cudaStream_t s = h->stream;
  // every vertex (owned or ghost) starts pending with tentative colour 1 (round 1)
  k_fill_u32<<<h->grid, BLOCK, 0, s>>>((uint32_t*)st, n_global, 1u);
  DK(cudaMemsetAsync(info, 0, sizeof(DevInfo), s));
  if (nl > 0) {
    k_prologue_count<true><<<h->grid, BLOCK, 0, s>>>(p);
    k_prologue_scatter<<<h->grid, BLOCK, 0, s>>>(p);
  }
  // halo adjacency: counts per remote vertex -> offsets -> lists
  DK(cudaMemsetAsync(hoff, 0, sizeof(uint32_t) * (size_t)(n_global + 1), s));
  if (nl > 0) k_halo_count<<<h->grid, BLOCK, 0, s>>>(p, nl, v_begin, v_end, (uint32_t*)hoff, (uint8_t*)bnd);
  h->boundary = (uint8_t*)bnd;
  {  // exclusive scan (CUB) of the n_global + 1 counters into hcur, then back to hoff
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (uint32_t*)hoff, (uint32_t*)hcur, (int)(n_global + 1), s);
    void* tmp;
    if ((e = alloc(&tmp, tmp_bytes)) != cudaSuccess) {
      gc_dist_destroy(h);
      return cuda_fail(e, "gc_dist_create: cudaMalloc");
    }
    DK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, (uint32_t*)hoff, (uint32_t*)hcur, (int)(n_global + 1), s));
    DK(cudaMemcpyAsync(hoff, hcur, sizeof(uint32_t) * (size_t)(n_global + 1), cudaMemcpyDeviceToDevice, s));
  }
  uint32_t nhalo = 0;
  DK(cudaMemcpyAsync(&nhalo, (uint32_t*)hoff + n_global, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  DK(cudaStreamSynchronize(s));
  void* hadj;
  if ((e = alloc(&hadj, sizeof(int32_t) * (size_t)(nhalo ? nhalo : 1))) != cudaSuccess) {
    gc_dist_destroy(h);
    return cuda_fail(e, "gc_dist_create: cudaMalloc");
  }
  DK(cudaMemcpyAsync(hcur, hoff, sizeof(uint32_t) * (size_t)(n_global + 1), cudaMemcpyDeviceToDevice, s));
  if (nl > 0) k_halo_fill<<<h->grid, BLOCK, 0, s>>>(p, nl, v_begin, v_end, (uint32_t*)hcur, (int32_t*)hadj);
  h->hoff = (uint32_t*)hoff;
  h->hadj = (int32_t*)hadj;
  DK(cudaGetLastError());
  DevInfo hi;
  DK(cudaMemcpyAsync(&hi, info, sizeof(DevInfo), cudaMemcpyDeviceToHost, s));
  DK(cudaStreamSynchronize(s));
  uint32_t acc = 0;
  for (int b = 0; b < NBIN; ++b) {
    h->off[b] = acc;
    acc += hi.binsize[b];
    h->cnt_in[b] = hi.binsize[b];
  }
  DK(cudaMemcpy(h->d_off, h->off, sizeof(h->off), cudaMemcpyHostToDevice));
  cudaSetDevice(prev);
  *out = h;
  return GC_OK;
}

gc_status gc_dist_phase_a(gc_dist* h) {
  g_err[0] = 0;
  if (!h) return GC_ERR_INVALID_ARGUMENT;
  if (h->round > 1 && h->p.n > 0) {
    k_phase_a<true, false><<<h->grid, BLOCK, 0, h->stream>>>(h->p, h->round, h->W[h->cur]);
    DK(cudaGetLastError());
  }
  DK(cudaStreamSynchronize(h->stream));
  return GC_OK;
}

gc_status gc_dist_phase_b(gc_dist* h, uint32_t* local_next) {
  g_err[0] = 0;
  if (!h || !local_next) return GC_ERR_INVALID_ARGUMENT;
  if (h->round > h->max_rounds) {
    set_err("gc_dist_phase_b: no convergence within max_rounds=%u", h->max_rounds);
    return GC_ERR_NO_CONVERGENCE;
  }
  *local_next = 0;
  if (h->p.n > 0) {
    launch_dist_b(h, h->grid, h->p, h->round, h->W[h->cur], h->W[h->cur ^ 1]);
    DK(cudaGetLastError());
    uint32_t cnt[3][NBIN];
    DK(cudaMemcpyAsync(cnt, h->p.info->cnt, sizeof(cnt), cudaMemcpyDeviceToHost, h->stream));
    DK(cudaStreamSynchronize(h->stream));
    for (int b = 0; b < NBIN; ++b) *local_next += cnt[(h->round + 1) % 3][b];
  }
  return GC_OK;
}

// what = 0: (v, word) of every local pending vertex of the current round (after Phase A);
// what = 1: the local winners of the current round (after Phase B).  pairs: device buffer of
// at least 2 * (v_end - v_begin) uint32.  *count = number of pairs written.
gc_status gc_dist_pack(gc_dist* h, int32_t what, uint32_t* pairs, uint64_t* count) {
  g_err[0] = 0;
  if (!h || !count || (what != 0 && what != 1)) return GC_ERR_INVALID_ARGUMENT;
  *count = 0;
  if (h->p.n == 0) return GC_OK;
  if (!pairs) return GC_ERR_INVALID_ARGUMENT;
  DK(cudaMemcpyAsync(h->d_cnt, h->cnt_in, sizeof(h->cnt_in), cudaMemcpyHostToDevice, h->stream));
  DK(cudaMemsetAsync(h->d_count, 0, sizeof(unsigned long long), h->stream));
  k_pack<<<h->grid, BLOCK, 0, h->stream>>>(h->W[h->cur], h->d_off, h->d_cnt, (const uint32_t*)h->p.st, what, pairs,
                                           h->d_count, h->boundary, h->p.v_base);
  DK(cudaGetLastError());
  unsigned long long c = 0;
  DK(cudaMemcpyAsync(&c, h->d_count, sizeof(c), cudaMemcpyDeviceToHost, h->stream));
  DK(cudaStreamSynchronize(h->stream));
  *count = c;
  return GC_OK;
}

gc_status gc_dist_unpack(gc_dist* h, const uint32_t* pairs, uint64_t count) {
  g_err[0] = 0;
  if (!h || (count && !pairs)) return GC_ERR_INVALID_ARGUMENT;
  if (count) {
    k_unpack<<<h->grid, BLOCK, 0, h->stream>>>(pairs, (int64_t)count, (uint32_t*)h->p.st);
    if (h->p.n > 0)
      k_halo_apply<<<h->grid, BLOCK, 0, h->stream>>>(pairs, (int64_t)count, h->v_begin, h->v_end, h->hoff, h->hadj,
                                                     h->p.fmp, h->p.plane, h->p.np);
    DK(cudaGetLastError());
  }
  DK(cudaStreamSynchronize(h->stream));
  return GC_OK;
}

// Advance to the next round (W_out becomes W_in); local_next = |W_out| from gc_dist_phase_b.
gc_status gc_dist_next_round(gc_dist* h) {
  g_err[0] = 0;
  if (!h) return GC_ERR_INVALID_ARGUMENT;
  if (h->p.n > 0) {
    uint32_t cnt[3][NBIN];
    DK(cudaMemcpy(cnt, h->p.info->cnt, sizeof(cnt), cudaMemcpyDeviceToHost));
    for (int b = 0; b < NBIN; ++b) h->cnt_in[b] = cnt[(h->round + 1) % 3][b];
  }
  h->cur ^= 1;
  h->round += 1;
  return GC_OK;
}

gc_status gc_dist_finalize(gc_dist* h, uint32_t* colors_local, uint32_t* max_color_local, uint32_t* rounds) {
  g_err[0] = 0;
  if (!h || !max_color_local || !rounds) return GC_ERR_INVALID_ARGUMENT;
  *max_color_local = 0;
  *rounds = h->round;
  if (h->p.n == 0) return GC_OK;
  if (!colors_local || is_device_ptr(colors_local) != 1) {
    set_err("gc_dist_finalize: colors_local must be device memory");
    return GC_ERR_INVALID_ARGUMENT;
  }
  Params p = h->p;
  p.colors_out = colors_local;
  DK(cudaMemsetAsync(&h->p.info->num_colors, 0, sizeof(uint32_t), h->stream));
  k_epilogue<<<h->grid, BLOCK, 0, h->stream>>>(p, h->round);
  DK(cudaGetLastError());
  DK(cudaMemcpyAsync(max_color_local, &h->p.info->num_colors, sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
  DK(cudaStreamSynchronize(h->stream));
  return GC_OK;
}

gc_status gc_dist_destroy(gc_dist* h) {
  if (!h) return GC_OK;
  for (int i = 0; i < h->nmem; ++i) cudaFreeAsync(h->mem[i], h->stream);
  if (h->stream) {
    cudaStreamSynchronize(h->stream);
    cudaStreamDestroy(h->stream);
  }
  delete h;
  return GC_OK;
}

}  // extern "C"
