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

namespace gcdev {

__global__ void __launch_bounds__(BLOCK) k_fill_u32(uint32_t* p, int64_t n, uint32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) p[i] = v;
}

// (vertex, state word) of every entry of the given worklist bins; with only_committed the
// entries whose word has the commit bit (this round's winners).
__global__ void __launch_bounds__(BLOCK) k_pack(const WE* W, const uint32_t* off, const uint32_t* cnt,
                                                const uint32_t* st, int only_committed, uint32_t* out,
                                                unsigned long long* out_count) {
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
        take = !only_committed || (s & SW<uint32_t>::COMMIT);
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
  void* mem[8] = {};
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
  if (h->policy == HIGHER_ID) k_phase_b<HIGHER_ID, false, false><<<grid, BLOCK, 0, h->stream>>>(p, r, W, Wo);
  else k_phase_b<LOWER_ID, false, false><<<grid, BLOCK, 0, h->stream>>>(p, r, W, Wo);
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
  auto alloc = [&](void** q, size_t bytes) {
    cudaError_t ee = cudaMalloc(q, bytes ? bytes : 16);
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
  memset(&h->p, 0, sizeof(h->p));
  Params& p = h->p;
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
  p.t3 = o.warp_bin_max ? o.warp_bin_max : 512;
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
    k_prologue_count<false><<<h->grid, BLOCK, 0, s>>>(p);
    k_prologue_scatter<<<h->grid, BLOCK, 0, s>>>(p);
  }
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
    k_phase_a<false, false><<<h->grid, BLOCK, 0, h->stream>>>(h->p, h->round, h->W[h->cur]);
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
                                           h->d_count);
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
  for (int i = 0; i < h->nmem; ++i) cudaFree(h->mem[i]);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return GC_OK;
}

}  // extern "C"
