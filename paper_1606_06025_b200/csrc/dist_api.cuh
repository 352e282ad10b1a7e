// dist_api.cuh — host side of include/gc_dist.h: multi-GPU SGR with a device-initiated
// exchange.  Included at the end of gc_api.cu (same translation unit: shares
// its host helpers and the persistent kernel instances).
//
// Per rank: one IPC-exportable window (cudaMalloc) laid out identically on every rank for a
// given n_global (WinLayout); every rank maps every other rank's window once (CUDA IPC, or
// plain pointers in the one-process emulation) and the persistent kernel receives the table of
// peer pointers (Params::peer).  NCCL is used only to all-gather small host records
// (arguments, IPC handles) — the bootstrap; the colouring itself never returns to the host.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <mutex>
#include <vector>

namespace {

// ---- NCCL, resolved at run time (the process may already hold torch's libnccl.so.2)
struct NcclApi {
  bool ok = false;
  char why[256] = "";
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi* nccl_api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(a.why, sizeof(a.why), "dlopen(libnccl.so.2): %s", dlerror());
      return;
    }
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.CommDestroy && a.GetErrorString;
    if (!a.ok) snprintf(a.why, sizeof(a.why), "libnccl.so.2 lacks a required symbol");
  });
  return &a;
}

// ---- one-process emulation: ranks are threads; the bootstrap all-gather is a memory exchange
// behind a generation barrier (two slot sets by generation parity, so a fast rank entering the
// next exchange never overwrites a slot a slow rank is still copying).
struct LocalGroup {
  int world = 0;
  int refs = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<std::vector<uint8_t>> slot[2];
  std::vector<Params> params;   // the ranks' kernel parameters of the shared launch
  float kernel_ms = 0;
};

constexpr size_t kBootBytes = 256;  // largest bootstrap record

// Window layout (byte offsets), identical on every rank for a given n_global.
struct WinLayout {
  int64_t pitch = 0;
  uint32_t np = 0;
  size_t xflag = 0, peers = 0, info = 0, st = 0, planes = 0, dirty = 0, ksplit = 0, bmask = 0, total = 0;
};
WinLayout win_layout(int64_t n_global) {
  WinLayout L;
  L.pitch = (n_global + 255) / 256 * 256;
  if (L.pitch == 0) L.pitch = 256;
  L.np = (uint32_t)MAX_PLANES;
  if ((uint64_t)L.np * (uint64_t)L.pitch > (16ull << 30)) {
    const uint64_t fit = (16ull << 30) / (uint64_t)L.pitch;
    L.np = fit < 16 ? 16u : (uint32_t)fit;
  }
  const size_t P = (size_t)L.pitch;
  L.xflag = 0;                                        // [MAX_RANKS][32] u32, persistent
  L.peers = 2048;                                     // Peer[MAX_RANKS], written per call
  static_assert(MAX_RANKS * 32 * 4 <= 2048 && MAX_RANKS * sizeof(Peer) <= 2048, "window header");
  L.info = 4096;                                      // DevInfo, zeroed per launch
  L.st = L.info + ((sizeof(DevInfo) + 4095) / 4096) * 4096;  // up to 4-byte words
  L.planes = L.st + 4 * P;
  L.dirty = L.planes + (size_t)L.np * P;
  L.ksplit = L.dirty + P;
  L.bmask = L.ksplit + 4 * P;
  L.total = L.bmask + P;
  return L;
}

}  // namespace

struct gc_comm {
  int rank = 0, world = 1, dev = 0;
  ncclComm_t nccl = nullptr;
  LocalGroup* lg = nullptr;
  cudaStream_t stream = nullptr;   // non-blocking; each call waits for the legacy stream's prior work
  void* boot = nullptr;            // NCCL bootstrap scratch: send [kBootBytes] + recv [world x kBootBytes]
  uint8_t* win = nullptr;          // this rank's window (cudaMalloc, IPC-exportable)
  size_t win_bytes = 0;
  uint8_t* peer[MAX_RANKS] = {};   // every rank's window in this process's address space
  bool mapped[MAX_RANKS] = {};     // peer[q] is an IPC mapping to close
  uint32_t epoch = 0;              // cross-rank barrier epochs used so far (same on every rank)
  DevInfo* hinfo = nullptr;        // pinned: read back after a launch without a staging copy
  void* dparams = nullptr;         // device Params of the launch this rank issues ([world] when emulating)
  bool broken = false;
};

namespace {

gc_status nccl_fail(ncclResult_t r, const char* what) {
  set_err("%s: %s", what, nccl_api()->GetErrorString ? nccl_api()->GetErrorString(r) : "NCCL error");
  return GC_ERR_NCCL;
}

// All-gather `bytes` (<= kBootBytes) per rank from every rank into all[world * bytes] (host).
gc_status boot_allgather(gc_comm* c, const void* mine, size_t bytes, void* all) {
  if (c->lg) {
    LocalGroup* g = c->lg;
    std::unique_lock<std::mutex> lk(g->mu);
    const uint64_t my_gen = g->gen;
    auto& slots = g->slot[my_gen & 1];
    slots[c->rank].assign((const uint8_t*)mine, (const uint8_t*)mine + bytes);
    if (++g->arrived == g->world) {
      g->arrived = 0;
      ++g->gen;
      g->cv.notify_all();
    } else {
      g->cv.wait(lk, [&] { return g->gen != my_gen; });
    }
    for (int q = 0; q < c->world; ++q) memcpy((uint8_t*)all + q * bytes, slots[q].data(), bytes);
    return GC_OK;
  }
  NcclApi* a = nccl_api();
  cudaError_t e;
  if ((e = cudaMemcpyAsync(c->boot, mine, bytes, cudaMemcpyHostToDevice, c->stream)) != cudaSuccess)
    return cuda_fail(e, "bootstrap H2D");
  uint8_t* recv = (uint8_t*)c->boot + kBootBytes;
  ncclResult_t r = a->AllGather(c->boot, recv, bytes, ncclUint8, c->nccl, c->stream);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  if ((e = cudaMemcpyAsync(all, recv, bytes * c->world, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(e, "bootstrap D2H");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(e, "bootstrap sync");
  return GC_OK;
}

// Agree on a status: every rank returns the worst (largest code) of all ranks' statuses.
gc_status agree(gc_comm* c, gc_status mine) {
  int32_t all[MAX_RANKS] = {};
  const int32_t m = (int32_t)mine;
  gc_status s = boot_allgather(c, &m, sizeof(m), all);
  if (s != GC_OK) {
    c->broken = true;
    return s;
  }
  gc_status worst = GC_OK;
  int who = -1;
  for (int q = 0; q < c->world; ++q)
    if (all[q] > (int32_t)worst) { worst = (gc_status)all[q]; who = q; }
  if (worst != GC_OK && mine == GC_OK) set_err("gc_color_dist: rank %d failed with %s", who, gc_status_string(worst));
  return worst;
}

void close_window(gc_comm* c) {
  for (int q = 0; q < MAX_RANKS; ++q) {
    if (c->mapped[q]) cudaIpcCloseMemHandle(c->peer[q]);
    c->mapped[q] = false;
    c->peer[q] = nullptr;
  }
  if (c->win) cudaFree(c->win);
  c->win = nullptr;
  c->win_bytes = 0;
}

// Make every rank's window hold `need` bytes and map the peers' windows (collective).
gc_status ensure_window(gc_comm* c, size_t need) {
  // every rank sees the same `need` (same n_global), so all decide alike
  if (c->win && c->win_bytes >= need) return GC_OK;
  close_window(c);
  gc_status mine = GC_OK;
  const size_t bytes = (need + (2u << 20) - 1) / (2u << 20) * (2u << 20);
  cudaError_t e = cudaMalloc((void**)&c->win, bytes);
  if (e == cudaSuccess) e = cudaMemset(c->win, 0, bytes);  // flags start at epoch 0
  if (e != cudaSuccess) {
    mine = cuda_fail(e, "gc_color_dist: window cudaMalloc");
    c->win = nullptr;
  } else {
    c->win_bytes = bytes;
  }
  c->epoch = 0;
  struct Rec {
    int32_t status;
    int32_t pad;
    uint64_t ptr;
    cudaIpcMemHandle_t h;
  } rec, all[MAX_RANKS];
  memset(&rec, 0, sizeof(rec));
  rec.status = (int32_t)mine;
  rec.ptr = (uint64_t)(uintptr_t)c->win;
  if (!c->lg && c->win && c->world > 1) {
    e = cudaIpcGetMemHandle(&rec.h, c->win);
    if (e != cudaSuccess) rec.status = (int32_t)cuda_fail(e, "cudaIpcGetMemHandle");
  }
  static_assert(sizeof(Rec) <= kBootBytes, "bootstrap record");
  gc_status s = boot_allgather(c, &rec, sizeof(rec), all);
  if (s != GC_OK) return s;
  gc_status worst = GC_OK;
  for (int q = 0; q < c->world; ++q)
    if (all[q].status > (int32_t)worst) worst = (gc_status)all[q].status;
  if (worst == GC_OK) {
    for (int q = 0; q < c->world; ++q) {
      if (q == c->rank) {
        c->peer[q] = c->win;
      } else if (c->lg) {
        c->peer[q] = (uint8_t*)(uintptr_t)all[q].ptr;
      } else {
        void* ptr = nullptr;
        e = cudaIpcOpenMemHandle(&ptr, all[q].h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          worst = cuda_fail(e, "cudaIpcOpenMemHandle");
          break;
        }
        c->peer[q] = (uint8_t*)ptr;
        c->mapped[q] = true;
      }
    }
  }
  worst = agree(c, worst);  // a failed mapping anywhere: every rank drops its window
  if (worst != GC_OK) close_window(c);
  return worst;
}

}  // namespace

extern "C" {

gc_status gc_nccl_unique_id(void* id_out) {
  g_err[0] = 0;
  if (!id_out) {
    set_err("gc_nccl_unique_id: NULL id_out");
    return GC_ERR_INVALID_ARGUMENT;
  }
  NcclApi* a = nccl_api();
  if (!a->ok) {
    set_err("gc_nccl_unique_id: %s", a->why);
    return GC_ERR_NCCL;
  }
  ncclUniqueId id;
  ncclResult_t r = a->GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(id) == GC_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof(id));
  return GC_OK;
}

static gc_status comm_common(gc_comm* c, int32_t device) {
  int prev = 0;
  cudaError_t e = cudaGetDevice(&prev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  c->dev = device >= 0 ? device : prev;
  if ((e = cudaSetDevice(c->dev)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  DevFacts f;
  if ((e = dev_facts(c->dev, &f)) != cudaSuccess) { cudaSetDevice(prev); return cuda_fail(e, "dev_facts"); }
  if (f.major != 10 || !f.coop) {
    cudaSetDevice(prev);
    set_err("gc_comm: device %d is not an sm_100-class device with cooperative launch", c->dev);
    return GC_ERR_UNSUPPORTED;
  }
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&c->hinfo, sizeof(DevInfo), cudaHostAllocDefault);
  if (e == cudaSuccess) e = cudaMalloc(&c->dparams, sizeof(Params) * MAX_RANKS);
  if (e == cudaSuccess && !c->lg) e = cudaMalloc(&c->boot, kBootBytes * (1 + MAX_RANKS));
  cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(e, "gc_comm: stream / bootstrap buffer");
  return GC_OK;
}

gc_status gc_comm_init(gc_comm** out, int32_t rank, int32_t world, const void* nccl_unique_id, int32_t device) {
  g_err[0] = 0;
  if (!out || !nccl_unique_id || world < 1 || world > MAX_RANKS || rank < 0 || rank >= world) {
    set_err("gc_comm_init: invalid argument (world must be 1..%d, 0 <= rank < world)", MAX_RANKS);
    return GC_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  NcclApi* a = nccl_api();
  if (!a->ok) {
    set_err("gc_comm_init: %s", a->why);
    return GC_ERR_NCCL;
  }
  gc_comm* c = new gc_comm();
  c->rank = rank;
  c->world = world;
  gc_status s = comm_common(c, device);
  if (s != GC_OK) { gc_comm_destroy(c); return s; }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->dev);
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  ncclResult_t r = a->CommInitRank(&c->nccl, world, id, rank);
  cudaSetDevice(prev);
  if (r != ncclSuccess) {
    c->nccl = nullptr;
    gc_comm_destroy(c);
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = c;
  return GC_OK;
}

gc_status gc_comm_init_local(gc_comm** comms_out, int32_t world, int32_t device) {
  g_err[0] = 0;
  if (!comms_out || world < 1 || world > MAX_RANKS) {
    set_err("gc_comm_init_local: world must be 1..%d", MAX_RANKS);
    return GC_ERR_INVALID_ARGUMENT;
  }
  LocalGroup* g = new LocalGroup();
  g->world = world;
  g->slot[0].resize(world);
  g->slot[1].resize(world);
  g->params.resize(world);
  for (int q = 0; q < world; ++q) comms_out[q] = nullptr;
  for (int q = 0; q < world; ++q) {
    gc_comm* c = new gc_comm();
    c->rank = q;
    c->world = world;
    c->lg = g;
    g->refs++;
    gc_status s = comm_common(c, device);
    if (s != GC_OK) {
      gc_comm_destroy(c);
      for (int k = 0; k < q; ++k) { gc_comm_destroy(comms_out[k]); comms_out[k] = nullptr; }
      return s;
    }
    comms_out[q] = c;
  }
  return GC_OK;
}

gc_status gc_comm_destroy(gc_comm* c) {
  if (!c) return GC_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->dev);
  if (c->stream) cudaStreamSynchronize(c->stream);
  close_window(c);
  if (c->boot) cudaFree(c->boot);
  if (c->hinfo) cudaFreeHost(c->hinfo);
  if (c->dparams) cudaFree(c->dparams);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->nccl && nccl_api()->CommDestroy) nccl_api()->CommDestroy(c->nccl);
  if (c->lg && --c->lg->refs == 0) delete c->lg;
  cudaSetDevice(prev);
  delete c;
  return GC_OK;
}

gc_status gc_color_dist(gc_comm* c, int64_t n_global, int64_t v_begin, int64_t v_end,
                        const int64_t* row_ptr_local, const int32_t* col_idx_local, const gc_opts* opts_in,
                        uint32_t* colors_out_local, uint32_t* num_colors, uint32_t* rounds) {
  g_err[0] = 0;
  if (!c) {
    set_err("gc_color_dist: NULL communicator");
    return GC_ERR_INVALID_ARGUMENT;
  }
  if (num_colors) *num_colors = 0;
  if (rounds) *rounds = 0;
  if (c->broken) {
    set_err("gc_color_dist: communicator unusable after an earlier failure (re-create it)");
    return GC_ERR_INVALID_ARGUMENT;
  }
  // ---- local argument checks; the verdict is agreed with the other ranks below
  gc_status local = GC_OK;
  gc_opts o;
  gc_opts_default(&o);
  Knobs kn;
  if (opts_in) {
    if (opts_in->struct_size != sizeof(gc_opts)) {
      set_err("gc_color_dist: opts->struct_size=%u, expected %zu", opts_in->struct_size, sizeof(gc_opts));
      local = GC_ERR_INVALID_ARGUMENT;
    } else {
      o = *opts_in;
    }
  }
  const int64_t nl = v_end - v_begin;
  if (local == GC_OK) {
    if (!num_colors || !rounds) set_err("gc_color_dist: num_colors and rounds must not be NULL");
    else if (o.policy > GC_POLICY_DEGREE) set_err("gc_color_dist: unknown policy %u", o.policy);
    else if (o.flags & (GC_FLAG_PULL_FIRSTFIT | GC_FLAG_HOST_ROUNDS | GC_FLAG_VALIDATE_SYMMETRY))
      set_err("gc_color_dist: PULL_FIRSTFIT / HOST_ROUNDS / VALIDATE_SYMMETRY are single-GPU only");
    else if (n_global < 0 || n_global > INT32_MAX || v_begin < 0 || v_end < v_begin || v_end > n_global)
      set_err("gc_color_dist: bad range [%lld, %lld) of n=%lld", (long long)v_begin, (long long)v_end, (long long)n_global);
    else if (nl > 0 && (!row_ptr_local || !col_idx_local || !colors_out_local))
      set_err("gc_color_dist: NULL row_ptr/col_idx/colors_out with a non-empty range");
    else if ((o.flags & GC_FLAG_TRACE) && o.trace_capacity && !o.trace_worklist)
      set_err("gc_color_dist: GC_FLAG_TRACE with NULL trace_worklist");
    else if ((o.flags & GC_FLAG_COUNT_WORK) && !o.work)
      set_err("gc_color_dist: GC_FLAG_COUNT_WORK with NULL work");
    else if (!resolve_knobs(o.tuning, &kn))
      set_err("gc_color_dist: bad opts->tuning");
    if (g_err[0]) local = GC_ERR_INVALID_ARGUMENT;
  }
  Scope sc;
  {
    cudaError_t e = cudaGetDevice(&sc.prev_dev);
    if (e == cudaSuccess) e = cudaSetDevice(c->dev);
    if (e == cudaSuccess) e = get_pool(c->dev, &sc.pool);
    if (e != cudaSuccess && local == GC_OK) local = cuda_fail(e, "gc_color_dist: device setup");
  }
  sc.stream = o.stream ? (cudaStream_t)o.stream : c->stream;
  cudaStream_t s = sc.stream;
  if (!o.stream && local == GC_OK) {  // inputs produced on the legacy default stream come first
    cudaError_t e = after_legacy(s);
    if (e != cudaSuccess) local = cuda_fail(e, "gc_color_dist: stream ordering");
  }
  // ---- agree on the arguments: same n_global / policy / flags / max_rounds, ranges tiling [0, n)
  struct Hello {
    int32_t status;
    uint32_t policy, flags, max_rounds;
    int64_t n_global, v_begin, v_end;
  } me{(int32_t)local, o.policy, o.flags & ~(uint32_t)(GC_FLAG_TRACE | GC_FLAG_COUNT_WORK), o.max_rounds, n_global,
       v_begin, v_end},
      all[MAX_RANKS];
  gc_status st = boot_allgather(c, &me, sizeof(me), all);
  if (st != GC_OK) { c->broken = true; return st; }
  for (int q = 0; q < c->world; ++q)
    if (all[q].status != GC_OK) {
      if (local == GC_OK) set_err("gc_color_dist: rank %d rejected its arguments", q);
      return GC_ERR_INVALID_ARGUMENT;
    }
  for (int q = 0; q < c->world; ++q) {
    const Hello& h = all[q];
    const bool tiles = h.v_begin == (q == 0 ? 0 : all[q - 1].v_end) && (q + 1 < c->world || h.v_end == n_global);
    if (h.n_global != n_global || h.policy != o.policy || h.flags != me.flags || h.max_rounds != o.max_rounds || !tiles) {
      set_err("gc_color_dist: ranks disagree (rank %d: n=%lld [%lld, %lld) policy %u flags %u max_rounds %u); "
              "ranges must tile [0, n) in rank order",
              q, (long long)h.n_global, (long long)h.v_begin, (long long)h.v_end, h.policy, h.flags, h.max_rounds);
      return GC_ERR_INVALID_ARGUMENT;
    }
  }
  if (n_global == 0) return GC_OK;

  // ---- window (replicas), mapped by every rank
  const WinLayout L = win_layout(n_global);
  if ((st = ensure_window(c, L.total)) != GC_OK) return st;

  // ---- private workspace and inputs
  // inputs
  const bool rp_dev = nl == 0 || is_device_ptr(row_ptr_local) == 1;
  const bool ci_dev = nl == 0 || is_device_ptr(col_idx_local) == 1;
  const bool out_dev = nl == 0 || is_device_ptr(colors_out_local) == 1;
  const int64_t* d_rp = row_ptr_local;
  const int32_t* d_ci = col_idx_local;
  int64_t m = 0;
  void *w0 = nullptr, *w1 = nullptr, *heavy = nullptr, *dcol = colors_out_local, *dtrace = nullptr, *dinfo_bad = nullptr;
  const uint32_t t3 = o.warp_bin_max ? o.warp_bin_max : 1024;
  const bool cw = (o.flags & GC_FLAG_COUNT_WORK) != 0;
  const bool trace = (o.flags & GC_FLAG_TRACE) && o.trace_capacity;
  const bool trace_dev = trace && is_device_ptr(o.trace_worklist) == 1;
  auto prepare = [&]() -> gc_status {
    if (nl > 0) {
      if (!rp_dev) {
        m = row_ptr_local[nl];
        void* p;
        CK(sc.alloc(&p, sizeof(int64_t) * (size_t)(nl + 1)));
        CK(cudaMemcpyAsync(p, row_ptr_local, sizeof(int64_t) * (size_t)(nl + 1), cudaMemcpyHostToDevice, s));
        d_rp = (const int64_t*)p;
      } else {
        CK(cudaMemcpyAsync(&m, d_rp + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
      }
      if (m < 0) {
        set_err("gc_color_dist: row_ptr_local[n_local]=%lld < 0", (long long)m);
        return GC_ERR_INVALID_GRAPH;
      }
      if (!ci_dev) {
        void* p;
        CK(sc.alloc(&p, sizeof(int32_t) * (size_t)(m ? m : 1)));
        if (m) CK(cudaMemcpyAsync(p, col_idx_local, sizeof(int32_t) * (size_t)m, cudaMemcpyHostToDevice, s));
        d_ci = (const int32_t*)p;
      }
    }
    const int64_t nla = nl ? nl : 1;
    const int64_t hcap = m / ((int64_t)t3 + 1) + 1;
    CK(sc.alloc(&w0, sizeof(WE) * (size_t)nla));
    CK(sc.alloc(&w1, sizeof(WE) * (size_t)nla));
    CK(sc.alloc(&heavy, sizeof(WE) * (size_t)(hcap < nla ? hcap : nla)));
    if (!out_dev) CK(sc.alloc(&dcol, sizeof(uint32_t) * (size_t)nla));
    if (trace && !trace_dev) CK(sc.alloc(&dtrace, sizeof(uint32_t) * o.trace_capacity));
    if (trace_dev) dtrace = o.trace_worklist;
    if (o.flags & GC_FLAG_VALIDATE) {
      CK(sc.alloc(&dinfo_bad, sizeof(DevInfo)));
      CK(cudaMemsetAsync(dinfo_bad, 0, sizeof(DevInfo), s));
      if (nl > 0) {
        DevFacts f;
        CK(dev_facts(c->dev, &f));
        k_validate<<<f.sms * 8, BLOCK, 0, s>>>((int32_t)nl, v_begin, n_global, d_rp, d_ci, 0, (DevInfo*)dinfo_bad);
        CK(cudaGetLastError());
      }
      unsigned long long bad = 0;
      CK(cudaMemcpyAsync(&bad, &((DevInfo*)dinfo_bad)->bad, sizeof(bad), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (bad) {
        bad = ~bad;
        set_err("gc_color_dist: invalid graph at vertex %llu: %s", bad >> 3, val_err_name((uint32_t)(bad & 7)));
        return GC_ERR_INVALID_GRAPH;
      }
    }
    return GC_OK;
  };
  if ((st = agree(c, prepare())) != GC_OK) return st;

  // ---- kernel parameters
  Params p;
  memset(&p, 0, sizeof(p));
  p.n = (int32_t)nl;
  p.v_base = (int32_t)v_begin;
  p.rp = d_rp;
  p.ci = d_ci;
  p.plane = L.pitch;
  p.np = L.np;
  p.fmp = c->win + L.planes;
  p.dirty = kn.n1 ? c->win + L.dirty : nullptr;
  p.ksplit = (int32_t*)(c->win + L.ksplit);
  p.heavy = (WE*)heavy;
  p.wl0 = (WE*)w0;
  p.wl1 = (WE*)w1;
  p.info = (DevInfo*)(c->win + L.info);
  p.trace = (uint32_t*)dtrace;
  p.trace_cap = trace ? o.trace_capacity : 0;
  p.colors_out = (uint32_t*)dcol;
  p.max_rounds = o.max_rounds ? o.max_rounds : (uint32_t)((uint64_t)n_global + 1 > 0xffffffffu ? 0xffffffffu : n_global + 1);
  p.t1 = o.thread_bin_max ? o.thread_bin_max : 16;
  p.t3 = t3;
  p.dense_div = kn.dense_div ? kn.dense_div : 3;  // the dense ingest (splits, degrees) is required
  p.dense_div_n1 = kn.dense_div_n1;
  p.dch = kn.dch;
  p.compact = kn.compact;
  p.n1 = kn.n1;
  p.n1chg = 0;       // a per-rank cost rule would make ranks mark differently: off
  p.list_ok = 0;     // list rounds are single-GPU only
  p.sfilter = 0;
  p.davg2 = nl > 0 && m > 0 ? (uint32_t)((m + 2 * nl - 1) / (2 * nl)) + 1u : 1u;
  p.timeout_ns = 60ull * 1000000000ull;
  p.nranks = c->world;
  p.rank = c->rank;
  p.n_global = (int32_t)n_global;
  p.bmask = c->win + L.bmask;
  for (int q = 0; q <= MAX_RANKS; ++q) p.rb[q] = q < c->world ? (int32_t)all[q].v_begin : INT32_MAX;
  Peer peers[MAX_RANKS];
  memset(peers, 0, sizeof(peers));
  for (int q = 0; q < c->world; ++q) {
    uint8_t* b = c->peer[q];
    peers[q].st = b + L.st;
    peers[q].fmp = b + L.planes;
    peers[q].dirty = b + L.dirty;
    peers[q].ksplit = (int32_t*)(b + L.ksplit);
    peers[q].info = (DevInfo*)(b + L.info);
    peers[q].xflag = (uint32_t*)(b + L.xflag);
  }
  p.peer = (const Peer*)(c->win + L.peers);
  if (kn.watchdog_ms) p.timeout_ns = (unsigned long long)kn.watchdog_ms * 1000000ull;
  {
    cudaError_t e = cudaMemcpyAsync(c->win + L.peers, peers, sizeof(peers), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return agree(c, cuda_fail(e, "peer table"));
  }

  // ---- launches: 8-bit state words first, wider on a (globally agreed) restart status
  DevFacts f;
  {
    cudaError_t e = dev_facts(c->dev, &f);
    if (e != cudaSuccess) return agree(c, cuda_fail(e, "dev_facts"));
  }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  struct EvGuard {
    cudaEvent_t* a;
    cudaEvent_t* b;
    ~EvGuard() { if (*a) cudaEventDestroy(*a); if (*b) cudaEventDestroy(*b); }
  } evg{&ev0, &ev1};
  int sbytes = kn.state_bytes, sbytes_used = sbytes, grid_used = 0;
  DevInfo hinfo;
  for (int attempt = 0; attempt < 3; ++attempt) {
    void* fn = pick_persistent_dist(sbytes, (int)o.policy, cw, kn.variant == 1);
    int per_sm = 0;
    auto prepare_launch = [&]() -> gc_status {
      // module loading of the instance, occupancy and events while no kernel runs; then this
      // rank's DevInfo is zeroed (before any rank's kernel can write into it: agreed below)
      cudaFuncAttributes fa;
      CK(cudaFuncGetAttributes(&fa, fn));
      CK(occupancy(c->dev, fn, &per_sm));
      if (o.kernel_ms && !ev0) {
        CK(cudaEventCreate(&ev0));
        CK(cudaEventCreate(&ev1));
      }
      CK(cudaMemsetAsync(p.info, 0, sizeof(DevInfo), s));
      CK(cudaStreamSynchronize(s));
      return GC_OK;
    };
    if ((st = agree(c, prepare_launch())) != GC_OK) return st;
    if (o.blocks_per_sm && (int)o.blocks_per_sm < per_sm) per_sm = (int)o.blocks_per_sm;
    // One launch per GPU.  Emulated ranks (one GPU) share ONE cooperative launch of
    // world x G CTAs, rank q taking CTAs [qG, (q+1)G): co-resident by construction.  (Separate
    // concurrent cooperative launches per rank were measured on B200 to leave some CTAs of a
    // rank's grid unscheduled while the other ranks' CTAs spin: a deadlock.)
    const int ranks_in_launch = c->lg ? c->world : 1;
    const int G = (f.sms * per_sm) / ranks_in_launch;
    grid_used = G;
    p.st = c->win + L.st;
    p.epoch_base = c->epoch;
    p.G = G;
    p.blk0 = c->lg ? c->rank * G : 0;
    p.nranks_in_launch = ranks_in_launch;
    cudaError_t e = cudaSuccess;
    if (c->lg) c->lg->params[c->rank] = p;
    if ((st = agree(c, GC_OK)) != GC_OK) return st;  // every rank's Params are in place
    if (!c->lg || c->rank == 0) {
      const Params* src = c->lg ? c->lg->params.data() : &p;
      e = cudaMemcpyAsync(c->dparams, src, sizeof(Params) * ranks_in_launch, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess && ev0 && attempt == 0) e = cudaEventRecord(ev0, s);
      const Params* dpp = (const Params*)c->dparams;
      void* args[] = {&dpp};
      if (e == cudaSuccess) e = cudaLaunchCooperativeKernel(fn, dim3(G * ranks_in_launch), dim3(BLOCK), args, 0, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) {
        c->broken = true;  // the other ranks may be waiting in a barrier of this launch
        cuda_fail(e, "gc_color_dist: persistent kernel");
      }
    }
    if (c->lg) {  // the emulated ranks learn that the shared launch ended (or failed)
      gc_status launched = e == cudaSuccess ? GC_OK : GC_ERR_CUDA;
      if ((st = agree(c, launched)) != GC_OK) {
        c->broken = true;
        return st;
      }
    } else if (e != cudaSuccess) {
      return GC_ERR_CUDA;
    }
    e = cudaMemcpyAsync(c->hinfo, p.info, sizeof(DevInfo), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      c->broken = true;
      return cuda_fail(e, "gc_color_dist: read-back");
    }
    memcpy(&hinfo, c->hinfo, sizeof(DevInfo));
    c->epoch += hinfo.bar_gen;  // every rank passed the same barriers
    sbytes_used = sbytes;
    if (hinfo.status == ST_NEED16 && sbytes < 2) sbytes = 2;
    else if (hinfo.status == ST_NEED32 && sbytes < 4) sbytes = 4;
    else break;
  }
  if (ev1) {  // (emulated ranks other than 0 launched nothing: they report rank 0's time)
    if (!c->lg || c->rank == 0) {
      cudaEventRecord(ev1, s);
      cudaEventSynchronize(ev1);
      cudaEventElapsedTime(o.kernel_ms, ev0, ev1);
      if (c->lg) c->lg->kernel_ms = *o.kernel_ms;
    }
    if (c->lg) {
      agree(c, GC_OK);
      *o.kernel_ms = c->lg->kernel_ms;
    }
  }
  if (hinfo.status == ST_WATCHDOG) {
    c->broken = true;
    {
      char buf[512];
      int o = 0;
      for (int b = 0; b < grid_used && b < 1024 && o < 400; ++b)
        if ((hinfo.stage[b] >> 20) != 1u || b == 0)
          o += snprintf(buf + o, sizeof(buf) - o, " cta%d:%x", b, hinfo.stage[b]);
      fprintf(stderr, "gc_color_dist watchdog rank %d stages:%s\n", c->rank, buf);
    }
    set_err("gc_color_dist: device watchdog fired (cross-rank barrier timeout; rank %d: waiting for rank %d "
            "at epoch %u, %u of %d local CTAs arrived, %u started; status word %u)", c->rank, (int)hinfo.diag[0] - 1,
            hinfo.diag[1], hinfo.diag[2], (int)grid_used, hinfo.diag[3], hinfo.status);
    return GC_ERR_CUDA;
  }
  if (hinfo.status == ST_NO_CONVERGENCE) {
    set_err("gc_color_dist: no convergence within max_rounds=%u", p.max_rounds);
    return GC_ERR_NO_CONVERGENCE;
  }
  {
    cudaError_t e = cudaSuccess;
    if (!out_dev && nl > 0)
      e = cudaMemcpyAsync(colors_out_local, dcol, sizeof(uint32_t) * (size_t)nl, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && trace && !trace_dev) {
      const uint32_t k = hinfo.rounds < o.trace_capacity ? hinfo.rounds : o.trace_capacity;
      if (k) e = cudaMemcpyAsync(o.trace_worklist, dtrace, sizeof(uint32_t) * k, cudaMemcpyDeviceToHost, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "gc_color_dist: outputs");
  }
  if (cw) {
    memset(o.work, 0, sizeof(gc_work));
    o.work->phase_a_vertices = hinfo.work[W_A_VERT];
    o.work->phase_a_edges = hinfo.work[W_A_EDGE];
    o.work->phase_b_vertices = hinfo.work[W_B_VERT];
    o.work->phase_b_edges = hinfo.work[W_B_EDGE];
    o.work->phase_b_gathers = hinfo.work[W_B_GATHER];
    o.work->commit_scatter = hinfo.work[W_SCATTER];
    o.work->pushes = hinfo.work[W_PUSH];
    o.work->scatter_reds = hinfo.work[W_SCATTER_RED];
    o.work->dense_a_swept = hinfo.work[W_DA_SWEEP];
    o.work->dense_b_swept = hinfo.work[W_DB_SWEEP];
    o.work->sparse_a_entries = hinfo.work[W_SA_ENT];
    o.work->sparse_b_entries = hinfo.work[W_SB_ENT];
    o.work->state_bytes = (uint64_t)sbytes_used;
    o.work->phase_b_evaluated = hinfo.work[W_B_EVAL];
    o.work->dense_b_evaluated = hinfo.work[W_DB_EVAL];
    o.work->dirty_marks = hinfo.work[W_MARK];
    o.work->tent_changes = hinfo.work[W_TCHG];
    o.work->pending_degree_sum = hinfo.work[W_WDEG];
  }
  *num_colors = hinfo.num_colors;
  *rounds = hinfo.rounds;
  return GC_OK;
}

}  // extern "C"
