// gc_api.cu — host side of the C ABI declared in include/gc.h.
// Argument checking, pointer-space detection, workspace from a per-device stream-ordered
// memory pool, one cooperative launch of the persistent SGR kernel, one stream sync.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <mutex>

#include "../../include/gc.h"
#include "../../include/gc_internal.h"
#include "sgr_kernels.cuh"
#include "sgr_inst.h"

using namespace gcdev;

namespace {

thread_local char g_err[1024] = "";

void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

constexpr int kMaxDev = 64;
std::mutex g_pool_mu;
cudaMemPool_t g_pool[kMaxDev] = {};

gc_status cuda_fail(cudaError_t e, const char* what) {
  set_err("%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? GC_ERR_OUT_OF_MEMORY : GC_ERR_CUDA;
}

#define CK(call)                                      \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

cudaError_t get_pool(int dev, cudaMemPool_t* out) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  if (!g_pool[dev]) {
    cudaMemPoolProps props;
    memset(&props, 0, sizeof(props));
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    cudaError_t e = cudaMemPoolCreate(&pool, &props);
    if (e != cudaSuccess) return e;
    uint64_t thr = UINT64_MAX;  // keep freed blocks cached across calls
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    g_pool[dev] = pool;
  }
  *out = g_pool[dev];
  return cudaSuccess;
}

// Per-device facts queried once (cudaGetDeviceProperties costs ~ms; attributes are cheap).
struct DevFacts {
  bool ready = false;
  int sms = 0, major = 0, minor = 0, coop = 0;
};
DevFacts g_facts[kMaxDev];

cudaError_t dev_facts(int dev, DevFacts* f) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  DevFacts& d = g_facts[dev];
  if (!d.ready) {
    cudaError_t e;
    if ((e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&d.coop, cudaDevAttrCooperativeLaunch, dev)) != cudaSuccess) return e;
    d.ready = true;
  }
  *f = d;
  return cudaSuccess;
}

// Max co-resident CTAs per SM of a kernel, cached per (device, kernel).
struct OccEntry { int dev; const void* fn; int per_sm; };
OccEntry g_occ[256];
int g_nocc = 0;

cudaError_t occupancy(int dev, const void* fn, int* per_sm) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (int i = 0; i < g_nocc; ++i)
    if (g_occ[i].dev == dev && g_occ[i].fn == fn) { *per_sm = g_occ[i].per_sm; return cudaSuccess; }
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, fn, BLOCK, 0);
  if (e == cudaSuccess && g_nocc < 256) g_occ[g_nocc++] = OccEntry{dev, fn, *per_sm};
  return e;
}

// Restores the caller's current device; frees pool allocations stream-ordered; owns an
// internal stream when the caller passed none.
struct Scope {
  static constexpr int kMaxPtr = 32;
  int prev_dev = -1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaMemPool_t pool = nullptr;
  void* ptrs[kMaxPtr];
  int nptr = 0;
  ~Scope() {
    for (int i = 0; i < nptr; ++i) cudaFreeAsync(ptrs[i], stream);
    if (stream) cudaStreamSynchronize(stream);
    if (own_stream) cudaStreamDestroy(stream);
    if (prev_dev >= 0) cudaSetDevice(prev_dev);
  }
  cudaError_t alloc(void** p, size_t bytes) {
    if (nptr >= kMaxPtr) return cudaErrorMemoryAllocation;  // bounded: never overflow ptrs[]
    if (bytes == 0) bytes = 16;
#ifdef GC_DEFAULT_POOL
    cudaError_t e = cudaMallocAsync(p, bytes, stream);
#else
    cudaError_t e = cudaMallocFromPoolAsync(p, bytes, pool, stream);
#endif
    if (e == cudaSuccess) ptrs[nptr++] = *p;
    return e;
  }
};

// A library-internal stream that starts after everything already queued on the legacy default
// stream (where callers such as torch produce row_ptr / col_idx) without the reverse implicit
// dependency a blocking stream would add: the stream is non-blocking and waits on an event
// recorded on the legacy stream.  (With blocking streams, the emulated ranks of gc_dist.h
// deadlock as soon as any thread queues work on the legacy stream: that work waits for the
// ranks' spinning kernels, and the next rank's kernel waits for it.)
cudaError_t after_legacy(cudaStream_t s);
cudaError_t internal_stream(cudaStream_t* s) {
  cudaError_t e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  return after_legacy(*s);
}
cudaError_t after_legacy(cudaStream_t s) {
  cudaEvent_t ev;
  cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e != cudaSuccess) return e;
  e = cudaEventRecord(ev, cudaStreamLegacy);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev, 0);
  cudaEventDestroy(ev);
  return e;
}

// 1 = device (or managed) memory usable by kernels, 0 = host memory, -1 = error
int is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? 1 : 0;
}

// The persistent kernel instances live in their own translation units (inst_*.cu, compiled
// in parallel); each returns the host stub of the requested instance.
void* pick_persistent(int sbytes, int pol, bool push, bool cw, bool fat = false) {
  if (fat && sbytes == 1 && push) return gc_inst_fat(pol, cw);
  if (sbytes == 1) return gc_inst_u8(pol, push, cw);
  if (sbytes == 2) return gc_inst_u16(pol, push, cw);
  return gc_inst_u32(pol, push, cw);
}
// multi-GPU instances (push First-Fit only), compiled with the cross-rank code
void* pick_persistent_dist(int sbytes, int pol, bool cw, bool fat) {
  if (fat && sbytes == 1) return gc_inst_dist_fat(pol, cw);
  if (sbytes == 1) return gc_inst_dist_u8(pol, cw);
  if (sbytes == 2) return gc_inst_dist_u16(pol, cw);
  return gc_inst_dist_u32(pol, cw);
}

template <int POL, bool PUSH, bool CW>
void launch_phase_b(int grid, cudaStream_t s, const Params& p, uint32_t r, WE* W, WE* Wo) {
  k_phase_b<POL, PUSH, CW><<<grid, BLOCK, 0, s>>>(p, r, W, Wo);
}
template <bool PUSH, bool CW>
void launch_phase_a(int grid, cudaStream_t s, const Params& p, uint32_t r, WE* W) {
  k_phase_a<PUSH, CW><<<grid, BLOCK, 0, s>>>(p, r, W);
}

void launch_b(int pol, bool push, bool cw, int grid, cudaStream_t s, const Params& p, uint32_t r, WE* W, WE* Wo) {
#define LB(P)                                                                   \
  if (pol == P) {                                                               \
    if (push) { if (cw) launch_phase_b<P, true, true>(grid, s, p, r, W, Wo); else launch_phase_b<P, true, false>(grid, s, p, r, W, Wo); } \
    else { if (cw) launch_phase_b<P, false, true>(grid, s, p, r, W, Wo); else launch_phase_b<P, false, false>(grid, s, p, r, W, Wo); } \
    return;                                                                     \
  }
  LB(HIGHER_ID) LB(LOWER_ID) LB(DEGREE)
#undef LB
}

// Schedule knobs (include/gc.h gc_tuning), resolved to the measured defaults.
struct Knobs {
  int state_bytes = 1;  // first attempt's state-word width
  uint32_t dense_div = 3, dense_div_n1 = 32, n1 = 1, list = 0, compact = 0, sfilter = 0, dch = 16, n1_chg = 0;
  int variant = -1;
  uint32_t watchdog_ms = 0;  // 0 = 60 s
  uint32_t widen = 1;        // 8-bit overflow: widen in place and resume (1) or restart (0)
};
bool resolve_knobs(const gc_tuning* t, Knobs* k) {
  *k = Knobs();
  if (!t) return true;
  if (t->struct_size != sizeof(gc_tuning)) return false;
  if (t->state_bytes == 2 || t->state_bytes == 4) k->state_bytes = t->state_bytes;
  else if (t->state_bytes != 0 && t->state_bytes != 1) return false;
  if (t->dense_div >= 0) k->dense_div = k->dense_div_n1 = (uint32_t)t->dense_div;
  if (t->dense_div_n1 >= 0) k->dense_div_n1 = (uint32_t)t->dense_div_n1;
  if (t->n1 >= 0) k->n1 = (uint32_t)t->n1;
  if (t->list >= 0) k->list = (uint32_t)t->list;
  if (t->compact >= 0) k->compact = (uint32_t)t->compact;
  if (t->scatter_filter >= 0) k->sfilter = (uint32_t)t->scatter_filter;
  if (t->dch > 0) k->dch = (uint32_t)t->dch;
  if (t->n1_chg >= 0) k->n1_chg = (uint32_t)t->n1_chg;
  k->variant = t->variant < 0 ? -1 : (t->variant ? 1 : 0);
  if (t->watchdog_ms > 0) k->watchdog_ms = (uint32_t)t->watchdog_ms;
  if (t->widen >= 0) k->widen = t->widen ? 1u : 0u;
  return true;
}

// Kernel-variant hints per graph (device, row_ptr address, n, m), a small direct-mapped cache.
struct HintEntry { int dev; const void* rp; int64_t n, m; int variant; };
HintEntry g_hint[64];
int variant_hint(int dev, const void* rp, int64_t n, int64_t m) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  const HintEntry& h = g_hint[((uintptr_t)rp >> 8 ^ (uint64_t)n) % 64];
  return (h.rp == rp && h.dev == dev && h.n == n && h.m == m) ? h.variant : -1;
}
void set_variant_hint(int dev, const void* rp, int64_t n, int64_t m, int variant) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_hint[((uintptr_t)rp >> 8 ^ (uint64_t)n) % 64] = HintEntry{dev, rp, n, m, variant};
}

const char* val_err_name(uint32_t code) {
  switch (code) {
    case VE_ROWPTR: return "row_ptr[0] != 0 or row_ptr decreasing";
    case VE_RANGE: return "col_idx entry out of range [0, n)";
    case VE_SELF: return "self loop";
    case VE_ORDER: return "row not strictly increasing (unsorted or duplicate entry)";
    case VE_ASYM: return "asymmetric edge (w in adj(v) but v not in adj(w))";
    default: return "invalid graph";
  }
}

}  // namespace

extern "C" {

int32_t gc_abi_version(void) { return GC_ABI_VERSION; }

void gc_tuning_default(gc_tuning* t) {
  if (!t) return;
  memset(t, 0, sizeof(*t));
  t->struct_size = sizeof(gc_tuning);
  t->state_bytes = 0;
  t->dense_div = t->dense_div_n1 = t->n1 = t->list = t->compact = t->scatter_filter = t->dch = t->n1_chg = -1;
  t->variant = -1;
  t->widen = -1;
}

void gc_opts_default(gc_opts* o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(gc_opts);
  o->policy = GC_POLICY_HIGHER_ID;
  o->flags = GC_FLAG_VALIDATE;
  o->max_rounds = 0;
  o->device = -1;
}

const char* gc_status_string(gc_status s) {
  switch (s) {
    case GC_OK: return "GC_OK";
    case GC_ERR_INVALID_ARGUMENT: return "GC_ERR_INVALID_ARGUMENT";
    case GC_ERR_INVALID_GRAPH: return "GC_ERR_INVALID_GRAPH";
    case GC_ERR_NO_CONVERGENCE: return "GC_ERR_NO_CONVERGENCE";
    case GC_ERR_OUT_OF_MEMORY: return "GC_ERR_OUT_OF_MEMORY";
    case GC_ERR_CUDA: return "GC_ERR_CUDA";
    case GC_ERR_NCCL: return "GC_ERR_NCCL";
    case GC_ERR_UNSUPPORTED: return "GC_ERR_UNSUPPORTED";
  }
  return "GC_ERR_UNKNOWN";
}

const char* gc_last_error_message(void) { return g_err; }

gc_status gc_partition_edge_balanced(int64_t n, const int64_t* row_ptr, int32_t parts, int64_t* bounds) {
  if (n < 0 || parts < 1 || !bounds || (n > 0 && !row_ptr)) {
    set_err("gc_partition_edge_balanced: invalid argument");
    return GC_ERR_INVALID_ARGUMENT;
  }
  const int64_t m = n > 0 ? row_ptr[n] : 0;
  bounds[0] = 0;
  for (int32_t k = 1; k < parts; ++k) {
    // target = ceil(k*m/parts) without overflow for m < 2^62
    const __int128 num = (__int128)k * m;
    const int64_t target = (int64_t)((num + parts - 1) / parts);
    int64_t lo = 0, hi = n;  // smallest v with row_ptr[v] >= target
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (row_ptr[mid] >= target) hi = mid; else lo = mid + 1;
    }
    bounds[k] = lo < bounds[k - 1] ? bounds[k - 1] : lo;
  }
  bounds[parts] = n;
  return GC_OK;
}

gc_status gc_color(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const gc_opts* opts_in,
                   uint32_t* colors_out, uint32_t* num_colors, uint32_t* rounds) {
  g_err[0] = 0;
  if (!num_colors || !rounds) {
    set_err("gc_color: num_colors and rounds must not be NULL");
    return GC_ERR_INVALID_ARGUMENT;
  }
  *num_colors = 0;
  *rounds = 0;
  gc_opts o;
  gc_opts_default(&o);
  if (opts_in) {
    if (opts_in->struct_size != sizeof(gc_opts)) {
      set_err("gc_color: opts->struct_size=%u, expected %zu", opts_in->struct_size, sizeof(gc_opts));
      return GC_ERR_INVALID_ARGUMENT;
    }
    o = *opts_in;
  }
  if (o.policy > GC_POLICY_DEGREE) {
    set_err("gc_color: unknown policy %u", o.policy);
    return GC_ERR_INVALID_ARGUMENT;
  }
  if (n < 0 || n > INT32_MAX) {
    set_err("gc_color: n=%lld out of range [0, 2^31-1]", (long long)n);
    return GC_ERR_INVALID_ARGUMENT;
  }
  if (n == 0) return GC_OK;
  if (!row_ptr || !col_idx || !colors_out) {
    set_err("gc_color: NULL row_ptr/col_idx/colors_out with n=%lld", (long long)n);
    return GC_ERR_INVALID_ARGUMENT;
  }
  if ((o.flags & GC_FLAG_TRACE) && o.trace_capacity && !o.trace_worklist) {
    set_err("gc_color: GC_FLAG_TRACE with NULL trace_worklist");
    return GC_ERR_INVALID_ARGUMENT;
  }
  if ((o.flags & GC_FLAG_COUNT_WORK) && !o.work) {
    set_err("gc_color: GC_FLAG_COUNT_WORK with NULL work");
    return GC_ERR_INVALID_ARGUMENT;
  }
  Knobs kn;
  if (!resolve_knobs(o.tuning, &kn)) {
    set_err("gc_color: bad opts->tuning (struct_size or state_bytes)");
    return GC_ERR_INVALID_ARGUMENT;
  }

  Scope sc;
  CK(cudaGetDevice(&sc.prev_dev));
  const int dev = o.device >= 0 ? o.device : sc.prev_dev;
  CK(cudaSetDevice(dev));
  DevFacts prop;
  CK(dev_facts(dev, &prop));
  if (prop.major != 10) {
    set_err("gc_color: device %d is sm_%d%d; this library is built for sm_100a", dev, prop.major, prop.minor);
    return GC_ERR_UNSUPPORTED;
  }
  if (o.stream) {
    sc.stream = (cudaStream_t)o.stream;
  } else {
    // ordered after the legacy default stream, where the caller's producers of row_ptr /
    // col_idx may still be running
    CK(internal_stream(&sc.stream));
    sc.own_stream = true;
  }
  CK(get_pool(dev, &sc.pool));
  cudaStream_t s = sc.stream;

  // ---- inputs in device memory
  const bool rp_dev = is_device_ptr(row_ptr) == 1;
  const bool ci_dev = is_device_ptr(col_idx) == 1;
  const bool out_dev = is_device_ptr(colors_out) == 1;
  const int64_t* d_rp = row_ptr;
  const int32_t* d_ci = col_idx;
  int64_t m = -1;
  if (!rp_dev) {
    m = row_ptr[n];
    void* p;
    CK(sc.alloc(&p, sizeof(int64_t) * (size_t)(n + 1)));
    CK(cudaMemcpyAsync(p, row_ptr, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyHostToDevice, s));
    d_rp = (const int64_t*)p;
  }
  if (!ci_dev) {
    if (m < 0) {
      CK(cudaMemcpyAsync(&m, d_rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    if (m < 0) {
      set_err("gc_color: row_ptr[n]=%lld < 0", (long long)m);
      return GC_ERR_INVALID_GRAPH;
    }
    void* p;
    CK(sc.alloc(&p, sizeof(int32_t) * (size_t)m));
    if (m) CK(cudaMemcpyAsync(p, col_idx, sizeof(int32_t) * (size_t)m, cudaMemcpyHostToDevice, s));
    d_ci = (const int32_t*)p;
  }

  // ---- workspace
  const bool push = !(o.flags & GC_FLAG_PULL_FIRSTFIT);
  const bool cw = (o.flags & GC_FLAG_COUNT_WORK) != 0;
  void *w0, *w1, *info, *dcol = colors_out, *dtrace = nullptr;
  uint8_t* planes = nullptr;
  // [st | plane 0 | plane 1 | ...] in one allocation: the state words (1, 2 or 4 bytes per
  // vertex, placed right before plane 0 whatever their width) and the forbidden-colour planes.
  const int64_t pitch = (n + 255) / 256 * 256;
  // up to MAX_PLANES planes (colours 1..512), at most ~16 GB of them; only the planes a run
  // reaches are ever touched (plane k from round 8k on)
  uint32_t np = push ? (uint32_t)MAX_PLANES : 0u;
  if (push && (uint64_t)np * (uint64_t)pitch > (16ull << 30)) {
    const uint64_t fit = (16ull << 30) / (uint64_t)pitch;
    np = fit < 16 ? 16u : (uint32_t)fit;
  }
  void* hot;
  CK(sc.alloc(&hot, (size_t)pitch * (4 + np)));
  planes = (uint8_t*)hot + 4 * pitch;
  // dense rounds (push mode, persistent driver): per-vertex split + static heavy-vertex list
  uint32_t dense_div = kn.dense_div;  // sweep on R-MAT s24 (2, 3, 4, 6 -> 3; dirty-set graphs use dense_div_n1)
  if (!push || (o.flags & GC_FLAG_HOST_ROUNDS)) dense_div = 0;
  const uint32_t t3 = o.warp_bin_max ? o.warp_bin_max : 1024;
  void *ksplit = nullptr, *heavy = nullptr, *dirty = nullptr, *wlw0 = nullptr, *wlw1 = nullptr, *dlist = nullptr;
  uint32_t list_ok = kn.list;  // list rounds (0 off (default: slower on every config measured),
                               // 1 cost rule, 2 from round 3 on)
  // dirty-set rounds: needs the per-vertex splits of the dense ingest
  uint32_t n1 = kn.n1;
  if (!dense_div) n1 = 0;
  if (dense_div) {
    if (m < 0) {
      CK(cudaMemcpyAsync(&m, d_rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    const int64_t hcap = m / ((int64_t)t3 + 1) + 1;  // vertices of degree > t3
    CK(sc.alloc(&ksplit, sizeof(int32_t) * (size_t)n));
    if (n1) CK(sc.alloc(&dirty, (size_t)pitch));
    if (n1 && list_ok) {
      CK(sc.alloc(&wlw0, sizeof(int32_t) * (size_t)n));
      CK(sc.alloc(&wlw1, sizeof(int32_t) * (size_t)n));
      CK(sc.alloc(&dlist, sizeof(int32_t) * (size_t)n));
    }
    CK(sc.alloc(&heavy, sizeof(WE) * (size_t)(hcap < n ? hcap : n)));
  }
  CK(sc.alloc(&w0, sizeof(WE) * (size_t)n));
  CK(sc.alloc(&w1, sizeof(WE) * (size_t)n));
  CK(sc.alloc(&info, sizeof(DevInfo)));
  CK(cudaMemsetAsync(info, 0, sizeof(DevInfo), s));
  if (!out_dev) CK(sc.alloc(&dcol, sizeof(uint32_t) * (size_t)n));
  const bool trace = (o.flags & GC_FLAG_TRACE) && o.trace_capacity;
  const bool trace_dev = trace && is_device_ptr(o.trace_worklist) == 1;
  if (trace) {
    if (trace_dev) dtrace = o.trace_worklist;
    else CK(sc.alloc(&dtrace, sizeof(uint32_t) * o.trace_capacity));
  }

  // ---- optional validation (C9): one warp per vertex
  if (o.flags & (GC_FLAG_VALIDATE | GC_FLAG_VALIDATE_SYMMETRY)) {
    const int vgrid = prop.sms * 8;
    k_validate<<<vgrid, BLOCK, 0, s>>>((int32_t)n, 0, n, d_rp, d_ci, (o.flags & GC_FLAG_VALIDATE_SYMMETRY) ? 1 : 0,
                                       (DevInfo*)info);
    CK(cudaGetLastError());
    unsigned long long bad = 0;
    CK(cudaMemcpyAsync(&bad, &((DevInfo*)info)->bad, sizeof(bad), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (bad) {
      bad = ~bad;
      set_err("gc_color: invalid graph at vertex %llu: %s", bad >> 3, val_err_name((uint32_t)(bad & 7)));
      return GC_ERR_INVALID_GRAPH;
    }
  }

  Params p;
  memset(&p, 0, sizeof(p));
  p.n = (int32_t)n;
  p.rp = d_rp;
  p.ci = d_ci;
  p.st = (uint8_t*)planes - 4 * pitch;
  p.fmp = push ? planes : nullptr;
  p.plane = pitch;
  p.np = np;
  p.sfilter = kn.sfilter;
  p.wl0 = (WE*)w0;
  p.wl1 = (WE*)w1;
  p.info = (DevInfo*)info;
  p.trace = (uint32_t*)dtrace;
  p.trace_cap = trace ? o.trace_capacity : 0;
  void* dphase = nullptr;
  if (trace && o.phase_ns) {
    CK(sc.alloc(&dphase, sizeof(uint64_t) * (4 * (size_t)o.trace_capacity + 1)));
    CK(cudaMemsetAsync(dphase, 0, sizeof(uint64_t) * (4 * (size_t)o.trace_capacity + 1), s));
    p.phase_ns = (unsigned long long*)dphase;
  }
  p.colors_out = (uint32_t*)dcol;
  p.max_rounds = o.max_rounds ? o.max_rounds : (uint32_t)((uint64_t)n + 1 > 0xffffffffu ? 0xffffffffu : n + 1);
  p.t1 = o.thread_bin_max ? o.thread_bin_max : 16;
  p.t3 = t3;   // sweep on R-MAT s24: 128/256/512/768/1024/1536/2048 -> 1024 best
  p.dense_div = dense_div;
  p.compact = kn.compact;
  p.dch = kn.dch;            // sweep 2..32 on the three configs: 16 (R-MAT s24 -1 %)
  p.n1chg = kn.n1_chg;
  p.dense_div_n1 = kn.dense_div_n1;  // sweep with dirty-set rounds (stencil, mesh): 4..256 -> 16 (round 1), 32 (round 2)
  p.ksplit = (int32_t*)ksplit;
  p.dirty = (uint8_t*)dirty;
  p.wlw0 = (int32_t*)wlw0;
  p.wlw1 = (int32_t*)wlw1;
  p.dl = (int32_t*)dlist;
  p.list_ok = dlist ? list_ok : 0u;
  p.n1 = dirty ? n1 : 0u;
  p.davg2 = n > 0 && m > 0 ? (uint32_t)((m + 2 * n - 1) / (2 * n)) + 1u : 1u;  // successors + 1
  p.n1gain = n > 0 ? (uint32_t)(m / (2 * n) < 8 ? m / (2 * n) : 8) : 0u;
  p.heavy = (WE*)heavy;
  p.timeout_ns = kn.watchdog_ms ? (unsigned long long)kn.watchdog_ms * 1000000ull : 60ull * 1000000000ull;

  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (o.kernel_ms) {
    CK(cudaEventCreate(&ev0));
    CK(cudaEventCreate(&ev1));
    CK(cudaEventRecord(ev0, s));
  }
  struct EvGuard {
    cudaEvent_t a, b;
    ~EvGuard() { if (a) cudaEventDestroy(a); if (b) cudaEventDestroy(b); }
  } evg{ev0, ev1};
  int sbytes = 4, sbytes_used = 4;
  bool fat_cand_for_hint = false;
  if (!(o.flags & GC_FLAG_HOST_ROUNDS)) {
    // ---- persistent cooperative kernel: the whole run in one launch
    if (!prop.coop) {
      set_err("gc_color: device %d does not support cooperative launch", dev);
      return GC_ERR_UNSUPPORTED;
    }
    // 8-bit state words first; a colour > 127 makes the kernel stop at the next barrier with
    // ST_NEED16 and a vertex of degree > 32766 stops it in its prologue with ST_NEED32; the
    // run is then repeated with the wider words (at most two restarts).
    // kernel variant: bounded degree (<= 64) and >= 8 entries per row -> 3 CTAs/SM (sgr_kernels.cuh).
    // The max degree is known only after the ingest, so the choice for a graph is remembered
    // from its previous call (variant_hint; the first call runs the default variant).  A stale
    // hint can only cost speed: every variant computes the same colouring.
    const bool fat_candidate = push && n1 && m >= 8 * n;
    fat_cand_for_hint = fat_candidate;
    bool fat = fat_candidate && variant_hint(dev, d_rp, n, m) == 1;
    if (kn.variant >= 0) fat = kn.variant == 1;
    sbytes = kn.state_bytes;
    for (int attempt = 0; attempt < 3; ++attempt) {
      p.st = (uint8_t*)planes - (int64_t)sbytes * pitch;
      void* fn = pick_persistent(sbytes, (int)o.policy, push, cw, fat);
      int per_sm = 0;
      CK(occupancy(dev, fn, &per_sm));
      if (per_sm < 1) {
        set_err("gc_color: persistent kernel cannot be resident");
        return GC_ERR_UNSUPPORTED;
      }
      if (o.blocks_per_sm && (int)o.blocks_per_sm < per_sm) per_sm = (int)o.blocks_per_sm;
      const int grid = prop.sms * per_sm;
      void* args[] = {&p};
      CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(BLOCK), args, 0, s));
      uint32_t status = 0, rsm[2] = {0, 0};
      DevInfo* I = (DevInfo*)info;
      CK(cudaMemcpyAsync(&status, &I->status, sizeof(status), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(rsm, &I->resume_r, sizeof(rsm), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      sbytes_used = sbytes;
      if (status == ST_NEED16 && sbytes < 2) {
        sbytes = 2;
        // The 8-bit run stopped at the barrier after Phase A of round rsm[0] (a colour > 127):
        // widen its state words in place and let the 16-bit kernel resume at that Phase A, instead
        // of repeating rounds 1..rsm[0]-1 (the words sit right before plane 0 in both widths, so
        // the 8-bit copy goes through a temporary).  Not with exact work counters (they would
        // count that Phase A twice): those runs restart.
        if (kn.widen && !cw && rsm[0] >= 2) {
          void* tmp;
          CK(sc.alloc(&tmp, (size_t)pitch));
          CK(cudaMemcpyAsync(tmp, planes - pitch, (size_t)pitch, cudaMemcpyDeviceToDevice, s));
          k_widen8<<<prop.sms * 8, BLOCK, 0, s>>>((const uint8_t*)tmp, (uint16_t*)(planes - 2 * pitch), pitch);
          CK(cudaGetLastError());
          // the run goes on: clear the stop status and the barrier counter (the 16-bit grid may
          // differ in size); the aborted Phase A's change count is redone
          CK(cudaMemsetAsync(&I->status, 0, sizeof(I->status), s));
          CK(cudaMemsetAsync(I->pstatus, 0, sizeof(I->pstatus), s));
          CK(cudaMemsetAsync(&I->bar_count, 0, sizeof(I->bar_count), s));
          CK(cudaMemsetAsync(&I->chg[rsm[0] % 3], 0, sizeof(uint32_t), s));
          CK(cudaMemsetAsync(&I->resume_r, 0, 2 * sizeof(uint32_t), s));
          p.resume_r = rsm[0];
          p.resume_dense = rsm[1];
          continue;
        }
      } else if (status == ST_NEED32 && sbytes < 4) {
        sbytes = 4;
      } else {
        break;
      }
      p.resume_r = 0;
      CK(cudaMemsetAsync(info, 0, sizeof(DevInfo), s));
    }
  } else {
    // ---- host-driven rounds (ablation): one launch per phase, |W| read every round
    p.st = (uint8_t*)planes - 4 * pitch;
    const int grid = prop.sms * 4;
    if (push) k_prologue_count<true><<<grid, BLOCK, 0, s>>>(p);
    else k_prologue_count<false><<<grid, BLOCK, 0, s>>>(p);
    k_prologue_scatter<<<grid, BLOCK, 0, s>>>(p);
    CK(cudaGetLastError());
    WE* W = p.wl0;
    WE* Wo = p.wl1;
    uint32_t r = 1;
    uint32_t cnt[3][NBIN];
    for (;;) {
      if (r > 1) {
        if (push) { if (cw) launch_phase_a<true, true>(grid, s, p, r, W); else launch_phase_a<true, false>(grid, s, p, r, W); }
        else { if (cw) launch_phase_a<false, true>(grid, s, p, r, W); else launch_phase_a<false, false>(grid, s, p, r, W); }
      }
#ifdef GC_HOSTDBG
      { cudaError_t e = cudaStreamSynchronize(s); fprintf(stderr, "HOSTDBG r=%u after A: %s\n", r, cudaGetErrorName(e)); }
#endif
      launch_b((int)o.policy, push, cw, grid, s, p, r, W, Wo);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(cnt, ((DevInfo*)info)->cnt, sizeof(cnt), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
#ifdef GC_HOSTDBG
      {
        const uint32_t* nx = cnt[(r + 1) % 3];
        uint32_t bs[NBIN];
        cudaMemcpy(bs, ((DevInfo*)info)->binsize, sizeof(bs), cudaMemcpyDeviceToHost);
        uint32_t off = 0;
        for (int b = 0; b < NBIN; ++b) {
          if (nx[b] > bs[b]) fprintf(stderr, "HOSTDBG r=%u bin %d count %u > cap %u\n", r, b, nx[b], bs[b]);
          WE* h = (WE*)malloc(sizeof(WE) * (nx[b] + 1));
          cudaMemcpy(h, Wo + off, sizeof(WE) * nx[b], cudaMemcpyDeviceToHost);
          for (uint32_t i = 0; i < nx[b]; ++i) {
            int64_t rb = 0;
            if (h[i].v < 0 || h[i].v >= n) { fprintf(stderr, "HOSTDBG r=%u bin %d i %u bad v %d\n", r, b, i, h[i].v); break; }
            cudaMemcpy(&rb, d_rp + h[i].v, 8, cudaMemcpyDeviceToHost);
            if (rb != h[i].beg || h[i].k < 0) { fprintf(stderr, "HOSTDBG r=%u bin %d i %u v %d k %d beg %lld rp %lld\n", r, b, i, h[i].v, h[i].k, h[i].beg, (long long)rb); break; }
            if (i > 64) break;
          }
          free(h);
          off += bs[b];
        }
        fprintf(stderr, "HOSTDBG r=%u after B: next=%u %u\n", r, nx[0], nx[1]);
      }
#endif
      const uint32_t* nx = cnt[(r + 1) % 3];
      if (nx[0] + nx[1] == 0) break;
      if (r >= p.max_rounds) {
        set_err("gc_color: no convergence within max_rounds=%u", p.max_rounds);
        return GC_ERR_NO_CONVERGENCE;
      }
      ++r;
      WE* t = W;
      W = Wo;
      Wo = t;
    }
    k_epilogue<<<grid, BLOCK, 0, s>>>(p, r);
  }
  CK(cudaGetLastError());
  if (ev1) CK(cudaEventRecord(ev1, s));

  DevInfo hinfo;
  CK(cudaMemcpyAsync(&hinfo, info, sizeof(DevInfo), cudaMemcpyDeviceToHost, s));
  if (!(o.flags & GC_FLAG_HOST_ROUNDS)) {
    CK(cudaStreamSynchronize(s));
    set_variant_hint(dev, d_rp, n, m, fat_cand_for_hint && hinfo.maxdeg <= 64u ? 1 : 0);
  }
  if (!out_dev) CK(cudaMemcpyAsync(colors_out, dcol, sizeof(uint32_t) * (size_t)n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (ev1) CK(cudaEventElapsedTime(o.kernel_ms, ev0, ev1));
  if (hinfo.status == ST_WATCHDOG) {
    set_err("gc_color: device watchdog fired (grid barrier timeout)");
    return GC_ERR_CUDA;
  }
  if (hinfo.status == ST_NO_CONVERGENCE) {
    set_err("gc_color: no convergence within max_rounds=%u", p.max_rounds);
    return GC_ERR_NO_CONVERGENCE;
  }
  if (trace && !trace_dev) {
    const uint32_t k = hinfo.rounds < o.trace_capacity ? hinfo.rounds : o.trace_capacity;
    if (k) {
      CK(cudaMemcpyAsync(o.trace_worklist, dtrace, sizeof(uint32_t) * k, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
  }
  if (dphase) {
    CK(cudaMemcpyAsync(o.phase_ns, dphase, sizeof(uint64_t) * (4 * (size_t)o.trace_capacity + 1),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
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

gc_status gc_verify(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const uint32_t* colors,
                    int32_t device, int64_t* bad_vertex) {
  g_err[0] = 0;
  if (!bad_vertex) {
    set_err("gc_verify: bad_vertex must not be NULL");
    return GC_ERR_INVALID_ARGUMENT;
  }
  *bad_vertex = -1;
  if (n < 0 || n > INT32_MAX) {
    set_err("gc_verify: n out of range");
    return GC_ERR_INVALID_ARGUMENT;
  }
  if (n == 0) return GC_OK;
  if (!row_ptr || !col_idx || !colors) {
    set_err("gc_verify: NULL pointer");
    return GC_ERR_INVALID_ARGUMENT;
  }
  Scope sc;
  CK(cudaGetDevice(&sc.prev_dev));
  const int dev = device >= 0 ? device : sc.prev_dev;
  CK(cudaSetDevice(dev));
  CK(internal_stream(&sc.stream));  // ordered after the legacy default stream
  sc.own_stream = true;
  CK(get_pool(dev, &sc.pool));
  cudaStream_t s = sc.stream;
  const int64_t* d_rp = row_ptr;
  const int32_t* d_ci = col_idx;
  const uint32_t* d_col = colors;
  int64_t m = -1;
  if (is_device_ptr(row_ptr) != 1) {
    m = row_ptr[n];
    void* p;
    CK(sc.alloc(&p, sizeof(int64_t) * (size_t)(n + 1)));
    CK(cudaMemcpyAsync(p, row_ptr, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyHostToDevice, s));
    d_rp = (const int64_t*)p;
  }
  if (is_device_ptr(col_idx) != 1) {
    if (m < 0) {
      CK(cudaMemcpyAsync(&m, d_rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    void* p;
    CK(sc.alloc(&p, sizeof(int32_t) * (size_t)m));
    if (m) CK(cudaMemcpyAsync(p, col_idx, sizeof(int32_t) * (size_t)m, cudaMemcpyHostToDevice, s));
    d_ci = (const int32_t*)p;
  }
  if (is_device_ptr(colors) != 1) {
    void* p;
    CK(sc.alloc(&p, sizeof(uint32_t) * (size_t)n));
    CK(cudaMemcpyAsync(p, colors, sizeof(uint32_t) * (size_t)n, cudaMemcpyHostToDevice, s));
    d_col = (const uint32_t*)p;
  }
  void* info;
  CK(sc.alloc(&info, sizeof(DevInfo)));
  CK(cudaMemsetAsync(info, 0, sizeof(DevInfo), s));
  DevFacts prop;
  CK(dev_facts(dev, &prop));
  k_verify<<<prop.sms * 8, BLOCK, 0, s>>>((int32_t)n, d_rp, d_ci, d_col, (DevInfo*)info);
  CK(cudaGetLastError());
  unsigned long long bad = 0;
  CK(cudaMemcpyAsync(&bad, &((DevInfo*)info)->bad, sizeof(bad), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bad) {
    bad = ~bad;
    *bad_vertex = (int64_t)(bad >> 3);
    set_err("gc_verify: vertex %lld violates %s", (long long)*bad_vertex,
            (bad & 7) == 1 ? "completeness/greedy bound" : "properness/First-Fit fixpoint");
    return GC_ERR_INVALID_GRAPH;
  }
  return GC_OK;
}

// Diagnostics (include/gc_internal.h): mean cost of one grid barrier of the persistent
// kernel, in microseconds, for blocks_per_sm CTAs per SM (0 = max co-resident).
gc_status gc__bench_grid_sync(int32_t device, int32_t blocks_per_sm, int32_t iters, float* us_per_sync) {
  g_err[0] = 0;
  if (!us_per_sync || iters < 1) return GC_ERR_INVALID_ARGUMENT;
  Scope sc;
  CK(cudaGetDevice(&sc.prev_dev));
  const int dev = device >= 0 ? device : sc.prev_dev;
  CK(cudaSetDevice(dev));
  CK(cudaStreamCreateWithFlags(&sc.stream, cudaStreamNonBlocking));
  sc.own_stream = true;
  CK(get_pool(dev, &sc.pool));
  DevFacts f;
  CK(dev_facts(dev, &f));
  void* info;
  CK(sc.alloc(&info, sizeof(DevInfo)));
  CK(cudaMemsetAsync(info, 0, sizeof(DevInfo), sc.stream));
  Params p;
  memset(&p, 0, sizeof(p));
  p.info = (DevInfo*)info;
  p.timeout_ns = 10ull * 1000000000ull;
  int per_sm = 0;
  CK(occupancy(dev, (const void*)k_bench_sync, &per_sm));
  if (blocks_per_sm > 0 && blocks_per_sm < per_sm) per_sm = blocks_per_sm;
  void* args[] = {&p, &iters};
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaLaunchCooperativeKernel((void*)k_bench_sync, dim3(f.sms * per_sm), dim3(BLOCK), args, 0, sc.stream));
  CK(cudaEventRecord(a, sc.stream));
  CK(cudaLaunchCooperativeKernel((void*)k_bench_sync, dim3(f.sms * per_sm), dim3(BLOCK), args, 0, sc.stream));
  CK(cudaEventRecord(b, sc.stream));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *us_per_sync = ms * 1000.f / iters;
  return GC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- multi-GPU partitions
#include "../../include/gc_dist.h"
#include "dist_api.cuh"
