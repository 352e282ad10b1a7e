/*
 * gc.h — C ABI of the B200-native round-synchronous speculative-greedy (SGR) graph
 * colouring library (arXiv 1606.06025).  Library: paper_1606_06025_b200/libgc.so.
 *
 * The library colours an undirected graph given in CSR form (§3 "The
 * column-indices array C ... The row-offsets R array contains n + 1 integers") with the
 * data-driven speculative greedy loop of Alg. 7 "Data-driven Parallel Graph Coloring"
 * = Alg. 2 GM with FirstFit (Alg. 4,
 * PAPER.md:327-338) and ConflictResolve (Alg. 5), made round-synchronous
 * (Jacobi) as the north star requires: every round, Phase A reads the colours committed
 * before the round, Phase B reads the round's tentative colours.  The result is therefore
 * a pure function of the graph and the policy, identical to the CPU oracle (oracle/),
 * independent of thread schedule, launch geometry and (for gc_color_dist) partitioning.
 *
 * Conventions common to every entry point:
 *  - The caller owns every buffer.  The library keeps no pointer after return.
 *  - Pointers may be host memory or device memory of the selected device; the space is
 *    detected with cudaPointerGetAttributes.  Host inputs are copied to the device and
 *    host outputs copied back inside the call.
 *  - Calls are synchronous: they return after every output is final (one stream sync).
 *    The call's work is ordered after work already queued on opts->stream, or, when that is
 *    NULL, after work already queued on the legacy default stream (an event on it is waited
 *    for; the internal stream itself is non-blocking).
 *  - On error every scalar output is set to 0, array outputs are unspecified, nothing is
 *    thrown or aborted, and a human-readable detail is available from
 *    gc_last_error_message() (thread-local).
 *  - No global mutable state other than a per-device workspace memory pool, per-device
 *    attribute caches and a small cache of the kernel variant chosen for recently seen graphs
 *    (keyed by device, row_ptr address, n and m; it affects speed only, never the result);
 *    no device- or context-wide setting (L2 limits, access-policy windows, ...) is changed.
 *    Concurrent calls on distinct streams are allowed.
 *  - No tuning choice is read from the environment: they are all in gc_opts / gc_tuning.
 */
#ifndef GC_H_
#define GC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GC_ABI_VERSION 2

typedef enum gc_status {
  GC_OK = 0,
  GC_ERR_INVALID_ARGUMENT = 1, /* NULL with n>0, n<0, n>INT32_MAX, bad struct_size/policy */
  GC_ERR_INVALID_GRAPH = 2,    /* row_ptr[0]!=0 / decreasing, col out of range, self loop,
                                  unsorted or duplicate row entry, asymmetric edge
                                  (only detected when the matching GC_FLAG_VALIDATE* is set) */
  GC_ERR_NO_CONVERGENCE = 3,   /* rounds would exceed max_rounds */
  GC_ERR_OUT_OF_MEMORY = 4,
  GC_ERR_CUDA = 5,             /* CUDA runtime error or device-side watchdog; see message */
  GC_ERR_NCCL = 6,
  GC_ERR_UNSUPPORTED = 7       /* no sm_100-class device, no cooperative launch, ... */
} gc_status;

/* Which endpoint of a same-colour edge {v, w} is re-queued (recolours). */
typedef enum gc_policy {
  GC_POLICY_HIGHER_ID = 0, /* default: the higher vertex id recolours (BASELINE north star) */
  GC_POLICY_LOWER_ID = 1,  /* Alg. 5 literal "color[v]=color[w] and v<w" clears v */
  GC_POLICY_DEGREE = 2     /* §3.2 heuristic: smaller static degree
                              recolours; equal degree -> the smaller id is picked (keeps it) */
} gc_policy;

enum {
  GC_FLAG_VALIDATE = 1u,          /* check CSR invariants S:22-32 (one pass over col_idx) */
  GC_FLAG_VALIDATE_SYMMETRY = 2u, /* also check w in adj(v) <=> v in adj(w) (O(m log deg)) */
  GC_FLAG_TRACE = 4u,             /* write |W_r| for r = 1..rounds into opts->trace_worklist */
  GC_FLAG_PULL_FIRSTFIT = 8u,     /* Phase A by a full neighbour scan each round (the paper's
                                     FirstFit) instead of the incremental forbidden-colour mask;
                                     same result, more traffic; ablation */
  GC_FLAG_HOST_ROUNDS = 16u,      /* one kernel launch per phase with the host reading |W| each
                                     round (the paper's baseline control) instead of
                                     the persistent kernel; same result; ablation */
  GC_FLAG_COUNT_WORK = 32u        /* fill opts->work with exact work counters (slower) */
};

/* Exact work counters (GC_FLAG_COUNT_WORK); the run is deterministic, so these are a pure
 * function of (graph, policy, flags).  Used for the algorithmic-byte roofline. */
typedef struct gc_work {
  uint64_t phase_a_vertices;   /* sum over rounds r >= 2 of |W_r| (round 1 needs no Phase A) */
  uint64_t phase_a_edges;      /* neighbour words gathered in Phase A (full scans/fallbacks) */
  uint64_t phase_b_vertices;   /* sum over rounds of |W_r| */
  uint64_t phase_b_edges;      /* col_idx entries examined by the conflict scans */
  uint64_t phase_b_gathers;    /* neighbour colour words gathered by the conflict scans */
  uint64_t commit_scatter;     /* neighbour entries visited by the commit scatters */
  uint64_t pushes;             /* vertices pushed into W_out over the run */
  uint64_t scatter_reds;       /* forbidden-mask atomics issued by the commit scatters (fewer than
                                   commit_scatter only with gc_tuning.scatter_filter) */
  uint64_t dense_a_swept;      /* vertices swept by dense (id-order) Phase A passes */
  uint64_t dense_b_swept;      /* vertices swept by dense Phase B passes */
  uint64_t sparse_a_entries;   /* worklist entries read by sparse Phase A passes */
  uint64_t sparse_b_entries;   /* worklist entries read by sparse Phase B passes */
  uint64_t state_bytes;        /* width of the state words of the final attempt (1, 2 or 4) */
  uint64_t phase_b_evaluated;  /* pending vertices whose conflict scan ran (dirty-set rounds skip
                                  the clean ones) */
  uint64_t dense_b_evaluated;  /* of which in dense rounds */
  uint64_t dirty_marks;        /* dirty marks written (changed vertices and their successors) */
  uint64_t tent_changes;       /* tentative colours changed by Phase A */
  uint64_t pending_degree_sum; /* sum over rounds r >= 2 of the degrees of the vertices in W_r
                                  (round 1 adds m): the units of SURVEY §8(d)'s pull model */
  uint64_t reserved[3];
} gc_work;

/* Schedule choices of the persistent kernel.  None of them changes the result (the colouring
 * is a pure function of graph and policy); they exist for ablations and tests.  -1 (or 0 for
 * state_bytes) = the measured default, stated per field. */
typedef struct gc_tuning {
  uint32_t struct_size;    /* = sizeof(gc_tuning) */
  int32_t state_bytes;     /* 0: 8-bit state words with restarts to 16/32 bits; 2 or 4: start wider */
  int32_t dense_div;       /* dense (id-order) rounds while |W_r| * dense_div > n; 0 = never dense;
                              default 3.  A non-negative value also sets dense_div_n1 unless that
                              is given explicitly */
  int32_t dense_div_n1;    /* the same in dirty-set rounds; default 32 */
  int32_t n1;              /* dirty-set rounds: 0 off, 1 when max degree <= 64 (default), 2 always */
  int32_t list;            /* explicit list rounds: 0 off (default), 1 cost rule, 2 from round 3 */
  int32_t compact;         /* dense Phase B lists pending vertices without marks: 0 (default) / 1 */
  int32_t scatter_filter;  /* commit scatter skips committed neighbours: 0 (default) / 1 */
  int32_t dch;             /* dense queue chunks of about n / (dch x warps) vertices; default 16 */
  int32_t n1_chg;          /* mark only when chg(r-1) * n1_chg < |W_r|; 0 = every round (default) */
  int32_t variant;         /* kernel: 0 = 4 CTAs/SM, 1 = 3 CTAs/SM (80 registers); -1 = chosen by a
                              max-degree pre-pass (bounded degree <= 64 and m >= 8n -> 1) */
  int32_t watchdog_ms;     /* device watchdog per grid barrier, ms (0 or -1: 60 000); tests use less */
  int32_t widen;           /* 8-bit words overflowing (a colour > 127): 1 (default) widen them to 16 bits
                              in place and resume at the Phase A that overflowed; 0 restart the run */
  int32_t reserved[3];
} gc_tuning;

/* Fill *t with "defaults" (-1 / 0 as above). */
void gc_tuning_default(gc_tuning* t);

typedef struct gc_opts {
  uint32_t struct_size;      /* = sizeof(gc_opts) (ABI check) */
  uint32_t policy;           /* gc_policy */
  uint32_t flags;            /* GC_FLAG_*; default GC_FLAG_VALIDATE */
  uint32_t max_rounds;       /* 0 -> n + 1 (reading C13) */
  int32_t device;            /* CUDA ordinal; -1 = the calling thread's current device */
  uint32_t thread_bin_max;   /* reserved: ignored since the commit scatters are warp-flattened
                                (kept for ABI stability) */
  uint32_t warp_bin_max;     /* degree <= this -> thread probe + warp continuation per vertex
                                (0 -> default 1024); larger degrees -> one CTA per vertex
                                (load balancing) */
  uint32_t blocks_per_sm;    /* persistent grid = SMs x this (0 -> max co-resident) */
  void* stream;              /* cudaStream_t to run on; NULL = library-internal stream */
  uint32_t* trace_worklist;  /* host or device, [trace_capacity]; used with GC_FLAG_TRACE */
  uint32_t trace_capacity;
  uint32_t group_bin_max;    /* reserved (ignored) */
  gc_work* work;             /* host pointer; used with GC_FLAG_COUNT_WORK */
  float* kernel_ms;          /* optional host pointer: device time (CUDA events on the call's
                                stream) from the first to the last colouring kernel, i.e.
                                excluding argument checks, copies and validation */
  uint64_t* phase_ns;        /* optional host pointer [4 * trace_capacity + 1] (diagnostics, with
                                GC_FLAG_TRACE): device globaltimer (ns) after the ingest; per
                                round r: [4r-3] last CTA done with Phase A's work, [4r-2] its
                                barrier passed, [4r-1] / [4r] the same for Phase B (persistent
                                driver only; adds a CTA barrier per phase) */
  const gc_tuning* tuning;   /* optional schedule overrides (NULL = measured defaults) */
  uint64_t reserved[1];
} gc_opts;

/* Fill *o with the defaults above (policy HIGHER_ID, flags GC_FLAG_VALIDATE). */
void gc_opts_default(gc_opts* o);

/*
 * gc_color — colour the undirected CSR graph (n, row_ptr, col_idx).
 *   n          number of vertices, 0 <= n <= INT32_MAX.
 *   row_ptr    int64[n+1], row offsets R; m = row_ptr[n] = directed
 *              adjacency entries (reading C15).
 *   col_idx    int32[m], column indices C; each row sorted strictly increasing, no self
 *              loop, symmetric (checked only under GC_FLAG_VALIDATE*).
 *   opts       NULL = gc_opts_default.
 *   colors_out uint32[n]: colour of every vertex, 1..Delta+1 (0 = sentinel never returned).
 *   num_colors max colour (= number of distinct colours, First-Fit fixpoint).
 *   rounds     number of SGR rounds (Phase-A passes; PAPER.md:427 loop iterations).
 * n = 0 returns GC_OK with num_colors = rounds = 0.
 * Workspace (device, from a per-device stream-ordered pool, freed before return): about
 * 110 bytes per vertex (state words + up to 64 forbidden-colour byte planes, of which only the
 * planes a run reaches are touched; splits; dirty marks; two 16-byte worklists) plus 16 bytes
 * per vertex of degree > 1024.  The colouring runs as one cooperative kernel occupying every SM;
 * concurrent calls on other streams wait for it (they never interleave).
 */
gc_status gc_color(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                   const gc_opts* opts, uint32_t* colors_out, uint32_t* num_colors,
                   uint32_t* rounds);

/*
 * gc_verify — device check that `colors` is complete (all >= 1), proper (no edge with equal
 * colours) and a First-Fit fixpoint (every colour is the smallest colour
 * absent from its neighbourhood, which every SGR result satisfies).
 *   *bad_vertex = first offending vertex found (any one), or -1 when valid.
 * Returns GC_OK when valid, GC_ERR_INVALID_GRAPH when a violation was found.
 */
gc_status gc_verify(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                    const uint32_t* colors, int32_t device, int64_t* bad_vertex);

const char* gc_status_string(gc_status s);
const char* gc_last_error_message(void);

/*
 * gc_partition_edge_balanced — host-only helper for the vertex-range multi-GPU path
 * (SURVEY §8(e)): bounds[k] = min{v : row_ptr[v] >= ceil(k*m/parts)} for k = 0..parts,
 * bounds[0] = 0, bounds[parts] = n.  row_ptr must be host memory.
 */
gc_status gc_partition_edge_balanced(int64_t n, const int64_t* row_ptr, int32_t parts,
                                     int64_t* bounds);

/* ABI version of the loaded library (== GC_ABI_VERSION it was built with). */
int32_t gc_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GC_H_ */
