/*
 * gc_dist.h — vertex-range partitioned SGR colouring (multi-GPU path), C ABI.
 * Library: paper_1606_06025_b200/csrc/libgc.so (same library as gc.h).
 *
 * SURVEY §8(e) / BASELINE north star: "The 8-GPU path partitions the graph by vertex range
 * with edge-balanced splits and ghost colors.  Each round, changed boundary colors are
 * exchanged ... and cross-partition conflicts are resolved by global id.  The result must
 * be bit-identical to 1 GPU."
 *
 * One partition per process/GPU.  A partition holds the rows [v_begin, v_end) of the global
 * CSR (row_ptr_local = row_ptr[v_begin..v_end] - row_ptr[v_begin], col_idx_local in GLOBAL
 * ids) and a replicated state word per global vertex.  The caller drives the rounds and
 * moves the packed (vertex, word) pairs between partitions (all-gather; the Python driver
 * paper_1606_06025_b200.dist does it with torch.distributed / NCCL):
 *
 *   create;  loop { phase_a; pack(0) -> all-gather -> unpack;          (round >= 2)
 *                   phase_b(&local_next); pack(1) -> all-gather -> unpack;
 *                   if sum over partitions of local_next == 0: break; next_round }
 *   finalize; destroy
 *
 * Round r reads exactly the state the single-GPU path reads (Jacobi rounds, reading C2), so
 * the colours are bit-identical to gc_color for every cover of [0, n).
 * First-Fit is incremental as on one GPU: each partition keeps forbidden-colour planes for its
 * own vertices; local winners OR their colour into them directly, and the commit pairs of
 * remote winners are applied through a halo adjacency (for every remote vertex, its local
 * neighbours) built by gc_dist_create.  Only boundary vertices (with a remote neighbour) are
 * packed: no other partition ever reads the others' words.  Policies HIGHER_ID
 * and LOWER_ID (global ids decide); DEGREE is single-GPU only (GC_ERR_UNSUPPORTED).
 * All pointers are device memory of opts->device; every call is synchronous on the
 * partition's internal stream.  Errors: see gc.h conventions.
 */
#ifndef GC_DIST_H_
#define GC_DIST_H_
#include <stdint.h>
#include "gc.h"
#ifdef __cplusplus
extern "C" {
#endif

typedef struct gc_dist gc_dist;

/* Allocate the partition state (replicated state words: 4 B x n_global; forbidden-colour
 * planes; halo adjacency, 4 B per cut edge) from the device's stream-ordered pool and build W_1. */
gc_status gc_dist_create(gc_dist** out, int64_t n_global, int64_t v_begin, int64_t v_end,
                         const int64_t* row_ptr_local, const int32_t* col_idx_local,
                         const gc_opts* opts);
/* Phase A (FirstFit) of the local pending vertices; no-op in round 1. */
gc_status gc_dist_phase_a(gc_dist* h);
/* Phase B (ConflictResolve + push); *local_next = local |W_{r+1}|. */
gc_status gc_dist_phase_b(gc_dist* h, uint32_t* local_next);
/* what 0: (v, word) of the local pending boundary vertices (after Phase A); what 1: the local
 * boundary winners (after Phase B).  pairs: device, >= 2*(v_end-v_begin) uint32; *count =
 * pairs written. */
gc_status gc_dist_pack(gc_dist* h, int32_t what, uint32_t* pairs, uint64_t* count);
/* Write gathered (v, word) pairs into the replicated state; committed words of remote
 * vertices also set their colour bit in the planes of their local neighbours (halo). */
gc_status gc_dist_unpack(gc_dist* h, const uint32_t* pairs, uint64_t count);
/* W_{r+1} becomes the input worklist of round r+1. */
gc_status gc_dist_next_round(gc_dist* h);
/* colors_local (device, [v_end-v_begin]); *max_color_local; *rounds = the current round. */
gc_status gc_dist_finalize(gc_dist* h, uint32_t* colors_local, uint32_t* max_color_local, uint32_t* rounds);
gc_status gc_dist_destroy(gc_dist* h);

#ifdef __cplusplus
}
#endif
#endif
