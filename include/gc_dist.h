/*
 * gc_dist.h — multi-GPU SGR colouring, one rank per GPU (C ABI; same library as gc.h:
 * paper_1606_06025_b200/csrc/libgc.so).  These are SURVEY §8(b)'s multi-GPU calls.
 *
 * What is computed: exactly gc_color's colouring (Alg. 7 Data-GC, with
 * FirstFit Alg. 4 PAPER.md:327-338 and ConflictResolve Alg. 5, in Jacobi
 * rounds).  The graph is partitioned by vertex range (BASELINE north star: "The 8-GPU path
 * partitions the graph by vertex range with edge-balanced splits and ghost colors ... cross-
 * partition conflicts are resolved by global id.  The result must be bit-identical to 1 GPU");
 * every cover of [0, n) gives bit-identical colours, num_colors, rounds and |W_r| trace.
 *
 * How (device-initiated exchange): every rank runs ONE persistent kernel for
 * the whole colouring — the paper's kernel fusion with a global barrier
 * taken across GPUs.  Each rank holds full-size replicas of the per-vertex state words,
 * forbidden-colour planes, dirty marks and (DEGREE) degrees in a window that every other rank
 * maps through CUDA IPC (NVLink peer memory).  Inside the kernel:
 *   - a changed tentative colour or a commit of a boundary vertex is stored straight into the
 *     replicas of the ranks that hold it as a ghost;
 *   - a winner ORs its colour bit into the owner's plane byte of every neighbour (peer RED);
 *   - dirty marks of successors across the cut are peer byte stores;
 *   - the two grid barriers per round span every rank's grid (system-scope fence, one flag per
 *     rank pair), and the barrier leader adds the rank's |W_{r+1}| into every rank's global
 *     count, so every rank leaves the round loop at the same round with no host involvement.
 * NCCL (loaded from libnccl.so.2 at run time) only bootstraps: it all-gathers the ranks'
 * ranges, arguments and IPC handles once per call (handles only when a window grows).
 *
 * Ownership and errors: as in gc.h.  Every call of gc_color_dist is collective: all ranks of
 * the communicator call it with the same n_global, policy, flags and max_rounds, and their
 * [v_begin, v_end) ranges, in rank order, must tile [0, n_global); otherwise every rank returns
 * GC_ERR_INVALID_ARGUMENT.  A failure on any rank (allocation, validation) is agreed by all
 * ranks before any kernel starts, so no rank is left waiting.  A device-side watchdog
 * (60 s per barrier) turns a lost rank into GC_ERR_CUDA and marks the communicator unusable.
 */
#ifndef GC_DIST_H_
#define GC_DIST_H_
#include <stdint.h>
#include "gc.h"
#ifdef __cplusplus
extern "C" {
#endif

#define GC_MAX_RANKS 8
#define GC_NCCL_UNIQUE_ID_BYTES 128

typedef struct gc_comm gc_comm;

/* ncclGetUniqueId into id_out[GC_NCCL_UNIQUE_ID_BYTES] (call on one rank, broadcast the bytes,
 * e.g. with torch.distributed).  GC_ERR_NCCL when libnccl.so.2 cannot be loaded. */
gc_status gc_nccl_unique_id(void* id_out);

/* Collective over `world` processes (1 <= world <= GC_MAX_RANKS): ncclCommInitRank on `device`
 * (-1 = current).  The communicator owns a stream and, after the first gc_color_dist, the
 * rank's IPC window (about 74 bytes per global vertex). */
gc_status gc_comm_init(gc_comm** out, int32_t rank, int32_t world, const void* nccl_unique_id,
                       int32_t device);

/* One-process emulation (tests, one GPU): comms_out[world] communicators whose ranks all live
 * on `device` and bootstrap through memory instead of NCCL.  The kernel code, windows, peer
 * stores and cross-rank barriers are the multi-GPU ones; each rank's gc_color_dist must be
 * called concurrently from its own host thread.  The emulated ranks run in ONE cooperative
 * launch (rank q on CTAs [qG, (q+1)G), issued by rank 0's thread), so that all of them are
 * co-resident by construction. */
gc_status gc_comm_init_local(gc_comm** comms_out, int32_t world, int32_t device);

/*
 * gc_color_dist — colour the rows [v_begin, v_end) owned by this rank.
 *   n_global          number of vertices of the whole graph (<= INT32_MAX).
 *   row_ptr_local     int64[v_end - v_begin + 1]: row_ptr[v_begin..v_end] - row_ptr[v_begin].
 *   col_idx_local     int32[row_ptr_local[v_end - v_begin]]: the rows' neighbours, GLOBAL ids,
 *                     sorted, loop-free, symmetric graph (GC_FLAG_VALIDATE checks range, order,
 *                     loops of the local rows; GC_FLAG_VALIDATE_SYMMETRY is rejected).
 *   opts              as gc_color (policy, flags GC_FLAG_VALIDATE / _TRACE / _COUNT_WORK, trace,
 *                     stream, kernel_ms, tuning); GC_FLAG_PULL_FIRSTFIT and GC_FLAG_HOST_ROUNDS
 *                     are rejected.  opts->device is ignored (the communicator's device).
 *   colors_out_local  uint32[v_end - v_begin], host or device.
 *   num_colors, rounds   global values, identical on every rank (trace: the global |W_r|).
 */
gc_status gc_color_dist(gc_comm* c, int64_t n_global, int64_t v_begin, int64_t v_end,
                        const int64_t* row_ptr_local, const int32_t* col_idx_local,
                        const gc_opts* opts, uint32_t* colors_out_local, uint32_t* num_colors,
                        uint32_t* rounds);

/* Release the window, peer mappings, stream and NCCL communicator (NULL: no-op). */
gc_status gc_comm_destroy(gc_comm* c);

#ifdef __cplusplus
}
#endif
#endif
