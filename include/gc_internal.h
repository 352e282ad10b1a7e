/*
 * gc_internal.h — diagnostics exported by libgc.so that are not part of the colouring
 * ABI (include/gc.h).  Stable only within one library build.
 */
#ifndef GC_INTERNAL_H_
#define GC_INTERNAL_H_
#include <stdint.h>
#include "gc.h"
#ifdef __cplusplus
extern "C" {
#endif

/* Mean device time of one grid-wide barrier of the persistent SGR kernel (the a4 round
 * control step, "global barrier"), measured with CUDA events over `iters`
 * barriers of a cooperative launch of SMs x blocks_per_sm CTAs (0 = max co-resident). */
gc_status gc__bench_grid_sync(int32_t device, int32_t blocks_per_sm, int32_t iters, float* us_per_sync);

#ifdef __cplusplus
}
#endif
#endif
