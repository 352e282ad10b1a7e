// inst_dist_u32.cu — multi-GPU persistent SGR kernel instances with 32-bit state words
// (GC_DIST_TU: namespace gcdev_dist, cross-rank exchange compiled in; see sgr_inst.h).
#define GC_INST_TU
#define GC_DIST_TU
#include "sgr_kernels.cuh"
#include "sgr_inst.h"

using namespace gcdev_dist;

void* gc_inst_dist_u32(int pol, bool cw) {
  if (pol == HIGHER_ID) return cw ? (void*)sgr_persistent<uint32_t, HIGHER_ID, true, true> : (void*)sgr_persistent<uint32_t, HIGHER_ID, true, false>;
  if (pol == LOWER_ID) return cw ? (void*)sgr_persistent<uint32_t, LOWER_ID, true, true> : (void*)sgr_persistent<uint32_t, LOWER_ID, true, false>;
  return cw ? (void*)sgr_persistent<uint32_t, DEGREE, true, true> : (void*)sgr_persistent<uint32_t, DEGREE, true, false>;
}
