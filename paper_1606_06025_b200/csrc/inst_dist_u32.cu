// inst_dist_u32.cu — multi-GPU persistent SGR kernel instances with 32-bit state words
// (GC_DIST_TU: namespace gcdev_dist, cross-rank exchange compiled in; see sgr_inst.h).
#define GC_INST_TU
#define GC_DIST_TU
#include "sgr_kernels.cuh"
#include "sgr_inst.h"

using namespace gcdev_dist;

void* gc_inst_dist_u32(int pol, bool cw) {
  if (pol == HIGHER_ID) return cw ? (void*)sgr_dist<uint32_t, HIGHER_ID, true> : (void*)sgr_dist<uint32_t, HIGHER_ID, false>;
  if (pol == LOWER_ID) return cw ? (void*)sgr_dist<uint32_t, LOWER_ID, true> : (void*)sgr_dist<uint32_t, LOWER_ID, false>;
  return cw ? (void*)sgr_dist<uint32_t, DEGREE, true> : (void*)sgr_dist<uint32_t, DEGREE, false>;
}
