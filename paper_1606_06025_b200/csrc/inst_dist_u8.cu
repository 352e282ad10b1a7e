// inst_dist_u8.cu — multi-GPU persistent SGR kernel instances with 8-bit state words (+ the 3-CTA/SM variant)
// (GC_DIST_TU: namespace gcdev_dist, cross-rank exchange compiled in; see sgr_inst.h).
#define GC_INST_TU
#define GC_DIST_TU
#include "sgr_kernels.cuh"
#include "sgr_inst.h"

using namespace gcdev_dist;

void* gc_inst_dist_u8(int pol, bool cw) {
  if (pol == HIGHER_ID) return cw ? (void*)sgr_dist<uint8_t, HIGHER_ID, true> : (void*)sgr_dist<uint8_t, HIGHER_ID, false>;
  if (pol == LOWER_ID) return cw ? (void*)sgr_dist<uint8_t, LOWER_ID, true> : (void*)sgr_dist<uint8_t, LOWER_ID, false>;
  return cw ? (void*)sgr_dist<uint8_t, DEGREE, true> : (void*)sgr_dist<uint8_t, DEGREE, false>;
}

void* gc_inst_dist_fat(int pol, bool cw) {
  if (pol == HIGHER_ID) return cw ? (void*)sgr_dist_fat<HIGHER_ID, true> : (void*)sgr_dist_fat<HIGHER_ID, false>;
  if (pol == LOWER_ID) return cw ? (void*)sgr_dist_fat<LOWER_ID, true> : (void*)sgr_dist_fat<LOWER_ID, false>;
  return cw ? (void*)sgr_dist_fat<DEGREE, true> : (void*)sgr_dist_fat<DEGREE, false>;
}
