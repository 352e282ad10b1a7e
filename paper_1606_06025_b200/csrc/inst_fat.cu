// inst_fat.cu — the 3-CTA/SM persistent SGR kernel instances (see sgr_inst.h).
#define GC_INST_TU
#include "sgr_kernels.cuh"
#include "sgr_inst.h"

using namespace gcdev;

void* gc_inst_fat(int pol, bool cw) {
  if (pol == HIGHER_ID) return cw ? (void*)sgr_persistent_fat<HIGHER_ID, true> : (void*)sgr_persistent_fat<HIGHER_ID, false>;
  if (pol == LOWER_ID) return cw ? (void*)sgr_persistent_fat<LOWER_ID, true> : (void*)sgr_persistent_fat<LOWER_ID, false>;
  return cw ? (void*)sgr_persistent_fat<DEGREE, true> : (void*)sgr_persistent_fat<DEGREE, false>;
}
