// inst_u8.cu — persistent SGR kernel instances with 8-bit state words (see sgr_inst.h).
#define GC_INST_TU
#include "sgr_kernels.cuh"
#include "sgr_inst.h"

using namespace gcdev;

namespace {
template <int POL, bool PUSH, bool CW>
void* ptr() { return (void*)sgr_persistent<uint8_t, POL, PUSH, CW>; }
template <int POL>
void* pick(bool push, bool cw) {
  if (push) return cw ? ptr<POL, true, true>() : ptr<POL, true, false>();
  return cw ? ptr<POL, false, true>() : ptr<POL, false, false>();
}
}  // namespace

void* gc_inst_u8(int pol, bool push, bool cw) {
  if (pol == HIGHER_ID) return pick<HIGHER_ID>(push, cw);
  if (pol == LOWER_ID) return pick<LOWER_ID>(push, cw);
  return pick<DEGREE>(push, cw);
}
