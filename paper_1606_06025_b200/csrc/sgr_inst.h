// sgr_inst.h — host stubs of the persistent kernel instances (one translation unit per
// state-word width, inst_*.cu, so that the library compiles in parallel).
#pragma once
void* gc_inst_u8(int pol, bool push, bool cw);
void* gc_inst_u16(int pol, bool push, bool cw);
void* gc_inst_u32(int pol, bool push, bool cw);
void* gc_inst_fat(int pol, bool cw);  // 3 CTAs/SM, 8-bit words, push First-Fit
// multi-GPU instances (namespace gcdev_dist, cross-rank code compiled in; push First-Fit)
void* gc_inst_dist_u8(int pol, bool cw);
void* gc_inst_dist_u16(int pol, bool cw);
void* gc_inst_dist_u32(int pol, bool cw);
void* gc_inst_dist_fat(int pol, bool cw);
