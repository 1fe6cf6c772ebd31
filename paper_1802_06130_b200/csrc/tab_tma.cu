// k_stage_tma instantiations (tables.h).
#include "tables.h"

#ifndef BLADE_TMA_GROUPS
#define BLADE_TMA_GROUPS 2
#endif
namespace blade {
namespace tables {
template <int NF, int NC, bool CH3 = false, bool WIDE = false, int RY = 2, int G = BLADE_TMA_GROUPS, int TR = 16>
static TmaVariant make_tma() {
  using SS = TmaShape<NF, NC, WIDE, RY, false, TR>;
  TmaVariant v{NF, NC, G, SS::BY, &k_stage_tma<NF, NC, G, CH3, WIDE, RY, false, TR>, SS::stage_bytes, SS::TROWS,
               SS::TCOLS, SS::FCB, SS::FR, SS::CCB, SS::CR, SS::RF, SS::RC, SS::S, false, CH3, WIDE};
  v.ry = RY;
  if constexpr (!CH3 && !WIDE && NC > 0 && RY == 4 && TR == 16) {  // fused-selector form (level 0, 4-row threads)
    using SF = TmaShape<NF, NC, WIDE, RY, true>;
    v.fsel_fn = &k_stage_tma<NF, NC, G, CH3, WIDE, RY, true>;
    v.fsel_stage_bytes = SF::stage_bytes;
    v.fsel_fr = SF::FR;
  }
  return v;
}
StageFixKernel stage_fixup_kernel(int nf, int nc) {
  if (nf == 5 && nc == 5) return &k_stage_fixup<5, 5>;
  if (nf == 3 && nc == 3) return &k_stage_fixup<3, 3>;
  if (nf == 5 && nc == 3) return &k_stage_fixup<5, 3>;
  return nullptr;
}
const std::vector<TmaVariant>& tma_variants() {
  static const std::vector<TmaVariant> v = {
      make_tma<3, 0>(), make_tma<5, 0>(), make_tma<7, 0>(), make_tma<9, 0>(),
      make_tma<3, 3>(), make_tma<5, 5>(), make_tma<5, 3>(),
      // 4 pixel rows per thread (fewer window wavefronts per pixel, 8 warps per SM)
      make_tma<3, 0, false, false, 4>(), make_tma<5, 0, false, false, 4>(), make_tma<7, 0, false, false, 4>(),
      make_tma<9, 0, false, false, 4>(), make_tma<3, 3, false, false, 4>(), make_tma<5, 5, false, false, 4>(),
      make_tma<5, 3, false, false, 4>(),
      // (three groups of 12-row tiles, 3 buffers: built and measured slower, c3 stage0 2.38 ->
      //  2.62 ms; profiles/r02_stage_groups.txt)
      make_tma<3, 0, true, false, 4>(), make_tma<5, 0, true, false, 4>(), make_tma<7, 0, true, false, 4>(),
      make_tma<9, 0, true, false, 4>(), make_tma<3, 3, true, false, 4>(), make_tma<5, 5, true, false, 4>(),
      make_tma<5, 3, true, false, 4>(),
      // per-channel YCbCr banks (NEXT f1): CTAs specialised by channel
      make_tma<3, 0, true>(), make_tma<5, 0, true>(), make_tma<7, 0, true>(), make_tma<9, 0, true>(),
      make_tma<3, 3, true>(), make_tma<5, 5, true>(), make_tma<5, 3, true>(),
      // K > 256 (NEXT f2): uint16 bucket tiles, bank read from global memory
      make_tma<3, 0, false, true>(), make_tma<5, 0, false, true>(), make_tma<7, 0, false, true>(),
      make_tma<9, 0, false, true>(), make_tma<5, 5, false, true>(), make_tma<7, 5, false, true>(),
      make_tma<7, 7, false, true>(), make_tma<9, 9, false, true>(), make_tma<5, 3, false, true>(),
      make_tma<9, 7, false, true>(),
  };
  return v;
}
#ifdef BLADE_TRACE
BT_DEFINE_ACCESS(trace_tma)
#endif
}  // namespace tables
}  // namespace blade
