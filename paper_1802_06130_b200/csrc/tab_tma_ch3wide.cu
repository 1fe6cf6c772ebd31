// k_stage_tma instantiations for per-channel (Y, Cb, Cr) banks with K > 256 (tables.h): the paper's
// own layout (16 x 16 x 16 buckets, one bank per channel, f1 x f2). CTAs are
// specialised by channel; uint16 bucket tiles; the bank is read from global memory (L2-resident).
#include "tables.h"

#ifndef BLADE_TMA_GROUPS
#define BLADE_TMA_GROUPS 2
#endif
namespace blade {
namespace tables {
template <int NF, int NC, int RY = 2, int G = BLADE_TMA_GROUPS, int TR = 16>
static TmaVariant make_tma_ch3_wide() {
  using SS = TmaShape<NF, NC, true, RY, false, TR>;
  TmaVariant v{NF, NC, G, SS::BY, &k_stage_tma<NF, NC, G, true, true, RY, false, TR>, SS::stage_bytes, SS::TROWS,
               SS::TCOLS, SS::FCB, SS::FR, SS::CCB, SS::CR, SS::RF, SS::RC, SS::S, false, true, true};
  v.ry = RY;
  return v;
}
const std::vector<TmaVariant>& tma_variants_ch3_wide() {
  static const std::vector<TmaVariant> v = {
      make_tma_ch3_wide<3, 0>(), make_tma_ch3_wide<5, 0>(), make_tma_ch3_wide<7, 0>(), make_tma_ch3_wide<9, 0>(),
      make_tma_ch3_wide<5, 5>(), make_tma_ch3_wide<7, 5>(), make_tma_ch3_wide<7, 7>(), make_tma_ch3_wide<9, 9>(),
      make_tma_ch3_wide<5, 3>(), make_tma_ch3_wide<9, 7>(),
  };
  return v;
}
}  // namespace tables
}  // namespace blade
