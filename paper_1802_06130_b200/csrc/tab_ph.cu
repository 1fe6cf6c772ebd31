// k_stage_ph instantiations (tables.h).
#include "tables.h"

namespace blade {
namespace tables {
template <int NF, int NC, bool CH3 = false>
static TmaVariant make_ph() {
  using SS = PhShape<NF, NC>;
  return TmaVariant{NF, NC, 2, 4, &k_stage_ph<NF, NC, CH3>, SS::stage_bytes, SS::TROWS, SS::TCOLS,
                    SS::FCB, SS::FR, SS::CCB, SS::CR, SS::RF, SS::RC, SS::S, true, CH3, false};
}
const std::vector<TmaVariant>& ph_variants() {
  static const std::vector<TmaVariant> v = {
      make_ph<7, 7>(), make_ph<9, 9>(), make_ph<7, 5>(), make_ph<9, 7>(), make_ph<5, 7>(), make_ph<7, 9>(),
      // per-channel YCbCr banks (NEXT f1) for the large footprints; smaller ones stay on the generic
      // kernel, where one CTA type (of 12) per tile leaves too little work per TMA tile
      make_ph<7, 7, true>(), make_ph<9, 9, true>(), make_ph<7, 5, true>(), make_ph<9, 7, true>(),
  };
  return v;
}
template <int NF, int NC>
static TmaVariant make_p2() {
  using SS = PhShape<NF, NC>;
  TmaVariant v{NF, NC, 2, 4, &k_stage_p2<NF, NC>, SS::stage_bytes, SS::TROWS, SS::TCOLS,
               SS::FCB, SS::FR, SS::CCB, SS::CR, SS::RF, SS::RC, SS::S, true, false, false};
  v.ptypes = 2;
  return v;
}
const std::vector<TmaVariant>& p2_variants() {
  // two phases fit next to two 16 x 128 tile buffers for these pair banks (7x7 + 7x7: 2 x 57.6 KB)
  static const std::vector<TmaVariant> v = {make_p2<7, 7>(), make_p2<7, 5>(), make_p2<5, 7>()};
  return v;
}
}  // namespace tables
}  // namespace blade
