// Generic k_stage instantiations (tables.h).
#include "tables.h"

namespace blade {
namespace tables {
template <int NF, int NC, int RS, int BY, bool CH3 = false, bool WIDE = false>
static StageVariant make_variant() {
  using SS = StageShape<NF, NC, RS, BY, CH3>;
  return StageVariant{NF, NC, RS, BY, &k_stage<NF, NC, RS, BY, CH3, WIDE>, SS::tile_floats, SS::threads,
                      SS::TROWS, SS::TCOLS, CH3, WIDE};
}
const std::vector<StageVariant>& stage_variants() {
  static const std::vector<StageVariant> v = {
      make_variant<3, 0, 1, 8>(), make_variant<5, 0, 1, 8>(), make_variant<7, 0, 1, 8>(),
      make_variant<9, 0, 1, 8>(), make_variant<3, 3, 2, 8>(), make_variant<5, 5, 2, 8>(),
      make_variant<7, 7, 2, 8>(), make_variant<7, 7, 2, 4>(), make_variant<9, 9, 2, 8>(),
      make_variant<9, 9, 2, 4>(), make_variant<9, 9, 2, 2>(), make_variant<7, 5, 2, 8>(),
      make_variant<7, 5, 2, 4>(), make_variant<5, 3, 2, 8>(), make_variant<9, 7, 2, 4>(),
      make_variant<9, 7, 2, 2>(),
      // per-channel YCbCr banks (NEXT f1)
      make_variant<3, 0, 1, 8, true>(), make_variant<5, 0, 1, 8, true>(), make_variant<7, 0, 1, 8, true>(),
      make_variant<9, 0, 1, 8, true>(), make_variant<3, 3, 2, 8, true>(), make_variant<5, 5, 2, 8, true>(),
      make_variant<7, 7, 2, 8, true>(), make_variant<7, 7, 2, 4, true>(), make_variant<9, 9, 2, 4, true>(),
      make_variant<9, 9, 2, 2, true>(), make_variant<7, 5, 2, 8, true>(), make_variant<7, 5, 2, 4, true>(),
      make_variant<5, 3, 2, 8, true>(), make_variant<9, 7, 2, 4, true>(), make_variant<9, 7, 2, 2, true>(),
      // K > 256 (NEXT f2): uint16 maps, bank in global memory
      make_variant<3, 0, 1, 8, false, true>(), make_variant<5, 0, 1, 8, false, true>(),
      make_variant<7, 0, 1, 8, false, true>(), make_variant<9, 0, 1, 8, false, true>(),
      make_variant<5, 5, 2, 8, false, true>(), make_variant<7, 5, 2, 8, false, true>(),
      make_variant<7, 7, 2, 8, false, true>(), make_variant<9, 9, 2, 8, false, true>(),
      make_variant<5, 3, 2, 8, false, true>(), make_variant<9, 7, 2, 8, false, true>(),
  };
  return v;
}
}  // namespace tables
}  // namespace blade
