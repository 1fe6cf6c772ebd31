// Generic k_stage instantiations for the remaining fine / coarse pairs of the ABI's range (odd sizes
// 1..9 each; tables.h): the pairs without a specialised TMA kernel run the generic stage kernel.
#include "tables.h"

namespace blade {
namespace tables {
template <int NF, int NC, int RS, int BY, bool CH3 = false, bool WIDE = false>
static StageVariant make_variant() {
  using SS = StageShape<NF, NC, RS, BY, CH3>;
  return StageVariant{NF, NC, RS, BY, &k_stage<NF, NC, RS, BY, CH3, WIDE>, SS::tile_floats, SS::threads,
                      SS::TROWS, SS::TCOLS, CH3, WIDE};
}
const std::vector<StageVariant>& stage_variants_pairs() {
  static const std::vector<StageVariant> v = {
      make_variant<1, 0, 1, 8>(),
      make_variant<1, 1, 2, 8>(), make_variant<1, 1, 2, 2>(),
      make_variant<1, 3, 2, 8>(), make_variant<1, 3, 2, 2>(),
      make_variant<1, 5, 2, 8>(), make_variant<1, 5, 2, 2>(),
      make_variant<1, 7, 2, 8>(), make_variant<1, 7, 2, 2>(),
      make_variant<1, 9, 2, 8>(), make_variant<1, 9, 2, 2>(),
      make_variant<3, 1, 2, 8>(), make_variant<3, 1, 2, 2>(),
      make_variant<3, 5, 2, 8>(), make_variant<3, 5, 2, 2>(),
      make_variant<3, 7, 2, 8>(), make_variant<3, 7, 2, 2>(),
      make_variant<3, 9, 2, 8>(), make_variant<3, 9, 2, 2>(),
      make_variant<5, 1, 2, 8>(), make_variant<5, 1, 2, 2>(),
      make_variant<5, 7, 2, 8>(), make_variant<5, 7, 2, 2>(),
      make_variant<5, 9, 2, 8>(), make_variant<5, 9, 2, 2>(),
      make_variant<7, 1, 2, 8>(), make_variant<7, 1, 2, 2>(),
      make_variant<7, 3, 2, 8>(), make_variant<7, 3, 2, 2>(),
      make_variant<7, 9, 2, 8>(), make_variant<7, 9, 2, 2>(),
      make_variant<9, 1, 2, 8>(), make_variant<9, 1, 2, 2>(),
      make_variant<9, 3, 2, 8>(), make_variant<9, 3, 2, 2>(),
      make_variant<9, 5, 2, 8>(), make_variant<9, 5, 2, 2>(),
  };
  return v;
}
}  // namespace tables
}  // namespace blade
