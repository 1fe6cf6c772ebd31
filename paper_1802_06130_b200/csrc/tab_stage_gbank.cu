// Generic k_stage instantiations that read the bank from global memory with uint8 maps (tables.h):
// the fallback for K <= 256 banks whose two phases do not fit the shared memory next to a tile.
#include "tables.h"

namespace blade {
namespace tables {
template <int NF, int NC, int RS, bool CH3>
static StageVariant make_gbank() {
  constexpr int BY = 8;
  using SS = StageShape<NF, NC, RS, BY, CH3>;
  StageVariant v{NF, NC, RS, BY, &k_stage<NF, NC, RS, BY, CH3, false, true>, SS::tile_floats, SS::threads,
                 SS::TROWS, SS::TCOLS, CH3, false};
  v.gbank = true;
  return v;
}
#define G(nf, nc, rs, ch3) make_gbank<nf, nc, rs, ch3>()
const std::vector<StageVariant>& stage_variants_gbank() {
  static const std::vector<StageVariant> v = {
      G(1, 0, 1, false), G(3, 0, 1, false), G(5, 0, 1, false), G(7, 0, 1, false), G(9, 0, 1, false),
      G(1, 0, 1, true), G(3, 0, 1, true), G(5, 0, 1, true), G(7, 0, 1, true), G(9, 0, 1, true),
      G(1, 1, 2, false), G(1, 1, 2, true),
      G(1, 3, 2, false), G(1, 3, 2, true),
      G(1, 5, 2, false), G(1, 5, 2, true),
      G(1, 7, 2, false), G(1, 7, 2, true),
      G(1, 9, 2, false), G(1, 9, 2, true),
      G(3, 1, 2, false), G(3, 1, 2, true),
      G(3, 3, 2, false), G(3, 3, 2, true),
      G(3, 5, 2, false), G(3, 5, 2, true),
      G(3, 7, 2, false), G(3, 7, 2, true),
      G(3, 9, 2, false), G(3, 9, 2, true),
      G(5, 1, 2, false), G(5, 1, 2, true),
      G(5, 3, 2, false), G(5, 3, 2, true),
      G(5, 5, 2, false), G(5, 5, 2, true),
      G(5, 7, 2, false), G(5, 7, 2, true),
      G(5, 9, 2, false), G(5, 9, 2, true),
      G(7, 1, 2, false), G(7, 1, 2, true),
      G(7, 3, 2, false), G(7, 3, 2, true),
      G(7, 5, 2, false), G(7, 5, 2, true),
      G(7, 7, 2, false), G(7, 7, 2, true),
      G(7, 9, 2, false), G(7, 9, 2, true),
      G(9, 1, 2, false), G(9, 1, 2, true),
      G(9, 3, 2, false), G(9, 3, 2, true),
      G(9, 5, 2, false), G(9, 5, 2, true),
      G(9, 7, 2, false), G(9, 7, 2, true),
      G(9, 9, 2, false), G(9, 9, 2, true),
  };
  return v;
}
#undef G
}  // namespace tables
}  // namespace blade
