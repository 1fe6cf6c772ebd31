// Generic k_stage instantiations for per-channel (Y, Cb, Cr) banks with K > 256 (tables.h): the
// paper's own layout, 16 x 16 x 16 buckets with one bank per channel (f1 x f2) —
// uint16 maps, the 3 x 4 x 4096-filter bank read from global memory (L2-resident).
#include "tables.h"

namespace blade {
namespace tables {
template <int NF, int NC, int RS>
static StageVariant make_ch3_wide() {
  constexpr int BY = 8;
  using SS = StageShape<NF, NC, RS, BY, true>;
  return StageVariant{NF, NC, RS, BY, &k_stage<NF, NC, RS, BY, true, true>, SS::tile_floats, SS::threads,
                      SS::TROWS, SS::TCOLS, true, true};
}
#define W(nf, nc, rs) make_ch3_wide<nf, nc, rs>()
const std::vector<StageVariant>& stage_variants_ch3_wide() {
  static const std::vector<StageVariant> v = {
      W(1, 0, 1), W(3, 0, 1), W(5, 0, 1), W(7, 0, 1), W(9, 0, 1),
      W(1, 1, 2), W(1, 3, 2), W(1, 5, 2), W(1, 7, 2), W(1, 9, 2),
      W(3, 1, 2), W(3, 3, 2), W(3, 5, 2), W(3, 7, 2), W(3, 9, 2),
      W(5, 1, 2), W(5, 3, 2), W(5, 5, 2), W(5, 7, 2), W(5, 9, 2),
      W(7, 1, 2), W(7, 3, 2), W(7, 5, 2), W(7, 7, 2), W(7, 9, 2),
      W(9, 1, 2), W(9, 3, 2), W(9, 5, 2), W(9, 7, 2), W(9, 9, 2),
  };
  return v;
}
#undef W
}  // namespace tables
}  // namespace blade
