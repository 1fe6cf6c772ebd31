// k_stage_ph instantiations (tables.h).
#include "tables.h"

namespace blade {
namespace tables {
template <int NF, int NC>
static TmaVariant make_ph() {
  using SS = PhShape<NF, NC>;
  return TmaVariant{NF, NC, 2, &k_stage_ph<NF, NC>, SS::stage_bytes, SS::TROWS, SS::TCOLS,
                    SS::FCB, SS::FR, SS::CCB, SS::CR, SS::RF, SS::RC, SS::S, true};
}
const std::vector<TmaVariant>& ph_variants() {
  static const std::vector<TmaVariant> v = {
      make_ph<7, 7>(), make_ph<9, 9>(), make_ph<7, 5>(), make_ph<9, 7>(), make_ph<5, 7>(), make_ph<7, 9>(),
  };
  return v;
}
}  // namespace tables
}  // namespace blade
