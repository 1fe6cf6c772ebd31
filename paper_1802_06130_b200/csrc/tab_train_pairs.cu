// Training kernel instantiations for the remaining footprints the Gram kernels hold (n_f^2 + n_c^2
// <= 123: upper 4 x 4 blocks of the normal equations over at most two passes of 256 threads;
// NEXT f4, tables.h). 7 + 9, 9 + 7 and 9 + 9 pairs stay BLADE_EUNSUPPORTED for training.
#include "tables.h"

namespace blade {
namespace tables {
template <int NF, int NC, bool WIDE>
static TrainVariant make_train() {
  return TrainVariant{NF, NC, TrainShape<NF, NC>::NTP, &k_train_gram_mma<NF, NC, WIDE>, WIDE,
                      &k_train_gram<NF, NC, WIDE>};
}
const std::vector<TrainVariant>& train_variants_pairs() {
  static const std::vector<TrainVariant> v = {
      make_train<1, 0, false>(), make_train<1, 1, false>(), make_train<1, 3, false>(), make_train<1, 5, false>(),
      make_train<1, 7, false>(), make_train<1, 9, false>(), make_train<3, 1, false>(), make_train<3, 5, false>(),
      make_train<3, 7, false>(), make_train<3, 9, false>(), make_train<5, 1, false>(), make_train<5, 7, false>(),
      make_train<5, 9, false>(), make_train<7, 1, false>(), make_train<7, 3, false>(), make_train<9, 1, false>(),
      make_train<9, 3, false>(), make_train<9, 5, false>(),
  };
  return v;
}
}  // namespace tables
}  // namespace blade
