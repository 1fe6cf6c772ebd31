// Training kernel instantiations (NEXT f4; tables.h).
#include "tables.h"

namespace blade {
namespace tables {
template <int NF, int NC, bool WIDE>
static TrainVariant make_train() {
  return TrainVariant{NF, NC, TrainShape<NF, NC>::NTP, &k_train_gram_mma<NF, NC, WIDE>, WIDE,
                      &k_train_gram<NF, NC, WIDE>};
}
const std::vector<TrainVariant>& train_variants() {
  static const std::vector<TrainVariant> v = {
      make_train<3, 0, false>(), make_train<5, 0, false>(), make_train<7, 0, false>(), make_train<9, 0, false>(),
      make_train<3, 3, false>(), make_train<5, 3, false>(), make_train<5, 5, false>(), make_train<7, 5, false>(),
      make_train<7, 7, false>(),
      make_train<5, 5, true>(), make_train<7, 5, true>(), make_train<7, 7, true>(), make_train<7, 0, true>(),
  };
  return v;
}
TrainKernel train_hist(bool wide) { return wide ? &k_train_hist<true> : &k_train_hist<false>; }
TrainKernel train_scatter(bool wide) { return wide ? &k_train_scatter<true> : &k_train_scatter<false>; }
TrainKernel train_scan() { return &k_train_scan<>; }
}  // namespace tables
}  // namespace blade
