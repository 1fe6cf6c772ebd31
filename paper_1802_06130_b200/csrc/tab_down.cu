// k_down / k_down_fixup instantiations (tables.h).
#include "tables.h"

namespace blade {
namespace tables {
template <bool FAST>
static DownKernel down_kernel_t(bool hilo, bool dec) {
  if (hilo) return dec ? &k_down<true, true, FAST> : &k_down<true, false, FAST>;
  return dec ? &k_down<false, true, FAST> : &k_down<false, false, FAST>;
}
DownKernel down_kernel(bool hilo, bool dec, bool fast) {
  return fast ? down_kernel_t<true>(hilo, dec) : down_kernel_t<false>(hilo, dec);
}
DownKernel fixup_kernel(bool hilo, bool fast) {
  if (hilo) return fast ? &k_down_fixup<true, true> : &k_down_fixup<true, false>;
  return fast ? &k_down_fixup<false, true> : &k_down_fixup<false, false>;
}
}  // namespace tables
}  // namespace blade
