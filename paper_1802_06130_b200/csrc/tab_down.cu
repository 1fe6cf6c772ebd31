// k_down / k_down_fixup instantiations (tables.h).
#include "tables.h"

namespace blade {
namespace tables {
template <bool FAST, bool WIDE>
static DownKernel down_kernel_t(bool hilo, bool dec, bool copy) {
  if (hilo) return dec ? &k_down<true, true, FAST, WIDE> : &k_down<true, false, FAST, WIDE>;
  if (copy) return dec ? &k_down<false, true, FAST, WIDE, true> : &k_down<false, false, FAST, WIDE, true>;
  return dec ? &k_down<false, true, FAST, WIDE> : &k_down<false, false, FAST, WIDE>;
}
DownKernel down_kernel(bool hilo, bool dec, bool fast, bool wide, bool copy) {
  if (wide) return down_kernel_t<false, true>(hilo, dec, copy);  // FAST implies K = 144
  return fast ? down_kernel_t<true, false>(hilo, dec, copy) : down_kernel_t<false, false>(hilo, dec, copy);
}
DownKernel dec_kernel(bool copy) {
  return copy ? &k_down<false, true, true, false, true, false> : &k_down<false, true, true, false, false, false>;
}
DownKernel fixup_kernel(bool hilo, bool fast, bool wide) {
  if (wide) return hilo ? &k_down_fixup<true, false, true> : &k_down_fixup<false, false, true>;
  if (hilo) return fast ? &k_down_fixup<true, true, false> : &k_down_fixup<true, false, false>;
  return fast ? &k_down_fixup<false, true, false> : &k_down_fixup<false, false, false>;
}
FixupMultiKernel fixup_multi_kernel(bool fast, bool wide) {
  if (wide) return &k_down_fixup_multi<false, true>;
  return fast ? &k_down_fixup_multi<true, false> : &k_down_fixup_multi<false, false>;
}
}  // namespace tables
}  // namespace blade
