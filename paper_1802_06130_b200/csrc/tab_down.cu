// k_down / k_down_fixup instantiations (tables.h).
#include "tables.h"

namespace blade {
namespace tables {
template <bool FAST, bool WIDE, bool IFIX>
static DownKernel down_kernel_t(bool hilo, bool dec, bool copy) {
  if (hilo) return dec ? &k_down<true, true, FAST, WIDE, false, true, IFIX> : &k_down<true, false, FAST, WIDE, false, true, IFIX>;
  if (copy) return dec ? &k_down<false, true, FAST, WIDE, true, true, IFIX> : &k_down<false, false, FAST, WIDE, true, true, IFIX>;
  return dec ? &k_down<false, true, FAST, WIDE, false, true, IFIX> : &k_down<false, false, FAST, WIDE, false, true, IFIX>;
}
template <bool IFIX>
static DownKernel down_kernel_i(bool hilo, bool dec, bool fast, bool wide, bool copy) {
  if (wide) return down_kernel_t<false, true, IFIX>(hilo, dec, copy);  // FAST implies K = 144
  return fast ? down_kernel_t<true, false, IFIX>(hilo, dec, copy) : down_kernel_t<false, false, IFIX>(hilo, dec, copy);
}
DownKernel down_kernel(bool hilo, bool dec, bool fast, bool wide, bool copy, bool ifix) {
  return ifix ? down_kernel_i<true>(hilo, dec, fast, wide, copy) : down_kernel_i<false>(hilo, dec, fast, wide, copy);
}
DownKernel down_tile_kernel(bool hilo, bool dec, bool wide) {
  if (wide)
    return hilo ? (dec ? &k_down_tile<true, true, true> : &k_down_tile<true, false, true>)
                : (dec ? &k_down_tile<false, true, true> : &k_down_tile<false, false, true>);
  return hilo ? (dec ? &k_down_tile<true, true, false> : &k_down_tile<true, false, false>)
              : (dec ? &k_down_tile<false, true, false> : &k_down_tile<false, false, false>);
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
#ifdef BLADE_TRACE
BT_DEFINE_ACCESS(trace_down)
#endif
}  // namespace tables
}  // namespace blade
