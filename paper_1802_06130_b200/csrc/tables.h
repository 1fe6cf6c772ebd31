// Kernel tables: every kernel instantiation the host orchestrator (blade_ms.cu) can launch,
// defined in its own translation unit (tab_down.cu, tab_stage.cu, tab_tma.cu, tab_ph.cu) so the
// library builds in parallel. Launches go through the typed __global__ function pointers.
#pragma once
#include <cuda.h>
#include <vector>

#include "k_down.cuh"
#include "k_down_tile.cuh"
#include "k_stage_ph.cuh"
#include "k_stage_tma.cuh"
#include "k_train.cuh"
#include "kernels.cuh"

namespace blade {
namespace tables {

using StageKernel = void (*)(StageArgs);
struct StageVariant {
  int nf, nc, rs, by;
  StageKernel fn;
  int tile_floats, threads, trows, tcols;
  bool ch3;   // per-channel (Y, Cb, Cr) banks: CTAs specialised by channel (NEXT f1)
  bool wide;  // K > 256: uint16 maps, bank read from global memory (NEXT f2)
  bool gbank = false;  // uint8 maps with the bank read from global memory (K <= 256 banks too large for shared memory)
};
// Generic stage kernels (any shape; row-parity CTAs for the big pair banks).
const std::vector<StageVariant>& stage_variants();
// the remaining fine / coarse pairs of the ABI's range (tab_stage_pairs.cu: shared banks;
// tab_stage_pairs2.cu: per-channel and K > 256 banks)
const std::vector<StageVariant>& stage_variants_pairs();
const std::vector<StageVariant>& stage_variants_pairs2();
// every footprint with uint8 maps and the bank in global memory (tab_stage_gbank.cu): the fallback
// when no shared-bank variant fits
const std::vector<StageVariant>& stage_variants_gbank();
// per-channel banks with K > 256 (tab_stage_ch3wide.cu): uint16 maps, bank in global memory
const std::vector<StageVariant>& stage_variants_ch3_wide();

using TmaKernel = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, StageTmaArgs);
struct TmaVariant {
  int nf, nc, groups;
  int by;  // warps per group (16 / pixel rows per thread); k_stage_ph: 4
  TmaKernel fn;
  int stage_bytes, trows, tcols, fcb, fr, ccb, cr, rf, rc, S;
  bool phase_split;  // k_stage_ph: CTAs specialised by output phase, one phase's bank each
  bool ch3;          // per-channel (Y, Cb, Cr) banks
  bool wide;         // K > 256: uint16 maps, bank read from global memory (NEXT f2)
  // the fused-selector form of the same kernel (level 0; nullptr if none): taller fine box
  TmaKernel fsel_fn = nullptr;
  int fsel_stage_bytes = 0, fsel_fr = 0;
  int ry = 2;  // pixel rows per thread (k_stage_tma)
  int ptypes = 4;  // phase-split kernels: CTA types per channel (k_stage_ph: 4 phases; k_stage_p2: 2
                   // row parities holding two phases each)
};
using StageFixKernel = void (*)(const StageFixArgs, const DownParams);
StageFixKernel stage_fixup_kernel(int nf, int nc);  // nullptr if none
// TMA stage kernels: the shapes whose whole (all-phase) bank fits next to two staging buffers.
const std::vector<TmaVariant>& tma_variants();
// the same for per-channel banks with K > 256 (tab_tma_ch3wide.cu)
const std::vector<TmaVariant>& tma_variants_ch3_wide();
// Phase-split TMA stage kernels: pair banks whose four phases do not fit one CTA.
const std::vector<TmaVariant>& ph_variants();
// Row-parity TMA stage kernels (two phases per CTA): pair banks whose two phases fit one CTA.
const std::vector<TmaVariant>& p2_variants();

using DownKernel = void (*)(const DownArgs, const DownParams);
// FAST: the configs' bucket layout (16 orientations x 3 strength x 3 coherence bins)
// wide: uint16 bucket maps (K > 256, NEXT f2)
DownKernel down_kernel(bool hilo, bool dec, bool fast, bool wide, bool copy = false, bool ifix = false);
DownKernel fixup_kernel(bool hilo, bool fast, bool wide);
// the small-level form of k_down (k_down_tile.cuh: 2-D tiles, inline fp64 fixes; FAST layout)
DownKernel down_tile_kernel(bool hilo, bool dec, bool wide);
// level-0 decimation (+ input copy) without the selector: the fused-selector stage computes s^0
DownKernel dec_kernel(bool copy);
using FixupMultiKernel = void (*)(const FixupMulti);
FixupMultiKernel fixup_multi_kernel(bool fast, bool wide);

// Training (NEXT f4): segmented fp64 SYRK of the normal equations.
using TrainKernel = void (*)(const TrainArgs);
struct TrainVariant {
  int nf, nc, ntp;
  TrainKernel gram;      // FP64 tensor-core (DMMA) accumulation
  bool wide;
  TrainKernel gram_dfma; // the same on the FP64 CUDA cores (BLADE_TRAIN_MMA=0)
};
const std::vector<TrainVariant>& train_variants();
const std::vector<TrainVariant>& train_variants_pairs();  // the other footprints with n_f^2 + n_c^2 <= 123
TrainKernel train_hist(bool wide);
TrainKernel train_scatter(bool wide);
TrainKernel train_scan();

#ifdef BLADE_TRACE
void trace_down(unsigned long long* out, bool reset);  // [16][3]: entry, waited, exit (ns)
void trace_tma(unsigned long long* out, bool reset);
#endif
}  // namespace tables
}  // namespace blade
