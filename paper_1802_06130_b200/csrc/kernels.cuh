// Shared definitions of the hot-path kernels (B200, sm_100a) and the generic stage kernel.
//
//   k_down      (k_down.cuh)      : fused decimation + selector at level l (K1 + K2)
//   k_stage_tma (k_stage_tma.cuh) : Eq. 9 / Eq. 1 stage with TMA double-buffered tiles (K3)
//   k_stage     (this file)       : Eq. 9 stage, generic fallback: CTAs specialised by output-row
//                                   parity so 7x7 / 9x9 pair banks fit; synchronous staging (K3')
//
// All arithmetic is FP32 on the CUDA cores (no fast-math flag: IEEE div, accurate atan2f; the one
// approximate operation is sqrt.approx.f32 in the FAST selector's strength / coherence tests,
// DESIGN.md R22).
// Tensor cores are not used: every pixel contracts with its own selected filter, so the
// contraction is a batched dot product, not a GEMM.
//
// Images are viewed through LevelView: a level of a batch, possibly a row band of it. Every
// index is GLOBAL (rows of the full level image); folds happen at the true image border
// (R2 / H7), so a band computes bit-identical values to the full image.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <type_traits>

namespace blade {

struct LevelView {
  float* p;         // frame 0, channel 0, buffer row 0
  int H, W;         // global level dims
  int row0, rows;   // the buffer holds global rows [row0, row0 + rows)
  long long plane;  // floats per channel plane of the buffer (rows * pitch)
  long long frame;  // floats per frame of the buffer (3 * plane)
  int pitch;        // floats per buffer row (>= W; padded to a multiple of 4 in the workspace)
};

// Programmatic dependent launch (sm_90+): the host launches every kernel of a cascade after the
// first with programmatic stream serialisation, so its CTAs can be scheduled (and do work that
// does not read the previous kernel's output, e.g. loading the bank) while the previous grid
// drains. pdl_wait() blocks until the previous grid has completed and its writes are visible;
// pdl_trigger() lets the next grid launch. Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// BLADE_TRACE builds (latency probes only): per kernel kind, the first CTA entry, the last
// griddepcontrol.wait return and the last warp exit (%globaltimer ns), read by blade_ms_trace().
#ifdef BLADE_TRACE
static __device__ unsigned long long g_trace[16][3];
__device__ __forceinline__ unsigned long long bt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BT_ENTRY(k) \
  if (threadIdx.x == 0 && threadIdx.y == 0) atomicMin(&g_trace[k][0], bt_now())
#define BT_WAITED(k) \
  if (threadIdx.x == 0 && threadIdx.y == 0) atomicMax(&g_trace[k][1], bt_now())
#define BT_EXIT(k) \
  if ((threadIdx.x & 31) == 0) atomicMax(&g_trace[k][2], bt_now())
#define BT_DEFINE_ACCESS(name)                                                              \
  void name(unsigned long long* out, bool reset) {                                          \
    if (out) cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace));                           \
    if (reset) {                                                                            \
      unsigned long long init[16][3];                                                       \
      for (int i = 0; i < 16; ++i) init[i][0] = ~0ull, init[i][1] = 0, init[i][2] = 0;      \
      cudaMemcpyToSymbol(g_trace, init, sizeof(init));                                      \
    }                                                                                       \
  }
#else
#define BT_ENTRY(k)
#define BT_WAITED(k)
#define BT_EXIT(k)
#endif
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// [R2] half-sample symmetric fold, periodic with period 2n.
__device__ __forceinline__ int fold_idx(int i, int n) {
  if (i >= 0 && i < n) return i;
  if (i < 0 && i >= -n) return -i - 1;
  if (i >= n && i < 2 * n) return 2 * n - 1 - i;
  int p = 2 * n;
  int m = i % p;
  if (m < 0) m += p;
  return m < n ? m : p - 1 - m;
}

// Buffer row of global row y (folded), clamped into the buffer as a safety net.
__device__ __forceinline__ int view_row(const LevelView& v, int y) {
  int r = fold_idx(y, v.H) - v.row0;
  return min(max(r, 0), v.rows - 1);
}

// ------------------------------------------------------------------------------------------
// K3' stage (Eq. 9 / Eq. 1), generic fallback. Persistent CTAs: each CTA copies the filterbank of its stage (the
// phases it needs) into shared memory ONCE and then loops over output tiles. Per tile it
// stages the fine patch of z^l (tile + r_f halo, 3 channels) and the coarse patch of u^{l+1}
// (tile/2 + r_c halo) in shared memory, folded at the true image border. Each thread computes
// a 2 x 2 pixel block: columns x, x+1 (same coarse column floor(x/2)) and rows y, y+RS.
//   RS == 1: a CTA holds all phases; its rows are contiguous (a 2x2 quad shares the coarse
//            centre).
//   RS == 2: CTAs are specialised by output-row parity (the bank of two phases fits in
//            shared memory for 7x7 / 9x9 pairs); a thread computes rows y and y + 2.
// The three colour channels share the taps [R13]: one tap load feeds 3 FMAs.
// ------------------------------------------------------------------------------------------
struct StageArgs {
  LevelView z;         // z^l
  LevelView u1;        // u^{l+1} (unused when NC == 0)
  LevelView out;       // u^l (output rows [out_r0, out_r0 + out_rn))
  const void* map;     // s^l, [N][map_rows][map_pitch] uint8 (uint16 when WIDE), row 0 = global row map_row0
  int map_row0, map_rows, map_pitch;
  const float* bank;   // device bank of this stage: [phase][PS floats: K x S taps, padded]
  int K, S, PS;        // buckets, padded tap stride (odd), phase stride (multiple of 4)
  int n_phases;        // 1 or 4
  int N;               // frames
  int out_r0, out_rn;  // global output rows
  int tiles_x, tiles_y, n_tiles;
  int clamp;           // clamp output to [0, 1]
  int u_rgb;           // CH3: the coarse input is RGB (z^{L-1}) rather than YCbCr planes
};

// Full-range BT.601 on the [0, 1] scale (R25), channel ch of (R, G, B).
__device__ __forceinline__ float rgb_to_ycc_ch(int ch, float R, float G, float B) {
  const float Y = fmaf(0.299f, R, fmaf(0.587f, G, 0.114f * B));
  const float kO = 128.0f / 255.0f;
  if (ch == 0) return Y;
  if (ch == 1) return fmaf(0.564f, B - Y, kO);
  return fmaf(0.713f, R - Y, kO);
}

template <int NF, int NC, int RS, int BY, bool CH3 = false>
struct StageShape {
  static constexpr int BX = 32;
  static constexpr int RF = NF / 2, RC = NC / 2;
  static constexpr int TCOLS = 2 * BX;             // output columns per tile
  static constexpr int TROWS = 2 * BY * RS;        // output rows per tile (span)
  static constexpr int FR = TROWS + 2 * RF;        // fine tile rows
  static constexpr int FC = TCOLS + 2 * RF;        // fine tile cols
  static constexpr int FCP = FC + ((FC & 1) ? 1 : 2);  // even pitch (float2 loads)
  static constexpr int CR = NC ? TROWS / 2 + 2 * RC : 0;
  static constexpr int CC = NC ? BX + 2 * RC : 0;
  static constexpr int CCP = NC ? CC + 1 : 0;
  static constexpr int NPH_CTA = RS == 2 ? 2 : 4;  // phases a CTA holds when n_phases == 4
  static constexpr int PL = CH3 ? 1 : 3;            // staged planes (CH3: the CTA's channel only)
  static constexpr int tile_floats = PL * FR * FCP + PL * CR * CCP;
  static constexpr int threads = BX * BY;
};

// CH3 (per-channel YCbCr banks, NEXT f1): CTAs are also specialised by channel c (Y, Cb, Cr); the
// fine patch (RGB z^l) is converted to channel c while staged, the coarse patch too when it is
// z^{L-1} (RGB), else it is plane c of the YCbCr u^{l+1}; the output is plane c of a YCbCr u^l
// (level 0 is converted back to RGB by k_ycc_to_rgb).
// WIDE (NEXT f2, K > 256): uint16 bucket maps and the bank read from global memory (L2-resident).
// GBANK: the bank read from global memory (default: when WIDE); with uint8 maps it serves the
// K <= 256 banks whose two phases do not fit next to a tile (e.g. 5 + 9 taps at K = 256: 219 KB).
template <int NF, int NC, int RS, int BY, bool CH3, bool WIDE = false, bool GBANK = WIDE>
__global__ void __launch_bounds__(32 * BY) k_stage(StageArgs a) {
  static_assert(GBANK || !WIDE, "K > 256 banks are read from global memory");
  using SS = StageShape<NF, NC, RS, BY, CH3>;
  using MT = typename std::conditional<WIDE, uint16_t, uint8_t>::type;
  constexpr int PL = SS::PL;
  constexpr int RF = SS::RF, RC = SS::RC;
  extern __shared__ __align__(16) float smem[];
  const int nph_cta = a.n_phases == 4 ? SS::NPH_CTA : 1;
  const int bank_floats = GBANK ? 0 : nph_cta * a.PS;
  float* sbank = smem;
  float* sfine = smem + ((bank_floats + 3) & ~3);
  float* scoarse = sfine + PL * SS::FR * SS::FCP;

  const int par = RS == 2 ? (int)(blockIdx.x & 1) : 0;  // output-row parity of this CTA
  const int rest = RS == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int chn = CH3 ? rest % 3 : 0;                    // filter channel of this CTA
  const int group = CH3 ? rest / 3 : rest;
  const int ngroups = (int)gridDim.x / (RS * (CH3 ? 3 : 1));
  const int tid = threadIdx.y * SS::BX + threadIdx.x;
  pdl_trigger();

  // ---- filterbank -> shared memory, once per CTA (GBANK: read in place from global memory)
  const int ph0 = (a.n_phases == 4 && RS == 2) ? 2 * par : 0;
  const long long boff = (long long)(chn * a.n_phases + ph0) * a.PS;
  const float* bank = GBANK ? a.bank + boff : sbank;
  if (!GBANK) {
    const float4* g4 = reinterpret_cast<const float4*>(a.bank + boff);
    float4* s4 = reinterpret_cast<float4*>(sbank);
    const int n4 = bank_floats >> 2;
    for (int i = tid; i < n4; i += SS::threads) s4[i] = __ldg(g4 + i);
    for (int i = (n4 << 2) + tid; i < bank_floats; i += SS::threads) sbank[i] = __ldg(a.bank + boff + i);
  }
  pdl_wait();  // the bank is constant; everything below reads the previous kernels' outputs

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int y_base = (a.out_r0 & ~1);  // tiles start on an even global row

  for (int t = group; t < a.n_tiles; t += ngroups) {
    const int n = t / (a.tiles_x * a.tiles_y);
    const int rem = t - n * a.tiles_x * a.tiles_y;
    const int tyi = rem / a.tiles_x, txi = rem - tyi * a.tiles_x;
    const int X0 = txi * SS::TCOLS;
    const int Y0 = y_base + tyi * SS::TROWS;

    __syncthreads();  // previous tile's reads of the staging buffers are done
    // ---- stage the fine patch (rows Y0-RF .., cols X0-RF ..)
    {
      const float* zp = a.z.p + (long long)n * a.z.frame;
      for (int i = tid; i < SS::FR * SS::FC; i += SS::threads) {
        const int r = i / SS::FC, q = i - r * SS::FC;
        const long long ro = (long long)view_row(a.z, Y0 - RF + r) * a.z.pitch + fold_idx(X0 - RF + q, a.z.W);
        if constexpr (CH3) {
          sfine[r * SS::FCP + q] =
              rgb_to_ycc_ch(chn, __ldg(zp + ro), __ldg(zp + a.z.plane + ro), __ldg(zp + 2 * a.z.plane + ro));
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            sfine[(c * SS::FR + r) * SS::FCP + q] = __ldg(zp + c * a.z.plane + ro);
        }
      }
    }
    if constexpr (NC > 0) {
      const float* up = a.u1.p + (long long)n * a.u1.frame;
      const int CY0 = Y0 / 2 - RC, CX0 = X0 / 2 - RC;
      for (int i = tid; i < SS::CR * SS::CC; i += SS::threads) {
        const int r = i / SS::CC, q = i - r * SS::CC;
        const long long ro = (long long)view_row(a.u1, CY0 + r) * a.u1.pitch + fold_idx(CX0 + q, a.u1.W);
        if constexpr (CH3) {
          scoarse[r * SS::CCP + q] =
              a.u_rgb ? rgb_to_ycc_ch(chn, __ldg(up + ro), __ldg(up + a.u1.plane + ro), __ldg(up + 2 * a.u1.plane + ro))
                      : __ldg(up + chn * a.u1.plane + ro);
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            scoarse[(c * SS::CR + r) * SS::CCP + q] = __ldg(up + c * a.u1.plane + ro);
        }
      }
    }
    __syncthreads();

    // ---- this thread's 2x2 block
    const int x = X0 + 2 * tx;                               // even column
    const int ly = RS == 2 ? 4 * ty + par : 2 * ty;          // local row of pixel row 0
    const int y0 = Y0 + ly;
    const bool row_ok[2] = {y0 >= a.out_r0 && y0 < a.out_r0 + a.out_rn,
                            y0 + RS >= a.out_r0 && y0 + RS < a.out_r0 + a.out_rn};
    const bool col_ok[2] = {x < a.z.W, x + 1 < a.z.W};
    if (!(row_ok[0] || row_ok[1]) || !col_ok[0]) continue;

    const float* tp[2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int yy = y0 + i * RS, xx = min(x + j, a.z.W - 1);
        int k = 0;
        if (row_ok[i])
          k = static_cast<const MT*>(a.map)[(long long)n * a.map_rows * a.map_pitch +
                                            (long long)(yy - a.map_row0) * a.map_pitch + xx];
        int ps = 0;
        if (a.n_phases == 4) ps = RS == 2 ? j : 2 * (yy & 1) + j;
        tp[i][j] = bank + ps * a.PS + k * a.S;
      }

    float acc[2][2][PL];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int c = 0; c < PL; ++c) acc[i][j][c] = 0.0f;

    // coarse term first (matches nothing in particular; any order is a valid fp32 sum)
    if constexpr (NC > 0) {
      // coarse centre row of pixel row i: (y0 + i*RS)/2 -> local (ly + i*RS)/2 + RC - RC
      const int cx = tx;  // local coarse col of the window start (centre tx + RC)
#pragma unroll
      for (int wr = 0; wr < NC + (RS == 2 ? 1 : 0); ++wr) {
        const int crow = (ly >> 1) + wr;  // local coarse row
        float v[PL][NC];
#pragma unroll
        for (int c = 0; c < PL; ++c)
#pragma unroll
          for (int q = 0; q < NC; ++q) v[c][q] = scoarse[(c * SS::CR + crow) * SS::CCP + cx + q];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int dy = wr - (RS == 2 ? i : 0);
          if (dy < 0 || dy >= NC) continue;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int dx = 0; dx < NC; ++dx) {
              const float tap = GBANK ? __ldg(tp[i][j] + NF * NF + dy * NC + dx) : tp[i][j][NF * NF + dy * NC + dx];
#pragma unroll
              for (int c = 0; c < PL; ++c) acc[i][j][c] = fmaf(tap, v[c][dx], acc[i][j][c]);
            }
        }
      }
    }
    // fine term
#pragma unroll
    for (int wr = 0; wr < NF + RS; ++wr) {
      const int frow = ly + wr;  // local fine row (tile origin is Y0 - RF)
      float v[PL][NF + 1];
#pragma unroll
      for (int c = 0; c < PL; ++c) {
        const float* rp = sfine + (c * SS::FR + frow) * SS::FCP + 2 * tx;
#pragma unroll
        for (int q = 0; q + 1 < NF + 1; q += 2) {
          const float2 t2 = *reinterpret_cast<const float2*>(rp + q);
          v[c][q] = t2.x;
          v[c][q + 1] = t2.y;
        }
        if ((NF + 1) & 1) v[c][NF] = rp[NF];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int dy = wr - i * RS;
        if (dy < 0 || dy >= NF) continue;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int dx = 0; dx < NF; ++dx) {
            const float tap = GBANK ? __ldg(tp[i][j] + dy * NF + dx) : tp[i][j][dy * NF + dx];
#pragma unroll
            for (int c = 0; c < PL; ++c) acc[i][j][c] = fmaf(tap, v[c][j + dx], acc[i][j][c]);
          }
      }
    }

    // ---- store
    float* op = a.out.p + (long long)n * a.out.frame;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (!row_ok[i]) continue;
      const long long ro = (long long)(y0 + i * RS - a.out.row0) * a.out.pitch;
#pragma unroll
      for (int c = 0; c < PL; ++c) {
        float v0 = acc[i][0][c], v1 = acc[i][1][c];
        if (a.clamp) {
          v0 = fminf(fmaxf(v0, 0.0f), 1.0f);
          v1 = fminf(fmaxf(v1, 0.0f), 1.0f);
        }
        float* d = op + (CH3 ? chn : c) * a.out.plane + ro + x;
        if (col_ok[1] && ((reinterpret_cast<uintptr_t>(d) & 7) == 0)) {
          *reinterpret_cast<float2*>(d) = make_float2(v0, v1);
        } else {
          d[0] = v0;
          if (col_ok[1]) d[1] = v1;
        }
      }
    }
  }
}

// Plane-by-plane row copy between pitches: dst[p][y][x] = src[p][y][x], x < W, for `planes`
// planes of H rows (the level-0 output of a full image whose rows are not 16-B multiples is
// staged in the workspace with 16-B rows for the TMA stage kernel, then copied out).
template <int = 0>
__global__ void k_copy_rows(float* dst, int dst_pitch, const float* src, int src_pitch, long long planes, int H,
                            int W) {
  pdl_trigger();
  pdl_wait();
  const long long total = planes * H * (long long)W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / W;
    const int x = (int)(i - row * W);
    dst[row * dst_pitch + x] = src[row * src_pitch + x];
  }
}

// YCbCr -> RGB in place over rows [0, rows) of a level view (exact inverse of rgb_to_ycc_ch up
// to fp32 rounding; R25), with the optional final clamp.
template <int = 0>
__global__ void k_ycc_to_rgb(float* p, long long plane, long long frame, long long per_frame, int N, int clamp) {
  pdl_trigger();
  pdl_wait();
  const long long total = (long long)N * per_frame;
  const float kO = 128.0f / 255.0f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long n = i / per_frame, o = i - n * per_frame;
    float* q = p + n * frame + o;
    const float Y = q[0], Cb = q[plane], Cr = q[2 * plane];
    float R = Y + (Cr - kO) / 0.713f;
    float B = Y + (Cb - kO) / 0.564f;
    float G = (Y - 0.299f * R - 0.114f * B) / 0.587f;
    if (clamp) {
      R = fminf(fmaxf(R, 0.0f), 1.0f);
      G = fminf(fmaxf(G, 0.0f), 1.0f);
      B = fminf(fmaxf(B, 0.0f), 1.0f);
    }
    q[0] = R;
    q[plane] = G;
    q[2 * plane] = B;
  }
}

}  // namespace blade
