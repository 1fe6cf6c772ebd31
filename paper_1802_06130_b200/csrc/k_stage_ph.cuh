// K3'' k_stage_ph: the stage of Eq. 9 (§4) for pair banks too large to keep all
// four phases in one CTA's shared memory (7x7 + 7x7: 226 KB, 9x9 + 9x9: 373 KB for 4 x 144 filters;
// BASELINE.json configs[2], configs[4]).
//
// CTAs are specialised by output phase p = 2 (y mod 2) + (x mod 2) (R9): a CTA keeps the
// 144 filters of its phase (58 / 94 KB, tma_tap_off layout) and computes only the pixels of that
// phase, so every thread block is a 2 x 2 block of the phase's sub-lattice (image pixels 2 apart).
// Two 128-thread groups per CTA each own one TMA tile buffer (fine patch of z^l, coarse patch of
// u^{l+1}, bucket tile of a 16 x 128 image tile) on an mbarrier and alternate tiles, so one
// group computes while the other's TMA is in flight. The four phase-CTAs of a tile read the same
// patches (L2 hits). Border cells are fixed up by the fold (R2) as in k_stage_tma.
// FP32 FMA on the CUDA cores; taps shared by R, G, B (R13); LDS.128 tap rows.
#pragma once
#include <cuda.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "k_stage_tma.cuh"

namespace blade {

template <int NF, int NC>
struct PhShape {
  static constexpr int BX = 32, BY = 4;             // threads per group
  static constexpr int threads = BX * BY;           // 128
  static constexpr int RF = NF / 2, RC = NC / 2;
  static constexpr int SUBR = 2 * BY, SUBC = 2 * BX;  // phase sub-lattice tile 8 x 64 (2 x 2 per thread)
  static constexpr int TROWS = 2 * SUBR, TCOLS = 2 * SUBC;  // image tile 16 x 128
  static constexpr int FM = 4, CM = 4;              // 16-B aligned TMA box starts (column margins)
  static constexpr int FR = TROWS - 1 + 2 * RF;     // fine rows Y0 + py - RF .. Y0 + py + TROWS - 2 + RF
  static constexpr int FCB = TCOLS + 2 * FM;        // 136: columns X0 - 4 .. X0 + 131
  static constexpr int CR = SUBR + 2 * RC;          // coarse rows Y0/2 - RC .. Y0/2 + SUBR - 1 + RC
  static constexpr int CCB = SUBC + 2 * CM;         // 72
  static constexpr int FW = 2 * RF + 3;             // fine window columns per thread
  static constexpr int CW = 2 * RC + 2;             // coarse window columns per thread
  static constexpr int fine_bytes = 3 * FR * FCB * 4;
  static constexpr int coarse_bytes = 3 * CR * CCB * 4;
  static constexpr int map_bytes = TROWS * TCOLS;
  static constexpr int al(int x) { return (x + 127) & ~127; }
  static constexpr int fine_off = 0;
  static constexpr int coarse_off = al(fine_bytes);
  static constexpr int map_off = coarse_off + al(coarse_bytes);
  static constexpr int stage_bytes = map_off + al(map_bytes);
  static constexpr int S = tma_tap_stride(NF, NC);
  static_assert(RF <= FM && RC <= CM, "halo wider than the TMA margin");
};

// One tile of phase (py, PX) by one 128-thread group: fix-up of border cells, then the 2 x 2
// sub-lattice block of each thread.
// CH3 (per-channel Y/Cb/Cr banks, NEXT f1): the CTA also serves one channel chn; after the
// fix-up the fine patch (RGB z^l) is converted to channel chn in plane 0, the coarse patch too
// when it is z^{L-1} (RGB), else plane chn of the YCbCr u^{l+1} is read; one accumulator per pixel.
template <int NF, int NC, int PX, bool CH3>
__device__ __forceinline__ void ph_tile(const StageTmaArgs& a, int n, int X0, int Y0, int py, float* sfine,
                                       float* scoarse, const uint8_t* smap, const float* sbank, int tid,
                                       int tx, int ty, int g, int chn) {
  using SS = PhShape<NF, NC>;
  constexpr int RF = SS::RF, RC = SS::RC;
  constexpr int PL = CH3 ? 1 : 3;
  auto group_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(SS::threads) : "memory"); };
  const int FY = Y0 + py - RF, FX = X0 - SS::FM;          // fine box origin
  const int CY = Y0 / 2 - RC, CX = X0 / 2 - SS::CM;       // coarse box origin
  const bool fine_border = FX < 0 || FX + SS::FCB > a.W || FY < 0 || FY + SS::FR > a.H;
  const bool coarse_border = CX < 0 || CX + SS::CCB > a.W1 || CY < 0 || CY + SS::CR > a.H1;
  if (fine_border || coarse_border) {
    if (fine_border) {
      const OobBox ob = oob_box(SS::FR, SS::FCB, FY, FX, a.H, a.W);
      for (int i = tid; i < ob.n; i += SS::threads) {
        int r, q;
        oob_cell(ob, i, r, q);
        const int gy = FY + r, gx = FX + q;
        const int fy = fold_idx(gy, a.H), fx = fold_idx(gx, a.W);
        const int ry = fy - FY, rx = fx - FX;
        const bool in_tile = ry >= 0 && ry < SS::FR && rx >= 0 && rx < SS::FCB;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float v;
          if (in_tile) {
            v = sfine[(c * SS::FR + ry) * SS::FCB + rx];
          } else {
            const int by = min(max(fy - a.z_row0, 0), a.z_rows - 1);
            v = a.z[(((long long)n * 3 + c) * a.z_rows + by) * a.z_pitch + fx];
          }
          sfine[(c * SS::FR + r) * SS::FCB + q] = v;
        }
      }
    }
    if (coarse_border) {
      const OobBox ob = oob_box(SS::CR, SS::CCB, CY, CX, a.H1, a.W1);
      for (int i = tid; i < ob.n; i += SS::threads) {
        int r, q;
        oob_cell(ob, i, r, q);
        const int gy = CY + r, gx = CX + q;
        const int fy = fold_idx(gy, a.H1), fx = fold_idx(gx, a.W1);
        const int ry = fy - CY, rx = fx - CX;
        const bool in_tile = ry >= 0 && ry < SS::CR && rx >= 0 && rx < SS::CCB;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float v;
          if (in_tile) {
            v = scoarse[(c * SS::CR + ry) * SS::CCB + rx];
          } else {
            const int by = min(max(fy - a.u_row0, 0), a.u_rows - 1);
            v = a.u1[(((long long)n * 3 + c) * a.u_rows + by) * a.u_pitch + fx];
          }
          scoarse[(c * SS::CR + r) * SS::CCB + q] = v;
        }
      }
    }
    group_sync();
  }
  const float* scoarse_c = scoarse;
  if constexpr (CH3) {  // colour conversion of the staged patches into plane 0
    for (int i = tid; i < SS::FR * SS::FCB; i += SS::threads)
      sfine[i] = rgb_to_ycc_ch(chn, sfine[i], sfine[SS::FR * SS::FCB + i], sfine[2 * SS::FR * SS::FCB + i]);
    if (a.u_rgb) {
      for (int i = tid; i < SS::CR * SS::CCB; i += SS::threads)
        scoarse[i] = rgb_to_ycc_ch(chn, scoarse[i], scoarse[SS::CR * SS::CCB + i], scoarse[2 * SS::CR * SS::CCB + i]);
    } else {
      scoarse_c = scoarse + chn * SS::CR * SS::CCB;
    }
    group_sync();
  }

  // ---- this thread's 2 x 2 sub-lattice block: image pixels (Y0 + py + 4 ty + 2 i, X0 + PX + 4 tx + 2 j);
  //      a block wholly outside the image / the output rows issues no shared-memory traffic
  {
    const int y0 = Y0 + py + 4 * ty, x0 = X0 + PX + 4 * tx;
    if (x0 >= a.W || y0 >= a.o_r0 + a.o_rn || y0 + 2 < a.o_r0) return;
  }
  const float* tp[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int k = smap[(py + 4 * ty + 2 * i) * SS::TCOLS + PX + 4 * tx + 2 * j];
      tp[i][j] = sbank + k * SS::S;
    }
  float acc[2][2][PL];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < PL; ++c) acc[i][j][c] = 0.0f;

  // coarse: pixel (i, j) has centre (Y0/2 + 2ty + i, X0/2 + 2tx + j); window rows 2ty + i + dy,
  // columns (box) 2tx + j + dx + CM - RC
  constexpr int CO = SS::CM - RC;
#pragma unroll
  for (int wr = 0; wr < NC + 1; ++wr) {
    float v[PL][SS::CW];
#pragma unroll
    for (int c = 0; c < PL; ++c)
      lds_run<(CO & 1), SS::CW, 2>(scoarse_c + (c * SS::CR + 2 * ty + wr) * SS::CCB + 2 * tx + CO, v[c]);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int dy = wr - i;
      if (dy < 0 || dy >= NC) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float t[NC];
        load_tap_row<NF, NC, 1>(tp[i][j], dy, t);
#pragma unroll
        for (int dx = 0; dx < NC; ++dx)
#pragma unroll
          for (int c = 0; c < PL; ++c) acc[i][j][c] = fmaf(t[dx], v[c][j + dx], acc[i][j][c]);
      }
    }
  }
  // fine: pixel (i, j) window rows 4ty + 2i + dy (box rows from Y0 + py - RF), columns (box)
  // PX + 4tx + 2j + dx + FM - RF
  constexpr int FO = PX + SS::FM - RF;
#pragma unroll
  for (int wr = 0; wr < NF + 2; ++wr) {
    float v[PL][SS::FW];
#pragma unroll
    for (int c = 0; c < PL; ++c)
      lds_run<(FO & 3), SS::FW>(sfine + (c * SS::FR + 4 * ty + wr) * SS::FCB + 4 * tx + FO, v[c]);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int dy = wr - 2 * i;
      if (dy < 0 || dy >= NF) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float t[NF];
        load_tap_row<NF, NC, 0>(tp[i][j], dy, t);
#pragma unroll
        for (int dx = 0; dx < NF; ++dx)
#pragma unroll
          for (int c = 0; c < PL; ++c) acc[i][j][c] = fmaf(t[dx], v[c][2 * j + dx], acc[i][j][c]);
      }
    }
  }

  // ---- store
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int yy = Y0 + py + 4 * ty + 2 * i;
    if (yy < a.o_r0 || yy >= a.o_r0 + a.o_rn) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int xx = X0 + PX + 4 * tx + 2 * j;
      if (xx >= a.W) continue;
      float* op = a.out + ((long long)n * 3 * a.out_rows + (yy - a.out_row0)) * a.out_pitch + xx;
#pragma unroll
      for (int c = 0; c < PL; ++c) {
        float v = acc[i][j][c];
        if (a.clamp) v = fminf(fmaxf(v, 0.0f), 1.0f);
        op[(long long)(CH3 ? chn : c) * a.out_rows * a.out_pitch] = v;
      }
    }
  }
}

// grid: 4 * m CTAs (CTA b serves phase b % 4; with CH3 12 * m, channel (b / 4) % 3), 256 threads =
// 2 groups of 128; n_tiles counts the 16 x 128 image tiles; each type's 2m workers stride over them.
template <int NF, int NC, bool CH3>
__global__ void __launch_bounds__(256, 1)
    k_stage_ph(const __grid_constant__ CUtensorMap tm_z, const __grid_constant__ CUtensorMap tm_u,
               const __grid_constant__ CUtensorMap tm_map, StageTmaArgs a) {
  using SS = PhShape<NF, NC>;
  constexpr int RF = SS::RF, RC = SS::RC;
  extern __shared__ __align__(128) unsigned char ph_smem[];
  unsigned char* buf0 = ph_smem;
  float* sbank = reinterpret_cast<float*>(ph_smem + 2 * SS::stage_bytes);
  const int bank_floats = a.K * SS::S;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(ph_smem + 2 * SS::stage_bytes + ((bank_floats * 4 + 127) & ~127));

  const int p = blockIdx.x & 3, py = p >> 1, px = p & 1;
  const int chn = CH3 ? (int)(blockIdx.x >> 2) % 3 : 0;   // filter channel (CH3)
  const int ci = CH3 ? (int)(blockIdx.x >> 2) / 3 : (int)(blockIdx.x >> 2);  // CTA index within its type
  const int g = threadIdx.y >> 2;                          // group (0, 1)
  const int tx = threadIdx.x, ty = threadIdx.y & 3;
  const int tid = ty * SS::BX + tx;                        // within the group
  const int ctid = threadIdx.y * SS::BX + threadIdx.x;
  const int cpp = gridDim.x / (CH3 ? 12 : 4);              // CTAs per (phase, channel) type
  const int workers = 2 * cpp;
  constexpr uint32_t tx_bytes = SS::fine_bytes + SS::coarse_bytes + SS::map_bytes;

  auto tile_coords = [&](int t, int& n, int& X0, int& Y0) {
    n = t / (a.tiles_x * a.tiles_y);
    const int rem = t - n * a.tiles_x * a.tiles_y;
    const int tyi = rem / a.tiles_x;
    X0 = (rem - tyi * a.tiles_x) * SS::TCOLS;
    Y0 = a.y_base + tyi * SS::TROWS;
  };
  auto issue = [&](int t) {
    int n, X0, Y0;
    tile_coords(t, n, X0, Y0);
    unsigned char* sb = buf0 + g * SS::stage_bytes;
    mbar_expect_tx(&mbar[g], tx_bytes);
    tma_load_3d(sb + SS::fine_off, &tm_z, X0 - SS::FM, Y0 + py - RF - a.z_row0, n * 3, &mbar[g]);
    tma_load_3d(sb + SS::coarse_off, &tm_u, X0 / 2 - SS::CM, Y0 / 2 - RC - a.u_row0, n * 3, &mbar[g]);
    tma_load_3d(sb + SS::map_off, &tm_map, X0, Y0 - a.map_row0, n, &mbar[g]);
  };

  // large levels: a CTA's two groups take adjacent tiles (shared halo rows in L2); small levels
  // (fewer tiles than groups): group 1 starts after every CTA's group 0, one tile per SM
  int t = a.n_tiles >= 2 * cpp ? ci * 2 + g : ci + g * cpp;
  pdl_trigger();
  if (ctid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&mbar[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the bank (constant data): one bulk copy, issued before waiting on the previous grid
    mbar_expect_tx(&mbar[2], (uint32_t)bank_floats * 4u);
    bulk_g2s(sbank, a.bank + (long long)(chn * 4 + p) * a.PS, (uint32_t)bank_floats * 4u, &mbar[2]);
  }
  pdl_wait();
  __syncthreads();
  if (tid == 0 && t < a.n_tiles) issue(t);
  mbar_wait(&mbar[2], 0);

  for (int it = 0; t < a.n_tiles; ++it, t += workers) {
    int n, X0, Y0;
    tile_coords(t, n, X0, Y0);
    mbar_wait(&mbar[g], it & 1);
    float* sfine = reinterpret_cast<float*>(buf0 + g * SS::stage_bytes + SS::fine_off);
    float* scoarse = reinterpret_cast<float*>(buf0 + g * SS::stage_bytes + SS::coarse_off);
    const uint8_t* smap = buf0 + g * SS::stage_bytes + SS::map_off;
    if (px)
      ph_tile<NF, NC, 1, CH3>(a, n, X0, Y0, py, sfine, scoarse, smap, sbank, tid, tx, ty, g, chn);
    else
      ph_tile<NF, NC, 0, CH3>(a, n, X0, Y0, py, sfine, scoarse, smap, sbank, tid, tx, ty, g, chn);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(SS::threads) : "memory");  // buffer free
    if (tid == 0 && t + workers < a.n_tiles) {
      fence_proxy_async();
      issue(t + workers);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// K3 (two-phase form) k_stage_p2: the same stage for pair banks whose TWO phases of one output-row
// parity fit a CTA next to two tile buffers (7x7 + 7x7: 2 x 57.6 KB; BASELINE.json configs[2]).
// CTAs are specialised by row parity py (phases 2 py and 2 py + 1, one bulk copy); a thread
// computes 2 rows of parity py (image rows 2 apart) x 4 CONSECUTIVE columns (both column phases),
// so a window row segment (NF + 3 fine / NC + 1 coarse values) feeds 4 pixels instead of 2: 45%
// fewer window loads per pixel than k_stage_ph's 2 x 2 sub-lattice blocks. Same boxes, groups,
// tile order and per-pixel fmaf order (coarse then fine, dy then dx) as k_stage_ph: bit-identical.
template <int NF, int NC>
__device__ __forceinline__ void p2_tile(const StageTmaArgs& a, int n, int X0, int Y0, int py, float* sfine,
                                       float* scoarse, const uint8_t* smap, const float* sbank, int tid, int tx,
                                       int ty, int g) {
  using SS = PhShape<NF, NC>;
  constexpr int RF = SS::RF, RC = SS::RC;
  auto group_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(SS::threads) : "memory"); };
  const int FY = Y0 + py - RF, FX = X0 - SS::FM;          // fine box origin
  const int CY = Y0 / 2 - RC, CX = X0 / 2 - SS::CM;       // coarse box origin
  const bool fine_border = FX < 0 || FX + SS::FCB > a.W || FY < 0 || FY + SS::FR > a.H;
  const bool coarse_border = CX < 0 || CX + SS::CCB > a.W1 || CY < 0 || CY + SS::CR > a.H1;
  if (fine_border || coarse_border) {
    if (fine_border) {
      const OobBox ob = oob_box(SS::FR, SS::FCB, FY, FX, a.H, a.W);
      for (int i = tid; i < ob.n; i += SS::threads) {
        int r, q;
        oob_cell(ob, i, r, q);
        const int fy = fold_idx(FY + r, a.H), fx = fold_idx(FX + q, a.W);
        const int ry = fy - FY, rx = fx - FX;
        const bool in_tile = ry >= 0 && ry < SS::FR && rx >= 0 && rx < SS::FCB;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float v;
          if (in_tile) {
            v = sfine[(c * SS::FR + ry) * SS::FCB + rx];
          } else {
            const int by = min(max(fy - a.z_row0, 0), a.z_rows - 1);
            v = a.z[(((long long)n * 3 + c) * a.z_rows + by) * a.z_pitch + fx];
          }
          sfine[(c * SS::FR + r) * SS::FCB + q] = v;
        }
      }
    }
    if (coarse_border) {
      const OobBox ob = oob_box(SS::CR, SS::CCB, CY, CX, a.H1, a.W1);
      for (int i = tid; i < ob.n; i += SS::threads) {
        int r, q;
        oob_cell(ob, i, r, q);
        const int fy = fold_idx(CY + r, a.H1), fx = fold_idx(CX + q, a.W1);
        const int ry = fy - CY, rx = fx - CX;
        const bool in_tile = ry >= 0 && ry < SS::CR && rx >= 0 && rx < SS::CCB;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float v;
          if (in_tile) {
            v = scoarse[(c * SS::CR + ry) * SS::CCB + rx];
          } else {
            const int by = min(max(fy - a.u_row0, 0), a.u_rows - 1);
            v = a.u1[(((long long)n * 3 + c) * a.u_rows + by) * a.u_pitch + fx];
          }
          scoarse[(c * SS::CR + r) * SS::CCB + q] = v;
        }
      }
    }
    group_sync();
  }

  // ---- this thread's block: image rows Y0 + py + 4 ty + 2 i (i < 2), columns X0 + 4 tx + j (j < 4)
  const int y0 = Y0 + py + 4 * ty, x0 = X0 + 4 * tx;
  if (x0 >= a.W || y0 >= a.o_r0 + a.o_rn || y0 + 2 < a.o_r0) return;
  int toff[2][4];  // column phase (j & 1) x PS + bucket x S
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const uint32_t mrow = *reinterpret_cast<const uint32_t*>(smap + (py + 4 * ty + 2 * i) * SS::TCOLS + 4 * tx);
#pragma unroll
    for (int j = 0; j < 4; ++j) toff[i][j] = (j & 1) * a.PS + (int)((mrow >> (8 * j)) & 0xff) * SS::S;
  }
  float acc[2][4][3];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[i][j][c] = 0.0f;

  // coarse: pixel (i, j) has centre (Y0/2 + 2ty + i, X0/2 + 2tx + j/2); window rows 2ty + i + dy,
  // box columns 2tx + CO + j/2 + dx
  constexpr int CO = SS::CM - RC, CWIN = NC + 1;
#pragma unroll
  for (int wr = 0; wr < NC + 1; ++wr) {
    float v[3][CWIN];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      lds_run<(CO & 1), CWIN, 2>(scoarse + (c * SS::CR + 2 * ty + wr) * SS::CCB + 2 * tx + CO, v[c]);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int dy = wr - i;
      if (dy < 0 || dy >= NC) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float t[NC];
        load_tap_row<NF, NC, 1>(sbank + toff[i][j], dy, t);
#pragma unroll
        for (int dx = 0; dx < NC; ++dx)
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[i][j][c] = fmaf(t[dx], v[c][(j >> 1) + dx], acc[i][j][c]);
      }
    }
  }
  // fine: pixel (i, j) window rows 4ty + 2i + dy (box rows from Y0 + py - RF), box columns
  // 4tx + FO + j + dx
  constexpr int FO = SS::FM - RF, FWIN = NF + 3;
#pragma unroll
  for (int wr = 0; wr < NF + 2; ++wr) {
    float v[3][FWIN];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      lds_run<(FO & 3), FWIN>(sfine + (c * SS::FR + 4 * ty + wr) * SS::FCB + 4 * tx + FO, v[c]);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int dy = wr - 2 * i;
      if (dy < 0 || dy >= NF) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float t[NF];
        load_tap_row<NF, NC, 0>(sbank + toff[i][j], dy, t);
#pragma unroll
        for (int dx = 0; dx < NF; ++dx)
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[i][j][c] = fmaf(t[dx], v[c][j + dx], acc[i][j][c]);
      }
    }
  }

  // ---- store (rows y0 + 2i; columns x0 .. x0 + 3; output rows are 16-B multiples)
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int yy = y0 + 2 * i;
    if (yy < a.o_r0 || yy >= a.o_r0 + a.o_rn) continue;
    float* op = a.out + ((long long)n * 3 * a.out_rows + (yy - a.out_row0)) * a.out_pitch + x0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float v0 = acc[i][0][c], v1 = acc[i][1][c], v2 = acc[i][2][c], v3 = acc[i][3][c];
      if (a.clamp) {
        v0 = fminf(fmaxf(v0, 0.0f), 1.0f);
        v1 = fminf(fmaxf(v1, 0.0f), 1.0f);
        v2 = fminf(fmaxf(v2, 0.0f), 1.0f);
        v3 = fminf(fmaxf(v3, 0.0f), 1.0f);
      }
      float* d = op + (long long)c * a.out_rows * a.out_pitch;
      if (x0 + 3 < a.W) {
        *reinterpret_cast<float4*>(d) = make_float4(v0, v1, v2, v3);
      } else {
        d[0] = v0;
        if (x0 + 1 < a.W) d[1] = v1;
        if (x0 + 2 < a.W) d[2] = v2;
      }
    }
  }
}

// grid: 2 * m CTAs (CTA b serves output-row parity b % 2), 256 threads = 2 groups of 128.
template <int NF, int NC>
__global__ void __launch_bounds__(256, 1)
    k_stage_p2(const __grid_constant__ CUtensorMap tm_z, const __grid_constant__ CUtensorMap tm_u,
               const __grid_constant__ CUtensorMap tm_map, StageTmaArgs a) {
  using SS = PhShape<NF, NC>;
  constexpr int RF = SS::RF, RC = SS::RC;
  extern __shared__ __align__(128) unsigned char p2_smem[];
  unsigned char* buf0 = p2_smem;
  float* sbank = reinterpret_cast<float*>(p2_smem + 2 * SS::stage_bytes);
  const int bank_floats = 2 * a.PS;  // phases 2 py, 2 py + 1
  uint64_t* mbar = reinterpret_cast<uint64_t*>(p2_smem + 2 * SS::stage_bytes + ((bank_floats * 4 + 127) & ~127));

  const int py = blockIdx.x & 1;
  const int ci = (int)(blockIdx.x >> 1);                   // CTA index within its parity
  const int g = threadIdx.y >> 2;                          // group (0, 1)
  const int tx = threadIdx.x, ty = threadIdx.y & 3;
  const int tid = ty * SS::BX + tx;                        // within the group
  const int ctid = threadIdx.y * SS::BX + threadIdx.x;
  const int cpp = gridDim.x / 2;                           // CTAs per parity
  const int workers = 2 * cpp;
  constexpr uint32_t tx_bytes = SS::fine_bytes + SS::coarse_bytes + SS::map_bytes;

  auto tile_coords = [&](int t, int& n, int& X0, int& Y0) {
    n = t / (a.tiles_x * a.tiles_y);
    const int rem = t - n * a.tiles_x * a.tiles_y;
    const int tyi = rem / a.tiles_x;
    X0 = (rem - tyi * a.tiles_x) * SS::TCOLS;
    Y0 = a.y_base + tyi * SS::TROWS;
  };
  auto issue = [&](int t) {
    int n, X0, Y0;
    tile_coords(t, n, X0, Y0);
    unsigned char* sb = buf0 + g * SS::stage_bytes;
    mbar_expect_tx(&mbar[g], tx_bytes);
    tma_load_3d(sb + SS::fine_off, &tm_z, X0 - SS::FM, Y0 + py - RF - a.z_row0, n * 3, &mbar[g]);
    tma_load_3d(sb + SS::coarse_off, &tm_u, X0 / 2 - SS::CM, Y0 / 2 - RC - a.u_row0, n * 3, &mbar[g]);
    tma_load_3d(sb + SS::map_off, &tm_map, X0, Y0 - a.map_row0, n, &mbar[g]);
  };

  int t = a.n_tiles >= 2 * cpp ? ci * 2 + g : ci + g * cpp;
  pdl_trigger();
  if (ctid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&mbar[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&mbar[2], (uint32_t)bank_floats * 4u);
    bulk_g2s(sbank, a.bank + (long long)(2 * py) * a.PS, (uint32_t)bank_floats * 4u, &mbar[2]);
  }
  pdl_wait();
  __syncthreads();
  if (tid == 0 && t < a.n_tiles) issue(t);
  mbar_wait(&mbar[2], 0);

  for (int it = 0; t < a.n_tiles; ++it, t += workers) {
    int n, X0, Y0;
    tile_coords(t, n, X0, Y0);
    mbar_wait(&mbar[g], it & 1);
    float* sfine = reinterpret_cast<float*>(buf0 + g * SS::stage_bytes + SS::fine_off);
    float* scoarse = reinterpret_cast<float*>(buf0 + g * SS::stage_bytes + SS::coarse_off);
    const uint8_t* smap = buf0 + g * SS::stage_bytes + SS::map_off;
    p2_tile<NF, NC>(a, n, X0, Y0, py, sfine, scoarse, smap, sbank, tid, tx, ty, g);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(SS::threads) : "memory");  // buffer free
    if (tid == 0 && t + workers < a.n_tiles) {
      fence_proxy_async();
      issue(t + workers);
    }
  }
}

}  // namespace blade
