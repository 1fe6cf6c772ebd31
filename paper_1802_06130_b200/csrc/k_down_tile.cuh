// K12' k_down_tile: the down pass at level l for SMALL levels (latency path), the
// same outputs as k_down bit for bit — the bucket map s^l (§3 Eq. 6) and
// z^{l+1} (8-tap decimation, §4) as the hi/lo fp32 pair — from a 2-D tile per
// CTA instead of k_down's vertical strip per warp.
//
// Why: k_down streams RB + 6 rows per warp, one long dependent chain per row (~400 instructions),
// so a small level costs ~10 rows of that chain whatever its size (c1: k_down0 9 us, k_down1
// 11 us on a 256 x 256 level, plus a 7 us fix-up launch; trace in profiles/r02_small_call_*).
// Here every phase is spread over all threads of a CTA with short independent chains:
//   load   the (TY + 6) x (TX + 6) box of z^l around a TY x TX output tile (folded at the image
//          border exactly as k_down folds: rows clamped into the buffer, columns mirrored);
//   P      the gradient products A = sum_c gx^2, B = sum_c gx gy, C = sum_c gy^2 of the
//          (TY + 4) x (TX + 4) window region (fp32, k_down's operation order, incl. the hi/lo
//          gradient (h1 - h0) + (l1 - l0) at l >= 1);
//   H      the horizontal 5-tap window of P: fmaf(w0, p-2 + p+2, fmaf(w1, p-1 + p+1, w2 p0));
//   V      the vertical window in k_down's ring order
//          fmaf(w0, h+2, fmaf(w1, h+1, fmaf(w2, h0, fmaf(w1, h-1, w0 h-2)))), bucket32 (FAST),
//          and the warp's uncertified pixels recomputed in fp64 right away (fix_bucket, as
//          k_down's IFIX form) — no fix-up launch;
//   D      decimation in fp64 from the box converted once: hp (8 taps, k_down's order) per box
//          row and output column, then the 8-row vertical sum in k_down's accumulation order
//          (rows 2Yd-3 .. 2Yd+4 with weights w0..w7), hi = (float)v, lo = (float)(v - hi).
// Identical arithmetic => identical maps and pyramids, so bands / batches / frame loops that
// pick different down kernels stay bit-identical (GPU test: test_down_tile_bit_identical).
// FAST bucket layout only (16 x 3 x 3), no input copy (ragged level-0 rows use k_down).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <type_traits>

#include "k_down.cuh"
#include "kernels.cuh"

namespace blade {

namespace dtile {
constexpr int TY = 16, TX = 32;              // output pixels of level l per CTA
constexpr int THREADS = 256;
constexpr int BR = TY + 6, BC = TX + 6;      // z box: rows Y0-3 .. Y0+TY+2, cols X0-3 .. X0+TX+2
constexpr int PR = TY + 4, PC = TX + 4;      // products: rows Y0-2 .. Y0+TY+1, cols X0-2 .. X0+TX+1
constexpr int DX = TX / 2, DY = TY / 2;      // decimated outputs per tile
__host__ __device__ constexpr size_t smem_bytes(bool hilo, bool dec) {
  return sizeof(float) * 3 * BR * BC * (hilo ? 2 : 1)                    // box (hi, lo)
         + sizeof(float) * 3 * PR * PC + sizeof(float) * 3 * PR * TX      // P, H
         + (dec ? sizeof(double) * 3 * BR * BC + sizeof(double) * 3 * BR * DX : 0);  // zd, hp
}
}  // namespace dtile

// fix_bucket (k_down.cuh) for a tile pixel at box coordinates (r0, q0), reading the staged box
// instead of global memory: the box holds the same folded samples, converted the same way
// ((double)hi + (double)lo), and the lanes, products, weights and butterfly order are
// fix_bucket's, so the fp64 decision is bit-identical — at shared-memory instead of L2 latency
// (the inline fixes were ~6 us of a 512 x 512 call's 47 us).
template <bool HILO, bool DEC>
__device__ __forceinline__ int fix_bucket_box(const float* bh, const float* bl, const double* zd, int r0, int q0,
                                              const DownParams& prm, int lane) {
  using namespace dtile;
  double pa = 0.0, pb = 0.0, pc = 0.0;
  if (lane < 25) {
    const int dy = lane / 5 - 2, dx = lane % 5 - 2;
    auto Z = [&](int c, int r, int q) -> double {
      const int e = (c * BR + r) * BC + q;
      if constexpr (DEC) return zd[e];
      return HILO ? (double)bh[e] + (double)bl[e] : (double)bh[e];
    };
    const int r = r0 + dy, q = q0 + dx;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double gx = Z(c, r, q + 1) - Z(c, r, q - 1);
      const double gy = Z(c, r + 1, q) - Z(c, r - 1, q);
      pa = fma(gx, gx, pa);
      pb = fma(gx, gy, pb);
      pc = fma(gy, gy, pc);
    }
    const double wgt = prm.wp[dy + 2] * prm.wp[dx + 2];
    pa *= wgt;
    pb *= wgt;
    pc *= wgt;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pa += __shfl_xor_sync(0xffffffffu, pa, o);
    pb += __shfl_xor_sync(0xffffffffu, pb, o);
    pc += __shfl_xor_sync(0xffffffffu, pc, o);
  }
  return bucket_of<true>(pa, pb, pc, prm);
}

// grid: ceil(W / TX) x ceil(span / TY) x N CTAs of 256 threads; tile rows from a.base (even).
template <bool HILO, bool DEC, bool WIDE>
__global__ void __launch_bounds__(dtile::THREADS) k_down_tile(const DownArgs a, const DownParams prm) {
  using namespace dtile;
  using MT = typename std::conditional<WIDE, uint16_t, uint8_t>::type;
  extern __shared__ __align__(16) unsigned char dts[];
  double* zd = reinterpret_cast<double*>(dts);                    // [3][BR][BC] (DEC)
  double* hp = zd + (DEC ? 3 * BR * BC : 0);                       // [3][BR][DX] (DEC)
  float* bh = reinterpret_cast<float*>(hp + (DEC ? 3 * BR * DX : 0));  // [3][BR][BC]
  float* bl = bh + 3 * BR * BC;                                    // [3][BR][BC] (HILO)
  float* P = bl + (HILO ? 3 * BR * BC : 0);                        // [3][PR][PC]
  float* Hs = P + 3 * PR * PC;                                     // [3][PR][TX]
  const int tid = threadIdx.x;
  const int X0 = blockIdx.x * TX, Y0 = a.base + blockIdx.y * TY, n = blockIdx.z;
  BT_ENTRY(HILO ? 1 : 0);
  pdl_trigger();
  pdl_wait();
  BT_WAITED(HILO ? 1 : 0);

  // ---- load the box (k_down's fold: buffer row of the folded global row, clamped; folded column)
  //      2-D mapping: lane -> columns tx, tx + 32; warp -> rows w, w + 8, ...; the folds and the
  //      row offsets are computed once per column / row, not per element. DEC converts to fp64
  //      as it stores (the decimation's (double)hi + (double)lo).
  const int tx = tid & 31, wp = tid >> 5;
  constexpr int NW = THREADS / 32;
  {
    const int fq0 = fold_idx(X0 - 3 + tx, a.W);
    const int fq1 = tx + 32 < BC ? fold_idx(X0 + 29 + tx, a.W) : 0;
    const float* fh = a.zhi + (long long)n * a.in_frame;
    const float* fl = HILO ? a.zlo + (long long)n * a.in_frame : nullptr;
#pragma unroll
    for (int rk = 0; rk < (BR + NW - 1) / NW; ++rk) {
      const int r = wp + rk * NW;
      if (r >= BR) break;
      int br = fold_idx(Y0 - 3 + r, a.H) - a.in_row0;
      br = min(max(br, 0), a.in_rows - 1);
      const long long ro = (long long)br * a.in_pitch;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const long long o = c * a.in_plane + ro;
        const int s0 = (c * BR + r) * BC + tx;
        const float h0 = fh[o + fq0];
        const float l0 = HILO ? fl[o + fq0] : 0.0f;
        bh[s0] = h0;
        if constexpr (HILO) bl[s0] = l0;
        if constexpr (DEC) zd[s0] = HILO ? (double)h0 + (double)l0 : (double)h0;
        if (tx + 32 < BC) {
          const float h1 = fh[o + fq1];
          const float l1 = HILO ? fl[o + fq1] : 0.0f;
          bh[s0 + 32] = h1;
          if constexpr (HILO) bl[s0 + 32] = l1;
          if constexpr (DEC) zd[s0 + 32] = HILO ? (double)h1 + (double)l1 : (double)h1;
        }
      }
    }
  }
  __syncthreads();

  // ---- P: products at (Y0 - 2 + i, X0 - 2 + j) <- box centre (i + 1, j + 1)
  auto product = [&](int i, int j) {
    float A = 0.0f, B = 0.0f, C = 0.0f;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float* h = bh + (c * BR + i + 1) * BC + j + 1;
      float gx = h[1] - h[-1], gy = h[BC] - h[-BC];
      if constexpr (HILO) {
        const float* l = bl + (c * BR + i + 1) * BC + j + 1;
        gx += l[1] - l[-1];
        gy += l[BC] - l[-BC];
      }
      A = fmaf(gx, gx, A);
      B = fmaf(gx, gy, B);
      C = fmaf(gy, gy, C);
    }
    const int e = i * PC + j;
    P[e] = A;
    P[PR * PC + e] = B;
    P[2 * PR * PC + e] = C;
  };
#pragma unroll
  for (int ik = 0; ik < (PR + NW - 1) / NW; ++ik) {
    const int i = wp + ik * NW;
    if (i >= PR) break;
    product(i, tx);
    if (tx + 32 < PC) product(i, tx + 32);
  }
  __syncthreads();
  const float w0 = (float)prm.wp[0], w1 = (float)prm.wp[1], w2 = (float)prm.wp[2];  // symmetric

  // ---- H: horizontal window at (Y0 - 2 + i, X0 + tx) over P columns tx .. tx + 4
#pragma unroll
  for (int ik = 0; ik < (PR + NW - 1) / NW; ++ik) {
    const int i = wp + ik * NW;
    if (i >= PR) break;
#pragma unroll
    for (int qd = 0; qd < 3; ++qd) {
      const float* p = P + (qd * PR + i) * PC + tx + 2;
      Hs[(qd * PR + i) * TX + tx] = fmaf(w0, p[-2] + p[2], fmaf(w1, p[-1] + p[1], w2 * p[0]));
    }
  }
  if constexpr (DEC) {
    // ---- D1: hp at box row r, decimated column X0/2 + k (input columns X0 + 2k - 3 .. + 4 =
    //      box columns 2k .. 2k + 7), k_down's order; (c, r) rows of 16 columns, two per warp
    constexpr double dw0 = -3.0 / 256.0, dw1 = -9.0 / 256.0, dw2 = 29.0 / 256.0, dw3 = 111.0 / 256.0;
    static_assert(DX == 16, "D1 maps 16 decimated columns to a half warp");
#pragma unroll
    for (int ek = 0; ek < (3 * BR * DX + THREADS - 1) / THREADS; ++ek) {
      const int e = tid + ek * THREADS;
      if (e >= 3 * BR * DX) break;
      const int cr = e >> 4, k = e & 15;  // cr = c * BR + r
      const double* z = zd + cr * BC + 2 * k + 3;  // input column X0 + 2k
      double h = dw0 * (z[-3] + z[4]);
      h = fma(dw1, z[-2] + z[3], h);
      h = fma(dw2, z[-1] + z[2], h);
      h = fma(dw3, z[0] + z[1], h);
      hp[e] = h;
    }
  }
  __syncthreads();

  // ---- V + bucket: pixel (Y0 + i, X0 + j); a warp = one tile row (coalesced map stores)
  MT* mapf = static_cast<MT*>(a.map) + (long long)n * a.s_rn * a.map_pitch;
  static_assert(TY % NW == 0, "V: whole warps per tile row");
#pragma unroll
  for (int ik = 0; ik < TY / NW; ++ik) {
    const int i = wp + ik * NW;
    const int j = tx;
    const int y = Y0 + i, x = X0 + j;
    float f[3];
#pragma unroll
    for (int qd = 0; qd < 3; ++qd) {
      const float* h = Hs + (qd * PR + i + 2) * TX + j;  // H row of y
      f[qd] = fmaf(w0, h[2 * TX], fmaf(w1, h[TX], fmaf(w2, h[0], fmaf(w1, h[-TX], w0 * h[-2 * TX]))));
    }
    bool safe = true;
    int bk = bucket32<true>(f[0], f[1], f[2], prm, safe);
    const bool emit = y >= a.s_r0 && y < a.s_r0 + a.s_rn && x < a.W;
#ifdef BLADE_TILE_NOFIX  // timing probe only: outputs invalid
    unsigned int m = 0;
#else
    unsigned int m = __ballot_sync(0xffffffffu, emit && !safe);  // rare: fp64 fix, whole warp
#endif
    const int lane = tx;
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const int k = fix_bucket_box<HILO, DEC>(bh, bl, zd, i + 3, src + 3, prm, lane);  // j = lane
      if (lane == src) bk = k;
    }
    if (emit) mapf[(long long)(y - a.s_r0) * a.map_pitch + x] = (MT)bk;
  }

  if constexpr (DEC) {
    // ---- D2: z^{l+1} row Yd = Y0/2 + i (rows 2Yd-3 .. 2Yd+4 = box rows 2i .. 2i+7), k_down's
    //      accumulation order (the ring adds w0 .. w7 in row order onto 0)
    constexpr double dw0 = -3.0 / 256.0, dw1 = -9.0 / 256.0, dw2 = 29.0 / 256.0, dw3 = 111.0 / 256.0;
    static_assert(DY == 8 && DX == 16, "D2 index by shifts");
#pragma unroll
    for (int ek = 0; ek < (3 * DY * DX + THREADS - 1) / THREADS; ++ek) {
      const int e = tid + ek * THREADS;
      if (e >= 3 * DY * DX) break;
      const int c = e >> 7, i = (e >> 4) & 7, k = e & 15;
      const int Yd = Y0 / 2 + i, Xd = X0 / 2 + k;
      if (Yd < a.d_r0 || Yd >= a.d_r0 + a.d_rn || Xd >= a.W1) continue;
      const double* h = hp + (c * BR + 2 * i) * DX + k;
      double v = fma(dw0, h[0], 0.0);
      v = fma(dw1, h[DX], v);
      v = fma(dw2, h[2 * DX], v);
      v = fma(dw3, h[3 * DX], v);
      v = fma(dw3, h[4 * DX], v);
      v = fma(dw2, h[5 * DX], v);
      v = fma(dw1, h[6 * DX], v);
      v = fma(dw0, h[7 * DX], v);
      const long long o = ((long long)n * 3 + c) * a.d_buf_rows * a.out_pitch + (long long)(Yd - a.d_buf_row0) * a.out_pitch + Xd;
      const float hi = (float)v;
      a.ohi[o] = hi;
      if (a.olo) a.olo[o] = (float)(v - (double)hi);
    }
  }
  BT_EXIT(HILO ? 1 : 0);
}

}  // namespace blade
