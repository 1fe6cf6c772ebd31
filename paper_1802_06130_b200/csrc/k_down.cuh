// K12 k_down: the fused down-pass at level l — ONE read of z^l produces
//   (a) the bucket map s^l (selector, §3 Eq. 6; R3-R8), and
//   (b) z^{l+1} = 8-tap antialiased bicubic 2x decimation of z^l (§4; R14),
//       written twice: fp64 (input of the next level's selector and decimation) and fp32 (input
//       of the stage kernel and the coarse base u^{L-1} = z^{L-1}).
//
// Precision (H1): the orientation theta = atan2(2B, D)/2 + pi/2 is
// ill-conditioned where the tensor is near-isotropic: an absolute error e in the window sums D, B
// moves theta by ~e / (lambda_1 - lambda_2). Plain fp32 sums (relative error ~1e-7 of the trace)
// flipped orientation buckets far (> 1e-5 rad) from a bin edge at ~1e-5 of pixels. Here the
// gradient differences, the products and the window sums of D = sum (gx^2 - gy^2) and
// B = sum gx gy are fp64, from an fp64 pyramid, so theta is accurate to ~1e-7 rad (the final
// atan2f on the fp32-rounded, well-conditioned vector (D, 2B)). The trace T and the strength /
// coherence decisions are well-conditioned and stay fp32:
//   S >= t  <=>  T/2 + r >= t^2,      C >= t  <=>  r (1 + t^2) >= 2 t T/2   (r = sqrt(D^2/4 + B^2)),
// (the second form avoids the l1 - l2 cancellation), C = 0 when l1 = 0 (R6), theta = 0 when
// D = B = 0 (R5). Gradients use UNSCALED differences (2 gx, 2 gy): every decision is invariant
// to a common positive scale of T, D, B except the strength test, which uses T/8 + r/4.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace blade {

constexpr int kMaxThr2 = 15;
struct DownParams {
  double w64[8];  // window weights e(d) / sum e (fp64)
  float w32[8];   // the same, rounded to fp32
  int n_o, n_s, n_c;
  float ts2[kMaxThr2];               // strength thresholds squared (fp32)
  float tcA[kMaxThr2], tcB[kMaxThr2];  // coherence: 1 + t^2, 2 t  (fp32)
  int tc_nonpos;                      // # coherence thresholds <= 0 (decides C == 0 pixels)
};

namespace down {
constexpr int TX = 32, TY = 16;   // selector outputs per block (level l)
constexpr int R = 3;              // image halo (1 gradient + 2 window) = decimation halo
constexpr int ZR = TY + 2 * R, ZC = TX + 2 * R;  // 22 x 38
constexpr int FR = TY + 4, FC = TX + 4;          // tensor fields 20 x 36
constexpr int DX = TX / 2, DY = TY / 2;          // decimation outputs 16 x 8
}  // namespace down

// Shared memory of one k_down block (dynamic, ~56 KB): t32 is dead once the fields are built, so
// the horizontal-window outputs reuse its space.
struct DownSmem {
  double t64[3][down::ZR][down::ZC];
  double fD[down::FR][down::FC], fB[down::FR][down::FC];
  double hp[3][down::ZR][down::DX];
  float fT[down::FR][down::FC + 1];
  union {
    struct { float t32[3][down::ZR][down::ZC + 1]; } a;
    struct {
      double hD[down::FR][down::TX], hB[down::FR][down::TX];
      float hT[down::FR][down::TX + 1];
    } b;
  } u;
};

template <typename T>
__device__ __forceinline__ T ld_nc(const T* p) { return __ldg(p); }

struct LevelView64 {
  const double* p;
  int H, W, row0, rows;
  long long plane, frame;
};

// grid: (ceil(W / TX), tiles over rows, N); block (32, 8).
// sel rows [s_r0, s_r0 + s_rn) of level l, dec rows [d_r0, d_r0 + d_rn) of level l+1; the block
// tile covers level-l rows [Y0, Y0 + TY) with Y0 = base + 16 * blockIdx.y (base even).
template <typename Tin, int WS, bool DEC>
__global__ void __launch_bounds__(256) k_down(const Tin* __restrict__ zin, int H, int W, int in_row0,
                                               int in_rows, long long in_plane, long long in_frame,
                                               int base, uint8_t* __restrict__ map, int s_r0, int s_rn,
                                               double* __restrict__ z64, float* __restrict__ z32,
                                               int H1, int W1, int d_buf_row0, int d_buf_rows, int d_r0,
                                               int d_rn, DownParams prm) {
  using namespace down;
  static_assert(WS == 5 || WS == 3 || WS == 1, "window radius must fit the 3-pixel halo");
  constexpr int RW = WS / 2;
  extern __shared__ __align__(16) unsigned char dsm[];
  DownSmem& sm = *reinterpret_cast<DownSmem*>(dsm);
  auto& t64 = sm.t64;
  auto& t32 = sm.u.a.t32;
  auto& hD = sm.u.b.hD;
  auto& hB = sm.u.b.hB;
  auto& hT = sm.u.b.hT;
  auto& fD = sm.fD;
  auto& fB = sm.fB;
  auto& fT = sm.fT;
  auto& hp = sm.hp;

  const int n = blockIdx.z;
  const int X0 = blockIdx.x * TX;
  const int Y0 = base + blockIdx.y * TY;
  const int lane = threadIdx.x, wid = threadIdx.y;
  const int tid = wid * 32 + lane;
  const Tin* src = zin + (long long)n * in_frame;

  // ---- stage the folded tile (rows Y0-3 .., cols X0-3 ..), fp64 and fp32 copies
  for (int r = wid; r < ZR; r += 8) {
    int gy = fold_idx(Y0 - R + r, H) - in_row0;
    gy = min(max(gy, 0), in_rows - 1);
    const Tin* rowp = src + (long long)gy * W;
    for (int q = lane; q < ZC; q += 32) {
      const int gx = fold_idx(X0 - R + q, W);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const Tin v = ld_nc(rowp + c * in_plane + gx);
        t64[c][r][q] = (double)v;
        t32[c][r][q] = (float)v;
      }
    }
  }
  __syncthreads();

  // ---- tensor fields at (TY+4) x (TX+4) positions: T (fp32), D, B (fp64); unscaled gradients
  for (int i = tid; i < FR * FC; i += 256) {
    const int r = i / FC, q = i - r * FC;
    float T = 0.0f;
    double D = 0.0, B = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double gx = t64[c][r + 1][q + 2] - t64[c][r + 1][q];
      const double gy = t64[c][r + 2][q + 1] - t64[c][r][q + 1];
      D = fma(gx - gy, gx + gy, D);
      B = fma(gx, gy, B);
      const float fx = t32[c][r + 1][q + 2] - t32[c][r + 1][q];
      const float fy = t32[c][r + 2][q + 1] - t32[c][r][q + 1];
      T = fmaf(fx, fx, fmaf(fy, fy, T));
    }
    fD[r][q] = D;
    fB[r][q] = B;
    fT[r][q] = T;
  }
  // ---- decimation, horizontal pass (independent of the fields)
  if constexpr (DEC) {
    for (int i = tid; i < 3 * ZR * DX; i += 256) {
      const int c = i / (ZR * DX);
      const int rem = i - c * ZR * DX;
      const int r = rem / DX, j = rem - r * DX;
      // output col X0/2 + j reads level cols 2(X0/2+j)-3 .. +4 = local 2j .. 2j+7
      const double* p = &t64[c][r][2 * j];
      double acc = 0.0;
      acc = fma(-3.0 / 256.0, p[0], acc);
      acc = fma(-9.0 / 256.0, p[1], acc);
      acc = fma(29.0 / 256.0, p[2], acc);
      acc = fma(111.0 / 256.0, p[3], acc);
      acc = fma(111.0 / 256.0, p[4], acc);
      acc = fma(29.0 / 256.0, p[5], acc);
      acc = fma(-9.0 / 256.0, p[6], acc);
      acc = fma(-3.0 / 256.0, p[7], acc);
      hp[c][r][j] = acc;
    }
  }
  __syncthreads();

  // ---- horizontal window (TY+4 rows x TX cols)
  for (int i = tid; i < FR * TX; i += 256) {
    const int r = i / TX, j = i - r * TX;
    double D = 0.0, B = 0.0;
    float T = 0.0f;
#pragma unroll
    for (int d = 0; d < WS; ++d) {
      const int q = j + 2 - RW + d;
      D = fma(prm.w64[d], fD[r][q], D);
      B = fma(prm.w64[d], fB[r][q], B);
      T = fmaf(prm.w32[d], fT[r][q], T);
    }
    hD[r][j] = D;
    hB[r][j] = B;
    hT[r][j] = T;
  }
  // ---- decimation, vertical pass -> z^{l+1} (fp64 + fp32)
  if constexpr (DEC) {
    for (int i = tid; i < 3 * DY * DX; i += 256) {
      const int c = i / (DY * DX);
      const int rem = i - c * DY * DX;
      const int r = rem / DX, j = rem - r * DX;
      const int oy = Y0 / 2 + r, ox = X0 / 2 + j;
      if (oy < d_r0 || oy >= d_r0 + d_rn || ox >= W1) continue;
      // output row Y0/2 + r reads level rows 2(Y0/2+r)-3 .. +4 = local 2r .. 2r+7
      double acc = 0.0;
      acc = fma(-3.0 / 256.0, hp[c][2 * r + 0][j], acc);
      acc = fma(-9.0 / 256.0, hp[c][2 * r + 1][j], acc);
      acc = fma(29.0 / 256.0, hp[c][2 * r + 2][j], acc);
      acc = fma(111.0 / 256.0, hp[c][2 * r + 3][j], acc);
      acc = fma(111.0 / 256.0, hp[c][2 * r + 4][j], acc);
      acc = fma(29.0 / 256.0, hp[c][2 * r + 5][j], acc);
      acc = fma(-9.0 / 256.0, hp[c][2 * r + 6][j], acc);
      acc = fma(-3.0 / 256.0, hp[c][2 * r + 7][j], acc);
      const long long o = (long long)n * 3 * d_buf_rows * W1 + ((long long)c * d_buf_rows + (oy - d_buf_row0)) * W1 + ox;
      if (z64) z64[o] = acc;
      z32[o] = (float)acc;
    }
  }
  __syncthreads();

  // ---- vertical window + eigen-features + quantiser
  const float kTwoPiInv = 0.15915494309189535f;
  for (int i = tid; i < TY * TX; i += 256) {
    const int r = i / TX, j = i - r * TX;
    const int oy = Y0 + r, ox = X0 + j;
    if (oy < s_r0 || oy >= s_r0 + s_rn || ox >= W) continue;
    double D = 0.0, B = 0.0;
    float T = 0.0f;
#pragma unroll
    for (int d = 0; d < WS; ++d) {
      const int rr = r + 2 - RW + d;
      D = fma(prm.w64[d], hD[rr][j], D);
      B = fma(prm.w64[d], hB[rr][j], B);
      T = fmaf(prm.w32[d], hT[rr][j], T);
    }
    // unscaled gradients: true (D, B, T) = (D, B, T) / 4
    const float Df = (float)D, Bf = (float)B;
    const float h = 0.125f * T;                                      // (T/4) / 2
    const float r_ = 0.25f * sqrtf(fmaf(0.25f * Df, Df, Bf * Bf));    // sqrt((D/2)^2 + B^2) / 4
    int o = 0;
    if (!(D == 0.0 && B == 0.0)) {
      const float phi = atan2f(2.0f * Bf, Df);
      o = (int)floorf(fmaf(phi, (float)prm.n_o * kTwoPiInv, 0.5f * (float)prm.n_o));
      o %= prm.n_o;
      if (o < 0) o += prm.n_o;
    }
    const float l1 = h + r_;
    int s = 0;
    for (int t = 0; t < prm.n_s - 1; ++t) s += (l1 >= prm.ts2[t]);
    int k;
    if (l1 > 0.0f) {
      k = 0;
      for (int t = 0; t < prm.n_c - 1; ++t) k += (r_ * prm.tcA[t] >= prm.tcB[t] * h);
    } else {
      k = prm.tc_nonpos;
    }
    map[(long long)n * s_rn * W + (long long)(oy - s_r0) * W + ox] = (uint8_t)((o * prm.n_s + s) * prm.n_c + k);
  }
}

}  // namespace blade
