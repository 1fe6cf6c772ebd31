// K12 k_down: the fused down-pass at level l (register-streaming). ONE read of z^l gives
//   (a) the bucket map s^l (selector; §3 Eq. 6; R3-R8), and
//   (b) z^{l+1} = 8-tap antialiased bicubic 2x decimation of z^l (§4; R14),
//       stored as an fp32 pair (hi = round(z), lo = round(z - hi)): hi is the stage input and the
//       coarse base u^{L-1}; hi + lo (exact to ~2^-48) feeds the next level's selector/decimation.
//
// Work decomposition: one WARP streams down a vertical strip of 64 columns of one
// frame, RB output rows at a time; lane j owns columns x = X0 + 2j, x + 1 (X0 = 56 s - 4) and the
// decimated column x / 2. Lanes 2..29 produce outputs (56 columns per strip); lanes 0, 1, 30, 31
// only supply the horizontal halo (gradient 1 + window 2 columns; decimation 3 / 4 columns).
// Horizontal neighbours come from warp shuffles, vertical neighbours from registers:
//   - each lane prefetches its own two columns of the next rows with 4-byte cp.async into a
//     lane-private ring in shared memory (RING rows deep, no cross-lane smem traffic, no barrier);
//   - gradients (unscaled: 2 g), the products A = sum_c gx^2, B = sum_c gx gy, C = sum_c gy^2
//     and the 5x5 Gaussian window are fp64 (the window runs as a horizontal pass over shuffled
//     neighbour products and a 5-deep vertical ring of pending output rows);
//   - decimation: horizontal 8 taps over shuffled neighbours, then a 4-deep vertical ring.
//
// Precision (DESIGN.md §6 H1): theta = atan2(2B, A - C) / 2 + pi / 2 is ill-conditioned where the
// tensor is near-isotropic (an absolute error e in the window sums moves theta by ~e/(l1 - l2)),
// so every sum that feeds theta is fp64 from an exact fp64 pyramid; the final atan2f runs on the
// fp32-rounded, well-conditioned vector (A - C, 2B). Strength and coherence decisions are
// well-conditioned and use the fp32 tests of k_down.cuh:
//   S >= t <=> T/2 + r >= t^2,   C >= t <=> r (1 + t^2) >= 2 t T/2   (r = sqrt((A-C)^2/4 + B^2)).
// fp32 -> fp64 conversions run at 16/clk/SM on B200 (measured, scripts/probes/tput.cu), so each
// element is converted exactly once, by the lane that loads it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace blade {

constexpr int kMaxThr2 = 15;
struct DownParams {
  double wp[5];                        // window weights at offsets -2..2 (zero-padded for WS < 5)
  int n_o, n_s, n_c;
  float ts2[kMaxThr2];   // strength thresholds squared (-inf for t <= 0, +inf padding)
  float kc2[kMaxThr2];   // positive coherence thresholds: (2t / (1 + t^2))^2 (+inf padding)
  int tc_nonpos;         // # coherence thresholds <= 0 (always passed)
  int quad_edges;        // n_o % 4 == 0 and n_o <= 64: quadrant + edge-count orientation
  float ecos[16], esin[16];  // interior edges 2 pi j / n_o, j = 1 .. n_o/4 - 1
};

namespace down {
constexpr int WARPS = 4;        // independent warps per CTA
constexpr int RING = 8;         // rows in flight per lane (cp.async ring)
constexpr int STRIP = 56;       // output columns per strip
constexpr int LANE_LO = 2, LANE_HI = 29;
}  // namespace down

struct DownArgs {
  const float* zhi;  // level l (hi plane, or the fp32 input at l = 0): [N][3][in_rows][W]
  const float* zlo;  // level l lo plane (nullptr at l = 0)
  int H, W, in_row0, in_rows;
  long long in_plane, in_frame;
  uint8_t* map;      // s^l rows [s_r0, s_r0 + s_rn), pitch W, frame stride s_rn * W
  int s_r0, s_rn;
  float* ohi;        // z^{l+1} hi: rows [d_buf_row0, + d_buf_rows), pitch W1 (nullptr: no dec)
  float* olo;        // z^{l+1} lo (nullptr: not needed, l + 1 is the coarsest level)
  int H1, W1, d_buf_row0, d_buf_rows, d_r0, d_rn;
  int base, RB, n_strips, n_bands, n_tasks;
};

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double shfl_up_d(double v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
__device__ __forceinline__ double shfl_dn_d(double v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }

// Bucket of one pixel from the windowed (unscaled x4) tensor sums a = sum w gx^2, b = sum w gx gy,
// c = sum w gy^2 (fp64), with no atan2 and no sqrt (DESIGN.md §6 k_down):
//   orientation: theta = (phi + pi) / 2 with phi = atan2(2b, a - c); o = floor(theta n_o / pi) is
//     the bin of psi = angle of (X, Y) = (c - a, -2b) in [0, 2 pi) with bins 2 pi / n_o. The
//     quadrant of (X, Y) gives q = floor(psi / (pi/2)); the vector is rotated into quadrant 0 and
//     the n_o/4 - 1 interior edges e_j = 2 pi j / n_o are counted by cross-product signs
//     (n_o % 4 != 0 falls back to atan2f). theta = 0 when a = c and b = 0 [R5].
//   strength:  S >= t  <=>  h + r >= t^2  <=>  t^2 - h <= 0  or  r^2 >= (t^2 - h)^2
//   coherence: C >= t (t > 0)  <=>  r (1 + t^2) >= 2 t h  <=>  r^2 >= kappa^2 h^2,
//              kappa = 2t / (1 + t^2); thresholds <= 0 always pass; C = 0 when h = 0 [R6]
// with h = (l1 + l2) / 2 = T/2 and r = (l1 - l2) / 2 = sqrt((a-c)^2/4 + b^2), all in fp32 on
// well-conditioned quantities. FAST: n_o = 16 (edges pi/8, pi/4, 3 pi/8 in the rotated quadrant,
// compile-time constants equal to the host's fp32 cos/sin) and <= 2 thresholds per feature.
template <bool FAST>
__device__ __forceinline__ int bucket_of(double a, double b, double c, const DownParams& prm) {
  constexpr int MAXT = FAST ? 2 : kMaxThr2;
  const float Df = (float)(a - c), Bf = (float)b;
  const float h = 0.125f * (float)(a + c);                          // unscaled x4 -> T/2
  const float q = 0.0625f * fmaf(0.25f * Df, Df, Bf * Bf);           // r^2
  int o = 0;
  if (!(Df == 0.0f && Bf == 0.0f)) {
    const float X = -Df, Y = -2.0f * Bf;
    if (FAST || prm.quad_edges) {
      int qd;
      float xr, yr;
      if (X > 0.0f && Y >= 0.0f) { qd = 0; xr = X; yr = Y; }
      else if (X <= 0.0f && Y > 0.0f) { qd = 1; xr = Y; yr = -X; }
      else if (X < 0.0f && Y <= 0.0f) { qd = 2; xr = -X; yr = -Y; }
      else { qd = 3; xr = -Y; yr = X; }
      if constexpr (FAST) {
        constexpr float c1 = 0.92387953251128674f, s1 = 0.38268343236508978f;  // pi/8
        constexpr float c2 = 0.70710678118654752f;                              // pi/4
        o = 4 * qd + (fmaf(c1, yr, -s1 * xr) >= 0.0f) + (fmaf(c2, yr, -c2 * xr) >= 0.0f) +
            (fmaf(s1, yr, -c1 * xr) >= 0.0f);
      } else {
        const int m = prm.n_o >> 2;
        o = qd * m;
        for (int j = 0; j < m - 1; ++j) o += (fmaf(prm.ecos[j], yr, -prm.esin[j] * xr) >= 0.0f);
      }
    } else {
      const float kTwoPiInv = 0.15915494309189535f;
      const float phi = atan2f(2.0f * Bf, Df);
      o = (int)floorf(fmaf(phi, (float)prm.n_o * kTwoPiInv, 0.5f * (float)prm.n_o));
      o %= prm.n_o;
      if (o < 0) o += prm.n_o;
    }
  }
  int s = 0;
#pragma unroll
  for (int t = 0; t < MAXT; ++t) {
    if (!FAST && t >= prm.n_s - 1) break;
    const float d = prm.ts2[t] - h;
    s += (d <= 0.0f) || (q >= d * d);
  }
  int k = prm.tc_nonpos;
  if (h > 0.0f) {
    const float h2 = h * h;
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      if (!FAST && t >= prm.n_c - 1) break;
      k += (q >= prm.kc2[t] * h2);
    }
  }
  return (o * prm.n_s + s) * prm.n_c + k;
}

// grid: ceil(n_tasks / WARPS) CTAs of 32 * WARPS threads; task = (frame, band, strip), strip fastest.
template <bool HILO, bool DEC, bool FAST>
__global__ void __launch_bounds__(32 * down::WARPS, 3) k_down(const DownArgs a, const DownParams prm) {
  using namespace down;
  constexpr int NP = HILO ? 6 : 3;  // planes per ring row (3 channels, x2 with lo)
  extern __shared__ __align__(16) float dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x * WARPS + warp;
  if (task >= a.n_tasks) return;
  float* ring = dsm + (size_t)warp * RING * NP * 64 + 2 * lane;  // this lane's 2 columns

  const int strip = task % a.n_strips;
  const int t2 = task / a.n_strips;
  const int band = t2 % a.n_bands;
  const int n = t2 / a.n_bands;
  const int X0 = strip * STRIP - 4;
  const int x = X0 + 2 * lane;
  const int Yb = a.base + band * a.RB;
  const int nrows = a.RB + 6;  // input rows Yb-3 .. Yb+RB+2
  const int fx0 = fold_idx(x, a.W), fx1 = fold_idx(x + 1, a.W);
  const float* hbase = a.zhi + (long long)n * a.in_frame;
  const float* lbase = HILO ? a.zlo + (long long)n * a.in_frame : nullptr;
  const bool out_lane = lane >= LANE_LO && lane <= LANE_HI;
  // one 8-byte copy when the two columns are adjacent in memory and 8-B aligned (interior, W even)
  const bool pair8 = fx1 == fx0 + 1 && ((fx0 | a.W | (int)(a.in_plane & 1)) & 1) == 0 &&
                     ((reinterpret_cast<uintptr_t>(a.zhi) | reinterpret_cast<uintptr_t>(HILO ? a.zlo : a.zhi)) & 7) == 0;

  auto issue = [&](int i) {
    const int r = Yb - 3 + i;
    int br = fold_idx(r, a.H) - a.in_row0;
    br = min(max(br, 0), a.in_rows - 1);
    float* dst = ring + (i % RING) * NP * 64;
    const long long ro = (long long)br * a.W;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float* s = hbase + c * a.in_plane + ro;
      if (pair8) {
        cp_async8(dst + c * 64, s + fx0);
      } else {
        cp_async4(dst + c * 64, s + fx0);
        cp_async4(dst + c * 64 + 1, s + fx1);
      }
      if constexpr (HILO) {
        const float* sl = lbase + c * a.in_plane + ro;
        if (pair8) {
          cp_async8(dst + (3 + c) * 64, sl + fx0);
        } else {
          cp_async4(dst + (3 + c) * 64, sl + fx0);
          cp_async4(dst + (3 + c) * 64 + 1, sl + fx1);
        }
      }
    }
  };
#pragma unroll
  for (int i = 0; i < RING - 1; ++i) {
    if (i < nrows) issue(i);
    cp_async_commit();
  }

  const double w0 = prm.wp[0], w1 = prm.wp[1], w2 = prm.wp[2], w3 = prm.wp[3], w4 = prm.wp[4];
  constexpr double dw0 = -3.0 / 256.0, dw1 = -9.0 / 256.0, dw2 = 29.0 / 256.0, dw3 = 111.0 / 256.0;

  double zm[3][2], zc[3][2];  // own columns of rows c-1, c (c = r-1 is the product row)
  double cL1[3], cR2[3];      // row c at columns x-1 and x+2
  double vA[4][2], vB[4][2], vC[4][2];  // pending window rows y = c-1 .. c+2 (after the shift)
  double dacc[4][3];          // pending decimated rows (4) x channels
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#pragma unroll
    for (int j = 0; j < 2; ++j) vA[k][j] = vB[k][j] = vC[k][j] = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) dacc[k][c] = 0.0;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    zm[c][0] = zm[c][1] = zc[c][0] = zc[c][1] = 0.0;
    cL1[c] = cR2[c] = 0.0;
  }

  uint8_t* mapf = a.map + (long long)n * a.s_rn * a.W;
  const long long oframe = (long long)n * 3 * a.d_buf_rows * a.W1;
  const int Xd = x >> 1;  // decimated column (x even)

#pragma unroll 2
  for (int i = 0; i < nrows; ++i) {
    if (i + RING - 1 < nrows) issue(i + RING - 1);
    cp_async_commit();
    cp_async_wait<RING - 1>();
    const float* src = ring + (i % RING) * NP * 64;
    double zn[3][2];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float2 h2 = *reinterpret_cast<const float2*>(src + c * 64);
      if constexpr (HILO) {
        const float2 l2 = *reinterpret_cast<const float2*>(src + (3 + c) * 64);
        zn[c][0] = (double)h2.x + (double)l2.x;
        zn[c][1] = (double)h2.y + (double)l2.y;
      } else {
        zn[c][0] = (double)h2.x;
        zn[c][1] = (double)h2.y;
      }
    }
    // horizontal neighbours of row r (x-1, x+2 for the next gradient row; x-3..x+4 for decimation)
    double nL1[3], nR2[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      nL1[c] = shfl_up_d(zn[c][1], 1);
      nR2[c] = shfl_dn_d(zn[c][0], 1);
    }
    const int r = Yb - 3 + i;

    if constexpr (DEC) {
      // ---- decimation: horizontal 8 taps at column Xd of row r, then the vertical ring
      const bool odd_r = (i & 1) == 0;  // Yb even => r = Yb - 3 + i is odd for even i
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double zL2 = shfl_up_d(zn[c][0], 1);   // x-2
        const double zL3 = shfl_up_d(zn[c][1], 2);   // x-3
        const double zR3 = shfl_dn_d(zn[c][1], 1);   // x+3
        const double zR4 = shfl_dn_d(zn[c][0], 2);   // x+4
        double hp = dw0 * zL3;
        hp = fma(dw1, zL2, hp);
        hp = fma(dw2, nL1[c], hp);
        hp = fma(dw3, zn[c][0], hp);
        hp = fma(dw3, zn[c][1], hp);
        hp = fma(dw2, nR2[c], hp);
        hp = fma(dw1, zR3, hp);
        hp = fma(dw0, zR4, hp);
        // pending rows Y' = Yb/2 + m - 3 + k (k = 0..3); weight index 6-2k (odd r) / 7-2k (even r)
        if (odd_r) {
          dacc[0][c] = fma(dw1, hp, dacc[0][c]);  // w[6] = w[1]
          dacc[1][c] = fma(dw3, hp, dacc[1][c]);  // w[4] = w[3]
          dacc[2][c] = fma(dw2, hp, dacc[2][c]);  // w[2]
          dacc[3][c] = fma(dw0, hp, dacc[3][c]);  // w[0]
        } else {
          dacc[0][c] = fma(dw0, hp, dacc[0][c]);  // w[7] = w[0]
          dacc[1][c] = fma(dw2, hp, dacc[1][c]);  // w[5] = w[2]
          dacc[2][c] = fma(dw3, hp, dacc[2][c]);  // w[3]
          dacc[3][c] = fma(dw1, hp, dacc[3][c]);  // w[1]
        }
      }
      // NB: w = [-3, -9, 29, 111, 111, 29, -9, -3] / 256 is symmetric: w[6] = w[1] = dw1 ...
      if (!odd_r) {
        const int Yd = (r - 4) / 2;  // completed row (r even)
        if (out_lane && Yd >= a.d_r0 && Yd < a.d_r0 + a.d_rn && Xd < a.W1 && i >= 7) {
          const long long o = oframe + (long long)(Yd - a.d_buf_row0) * a.W1 + Xd;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double v = dacc[0][c];
            const float hi = (float)v;
            a.ohi[o + (long long)c * a.d_buf_rows * a.W1] = hi;
            if (a.olo) a.olo[o + (long long)c * a.d_buf_rows * a.W1] = (float)(v - (double)hi);
          }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          dacc[0][c] = dacc[1][c];
          dacc[1][c] = dacc[2][c];
          dacc[2][c] = dacc[3][c];
          dacc[3][c] = 0.0;
        }
      }
    }

    if (i >= 2) {
      // ---- products at row c = r - 1 for columns x, x+1 (unscaled gradients 2g)
      double A0 = 0.0, B0 = 0.0, C0 = 0.0, A1 = 0.0, B1 = 0.0, C1 = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double gx0 = zc[c][1] - cL1[c], gx1 = cR2[c] - zc[c][0];
        const double gy0 = zn[c][0] - zm[c][0], gy1 = zn[c][1] - zm[c][1];
        A0 = fma(gx0, gx0, A0);
        B0 = fma(gx0, gy0, B0);
        C0 = fma(gy0, gy0, C0);
        A1 = fma(gx1, gx1, A1);
        B1 = fma(gx1, gy1, B1);
        C1 = fma(gy1, gy1, C1);
      }
      // ---- horizontal window: products at x-2, x-1 (lane-1) and x+2, x+3 (lane+1)
      const double Am2 = shfl_up_d(A0, 1), Am1 = shfl_up_d(A1, 1), Ap2 = shfl_dn_d(A0, 1), Ap3 = shfl_dn_d(A1, 1);
      const double Bm2 = shfl_up_d(B0, 1), Bm1 = shfl_up_d(B1, 1), Bp2 = shfl_dn_d(B0, 1), Bp3 = shfl_dn_d(B1, 1);
      const double Cm2 = shfl_up_d(C0, 1), Cm1 = shfl_up_d(C1, 1), Cp2 = shfl_dn_d(C0, 1), Cp3 = shfl_dn_d(C1, 1);
      double hA0 = w0 * Am2, hB0 = w0 * Bm2, hC0 = w0 * Cm2;
      hA0 = fma(w1, Am1, hA0); hB0 = fma(w1, Bm1, hB0); hC0 = fma(w1, Cm1, hC0);
      hA0 = fma(w2, A0, hA0);  hB0 = fma(w2, B0, hB0);  hC0 = fma(w2, C0, hC0);
      hA0 = fma(w3, A1, hA0);  hB0 = fma(w3, B1, hB0);  hC0 = fma(w3, C1, hC0);
      hA0 = fma(w4, Ap2, hA0); hB0 = fma(w4, Bp2, hB0); hC0 = fma(w4, Cp2, hC0);
      double hA1 = w0 * Am1, hB1 = w0 * Bm1, hC1 = w0 * Cm1;
      hA1 = fma(w1, A0, hA1);  hB1 = fma(w1, B0, hB1);  hC1 = fma(w1, C0, hC1);
      hA1 = fma(w2, A1, hA1);  hB1 = fma(w2, B1, hB1);  hC1 = fma(w2, C1, hC1);
      hA1 = fma(w3, Ap2, hA1); hB1 = fma(w3, Bp2, hB1); hC1 = fma(w3, Cp2, hC1);
      hA1 = fma(w4, Ap3, hA1); hB1 = fma(w4, Bp3, hB1); hC1 = fma(w4, Cp3, hC1);
      // ---- vertical window: pending rows y = c-2 .. c+2 get weight w[c - y + 2]
      const double hA[2] = {hA0, hA1}, hB[2] = {hB0, hB1}, hC[2] = {hC0, hC1};
      const int y = r - 3;  // = c - 2: completes now
      const bool emit = i >= 6 && out_lane && y >= a.s_r0 && y < a.s_r0 + a.s_rn;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const double fa = fma(w4, hA[j], vA[0][j]), fb = fma(w4, hB[j], vB[0][j]), fc = fma(w4, hC[j], vC[0][j]);
        if (emit && x + j < a.W)
          mapf[(long long)(y - a.s_r0) * a.W + x + j] = (uint8_t)bucket_of<FAST>(fa, fb, fc, prm);
        vA[0][j] = fma(w3, hA[j], vA[1][j]); vB[0][j] = fma(w3, hB[j], vB[1][j]); vC[0][j] = fma(w3, hC[j], vC[1][j]);
        vA[1][j] = fma(w2, hA[j], vA[2][j]); vB[1][j] = fma(w2, hB[j], vB[2][j]); vC[1][j] = fma(w2, hC[j], vC[2][j]);
        vA[2][j] = fma(w1, hA[j], vA[3][j]); vB[2][j] = fma(w1, hB[j], vB[3][j]); vC[2][j] = fma(w1, hC[j], vC[3][j]);
        vA[3][j] = w0 * hA[j];               vB[3][j] = w0 * hB[j];               vC[3][j] = w0 * hC[j];
      }
    }
    // ---- rotate the gradient rows
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      zm[c][0] = zc[c][0];
      zm[c][1] = zc[c][1];
      zc[c][0] = zn[c][0];
      zc[c][1] = zn[c][1];
      cL1[c] = nL1[c];
      cR2[c] = nR2[c];
    }
  }
}

}  // namespace blade
