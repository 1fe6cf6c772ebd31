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
//   - each lane prefetches its own two columns of the next rows with 4/8-byte cp.async into a
//     lane-private ring in shared memory (RING rows deep, no cross-lane smem traffic, no barrier);
//   - gradients (unscaled: 2 g), the products A = sum_c gx^2, B = sum_c gx gy, C = sum_c gy^2
//     and the 5x5 Gaussian window are fp32 (the window runs as a horizontal pass over shuffled
//     neighbour products and a 5-deep vertical ring of pending output rows);
//   - the bucket decision is fp32 with a certificate: a pixel whose orientation bin the fp32 error
//     bound cannot guarantee is queued for k_down_fixup, which recomputes it in fp64 (below);
//   - decimation is fp64 (the next level's selector needs the pyramid to ~1e-12): horizontal 8
//     taps over shuffled fp64 neighbours, then a 4-deep vertical ring; output hi/lo fp32 pair.
// fp32 -> fp64 conversions run at 16/clk/SM on B200 (measured, scripts/probes/tput.cu), so each
// element is converted exactly once, by the lane that loads it.
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include <type_traits>

#include "kernels.cuh"

namespace blade {

constexpr int kMaxThr2 = 15;
struct DownParams {
  double wp[5];                        // window weights at offsets -2..2 (zero-padded for WS < 5)
  int n_o, n_s, n_c;
  float ts2[kMaxThr2];   // strength thresholds squared (-inf for t <= 0, +inf padding)
  float kc2[kMaxThr2];   // positive coherence thresholds: (2t / (1 + t^2))^2 (+inf padding)
  int tc_nonpos;         // # coherence thresholds <= 0 (always passed)
  float tsR[2];          // FAST selector (bucket32_fast): 8 t^2 per strength threshold (-inf for t <= 0)
  float kcR[2];          // FAST selector: kappa = 2t / (1 + t^2) per positive coherence threshold (+inf padding)
  int quad_edges;        // n_o % 4 == 0 and n_o <= 64: quadrant + edge-count orientation
  float ecos[16], esin[16];  // interior edges 2 pi j / n_o, j = 1 .. n_o/4 - 1
};

// BLADE_DOWN_PACK (A/B builds, profiles/r02_down_pack.txt): 0 = scalar fp32 window arithmetic,
// 1 (default) = the vertical window ring
// as packed fp32x2 FMAs, 2 = products and horizontal window packed too (all bit-identical).
#ifndef BLADE_DOWN_PACK
#define BLADE_DOWN_PACK 1
#endif
// CTAs per SM the level >= 1 (hi/lo) variant is compiled for (A/B builds)
#ifndef BLADE_DOWN_HILO_MINB
#define BLADE_DOWN_HILO_MINB 3
#endif
#ifndef BLADE_DOWN_LO_MINB
#define BLADE_DOWN_LO_MINB 4
#endif
namespace down {
constexpr int WARPS = 4;        // independent warps per CTA
#ifndef BLADE_DOWN_RING
#define BLADE_DOWN_RING 8
#endif
constexpr int RING = BLADE_DOWN_RING;  // rows in flight per lane (cp.async ring)
constexpr int STRIP = 56;       // output columns per strip
constexpr int LANE_LO = 2, LANE_HI = 29;
}  // namespace down

struct DownArgs {
  const float* zhi;  // level l (hi plane, or the fp32 input at l = 0): [N][3][in_rows][W]
  const float* zlo;  // level l lo plane (nullptr at l = 0)
  int H, W, in_row0, in_rows;
  long long in_plane, in_frame;
  int in_pitch;      // floats per input row (>= W)
  void* map;         // s^l rows [s_r0, s_r0 + s_rn), pitch map_pitch (>= W; a multiple of 16 in
                     // the workspace so the stage can TMA it), frame stride s_rn * map_pitch;
                     // uint8 entries (K <= 256) or uint16 (WIDE, K <= 65536)
  int s_r0, s_rn, map_pitch;
  float* ohi;        // z^{l+1} hi: rows [d_buf_row0, + d_buf_rows), pitch W1 (nullptr: no dec)
  float* olo;        // z^{l+1} lo (nullptr: not needed, l + 1 is the coarsest level)
  int H1, W1, d_buf_row0, d_buf_rows, d_r0, d_rn;
  int out_pitch;     // floats per z^{l+1} row (>= W1)
  int base, RB, n_strips, n_bands, n_tasks;
  unsigned long long* fb_list;  // uncertified map entries (flat index into map), capacity fb_cap
  unsigned int* fb_count;       // zeroed before the launch; may exceed fb_cap (overflow)
  unsigned int fb_cap;
  int N;                        // frames of the launch
  float* zcopy;                 // level 0 only (nullptr: off): a copy of the input rows with row pitch
  int copy_pitch;               // copy_pitch (a multiple of 4) for the TMA stage, [N][3][H][copy_pitch]
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

// ---- fp32 selector with a certificate (DESIGN.md §6 H1)
//
// The window sums a = sum w gx^2, b = sum w gx gy, c = sum w gy^2 (unscaled gradients 2g, fp32 from
// exact fp32 inputs or from the hi/lo pyramid) carry absolute errors |da|, |dc| <= ~11 u T and
// |db| <= ~8 u T (T = a + c, u = 2^-24: every product and weight is rounded once, all sums of
// a and c have positive terms, |gx gy| <= (gx^2 + gy^2) / 2). So X = c - a and Y = -2b, whose angle
// psi decides the orientation bin, are each off by <= 16 u T, and every sign test below (the
// quadrant signs of X, Y and the cross products with the bin edges, |v| <= T) is off by at most
// 32 u T. A test whose |value| exceeds kCert T = 64 u T therefore has the sign of the exact test;
// a pixel with any closer test is queued and recomputed in fp64 (k_down_fixup). Strength and coherence are
// well-conditioned: their fp32 errors (~1e-6 relative) stay far inside the 1e-5 parity window.
constexpr float kCert = 64.0f * 5.9604644775390625e-8f;

__host__ __device__ __forceinline__ unsigned int f32_bits(float x) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(x);
#else
  unsigned int u;
  memcpy(&u, &x, 4);
  return u;
#endif
}
__host__ __device__ __forceinline__ float sqrt_approx(float x) {
#ifdef __CUDA_ARCH__
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
#else
  return sqrtf(x);
#endif
}

// FAST layout (16 orientations x 3 strengths x 3 coherences), the same decisions as the generic
// bucket32 below with about half the instructions (the selector's largest cost, ncu/SASS of
// k_down: 70 instructions per pixel -> ~40):
//   orientation: the bin of psi = angle of (X, Y) = (-D, -2b) (D = a - c) is found by REFLECTION
//     instead of rotation: alpha = angle of (|X|, |Y|) in [0, pi/2], m = # of the interior edges
//     pi/8, pi/4, 3 pi/8 at or below alpha (three cross-product signs, read from sign bits), and
//     o = 8 [Y < 0] + (m, or 7 - m when X and Y have opposite signs: psi = pi - alpha or
//     2 pi - alpha). The sign tests are the rotated form's up to the order of the two operands
//     (the same error bound); a certified pixel clears every one by 64 u T, so no test is a tie
//     and the reflection gives the exact bin. T = 0 (no gradient anywhere in the window) is
//     theta = 0, certified [R5]; any other isotropic tensor (D = b = 0) fails the certificate.
//   strength / coherence with R = sqrt(D^2 + 4 b^2) (sqrt.approx, ~2 ulp): with the unscaled x4
//     sums, l1 = (T + R) / 8 and r / h = R / T, so S >= t <=> T + R >= 8 t^2 (tsR) and
//     C >= t <=> R > kappa T (kcR; strict, so T = 0 gives C = 0 [R6]). These features are
//     well-conditioned: the fp32 error (~3e-7 relative) stays far inside the 1e-5 parity window.
__host__ __device__ __forceinline__ int bucket32_fast(float a, float b, float c, const float* tsR, const float* kcR,
                                                      int tc_nonpos, bool& safe) {
  const float T = a + c, D = a - c, B2 = b + b;
  const float ax = fabsf(D), ay = fabsf(B2);
  constexpr float c1 = 0.92387953251128674f, s1 = 0.38268343236508978f;  // pi/8
  constexpr float c2 = 0.70710678118654752f;                              // pi/4
  const float e1 = fmaf(c1, ay, -s1 * ax), e2 = fmaf(c2, ay, -c2 * ax), e3 = fmaf(s1, ay, -c1 * ax);
  const float mn = fminf(fminf(fminf(ax, ay), fminf(fabsf(e1), fabsf(e2))), fabsf(e3));
  const bool zero = T == 0.0f && b == 0.0f;
  safe = zero || mn > kCert * T;
  // t = m = 3 - # negative edge tests; flip (X, Y of opposite signs) -> 7 - t; + 8 when Y < 0
  const int t = 3 - (int)((f32_bits(e1) >> 31) + (f32_bits(e2) >> 31) + (f32_bits(e3) >> 31));
  const int fm = (int)(f32_bits(D) ^ f32_bits(b)) >> 31;  // X = -D, Y = -2b: sign(X) != sign(Y)
  const int lm = ~((int)f32_bits(b) >> 31);                // Y < 0 <=> b > 0
  int o = (t ^ fm) + (fm & 8) + (lm & 8);
  o = zero ? 0 : o;
  const float R = sqrt_approx(fmaf(B2, B2, D * D));
  const float TR = T + R;
  const int s = (TR >= tsR[0]) + (TR >= tsR[1]);
  const int k = tc_nonpos + (R > kcR[0] * T) + (R > kcR[1] * T);
  return (o * 3 + s) * 3 + k;
}

template <bool FAST>
__device__ __forceinline__ int bucket32(float a, float b, float c, const DownParams& prm, bool& safe) {
  if constexpr (FAST) return bucket32_fast(a, b, c, prm.tsR, prm.kcR, prm.tc_nonpos, safe);
  constexpr int MAXT = FAST ? 2 : kMaxThr2;
  const float T = a + c;
  const float Df = a - c;
  const float h = 0.125f * T;                                    // unscaled x4 -> T/2
  const float q = 0.0625f * fmaf(0.25f * Df, Df, b * b);         // r^2
  const float bound = kCert * T;
  const float X = -Df, Y = -2.0f * b;
  const bool zero = Df == 0.0f && b == 0.0f;
  int o;
  float mn;
  if constexpr (FAST) {
    // branch-free: rotate (X, Y) by pi into the upper half plane, then by -pi/2 into quadrant 0
    const bool lower = Y < 0.0f || (Y == 0.0f && X < 0.0f);
    const float X1 = lower ? -X : X, Y1 = lower ? -Y : Y;
    const bool left = X1 <= 0.0f;
    const float xr = left ? Y1 : X1, yr = left ? -X1 : Y1;
    constexpr float c1 = 0.92387953251128674f, s1 = 0.38268343236508978f;  // pi/8
    constexpr float c2 = 0.70710678118654752f;                              // pi/4
    const float e1 = fmaf(c1, yr, -s1 * xr), e2 = fmaf(c2, yr, -c2 * xr), e3 = fmaf(s1, yr, -c1 * xr);
    o = (lower ? 8 : 0) + (left ? 4 : 0) + (e1 >= 0.0f) + (e2 >= 0.0f) + (e3 >= 0.0f);
    mn = fminf(fminf(fabsf(X), fabsf(Y)), fminf(fabsf(e1), fminf(fabsf(e2), fabsf(e3))));
    o = zero ? 0 : o;
  } else {
    o = 0;
    mn = fminf(fabsf(X), fabsf(Y));
    if (!zero) {
      if (prm.quad_edges) {
        int qd;
        float xr, yr;
        if (X > 0.0f && Y >= 0.0f) { qd = 0; xr = X; yr = Y; }
        else if (X <= 0.0f && Y > 0.0f) { qd = 1; xr = Y; yr = -X; }
        else if (X < 0.0f && Y <= 0.0f) { qd = 2; xr = -X; yr = -Y; }
        else { qd = 3; xr = -Y; yr = X; }
        const int m = prm.n_o >> 2;
        o = qd * m;
        for (int j = 0; j < m - 1; ++j) {
          const float e = fmaf(prm.ecos[j], yr, -prm.esin[j] * xr);
          o += (e >= 0.0f);
          mn = fminf(mn, fabsf(e));
        }
      } else {
        // generic n_o: atan2f (~2 ulp) and the distance to the nearest edge in psi
        const float kTwoPiInv = 0.15915494309189535f;
        const float phi = atan2f(-Y, -X);  // = atan2(2b, a - c)
        const float f = fmaf(phi, (float)prm.n_o * kTwoPiInv, 0.5f * (float)prm.n_o);
        o = (int)floorf(f);
        const float fr = f - floorf(f);
        const float dist = fminf(fr, 1.0f - fr) * 6.283185307179586f / (float)prm.n_o;  // radians in psi
        mn = fminf(mn, (dist - 2e-6f) * sqrtf(fmaf(X, X, Y * Y)));
        o %= prm.n_o;
        if (o < 0) o += prm.n_o;
      }
    }
  }
  // certified iff every sign test clears the error bound; exact zero gradients => theta = 0 [R5]
  safe = zero ? !(T > 0.0f) : (mn > bound);
  const float h2 = h * h;
  int s = 0, k = 0;
  if constexpr (FAST) {
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      const float d = prm.ts2[t] - h;
      s += (d <= 0.0f) || (q >= d * d);
    }
#pragma unroll
    for (int t = 0; t < MAXT; ++t) k += (q >= prm.kc2[t] * h2);
  } else {
    // the tests are monotone in t (ascending thresholds, +inf padding up to kMaxThr2 = 15):
    // binary search for the count of passed thresholds
#pragma unroll
    for (int step = 8; step >= 1; step >>= 1) {
      const int t = s + step - 1;
      if (t < kMaxThr2) {
        const float d = prm.ts2[t] - h;
        if ((d <= 0.0f) || (q >= d * d)) s += step;
      }
      const int u = k + step - 1;
      if (u < kMaxThr2 && q >= prm.kc2[u] * h2) k += step;
    }
  }
  k = prm.tc_nonpos + (h > 0.0f ? k : 0);  // C = 0 when l1 = 0 [R6]
  if constexpr (FAST) return (o * 3 + s) * 3 + k;  // FAST layout: 16 x 3 x 3
  return (o * prm.n_s + s) * prm.n_c + k;
}

// The fields of one level a fix-up needs, read once per pixel from the (dynamically indexed)
// kernel parameters into registers.
struct FixLevel {
  const float* zhi;
  const float* zlo;
  void* map;
  const unsigned long long* fb_list;
  long long in_frame, in_plane;
  int H, W, in_row0, in_rows, in_pitch, s_r0, s_rn, map_pitch;
  __device__ __forceinline__ explicit FixLevel(const DownArgs& a)
      : zhi(a.zhi), zlo(a.zlo), map(a.map), fb_list(a.fb_list), in_frame(a.in_frame), in_plane(a.in_plane),
        H(a.H), W(a.W), in_row0(a.in_row0), in_rows(a.in_rows), in_pitch(a.in_pitch), s_r0(a.s_r0), s_rn(a.s_rn),
        map_pitch(a.map_pitch) {}
};

// The fp64 bucket of pixel (n, y, xx) of a level (whole warp; lane t < 25 evaluates window tap
// (t / 5 - 2, t % 5 - 2)); every lane returns it.
template <bool FAST>
__device__ __forceinline__ int fix_bucket(const FixLevel& a, const DownParams& prm, int n, int y, int xx, int lane) {
  const bool hilo = a.zlo != nullptr;
  double pa = 0.0, pb = 0.0, pc = 0.0;
  if (lane < 25) {
    const int dy = lane / 5 - 2, dx = lane % 5 - 2;
    auto Z = [&](int c, int yy, int xq) -> double {
      int br = fold_idx(yy, a.H) - a.in_row0;
      br = min(max(br, 0), a.in_rows - 1);
      const long long o = (long long)n * a.in_frame + c * a.in_plane + (long long)br * a.in_pitch + fold_idx(xq, a.W);
      double v = (double)a.zhi[o];
      if (hilo) v += (double)a.zlo[o];
      return v;
    };
    const int yy = y + dy, xq = xx + dx;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double gx = Z(c, yy, xq + 1) - Z(c, yy, xq - 1);
      const double gy = Z(c, yy + 1, xq) - Z(c, yy - 1, xq);
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
  return bucket_of<FAST>(pa, pb, pc, prm);
}

// grid: ceil(n_tasks / WARPS) CTAs of 32 * WARPS threads; task = (frame, band, strip), strip fastest.
// COPY (level 0 only): also write the input rows into a.zcopy (16-B row pitch) for the TMA stage
// when the caller's rows are not 16-B multiples.
// SEL = false (level 0 when the stage computes the selector itself, DESIGN.md §6 "fused
// selector"): decimation (and COPY) only; no map, no fix-up list.
// IFIX (small calls): an uncertified pixel is recomputed in fp64 by the whole warp right away
// (fix_bucket, the fix-up kernel's arithmetic) instead of being queued for a fix-up launch.
template <bool HILO, bool DEC, bool FAST, bool WIDE, bool COPY = false, bool SEL = true, bool IFIX = false>
__global__ void __launch_bounds__(32 * down::WARPS, HILO ? BLADE_DOWN_HILO_MINB : BLADE_DOWN_LO_MINB) k_down(const DownArgs a, const DownParams prm) {
  using MT = typename std::conditional<WIDE, uint16_t, uint8_t>::type;  // bucket map entry
  using namespace down;
  constexpr int NP = HILO ? 6 : 3;  // planes per ring row (3 channels, x2 with lo)
  extern __shared__ __align__(16) float dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x * WARPS + warp;
  BT_ENTRY(HILO ? 1 : 0);
  pdl_trigger();
  if (task >= a.n_tasks) return;
  pdl_wait();
  BT_WAITED(HILO ? 1 : 0);
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
  const bool pair8 = fx1 == fx0 + 1 && ((fx0 | a.in_pitch | (int)(a.in_plane & 1)) & 1) == 0 &&
                     ((reinterpret_cast<uintptr_t>(a.zhi) | reinterpret_cast<uintptr_t>(HILO ? a.zlo : a.zhi)) & 7) == 0;
  const bool all_pair8 = __all_sync(0xffffffffu, pair8);

  // interior task: every input row it streams lies inside the image and the buffer (no fold)
  const bool interior = Yb - 3 >= 0 && Yb - 3 + nrows <= a.H && Yb - 3 >= a.in_row0 &&
                        Yb - 3 + nrows <= a.in_row0 + a.in_rows;
  auto issue = [&](int i) {
    const int r = Yb - 3 + i;
    int br;
    if (interior) {
      br = r - a.in_row0;
    } else {
      br = fold_idx(r, a.H) - a.in_row0;
      br = min(max(br, 0), a.in_rows - 1);
    }
    float* dst = ring + (i % RING) * NP * 64;
    const long long ro = (long long)br * a.in_pitch;
    if (all_pair8) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        cp_async8(dst + c * 64, hbase + c * a.in_plane + ro + fx0);
        if constexpr (HILO) cp_async8(dst + (3 + c) * 64, lbase + c * a.in_plane + ro + fx0);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float* s = hbase + c * a.in_plane + ro;
        cp_async4(dst + c * 64, s + fx0);
        cp_async4(dst + c * 64 + 1, s + fx1);
        if constexpr (HILO) {
          const float* sl = lbase + c * a.in_plane + ro;
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

  const float w0 = (float)prm.wp[0], w1 = (float)prm.wp[1], w2 = (float)prm.wp[2];  // symmetric
  constexpr double dw0 = -3.0 / 256.0, dw1 = -9.0 / 256.0, dw2 = 29.0 / 256.0, dw3 = 111.0 / 256.0;

  // fp32 gradient rows (own columns of rows c-1, c; row c at columns x-1, x+2); hi and lo parts
  float hm[3][2], hc[3][2], hL[3], hR[3];
  float lm[3][2], lc[3][2], lL[3], lR[3];
  // pending window rows y = c-1 .. c+2 (after the shift); (x, y) = the lane's two columns, so the
  // window arithmetic runs as packed fp32x2 FMAs (FFMA2; element-wise identical to fmaf)
  float2 vA[4], vB[4], vC[4];
  double dacc[4][3];                   // pending decimated rows (4) x channels
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    vA[k] = vB[k] = vC[k] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int c = 0; c < 3; ++c) dacc[k][c] = 0.0;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    hm[c][0] = hm[c][1] = hc[c][0] = hc[c][1] = hL[c] = hR[c] = 0.0f;
    lm[c][0] = lm[c][1] = lc[c][0] = lc[c][1] = lL[c] = lR[c] = 0.0f;
  }

  MT* mapf = static_cast<MT*>(a.map) + (long long)n * a.s_rn * a.map_pitch;
  // channel plane of z^{l+1} (< 2^31 floats: a level-1 plane that large would need > 180 GB of
  // level-0 input and output)
  const int ostr32 = a.d_buf_rows * a.out_pitch;
  const int Xd = x >> 1;  // decimated column (x even)
  // offset of z^{l+1} row Yd = (r - 4) / 2 at the lane's column, for the even rows r (odd i; the
  // first is i = 1, r = Yb - 2); advanced by one row per even r
  long long oo = 3 * (long long)n * ostr32 + (long long)((Yb - 6) / 2 - a.d_buf_row0) * a.out_pitch + Xd;
  const bool has_lo = a.olo != nullptr;
  // 2-byte map stores when every map row starts 2-B aligned (x is even)
  const bool map16 = (a.map_pitch & 1) == 0 && (reinterpret_cast<uintptr_t>(a.map) & (2 * sizeof(MT) - 1)) == 0;

  // map entry of this lane for the window row completing at iteration i (y = Yb - 6 + i)
  MT* mrow_i = mapf + (long long)(Yb - 6 - a.s_r0) * a.map_pitch + x;
#pragma unroll 2
  for (int i = 0; i < nrows; ++i, mrow_i += a.map_pitch) {
    if (i + RING - 1 < nrows) issue(i + RING - 1);
    cp_async_commit();
    cp_async_wait<RING - 1>();
    const float* src = ring + (i % RING) * NP * 64;
    float hn[3][2], ln[3][2], nL[3], nR[3], nlL[3], nlR[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float2 h2 = *reinterpret_cast<const float2*>(src + c * 64);
      hn[c][0] = h2.x;
      hn[c][1] = h2.y;
      if constexpr (HILO) {
        const float2 l2 = *reinterpret_cast<const float2*>(src + (3 + c) * 64);
        ln[c][0] = l2.x;
        ln[c][1] = l2.y;
      } else {
        ln[c][0] = ln[c][1] = 0.0f;
      }
      // columns x-1 and x+2 of row r (fp32 parts): gradients of the next product row
      nL[c] = __shfl_up_sync(0xffffffffu, hn[c][1], 1);
      nR[c] = __shfl_down_sync(0xffffffffu, hn[c][0], 1);
      if constexpr (HILO) {
        nlL[c] = __shfl_up_sync(0xffffffffu, ln[c][1], 1);
        nlR[c] = __shfl_down_sync(0xffffffffu, ln[c][0], 1);
      } else {
        nlL[c] = nlR[c] = 0.0f;
      }
    }
    const int r = Yb - 3 + i;
    if (COPY && out_lane && r >= Yb && r < Yb + a.RB && r < a.H && x < a.W) {
      // the band's own rows, the strip's own columns: every input sample is written exactly once
      float* cp = a.zcopy + ((long long)n * 3 * a.H + r) * a.copy_pitch + x;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        cp[(long long)c * a.H * a.copy_pitch] = hn[c][0];
        if (x + 1 < a.W) cp[(long long)c * a.H * a.copy_pitch + 1] = hn[c][1];
      }
    }

    if constexpr (DEC) {
      // ---- decimation (fp64): horizontal 8 taps at column Xd of row r, then the vertical ring
      const bool odd_r = (i & 1) == 0;  // Yb even => r = Yb - 3 + i is odd for even i
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        // level 0 has no lo part: skip the (useless, issue-slot costing) fp64 adds of zero
        const double z0 = HILO ? (double)hn[c][0] + (double)ln[c][0] : (double)hn[c][0];
        const double z1 = HILO ? (double)hn[c][1] + (double)ln[c][1] : (double)hn[c][1];
        const double zL1 = HILO ? (double)nL[c] + (double)nlL[c] : (double)nL[c];
        const double zR2 = HILO ? (double)nR[c] + (double)nlR[c] : (double)nR[c];
        const double zL2 = shfl_up_d(z0, 1);   // x-2
        const double zL3 = shfl_up_d(z1, 2);   // x-3
        const double zR3 = shfl_dn_d(z1, 1);   // x+3
        const double zR4 = shfl_dn_d(z0, 2);   // x+4
        double hp = dw0 * (zL3 + zR4);
        hp = fma(dw1, zL2 + zR3, hp);
        hp = fma(dw2, zL1 + zR2, hp);
        hp = fma(dw3, z0 + z1, hp);
        if (odd_r) {
          dacc[0][c] = fma(dw1, hp, dacc[0][c]);  // w[6]
          dacc[1][c] = fma(dw3, hp, dacc[1][c]);  // w[4]
          dacc[2][c] = fma(dw2, hp, dacc[2][c]);  // w[2]
          dacc[3][c] = fma(dw0, hp, dacc[3][c]);  // w[0]
        } else {
          dacc[0][c] = fma(dw0, hp, dacc[0][c]);  // w[7]
          dacc[1][c] = fma(dw2, hp, dacc[1][c]);  // w[5]
          dacc[2][c] = fma(dw3, hp, dacc[2][c]);  // w[3]
          dacc[3][c] = fma(dw1, hp, dacc[3][c]);  // w[1]
        }
      }
      if (!odd_r) {
        const int Yd = (r - 4) / 2;  // completed row (r even)
        if (out_lane && Yd >= a.d_r0 && Yd < a.d_r0 + a.d_rn && Xd < a.W1 && i >= 7) {
          float* ph = a.ohi + oo;  // channel planes at +ostr32 (one IMAD.WIDE per store)
          float hi[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            hi[c] = (float)dacc[0][c];
            ph[c * ostr32] = hi[c];
          }
          if (has_lo) {
            float* pl = a.olo + oo;
#pragma unroll
            for (int c = 0; c < 3; ++c) pl[c * ostr32] = (float)(dacc[0][c] - (double)hi[c]);
          }
        }
        oo += a.out_pitch;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          dacc[0][c] = dacc[1][c];
          dacc[1][c] = dacc[2][c];
          dacc[2][c] = dacc[3][c];
          dacc[3][c] = 0.0;
        }
      }
    }

    if (SEL && i >= 2) {
      // ---- fp32 products at row c = r - 1 for columns x, x+1 (unscaled gradients 2g; at l >= 1
      //      (hi1 - hi0) + (lo1 - lo0), relative error ~2u of the exact fp64-level difference).
      //      Packed over the column pair: __ffma2_rn / __fmul2_rn / __fadd2_rn round each element
      //      exactly as fmaf / * / + do, so the results are those of the scalar form.
#if BLADE_DOWN_PACK >= 2
      const float2 m1 = make_float2(-1.0f, -1.0f);
      float2 A = make_float2(0.0f, 0.0f), B = A, C = A;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float2 gx = __ffma2_rn(make_float2(hL[c], hc[c][0]), m1, make_float2(hc[c][1], hR[c]));
        float2 gy = __ffma2_rn(make_float2(hm[c][0], hm[c][1]), m1, make_float2(hn[c][0], hn[c][1]));
        if constexpr (HILO) {
          gx = __fadd2_rn(gx, __ffma2_rn(make_float2(lL[c], lc[c][0]), m1, make_float2(lc[c][1], lR[c])));
          gy = __fadd2_rn(gy, __ffma2_rn(make_float2(lm[c][0], lm[c][1]), m1, make_float2(ln[c][0], ln[c][1])));
        }
        A = __ffma2_rn(gx, gx, A);
        B = __ffma2_rn(gx, gy, B);
        C = __ffma2_rn(gy, gy, C);
      }
#else
      float A0 = 0.0f, B0 = 0.0f, C0 = 0.0f, A1 = 0.0f, B1 = 0.0f, C1 = 0.0f;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float gx0 = hc[c][1] - hL[c], gx1 = hR[c] - hc[c][0];
        float gy0 = hn[c][0] - hm[c][0], gy1 = hn[c][1] - hm[c][1];
        if constexpr (HILO) {
          gx0 += lc[c][1] - lL[c];
          gx1 += lR[c] - lc[c][0];
          gy0 += ln[c][0] - lm[c][0];
          gy1 += ln[c][1] - lm[c][1];
        }
        A0 = fmaf(gx0, gx0, A0);
        B0 = fmaf(gx0, gy0, B0);
        C0 = fmaf(gy0, gy0, C0);
        A1 = fmaf(gx1, gx1, A1);
        B1 = fmaf(gx1, gy1, B1);
        C1 = fmaf(gy1, gy1, C1);
      }
      const float2 A = make_float2(A0, A1), B = make_float2(B0, B1), C = make_float2(C0, C1);
#endif
      // ---- horizontal window: products at x-2, x-1 (lane-1) and x+2, x+3 (lane+1); w symmetric:
      //      h[j] = w0 (p[j-2] + p[j+2]) + (w1 (p[j-1] + p[j+1]) + w2 p[j])
      const float2 w0v = make_float2(w0, w0), w1v = make_float2(w1, w1), w2v = make_float2(w2, w2);
      auto hwin = [&](float2 P) {
        const float2 M = make_float2(__shfl_up_sync(0xffffffffu, P.x, 1), __shfl_up_sync(0xffffffffu, P.y, 1));
        const float2 Q = make_float2(__shfl_down_sync(0xffffffffu, P.x, 1), __shfl_down_sync(0xffffffffu, P.y, 1));
#if BLADE_DOWN_PACK >= 2
        const float2 s2 = __fadd2_rn(M, Q);                                         // (m2+p2, m1+p3)
        const float2 s1 = __fadd2_rn(make_float2(M.y, P.x), make_float2(P.y, Q.x));  // (m1+p1, p0+p2)
        return __ffma2_rn(w0v, s2, __ffma2_rn(w1v, s1, __fmul2_rn(w2v, P)));
#else
        return make_float2(fmaf(w0, M.x + Q.x, fmaf(w1, M.y + P.y, w2 * P.x)),
                           fmaf(w0, M.y + Q.y, fmaf(w1, P.x + Q.x, w2 * P.y)));
#endif
      };
      const float2 hA = hwin(A), hB = hwin(B), hC = hwin(C);
      // ---- vertical window: pending rows y = c-2 .. c+2 get weight w[c - y + 2]
      const int y = r - 3;  // = c - 2: completes now
#if BLADE_DOWN_PACK >= 1
      const float2 fa = __ffma2_rn(w0v, hA, vA[0]), fb = __ffma2_rn(w0v, hB, vB[0]), fc = __ffma2_rn(w0v, hC, vC[0]);
      vA[0] = __ffma2_rn(w1v, hA, vA[1]); vB[0] = __ffma2_rn(w1v, hB, vB[1]); vC[0] = __ffma2_rn(w1v, hC, vC[1]);
      vA[1] = __ffma2_rn(w2v, hA, vA[2]); vB[1] = __ffma2_rn(w2v, hB, vB[2]); vC[1] = __ffma2_rn(w2v, hC, vC[2]);
      vA[2] = __ffma2_rn(w1v, hA, vA[3]); vB[2] = __ffma2_rn(w1v, hB, vB[3]); vC[2] = __ffma2_rn(w1v, hC, vC[3]);
      vA[3] = __fmul2_rn(w0v, hA);        vB[3] = __fmul2_rn(w0v, hB);        vC[3] = __fmul2_rn(w0v, hC);
#else
      auto f2 = [](float w, float2 h, float2 v) { return make_float2(fmaf(w, h.x, v.x), fmaf(w, h.y, v.y)); };
      const float2 fa = f2(w0, hA, vA[0]), fb = f2(w0, hB, vB[0]), fc = f2(w0, hC, vC[0]);
      vA[0] = f2(w1, hA, vA[1]); vB[0] = f2(w1, hB, vB[1]); vC[0] = f2(w1, hC, vC[1]);
      vA[1] = f2(w2, hA, vA[2]); vB[1] = f2(w2, hB, vB[2]); vC[1] = f2(w2, hC, vC[2]);
      vA[2] = f2(w1, hA, vA[3]); vB[2] = f2(w1, hB, vB[3]); vC[2] = f2(w1, hC, vC[3]);
      vA[3] = make_float2(w0 * hA.x, w0 * hA.y); vB[3] = make_float2(w0 * hB.x, w0 * hB.y);
      vC[3] = make_float2(w0 * hC.x, w0 * hC.y);
#endif
      // the first six rows of a task are its top halo: their window sums are incomplete and never
      // emitted, so their buckets are not evaluated (warp-uniform)
      if (i >= 6) {
        const bool emit = out_lane && y >= a.s_r0 && y < a.s_r0 + a.s_rn;
        bool safe0 = true, safe1 = true;
        const int bk0 = bucket32<FAST>(fa.x, fb.x, fc.x, prm, safe0);
        const int bk1 = bucket32<FAST>(fa.y, fb.y, fc.y, prm, safe1);
        const bool need_fb = emit && ((x < a.W && !safe0) || (x + 1 < a.W && !safe1));
        int b0 = bk0, b1 = bk1;
        if constexpr (IFIX) {  // rare: the uncertified pixels of this row, one fp64 warp pass each
          unsigned int m0 = __ballot_sync(0xffffffffu, emit && x < a.W && !safe0);
          unsigned int m1 = __ballot_sync(0xffffffffu, emit && x + 1 < a.W && !safe1);
          while (m0 | m1) {  // warp-uniform
            const int j = m0 ? 0 : 1;
            const int src = __ffs(j == 0 ? m0 : m1) - 1;
            if (j == 0) m0 &= m0 - 1; else m1 &= m1 - 1;
            const int xx = __shfl_sync(0xffffffffu, x, src) + j;
            const int k = fix_bucket<FAST>(FixLevel(a), prm, n, y, xx, lane);
            if (lane == src) {
              if (j == 0) b0 = k; else b1 = k;
            }
          }
        } else if (need_fb) {  // rare: queue the uncertified pixel(s) for the fp64 fix-up kernel
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (x + j >= a.W) continue;
            const unsigned int slot = atomicAdd(a.fb_count, 1u);
            if (slot < a.fb_cap)
              a.fb_list[slot] = ((unsigned long long)n * a.s_rn + (unsigned long long)(y - a.s_r0)) * a.W + x + j;
          }
        }
        if (emit && x < a.W) {
          MT* mrow = mrow_i;
          if (map16 && x + 1 < a.W) {  // both entries in one store
            if constexpr (WIDE)
              *reinterpret_cast<uint32_t*>(mrow) = (uint32_t)b0 | ((uint32_t)b1 << 16);
            else
              *reinterpret_cast<uint16_t*>(mrow) = (uint16_t)(b0 | (b1 << 8));
          } else {
            mrow[0] = (MT)b0;
            if (x + 1 < a.W) mrow[1] = (MT)b1;
          }
        }
      }
    }
    // ---- rotate the gradient rows
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      hm[c][0] = hc[c][0];
      hm[c][1] = hc[c][1];
      hc[c][0] = hn[c][0];
      hc[c][1] = hn[c][1];
      hL[c] = nL[c];
      hR[c] = nR[c];
      lm[c][0] = lc[c][0];
      lm[c][1] = lc[c][1];
      lc[c][0] = ln[c][0];
      lc[c][1] = ln[c][1];
      lL[c] = nlL[c];
      lR[c] = nlR[c];
    }
  }
  BT_EXIT(HILO ? 1 : 0);
}

// Fix-up of the uncertified pixels of one k_down launch: fp64 (a, b, c) and the bucket rule in
// fp64-derived fp32 as the fp64 selector. If the list overflowed (pathological inputs with many
// exactly isotropic tensors), every map entry of the launch is recomputed.
template <bool HILO, bool FAST, bool WIDE>
__global__ void __launch_bounds__(128) k_down_fixup(const DownArgs a, const DownParams prm) {
  using MT = typename std::conditional<WIDE, uint16_t, uint8_t>::type;
  // one warp per pixel: lane t < 25 evaluates the gradient products at window offset
  // (t / 5 - 2, t % 5 - 2) in fp64, the weighted products are summed over the warp (fp64)
  pdl_trigger();
  pdl_wait();
  const unsigned int cnt = *a.fb_count;
  const bool all = cnt > a.fb_cap;
  const unsigned long long per_frame = (unsigned long long)a.s_rn * a.W;
  const unsigned long long items = all ? (unsigned long long)a.N * per_frame : (unsigned long long)cnt;
  const int lane = threadIdx.x & 31;
  const unsigned long long warps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
  for (unsigned long long i = blockIdx.x * (unsigned long long)(blockDim.x >> 5) + (threadIdx.x >> 5); i < items;
       i += warps) {
    const unsigned long long e = all ? i : a.fb_list[i];
    const int n = (int)(e / per_frame);
    const unsigned long long r = e - (unsigned long long)n * per_frame;
    const int y = a.s_r0 + (int)(r / a.W), xx = (int)(r % a.W);
    double pa = 0.0, pb = 0.0, pc = 0.0;
    if (lane < 25) {
      const int dy = lane / 5 - 2, dx = lane % 5 - 2;
      auto Z = [&](int c, int yy, int xq) -> double {
        int br = fold_idx(yy, a.H) - a.in_row0;
        br = min(max(br, 0), a.in_rows - 1);
        const long long o = (long long)n * a.in_frame + c * a.in_plane + (long long)br * a.in_pitch + fold_idx(xq, a.W);
        double v = (double)a.zhi[o];
        if constexpr (HILO) v += (double)a.zlo[o];
        return v;
      };
      const int yy = y + dy, xq = xx + dx;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double gx = Z(c, yy, xq + 1) - Z(c, yy, xq - 1);
        const double gy = Z(c, yy + 1, xq) - Z(c, yy - 1, xq);
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
    if (lane == 0)
      static_cast<MT*>(a.map)[((unsigned long long)n * a.s_rn + (unsigned long long)(y - a.s_r0)) * a.map_pitch + xx] =
          (MT)bucket_of<FAST>(pa, pb, pc, prm);
  }
}

// All selector levels' fix-ups of one cascade in ONE launch (up to kFixMax levels): the lists
// are only needed by the stages, which run after every k_down, so the per-level fix-up launches
// merge into one after the down pass (one launch instead of L-1; c1: -7 us of 64).
constexpr int kFixMax = 4;
struct FixupMulti {
  DownArgs a[kFixMax];
  DownParams prm[kFixMax];
  int n;  // levels in use
};

template <bool FAST, bool WIDE>
__device__ __forceinline__ void fixup_pixel(const FixLevel& a, const DownParams& prm, unsigned long long i,
                                            bool all, int lane) {
  using MT = typename std::conditional<WIDE, uint16_t, uint8_t>::type;
  const unsigned long long per_frame = (unsigned long long)a.s_rn * a.W;
  const unsigned long long e = all ? i : a.fb_list[i];
  const int n = (int)(e / per_frame);
  const unsigned long long r = e - (unsigned long long)n * per_frame;
  const int y = a.s_r0 + (int)(r / a.W), xx = (int)(r % a.W);
  const int k = fix_bucket<FAST>(a, prm, n, y, xx, lane);
  if (lane == 0)
    static_cast<MT*>(a.map)[((unsigned long long)n * a.s_rn + (unsigned long long)(y - a.s_r0)) * a.map_pitch + xx] =
        (MT)k;
}

template <bool FAST, bool WIDE>
__global__ void __launch_bounds__(128) k_down_fixup_multi(const __grid_constant__ FixupMulti m) {
  BT_ENTRY(2);
  pdl_trigger();
  pdl_wait();
  BT_WAITED(2);
  unsigned long long items[kFixMax];
  bool all[kFixMax];
  unsigned long long total = 0;
#pragma unroll
  for (int l = 0; l < kFixMax; ++l) {
    items[l] = 0;
    all[l] = false;
    if (l < m.n) {
      const unsigned int cnt = *m.a[l].fb_count;
      all[l] = cnt > m.a[l].fb_cap;  // overflow: the whole map of that level
      items[l] = all[l] ? (unsigned long long)m.a[l].N * m.a[l].s_rn * m.a[l].W : (unsigned long long)cnt;
      total += items[l];
    }
  }
  // one pass over the concatenated lists: every warp takes at most ceil(total / warps) pixels of
  // any level (the calls this serves are small: one pixel latency per warp)
  const int lane = threadIdx.x & 31;
  const unsigned long long warps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
  for (unsigned long long i = blockIdx.x * (unsigned long long)(blockDim.x >> 5) + (threadIdx.x >> 5); i < total;
       i += warps) {
    unsigned long long j = i;
    int l = 0;
    while (l + 1 < m.n && j >= items[l]) {  // warp-uniform
      j -= items[l];
      ++l;
    }
    fixup_pixel<FAST, WIDE>(FixLevel(m.a[l]), m.prm[l], j, all[l], lane);
  }
  BT_EXIT(2);
}

}  // namespace blade
