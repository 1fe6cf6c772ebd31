// K3 k_stage_tma: the stage of Eq. 9 (§4) / Eq. 1 (§3) with
// TMA-staged, double-buffered tiles. Used whenever the whole bank of a stage (all phases) fits in
// shared memory next to two staging buffers (5x5 / 3x3 pairs, every single-level footprint).
//
// Persistent CTA (1 per SM): copy the stage's bank (4 phases x K filters, odd tap stride) into
// shared memory once, then loop over 16 x 128 output tiles. For tile i+1 one elected thread
// issues three cp.async.bulk.tensor loads (fine patch of z^l with an r_f halo, coarse patch of
// u^{l+1} with an r_c halo, the uint8 bucket tile) into the other buffer, completing on an
// mbarrier, while all threads compute tile i. TMA fills out-of-image cells with zeros; on border
// tiles a fix-up pass overwrites them with the folded sample (R2), taken from the tile
// itself or, for tiny levels, from global memory.
//
// Each thread computes an RY x 4 pixel block (RY = 2 or 4 rows from an even row y; columns
// x..x+3): all four 2x2 output phases, so phase(i, j) = 2 (i & 1) + (j & 1) is static and the two
// coarse centres floor(x/2), floor(x/2)+1 are shared by column pairs. Per input row the thread
// loads its window segment once (LDS.128 / LDS.64, conflict-free) and feeds it to up to RY pixel
// rows; the taps are loaded per pixel (LDS.128 rows at per-pixel addresses) and shared by the
// three colour channels (R13). FP32 FMA on the CUDA cores. RY = 4 (4 warps per group, 8 per SM)
// is used on large, wide levels: 16% fewer shared-memory wavefronts per pixel.
#pragma once
#include <cuda.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "k_down.cuh"
#include "kernels.cuh"

namespace blade {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// One bulk (non-tensor) copy global -> shared of `bytes` (multiple of 16, both ends 16-B aligned)
// by the TMA engine, completing on an mbarrier: the whole bank in one instruction.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// The cells of a rows x cols staging box with image origin (gy0, gx0) that fall outside
// [0, H) x [0, W): top rows, then the left / right columns of the middle rows, then bottom rows.
// oob_count() sizes the enumeration, oob_cell() maps its index e to the box cell (r, q), so a
// border fix-up touches only the out-of-image cells instead of testing the whole box.
struct OobBox {
  int cols, top, mid, left, right, n;
};
__device__ __forceinline__ OobBox oob_box(int rows, int cols, int gy0, int gx0, int H, int W) {
  OobBox b;
  b.cols = cols;
  b.top = min(rows, max(0, -gy0));
  const int bot = rows - max(b.top, min(rows, H - gy0));
  b.mid = rows - b.top - bot;
  b.left = min(cols, max(0, -gx0));
  b.right = cols - max(b.left, min(cols, W - gx0));
  b.n = (b.top + bot) * cols + b.mid * (b.left + b.right);
  return b;
}
__device__ __forceinline__ void oob_cell(const OobBox& b, int e, int& r, int& q) {
  const int nt = b.top * b.cols;
  if (e < nt) {
    r = e / b.cols;
    q = e - r * b.cols;
    return;
  }
  e -= nt;
  const int lr = b.left + b.right;
  if (e < b.mid * lr) {
    const int rr = e / lr, k = e - rr * lr;
    r = b.top + rr;
    q = k < b.left ? k : b.cols - b.right + (k - b.left);
    return;
  }
  e -= b.mid * lr;
  const int rb = e / b.cols;
  r = b.top + b.mid + rb;
  q = e - rb * b.cols;
}

// Loads N consecutive floats from p into v[0..N). The address of p is congruent to A floats
// modulo 4 (i.e. p - A is 16-B aligned when MAXV == 4, 8-B aligned when MAXV == 2); at each
// position the widest naturally aligned LDS (up to MAXV floats) is used. Compile-time recursion.
template <int A, int I, int N, int MAXV>
__device__ __forceinline__ void lds_run_at(const float* p, float* v) {
  if constexpr (I < N) {
    if constexpr (MAXV >= 4 && ((A + I) & 3) == 0 && I + 3 < N) {
      const float4 t = *reinterpret_cast<const float4*>(p + I);
      v[I] = t.x; v[I + 1] = t.y; v[I + 2] = t.z; v[I + 3] = t.w;
      lds_run_at<A, I + 4, N, MAXV>(p, v);
    } else if constexpr (MAXV >= 2 && ((A + I) & 1) == 0 && I + 1 < N) {
      const float2 t = *reinterpret_cast<const float2*>(p + I);
      v[I] = t.x; v[I + 1] = t.y;
      lds_run_at<A, I + 2, N, MAXV>(p, v);
    } else {
      v[I] = p[I];
      lds_run_at<A, I + 1, N, MAXV>(p, v);
    }
  }
}
template <int A, int N, int MAXV = 4>
__device__ __forceinline__ void lds_run(const float* p, float* v) {
  lds_run_at<A, 0, N, MAXV>(p, v);
}

// The fine window row of a thread (N floats from a column congruent to A mod 4). For the 5 x 5
// fine block (A = 2, N = 8: LDS.64, LDS.128, LDS.64) the two 8-byte end loads of a half warp
// (lanes 16 B apart) hit every bank twice: lanes tx and tx + 8 share banks. Lanes 8..15 of each
// half warp therefore load the right pair first and the left pair second, so each LDS.64 covers
// the 32 banks once (2 wavefronts instead of 4; the values are swapped back by 4 selects).
// Other shapes: lds_run.
template <int A, int N>
__device__ __forceinline__ void lds_fine(const float* p, float* v, bool swap) {
  if constexpr (A == 2 && N == 8) {
    const float2 P = *reinterpret_cast<const float2*>(p + (swap ? 6 : 0));
    const float4 M = *reinterpret_cast<const float4*>(p + 2);
    const float2 Q = *reinterpret_cast<const float2*>(p + (swap ? 0 : 6));
    v[0] = swap ? Q.x : P.x;
    v[1] = swap ? Q.y : P.y;
    v[2] = M.x; v[3] = M.y; v[4] = M.z; v[5] = M.w;
    v[6] = swap ? P.x : Q.x;
    v[7] = swap ? P.y : Q.y;
  } else {
    lds_run<A, N>(p, v);
  }
}

// Tap layout of one (phase, bucket) filter for this kernel (LDS.128-friendly): for every row of
// the fine block (NF x NF) and then of the coarse block (NC x NC), the first 4 floor(n / 4) taps as
// float4 chunks; after all chunks, the remaining n % 4 taps of every row. The filter stride S is
// rounded up to a multiple of 4 floats with S / 4 odd (spreads the per-pixel 16-B tap loads over
// the 8 bank groups). Used by the host re-layout (blade_ms_create) and, with compile-time
// arguments, by the kernel.
__host__ __device__ constexpr int tma_tap_off(int nf, int nc, int block, int dy, int dx) {
  const int qf = nf / 4, qc = nc / 4, vec = 4 * (nf * qf + nc * qc);
  if (block == 0)
    return dx < 4 * qf ? 4 * (dy * qf + dx / 4) + dx % 4 : vec + dy * (nf % 4) + (dx - 4 * qf);
  return dx < 4 * qc ? 4 * (nf * qf + dy * qc + dx / 4) + dx % 4
                     : vec + nf * (nf % 4) + dy * (nc % 4) + (dx - 4 * qc);
}
__host__ __device__ constexpr int tma_tap_stride(int nf, int nc) {
  const int r = (nf * nf + nc * nc + 3) & ~3;
  return ((r / 4) & 1) ? r : r + 4;
}

// Loads the NB taps of row dy of `block` of the filter at tp (16-B aligned) into t[0..NB).
// GL: the bank lives in global memory (L2-resident, read-only path) instead of shared memory.
template <int NF, int NC, int BLOCK, bool GL = false>
__device__ __forceinline__ void load_tap_row(const float* tp, int dy, float* t) {
  constexpr int NB = BLOCK == 0 ? NF : NC;
#pragma unroll
  for (int q = 0; q < NB / 4; ++q) {
    const float4* p4 = reinterpret_cast<const float4*>(tp + tma_tap_off(NF, NC, BLOCK, dy, 4 * q));
    const float4 v = GL ? __ldg(p4) : *p4;
    t[4 * q] = v.x;
    t[4 * q + 1] = v.y;
    t[4 * q + 2] = v.z;
    t[4 * q + 3] = v.w;
  }
#pragma unroll
  for (int k = 4 * (NB / 4); k < NB; ++k) {
    const float* p = tp + tma_tap_off(NF, NC, BLOCK, dy, k);
    t[k] = GL ? __ldg(p) : *p;
  }
}

// RY: pixel rows per thread (2 or 4); a tile is always 16 x 128 outputs, so RY = 4 runs 4 warps
// per group (one window row then feeds 4 pixel rows instead of 2: fewer shared-memory wavefronts
// per pixel, 8 warps per SM).
// FSEL (fused selector, level 0): the fine box carries FH = max(RF, 3) halo rows so that the
// kernel computes the bucket map of its own tile (gradient 1 + window 2 rows) instead of loading
// it; the FIR reads the box from row FRO = FH - RF.
template <int NF, int NC, bool WIDE = false, int RY_ = 2, bool FSEL = false, int TR = 16>
struct TmaShape {
  static constexpr int RX = 4, RY = RY_, BX = 32, BY = TR / RY_;
  static constexpr int threads = BX * BY;
  static constexpr int RF = NF / 2, RC = NC / 2;
  static constexpr int FH = FSEL ? (RF > 3 ? RF : 3) : RF;
  static constexpr int FRO = FH - RF;
  static constexpr int TCOLS = BX * RX, TROWS = BY * RY;  // 128 x 16 outputs per tile
  // TMA box starts must be 16-B aligned in the innermost dimension (a box at column 2 faults with
  // an illegal instruction: scripts/probes/tma_probe.cu), so both boxes start 4 columns left of
  // the tile (covers halos up to 4) and the windows start at FO / CO inside.
  static constexpr int FM = 4, CM = 4;
  static constexpr int FO = FM - RF, CO = CM - RC;
  static constexpr int FR = TROWS + 2 * FH;
  static constexpr int FCB = TCOLS + 2 * FM;            // 136
  static constexpr int CR = NC ? TROWS / 2 + 2 * RC : 0;
  static constexpr int CCB = NC ? TCOLS / 2 + 2 * CM : 0;  // 72
  static_assert(RF <= FM && RC <= CM, "halo wider than the TMA margin");
  static constexpr int fine_bytes = 3 * FR * FCB * 4;
  static constexpr int coarse_bytes = 3 * CR * CCB * 4;
  static constexpr int map_bytes = TROWS * TCOLS * (WIDE ? 2 : 1);  // uint16 buckets when WIDE
  static constexpr int al(int x) { return (x + 127) & ~127; }
  static constexpr int fine_off = 0;
  static constexpr int coarse_off = al(fine_bytes);
  static constexpr int map_off = coarse_off + al(coarse_bytes);
  static constexpr int stage_bytes = map_off + al(map_bytes);
  static constexpr int FWIN = NF + RX - 1;  // fine window columns per thread
  static constexpr int CWIN = NC + 1;       // coarse window columns per thread
  static constexpr int S = tma_tap_stride(NF, NC);
};

struct StageTmaArgs {
  int H, W;            // level l dims (global)
  int H1, W1;          // level l+1 dims
  int z_row0, z_rows;  // rows of the z^l buffer
  int u_row0, u_rows;  // rows of the u^{l+1} buffer
  int map_row0, map_rows;
  const float* z;      // z^l buffer (generic pointer, fix-up path for tiny levels)
  const float* u1;
  float* out;          // u^l buffer, rows [out_row0, out_row0 + out_rows)
  int out_row0, out_rows;
  const float* bank;   // [phase][PS] for this stage
  int K, S, PS, n_phases;
  int N;
  int y_base;          // first tile row (even)
  int o_r0, o_rn;      // output rows computed
  int tiles_x, tiles_y, n_tiles;
  int clamp;
  int u_rgb;           // CH3 (k_stage_ph): the coarse input is RGB z^{L-1}, not YCbCr planes
  int z_pitch, u_pitch, out_pitch;  // floats per row of the z^l, u^{l+1} and output buffers
  // FSEL: the selector of the tile (FAST layout), fp32 with the certificate of k_down; the
  // uncertified in-range pixels are queued (map-index format of k_down) for k_stage_fixup
  float sw0, sw1, sw2;            // window weights at offsets 2, 1, 0 (symmetric)
  float tsR[2], kcR[2];           // DownParams' transformed thresholds (FAST selector)
  int tc_nonpos;
  unsigned long long* fb_list;
  unsigned int* fb_count;
  unsigned int fb_cap;
};

// FSEL: buckets of the thread's RY x 4 pixels (rows y .. y+RY-1, cols x .. x+3) from the box
// `sf` (3 planes of FR x FCB, box origin (Y0 - FH, X0 - FM)): the arithmetic of k_down (level 0:
// exact fp32 inputs) — unscaled central differences, products summed over the channels with
// fmaf, the 5-tap horizontal window, then the vertical window as the same 4-deep ring of fmaf —
// and its certified fp32 decision. Streams the RY + 6 box rows y-3 .. y+RY+2 (columns x-4 ..
// x+7, three LDS.128 per row and channel), one product row per (not unrolled) iteration; the
// buckets go to the tile's shared map (the thread's own entries, read back by the same thread)
// and the uncertified in-range pixels to the fix-up list.
template <int RY, int FR, int FCB, int FH, int TCOLS>
__device__ __forceinline__ void fused_buckets(const float* sf, uint8_t* smap, int ty, int tx, int n, int y, int x,
                                              const StageTmaArgs& a) {
  DownParams prm;
  prm.tsR[0] = a.tsR[0];
  prm.tsR[1] = a.tsR[1];
  prm.kcR[0] = a.kcR[0];
  prm.kcR[1] = a.kcR[1];
  prm.tc_nonpos = a.tc_nonpos;
  const float* zb = sf + (RY * ty + FH - 3) * FCB + 4 * tx;  // box row of y - 3, column of x - 4
  float zp[3][8], zc[3][10];  // Z(r - 1) at columns x-2 .. x+5, Z(r) at x-3 .. x+6
  auto load_row = [&](int rr, int c, float* v12) {
    const float* p = zb + (c * FR + rr) * FCB;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const float4 t = *reinterpret_cast<const float4*>(p + 4 * q);
      v12[4 * q] = t.x; v12[4 * q + 1] = t.y; v12[4 * q + 2] = t.z; v12[4 * q + 3] = t.w;
    }
  };
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float v[12];
    load_row(0, c, v);  // y - 3
#pragma unroll
    for (int k = 0; k < 8; ++k) zp[c][k] = v[k + 2];
    load_row(1, c, v);  // y - 2
#pragma unroll
    for (int k = 0; k < 10; ++k) zc[c][k] = v[k + 1];
  }
  float vA[4][4], vB[4][4], vC[4][4];  // pending window rows (k_down's ring), 4 columns
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) vA[k][j] = vB[k][j] = vC[k][j] = 0.0f;
  const float w0 = a.sw0, w1 = a.sw1, w2 = a.sw2;
  // product rows pr = y-2 .. y+RY+1; output row pr - 2 completes from s = 4 on
#pragma unroll 1
  for (int s = 0; s < RY + 4; ++s) {
    float A[8], B[8], C[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) A[k] = B[k] = C[k] = 0.0f;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float zn[12];
      load_row(s + 2, c, zn);  // Z(pr + 1) at columns x-4 .. x+7
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // column x - 2 + k
        const float gx = zc[c][k + 2] - zc[c][k];
        const float gy = zn[k + 2] - zp[c][k];
        A[k] = fmaf(gx, gx, A[k]);
        B[k] = fmaf(gx, gy, B[k]);
        C[k] = fmaf(gy, gy, C[k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) zp[c][k] = zc[c][k + 1];
#pragma unroll
      for (int k = 0; k < 10; ++k) zc[c][k] = zn[k + 1];
    }
    const int yy = y + s - 4;
    uint32_t word = 0;
    bool emit = s >= 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // output column x + j <-> products k = j + 2
      const float hA = fmaf(w0, A[j] + A[j + 4], fmaf(w1, A[j + 1] + A[j + 3], w2 * A[j + 2]));
      const float hB = fmaf(w0, B[j] + B[j + 4], fmaf(w1, B[j + 1] + B[j + 3], w2 * B[j + 2]));
      const float hC = fmaf(w0, C[j] + C[j + 4], fmaf(w1, C[j + 1] + C[j + 3], w2 * C[j + 2]));
      const float fa = fmaf(w0, hA, vA[0][j]), fb = fmaf(w0, hB, vB[0][j]), fc = fmaf(w0, hC, vC[0][j]);
      if (emit) {
        bool ok = true;
        const int bk = bucket32<true>(fa, fb, fc, prm, ok);
        word |= (uint32_t)bk << (8 * j);
        if (!ok && yy >= a.o_r0 && yy < a.o_r0 + a.o_rn && x + j < a.W) {  // rare
          const unsigned int slot = atomicAdd(a.fb_count, 1u);
          if (slot < a.fb_cap)
            a.fb_list[slot] = ((unsigned long long)n * a.o_rn + (unsigned long long)(yy - a.o_r0)) * a.W + x + j;
        }
      }
      vA[0][j] = fmaf(w1, hA, vA[1][j]); vB[0][j] = fmaf(w1, hB, vB[1][j]); vC[0][j] = fmaf(w1, hC, vC[1][j]);
      vA[1][j] = fmaf(w2, hA, vA[2][j]); vB[1][j] = fmaf(w2, hB, vB[2][j]); vC[1][j] = fmaf(w2, hC, vC[2][j]);
      vA[2][j] = fmaf(w1, hA, vA[3][j]); vB[2][j] = fmaf(w1, hB, vB[3][j]); vC[2][j] = fmaf(w1, hC, vC[3][j]);
      vA[3][j] = w0 * hA;                vB[3][j] = w0 * hB;                vC[3][j] = w0 * hC;
    }
    if (emit) *reinterpret_cast<uint32_t*>(smap + (RY * ty + s - 4) * TCOLS + 4 * tx) = word;
  }
}

// G = 1: one 256-thread group, double-buffered tiles (TMA of tile i+1 overlaps tile i).
// G >= 3 (A/B builds): G groups, one buffer each — e.g. three 3-warp groups on 12-row tiles fill
//        the shared memory (3 x 36 KB + the 120 KB bank) so that two groups compute while one
//        waits for its TMA; measured slower than two 4-warp groups (profiles/r02_stage_groups.txt).
// G = 2: two 256-thread groups (16 warps) share the bank; each group owns one tile buffer and works
//        on every other tile, so one group computes while the other waits for its TMA (twice the
//        resident warps for the same shared memory).
// CH3 (per-channel Y/Cb/Cr banks, NEXT f1): CTA b serves channel b % 3 (all four phases of that
// channel's bank); the staged patches are converted to that channel in plane 0 after the fix-up
// (the coarse patch only when it is the RGB z^{L-1}; else plane chn of the YCbCr u^{l+1} is read).
// WIDE (NEXT f2, K > 256): uint16 bucket tiles and the bank read from global memory (the paper's
// 16 x 16 x 16 layout is 4.8 MB per stage: L2-resident, not shared-memory resident).
// BLADE_STAGE_MAXNREG (A/B builds): cap the registers instead of the launch bounds, so that a
// k_down CTA fits next to the stage CTA on one SM (co-scheduled down / up passes).
#ifdef BLADE_STAGE_MAXNREG
#define BLADE_STAGE_BOUNDS(threads) \
  __maxnreg__((threads) <= 256 ? BLADE_STAGE_MAXNREG : (65536 / (threads)) & ~7)
#else
#define BLADE_STAGE_BOUNDS(threads) __launch_bounds__(threads, 1)
#endif
template <int NF, int NC, int G, bool CH3, bool WIDE = false, int RY = 2, bool FSEL = false, int TR = 16>
__global__ void BLADE_STAGE_BOUNDS(32 * (TR / RY) * G)
    k_stage_tma(const __grid_constant__ CUtensorMap tm_z, const __grid_constant__ CUtensorMap tm_u,
                const __grid_constant__ CUtensorMap tm_map, StageTmaArgs a) {
  using SS = TmaShape<NF, NC, WIDE, RY, FSEL, TR>;
  static_assert(!FSEL || (!WIDE && !CH3 && NC > 0), "fused selector: shared-bank pair stages only");
  constexpr int RF = SS::RF, RC = SS::RC;
  constexpr int PL = CH3 ? 1 : 3;
  const int chn = CH3 ? (int)(blockIdx.x % 3) : 0;
  const int cta = CH3 ? (int)(blockIdx.x / 3) : (int)blockIdx.x;
  const int nctas = CH3 ? (int)(gridDim.x / 3) : (int)gridDim.x;
  extern __shared__ __align__(128) unsigned char tma_smem[];
  // layout: [stage buffers x2][bank][mbarriers]
  unsigned char* buf0 = tma_smem;
  const int bank_floats = a.n_phases * a.PS;
  constexpr int NB = G >= 2 ? G : 2;  // tile buffers: one per group, or a double buffer (G = 1)
  float* sbank = reinterpret_cast<float*>(tma_smem + NB * SS::stage_bytes);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(tma_smem + NB * SS::stage_bytes +
                                               (WIDE ? 0 : ((bank_floats * 4 + 127) & ~127)));
  const float* bank = WIDE ? a.bank + (long long)chn * bank_floats : sbank;

  const int g = G >= 2 ? (int)(threadIdx.y / SS::BY) : 0;  // thread group
  const int ty = (int)(threadIdx.y % SS::BY), tx = threadIdx.x;
  const int tid = ty * SS::BX + tx;  // thread index within the group
  auto group_sync = [&]() {
    if constexpr (G >= 2)
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(SS::threads) : "memory");
    else
      __syncthreads();
  };
  constexpr uint32_t tx_bytes = SS::fine_bytes + SS::coarse_bytes + (FSEL ? 0 : SS::map_bytes);

  auto tile_coords = [&](int t, int& n, int& X0, int& Y0) {
    n = t / (a.tiles_x * a.tiles_y);
    const int rem = t - n * a.tiles_x * a.tiles_y;
    const int tyi = rem / a.tiles_x;
    X0 = (rem - tyi * a.tiles_x) * SS::TCOLS;
    Y0 = a.y_base + tyi * SS::TROWS;
  };
  auto issue = [&](int t, int b) {
    int n, X0, Y0;
    tile_coords(t, n, X0, Y0);
    unsigned char* sb = buf0 + b * SS::stage_bytes;
    mbar_expect_tx(&mbar[b], tx_bytes);
    tma_load_3d(sb + SS::fine_off, &tm_z, X0 - SS::FM, Y0 - SS::FH - a.z_row0, n * 3, &mbar[b]);
    if constexpr (NC > 0)
      tma_load_3d(sb + SS::coarse_off, &tm_u, X0 / 2 - SS::CM, Y0 / 2 - RC - a.u_row0, n * 3, &mbar[b]);
    if constexpr (!FSEL) tma_load_3d(sb + SS::map_off, &tm_map, X0, Y0 - a.map_row0, n, &mbar[b]);
  };

  const int ctid = threadIdx.y * SS::BX + threadIdx.x;
  int t = cta + g * nctas;
  const int tstride = G * nctas;
  [[maybe_unused]] const int bt_k = 8 + 2 * (a.W >= 512 ? 1 : 0);  // trace kind (probe builds)
  BT_ENTRY(bt_k);
  pdl_trigger();
  if (ctid == 0) {
#pragma unroll
    for (int q = 0; q <= NB; ++q) mbar_init(&mbar[q], 1);  // [0, NB): tile buffers, NB: the bank
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // ---- the bank -> shared memory, once, by one bulk copy (constant data: issued before
    //      waiting on the previous grid)
    if (!WIDE) {
      mbar_expect_tx(&mbar[NB], (uint32_t)bank_floats * 4u);
      bulk_g2s(sbank, a.bank + (long long)chn * bank_floats, (uint32_t)bank_floats * 4u, &mbar[NB]);
    }
  }
  pdl_wait();
  BT_WAITED(bt_k);
  __syncthreads();
  if (tid == 0 && t < a.n_tiles) issue(t, g);
  if (!WIDE) mbar_wait(&mbar[NB], 0);
  BT_WAITED(bt_k + 1);  // bank resident

  for (int it = 0; t < a.n_tiles; ++it, t += tstride) {
    const int b = G >= 2 ? g : (it & 1);
    const int tn = t + tstride;
    if (G == 1 && tid == 0 && tn < a.n_tiles) {
      fence_proxy_async();  // generic-proxy accesses of buffer b^1 (previous tile) are ordered
      issue(tn, b ^ 1);
    }
    int n, X0, Y0;
    tile_coords(t, n, X0, Y0);
    mbar_wait(&mbar[b], G >= 2 ? (it & 1) : ((it >> 1) & 1));
    float* sfine = reinterpret_cast<float*>(buf0 + b * SS::stage_bytes + SS::fine_off);
    float* scoarse = reinterpret_cast<float*>(buf0 + b * SS::stage_bytes + SS::coarse_off);
    const uint8_t* smap = buf0 + b * SS::stage_bytes + SS::map_off;

    // ---- border fix-up: out-of-image cells <- folded samples
    const int FX = X0 - SS::FM, CX = X0 / 2 - SS::CM;  // box origins (columns)
    const bool fine_border = FX < 0 || FX + SS::FCB > a.W || Y0 - SS::FH < 0 || Y0 + SS::TROWS + SS::FH > a.H;
    const bool coarse_border = NC > 0 && (CX < 0 || CX + SS::CCB > a.W1 || Y0 / 2 - RC < 0 ||
                                          Y0 / 2 - RC + SS::CR > a.H1);
    // only the box cells some in-range output pixel reads are fixed up (the output rows of the
    // tile and its in-image columns, +- the footprint): on levels narrower or shorter than a tile
    // most of the box lies outside the image and is never read (c0: 64 x 64 in a 20 x 136 box)
    const int py_lo = max(Y0, a.o_r0), py_hi = min(Y0 + SS::TROWS, a.o_r0 + a.o_rn);
    const int px_hi = min(X0 + SS::TCOLS, a.W);
    if ((fine_border || coarse_border) && py_lo < py_hi) {
      if (fine_border) {
        const int r0 = max(0, py_lo - SS::FH - (Y0 - SS::FH)), r1 = min(SS::FR, py_hi + SS::FH - (Y0 - SS::FH));
        const int c0 = max(0, X0 - SS::FH - FX), c1 = min(SS::FCB, px_hi + SS::FH - FX);
        const OobBox ob = oob_box(r1 - r0, c1 - c0, Y0 - SS::FH + r0, FX + c0, a.H, a.W);
        for (int i = tid; i < ob.n; i += SS::threads) {
          int r, q;
          oob_cell(ob, i, r, q);
          r += r0;
          q += c0;
          const int gy = Y0 - SS::FH + r, gx = FX + q;
          const int fy = fold_idx(gy, a.H), fx = fold_idx(gx, a.W);
          const int ry = fy - (Y0 - SS::FH), rx = fx - FX;
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
      if constexpr (NC > 0) {
        if (coarse_border) {
          const int CY0 = Y0 / 2 - RC, CX0 = CX;
          const int r0 = max(0, py_lo / 2 - RC - CY0), r1 = min(SS::CR, (py_hi - 1) / 2 + RC + 1 - CY0);
          const int c0 = max(0, X0 / 2 - RC - CX0), c1 = min(SS::CCB, (px_hi - 1) / 2 + RC + 1 - CX0);
          const OobBox ob = oob_box(r1 - r0, c1 - c0, CY0 + r0, CX0 + c0, a.H1, a.W1);
          for (int i = tid; i < ob.n; i += SS::threads) {
            int r, q;
            oob_cell(ob, i, r, q);
            r += r0;
            q += c0;
            const int gy = CY0 + r, gx = CX0 + q;
            const int fy = fold_idx(gy, a.H1), fx = fold_idx(gx, a.W1);
            const int ry = fy - CY0, rx = fx - CX0;
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
      }
      group_sync();
    }
    const float* scoarse_c = scoarse;
    if constexpr (CH3) {  // colour conversion of the staged patches into plane 0
      for (int i = tid; i < SS::FR * SS::FCB; i += SS::threads)
        sfine[i] = rgb_to_ycc_ch(chn, sfine[i], sfine[SS::FR * SS::FCB + i], sfine[2 * SS::FR * SS::FCB + i]);
      if constexpr (NC > 0) {
        if (a.u_rgb) {
          for (int i = tid; i < SS::CR * SS::CCB; i += SS::threads)
            scoarse[i] = rgb_to_ycc_ch(chn, scoarse[i], scoarse[SS::CR * SS::CCB + i], scoarse[2 * SS::CR * SS::CCB + i]);
        } else {
          scoarse_c = scoarse + chn * SS::CR * SS::CCB;
        }
      }
      group_sync();
    }

    // ---- this thread's RY x 4 block (rows y .. y+RY-1, y even; cols x .. x+3)
    const int x = X0 + SS::RX * tx;
    const int y = Y0 + RY * ty;
    constexpr int KB = WIDE ? 16 : 8;
    constexpr uint64_t KM = WIDE ? 0xffff : 0xff;
    int toff[RY][4];  // filter offsets in the bank: phase (2 (i & 1) + (j & 1)) x PS + bucket x S
    if constexpr (FSEL)  // this thread's buckets, from the staged tile, into its own map entries
      fused_buckets<RY, SS::FR, SS::FCB, SS::FH, SS::TCOLS>(sfine, const_cast<uint8_t*>(smap), ty, tx, n, y, x, a);
#pragma unroll
    for (int i = 0; i < RY; ++i) {
      uint64_t mrow;
      if constexpr (WIDE)
        mrow = *reinterpret_cast<const uint64_t*>(smap + 2 * ((RY * ty + i) * SS::TCOLS + 4 * tx));
      else
        mrow = *reinterpret_cast<const uint32_t*>(smap + (RY * ty + i) * SS::TCOLS + 4 * tx);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = (int)((mrow >> (KB * j)) & KM);
        const int ph = a.n_phases == 4 ? 2 * (i & 1) + (j & 1) : 0;
        toff[i][j] = ph * a.PS + k * SS::S;
      }
    }
    float acc[RY][4][PL];
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < PL; ++c) acc[i][j][c] = 0.0f;

    // threads whose block lies wholly outside the image (the right part of a partial last tile
    // column, rows past the last output row) issue no shared-memory traffic at all
    const bool active = x < a.W && y < a.o_r0 + a.o_rn && y + RY > a.o_r0;
    if (active) {
    if constexpr (NC > 0) {
      // coarse rows local ty RY/2 .. + NC + RY/2 - 1 (pixel row i sits on coarse row wr - i/2 of its
      // window); cols 2tx .. 2tx+NC
#pragma unroll
      for (int wr = 0; wr < NC + RY / 2 - 1; ++wr) {
        float v[PL][SS::CWIN];
#pragma unroll
        for (int c = 0; c < PL; ++c)
          lds_run<(SS::CO & 1), SS::CWIN, 2>(
              scoarse_c + (c * SS::CR + (RY / 2) * ty + wr) * SS::CCB + 2 * tx + SS::CO, v[c]);
#pragma unroll
        for (int i = 0; i < RY; ++i) {
          const int dy = wr - (i >> 1);
          if (dy < 0 || dy >= NC) continue;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float t[NC > 0 ? NC : 1];
            load_tap_row<NF, NC, 1, WIDE>(bank + toff[i][j], dy, t);
#pragma unroll
            for (int dx = 0; dx < NC; ++dx) {
#pragma unroll
              for (int c = 0; c < PL; ++c) acc[i][j][c] = fmaf(t[dx], v[c][(j >> 1) + dx], acc[i][j][c]);
            }
          }
        }
      }
    }
    // fine rows local RY ty .. RY ty + NF + RY - 2, cols 4tx .. 4tx+NF+2
    const bool swap8 = (tx >> 3) & 1;  // lds_fine: half-warp halves take the two end pairs in turn
#pragma unroll
    for (int wr = 0; wr < NF + RY - 1; ++wr) {
      float v[PL][SS::FWIN];
#pragma unroll
      for (int c = 0; c < PL; ++c)
        lds_fine<SS::FO, SS::FWIN>(sfine + (c * SS::FR + RY * ty + wr + SS::FRO) * SS::FCB + 4 * tx + SS::FO, v[c],
                                   swap8);
#pragma unroll
      for (int i = 0; i < RY; ++i) {
        const int dy = wr - i;
        if (dy < 0 || dy >= NF) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float t[NF];
          load_tap_row<NF, NC, 0, WIDE>(bank + toff[i][j], dy, t);
#pragma unroll
          for (int dx = 0; dx < NF; ++dx) {
#pragma unroll
            for (int c = 0; c < PL; ++c) acc[i][j][c] = fmaf(t[dx], v[c][j + dx], acc[i][j][c]);
          }
        }
      }
    }

    // ---- store (rows y .. y+RY-1; cols x .. x+3)
#pragma unroll
    for (int i = 0; i < RY; ++i) {
      const int yy = y + i;
      if (yy < a.o_r0 || yy >= a.o_r0 + a.o_rn || x >= a.W) continue;
      float* op = a.out + ((long long)n * 3 * a.out_rows + (yy - a.out_row0)) * a.out_pitch + x;
#pragma unroll
      for (int c = 0; c < PL; ++c) {
        float v0 = acc[i][0][c], v1 = acc[i][1][c], v2 = acc[i][2][c], v3 = acc[i][3][c];
        if (a.clamp) {
          v0 = fminf(fmaxf(v0, 0.0f), 1.0f);
          v1 = fminf(fmaxf(v1, 0.0f), 1.0f);
          v2 = fminf(fmaxf(v2, 0.0f), 1.0f);
          v3 = fminf(fmaxf(v3, 0.0f), 1.0f);
        }
        float* d = op + (long long)(CH3 ? chn : c) * a.out_rows * a.out_pitch;
        if (x + 3 < a.W) {
          *reinterpret_cast<float4*>(d) = make_float4(v0, v1, v2, v3);  // output rows are 16-B multiples
        } else {
          d[0] = v0;
          if (x + 1 < a.W) d[1] = v1;
          if (x + 2 < a.W) d[2] = v2;
        }
      }
    }
    }  // active
    group_sync();  // buffer b is free for the next TMA into it
    if (G >= 2 && tid == 0 && tn < a.n_tiles) {
      fence_proxy_async();
      issue(tn, b);
    }
  }
  BT_EXIT(bt_k);
}

// Fix-up of the fused-selector stage (level 0): the pixels whose fp32 orientation the certificate
// could not guarantee get their bucket in fp64 (the k_down_fixup arithmetic: one warp per pixel,
// lanes 0..24 the window taps) and their output recomputed with it: lanes take the taps t = lane,
// lane + 32, ... of the filter (ABI order: fine block then coarse block, generic bank layout) and
// the warp sums the three channels' partial dot products. If the list overflowed, every pixel of
// the launch is recomputed this way.
struct StageFixArgs {
  const float* z;  // level-0 input view: [N][3][z_rows][z_pitch], global rows from z_row0
  int z_row0, z_rows, z_pitch;
  const float* u1;  // u^1 buffer: [N][3][u_rows][u_pitch], global rows from u_row0
  int u_row0, u_rows, u_pitch;
  float* out;       // output view: [N][3][out_rows][out_pitch], global rows from out_row0
  int out_row0, out_rows, out_pitch;
  int H, W, H1, W1;
  int N, o_r0, o_rn;  // computed rows (the list's map-index space: [N][o_rn][W])
  const float* bank;  // generic layout of this stage: [phase][PS], filter k at k * S
  int S, PS, n_phases, clamp;
  const unsigned long long* fb_list;
  const unsigned int* fb_count;
  unsigned int fb_cap;
};

template <int NF, int NC>
__global__ void __launch_bounds__(128) k_stage_fixup(const StageFixArgs a, const DownParams prm) {
  constexpr int RF = NF / 2, RC = NC / 2;
  pdl_trigger();
  pdl_wait();
  const unsigned int cnt = *a.fb_count;
  const bool all = cnt > a.fb_cap;
  const unsigned long long per_frame = (unsigned long long)a.o_rn * a.W;
  const unsigned long long items = all ? (unsigned long long)a.N * per_frame : (unsigned long long)cnt;
  const int lane = threadIdx.x & 31;
  const unsigned long long warps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
  const long long zpl = (long long)a.z_rows * a.z_pitch, upl = (long long)a.u_rows * a.u_pitch;
  auto Z = [&](int n, int c, int yy, int xq) -> float {
    const int br = min(max(fold_idx(yy, a.H) - a.z_row0, 0), a.z_rows - 1);
    return a.z[((long long)n * 3 + c) * zpl + (long long)br * a.z_pitch + fold_idx(xq, a.W)];
  };
  for (unsigned long long i = blockIdx.x * (unsigned long long)(blockDim.x >> 5) + (threadIdx.x >> 5); i < items;
       i += warps) {
    const unsigned long long e = all ? i : a.fb_list[i];
    const int n = (int)(e / per_frame);
    const unsigned long long r = e - (unsigned long long)n * per_frame;
    const int y = a.o_r0 + (int)(r / a.W), x = (int)(r % a.W);
    // ---- fp64 bucket (k_down_fixup)
    double pa = 0.0, pb = 0.0, pc = 0.0;
    if (lane < 25) {
      const int dy = lane / 5 - 2, dx = lane % 5 - 2, yy = y + dy, xq = x + dx;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double gx = (double)Z(n, c, yy, xq + 1) - (double)Z(n, c, yy, xq - 1);
        const double gy = (double)Z(n, c, yy + 1, xq) - (double)Z(n, c, yy - 1, xq);
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
    const int k = __shfl_sync(0xffffffffu, bucket_of<true>(pa, pb, pc, prm), 0);
    // ---- Eq. 9 for this pixel with bucket k: lane c < 3 sums channel c with the stage kernels'
    //      fmaf order (coarse rows, then fine rows; dy, then dx ascending), so the output is the
    //      one those kernels give with the fp64 bucket (bands and batches stay bit-identical)
    const int ph = a.n_phases == 4 ? 2 * (y & 1) + (x & 1) : 0;
    const float* f = a.bank + (long long)ph * a.PS + (long long)k * a.S;
    if (lane < 3) {
      const int c = lane;
      float acc = 0.0f;
      for (int dy = 0; dy < NC; ++dy) {
        const int br = min(max(fold_idx(y / 2 + dy - RC, a.H1) - a.u_row0, 0), a.u_rows - 1);
        const float* urow = a.u1 + ((long long)n * 3 + c) * upl + (long long)br * a.u_pitch;
        for (int dx = 0; dx < NC; ++dx) acc = fmaf(f[NF * NF + dy * NC + dx], urow[fold_idx(x / 2 + dx - RC, a.W1)], acc);
      }
      for (int dy = 0; dy < NF; ++dy)
        for (int dx = 0; dx < NF; ++dx) acc = fmaf(f[dy * NF + dx], Z(n, c, y + dy - RF, x + dx - RF), acc);
      if (a.clamp) acc = fminf(fmaxf(acc, 0.0f), 1.0f);
      a.out[((long long)n * 3 + c) * a.out_rows * a.out_pitch + (long long)(y - a.out_row0) * a.out_pitch + x] = acc;
    }
  }
}

}  // namespace blade
