// NEXT f4: filter learning of PAPER.md:186-198 (§3, Eqs. 7-8) on the GPU — the per-(phase, bucket)
// normal equations G = sum x x^T, m = sum x u of the stacked sample x = [R_i z^l ; R_{i/2} u^{l+1}]
// (ABI tap order, R27), accumulated in fp64 as a segmented SYRK:
//   k_train_hist    count the pixels of every segment s = phase * K + bucket
//   k_train_scan    exclusive scan of the counts (one CTA)
//   k_train_scatter counting sort of the pixel indices by segment
//   k_train_gram    each CTA walks a slice of the sorted pixels in batches of 32: it gathers the
//                   samples of the three channels (fine patch, coarse patch, target appended as
//                   column nt) into shared memory as fp64, every thread accumulates 4 x 4 blocks of
//                   the extended matrix E = sum [x; u][x; u]^T in registers (upper block triangle),
//                   and flushes them with fp64 atomics to E[segment] when the segment changes.
// E[s] (NTP x NTP, NTP = nt + 1 rounded up to 4) holds G in [0, nt)^2 and m in column nt.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <type_traits>

#include "kernels.cuh"

namespace blade {

struct TrainArgs {
  const float* z;       // noisy level l [N][3][H][W]
  const float* uc;      // clean target at level l [N][3][H][W]
  const float* u1;      // u^{l+1} [N][3][H1][W1] (nullptr when single-level)
  const void* map;      // bucket map [N][H][W] (uint8, or uint16 when WIDE)
  int N, H, W, H1, W1;
  int n_phases, K, n_seg;
  unsigned int* count;  // [n_seg] (per call)
  unsigned int* cursor; // [n_seg]
  unsigned int* sorted; // [N H W] pixel indices sorted by segment
  double* E;            // [n_seg][NTP][NTP] (accumulated)
  unsigned long long* count_out;  // [n_seg] (accumulated)
  int pix_per_cta;
};

template <bool WIDE>
__device__ __forceinline__ int train_seg(const TrainArgs& a, unsigned int i) {
  using MT = typename std::conditional<WIDE, uint16_t, uint8_t>::type;
  const unsigned int hw = (unsigned int)a.H * (unsigned int)a.W;  // N H W < 2^32 (host check)
  const unsigned int r = i % hw;
  const int y = (int)(r / (unsigned int)a.W), x = (int)(r - (unsigned int)y * (unsigned int)a.W);
  const int k = static_cast<const MT*>(a.map)[i];
  const int p = a.n_phases == 4 ? 2 * (y & 1) + (x & 1) : 0;
  return p * a.K + k;
}

template <bool WIDE>
__global__ void __launch_bounds__(256) k_train_hist(const TrainArgs a) {
  extern __shared__ unsigned int hist[];
  for (int i = threadIdx.x; i < a.n_seg; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const long long total = (long long)a.N * a.H * a.W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
    atomicAdd(&hist[train_seg<WIDE>(a, (unsigned int)i)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < a.n_seg; i += blockDim.x)
    if (hist[i]) atomicAdd(&a.count[i], hist[i]);
}

// one CTA of 1024 threads: cursor = exclusive scan of count; count_out += count
template <int = 0>
__global__ void __launch_bounds__(1024) k_train_scan(const TrainArgs a) {
  __shared__ unsigned int part[1024];
  const int t = threadIdx.x;
  const int per = (a.n_seg + 1023) / 1024;
  const int b0 = t * per, b1 = min(b0 + per, a.n_seg);
  unsigned int s = 0;
  for (int i = b0; i < b1; ++i) s += a.count[i];
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele scan
    const unsigned int v = t >= off ? part[t - off] : 0u;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  unsigned int run = part[t] - s;  // exclusive prefix of this thread's range
  for (int i = b0; i < b1; ++i) {
    a.cursor[i] = run;
    run += a.count[i];
    a.count_out[i] += a.count[i];
  }
}

// Counting-sort scatter by chunks of consecutive pixels: a CTA counts its chunk's pixels per
// segment in shared memory, reserves one contiguous run per segment with a single global atomic,
// then places the chunk's pixels inside those runs (shared-memory atomics). One global atomic per
// (chunk, segment) instead of per pixel; a segment's list is a sequence of per-chunk runs.
template <bool WIDE>
__global__ void __launch_bounds__(512) k_train_scatter(const TrainArgs a) {
  extern __shared__ unsigned int sc[];  // [n_seg] chunk counts / placement cursors, [n_seg] bases
  unsigned int* cnt = sc;
  unsigned int* base = sc + a.n_seg;
  constexpr int CHUNK = 8192;
  const long long total = (long long)a.N * a.H * a.W;
  for (long long c0 = (long long)blockIdx.x * CHUNK; c0 < total; c0 += (long long)gridDim.x * CHUNK) {
    const long long c1 = min(total, c0 + CHUNK);
    for (int i = threadIdx.x; i < a.n_seg; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) atomicAdd(&cnt[train_seg<WIDE>(a, (unsigned int)i)], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < a.n_seg; i += blockDim.x) {
      const unsigned int n = cnt[i];
      base[i] = n ? atomicAdd(&a.cursor[i], n) : 0u;
      cnt[i] = 0;
    }
    __syncthreads();
    for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
      const int sg = train_seg<WIDE>(a, (unsigned int)i);
      a.sorted[base[sg] + atomicAdd(&cnt[sg], 1u)] = (unsigned int)i;
    }
    __syncthreads();
  }
}

template <int NF, int NC>
struct TrainShape {
  static constexpr int NT = NF * NF + NC * NC;
  static constexpr int NTP = (NT + 1 + 3) & ~3;  // + target column, 4-aligned
  static constexpr int NB = NTP / 4;
  static constexpr int UB = NB * (NB + 1) / 2;    // upper 4 x 4 blocks
  static constexpr int THREADS = 256;
  static constexpr int BPT = (UB + THREADS - 1) / THREADS;  // blocks per thread
  static constexpr int GROUPS = UB <= THREADS ? THREADS / UB : 1;  // thread groups splitting the samples
  static constexpr int BATCH = NTP <= 64 ? 32 : 16;  // pixels per gather (<= 40 KB of fp64)
  static_assert(BPT <= 2, "training supports nt + 1 <= 88 (up to 7x7 + 5x5 pairs / 9x9 single)");
};

template <int NF, int NC, bool WIDE>
__global__ void __launch_bounds__(256) k_train_gram(const TrainArgs a) {
  using TS = TrainShape<NF, NC>;
  constexpr int NTP = TS::NTP, NT = TS::NT, B = TS::BATCH;
  constexpr int RF = NF / 2, RC = NC / 2;
  __shared__ double xs[B][3][NTP];
  __shared__ int segs[B];
  const int t = threadIdx.x;
  // this thread's upper blocks (ra, cb); with GROUPS > 1 the blocks are replicated over thread
  // groups that take every GROUPS-th pixel of a batch (no idle threads for small filters)
  const int grp = TS::GROUPS > 1 ? t / TS::UB : 0;
  const int tb = TS::GROUPS > 1 ? t - grp * TS::UB : t;
  int ba[TS::BPT], bb[TS::BPT];
  bool act[TS::BPT];
#pragma unroll
  for (int q = 0; q < TS::BPT; ++q) {
    int blk = tb + q * TS::THREADS;
    act[q] = blk < TS::UB && grp < TS::GROUPS;
    int r = 0;
    while (act[q] && blk >= TS::NB - r) {
      blk -= TS::NB - r;
      ++r;
    }
    ba[q] = r;
    bb[q] = r + blk;
  }
  double acc[TS::BPT][4][4];
#pragma unroll
  for (int q = 0; q < TS::BPT; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[q][i][j] = 0.0;

  const long long total = (long long)a.N * a.H * a.W;
  const long long r0 = (long long)blockIdx.x * a.pix_per_cta;
  const long long r1 = min(total, r0 + a.pix_per_cta);
  int cur = -1;
  auto flush = [&]() {
    if (cur < 0) return;
    double* Es = a.E + (long long)cur * NTP * NTP;
#pragma unroll
    for (int q = 0; q < TS::BPT; ++q) {
      if (!act[q]) continue;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          atomicAdd(Es + (4 * ba[q] + i) * NTP + 4 * bb[q] + j, acc[q][i][j]);
          acc[q][i][j] = 0.0;
        }
    }
  };
  const unsigned int hw = (unsigned int)a.H * (unsigned int)a.W;  // N H W < 2^32 (checked on the host)
  __shared__ int pn[B];
  // per batch pixel: folded row offsets (row * W, into the frame's plane) and folded columns of its
  // fine and coarse windows, computed once per pixel instead of once per gathered sample
  __shared__ int frow[B][NF], fcol[B][NF];
  __shared__ int crow[B][NC > 0 ? NC : 1], ccol[B][NC > 0 ? NC : 1];
  __shared__ int ctr[B];  // offset of the centre pixel in its plane
  for (int e = t; e < B * 3 * (NTP - NT - 1); e += TS::THREADS) {  // padding columns stay zero
    const int j = e / (3 * (NTP - NT - 1)), rem = e - j * 3 * (NTP - NT - 1);
    const int c = rem / (NTP - NT - 1), q = rem - c * (NTP - NT - 1);
    xs[j][c][NT + 1 + q] = 0.0;
  }
  for (long long b0 = r0; b0 < r1; b0 += B) {
    const int nb = (int)min((long long)B, r1 - b0);
    __syncthreads();  // previous batch consumed
    // ---- decode the batch's pixels once (32-bit), with their segments
    if (t < nb) {
      const unsigned int pix = a.sorted[b0 + t];
      const unsigned int n = pix / hw, r = pix - n * hw;
      const unsigned int y = r / (unsigned int)a.W;
      pn[t] = (int)n;
      ctr[t] = (int)r;
      segs[t] = train_seg<WIDE>(a, pix);
      const int yy = (int)y, xx = (int)(r - y * (unsigned int)a.W);
#pragma unroll
      for (int d = 0; d < NF; ++d) {
        frow[t][d] = fold_idx(yy + d - RF, a.H) * a.W;
        fcol[t][d] = fold_idx(xx + d - RF, a.W);
      }
      if constexpr (NC > 0) {
#pragma unroll
        for (int d = 0; d < NC; ++d) {
          crow[t][d] = fold_idx(yy / 2 + d - RC, a.H1) * a.W1;
          ccol[t][d] = fold_idx(xx / 2 + d - RC, a.W1);
        }
      }
    }
    __syncthreads();
    // ---- gather the samples (fp64): fine taps, coarse taps, target (column NT); three
    //      branch-free loops so the lanes of a warp stay converged
    const long long plane = (long long)a.H * a.W, plane1 = (long long)a.H1 * a.W1;
    for (int e = t; e < nb * 3 * NF * NF; e += TS::THREADS) {
      const int j = e / (3 * NF * NF), rem = e - j * (3 * NF * NF);
      const int c = rem / (NF * NF), tap = rem - c * (NF * NF);
      const int dy = tap / NF, dx = tap - dy * NF;
      xs[j][c][tap] = (double)__ldg(a.z + ((long long)pn[j] * 3 + c) * plane + frow[j][dy] + fcol[j][dx]);
    }
    if constexpr (NC > 0) {
      for (int e = t; e < nb * 3 * NC * NC; e += TS::THREADS) {
        const int j = e / (3 * NC * NC), rem = e - j * (3 * NC * NC);
        const int c = rem / (NC * NC), tc = rem - c * (NC * NC);
        const int dy = tc / NC, dx = tc - dy * NC;
        xs[j][c][NF * NF + tc] = (double)__ldg(a.u1 + ((long long)pn[j] * 3 + c) * plane1 + crow[j][dy] + ccol[j][dx]);
      }
    }
    for (int e = t; e < nb * 3; e += TS::THREADS) {
      const int j = e / 3, c = e - 3 * j;
      xs[j][c][NT] = (double)__ldg(a.uc + ((long long)pn[j] * 3 + c) * plane + ctr[j]);
    }
    __syncthreads();
    // ---- accumulate (uniform over the CTA: segment changes flush)
    for (int j = grp; j < nb; j += TS::GROUPS) {
      const int sg = segs[j];
      if (sg != cur) {
        flush();
        cur = sg;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int q = 0; q < TS::BPT; ++q) {
          if (!act[q]) continue;
          const double* xa = &xs[j][c][4 * ba[q]];
          const double* xb = &xs[j][c][4 * bb[q]];
          double va[4], vb[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            va[i] = xa[i];
            vb[i] = xb[i];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[q][i][k] = fma(va[i], vb[k], acc[q][i][k]);
        }
      }
    }
  }
  flush();
}


// ---- k_train_gram_mma: the same accumulation on the FP64 tensor cores (DMMA, mma.sync
// m8n8k4 .f64). The batch's samples (pixel j, channel c) are the K dimension: for an 8 x 8 block
// (I, J) of the upper block triangle, D += A B with A[r][k] = x_k[8I + r], B[k][c] = x_k[8J + c]
// over steps of 4 samples. One warp owns every 8th block; its fragments are loaded straight
// from the shared sample rows (stride NTPX doubles: the 16 lanes of a half warp hit distinct
// bank pairs). Samples of another segment inside a 4-sample step are masked to zero, so every
// MMA adds only the current segment's samples; the segment changes flush with fp64 atomics as
// before. Entries written: (r, c) with r / 8 <= c / 8 (a superset of E's upper 4 x 4-block
// triangle contract); rows / columns >= NTP do not exist in E and are skipped.
template <int NF, int NC>
struct TrainMmaShape {
  static constexpr int NT = NF * NF + NC * NC;
  static constexpr int NTP = (NT + 1 + 3) & ~3;     // E's row pitch (TrainShape)
  static constexpr int NTP8 = (NT + 1 + 7) & ~7;    // 8-aligned columns of a sample row
  // sample-row stride in doubles, = 4 (mod 8): the 4 rows x 4 columns a half warp's fragment
  // loads touch land on 16 distinct 8-byte bank pairs
  static constexpr int NTPX = NTP8 + 4;
  static constexpr int NB = NTP8 / 8;
  static constexpr int UB = NB * (NB + 1) / 2;      // upper 8 x 8 blocks
  static constexpr int WARPS = 8;
  static constexpr int BPW = (UB + WARPS - 1) / WARPS;  // blocks per warp
  static constexpr int BATCH = NTPX <= 64 ? 24 : 16;    // pixels per gather (<= 48 KB static smem)
};

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NF, int NC, bool WIDE>
__global__ void __launch_bounds__(256) k_train_gram_mma(const TrainArgs a) {
  using TS = TrainMmaShape<NF, NC>;
  constexpr int NTP = TS::NTP, NTPX = TS::NTPX, NT = TS::NT, B = TS::BATCH;
  constexpr int RF = NF / 2, RC = NC / 2;
  static_assert(NTPX % 8 == 4, "sample stride");
  __shared__ double xs[B * 3][NTPX];
  __shared__ int segs[B];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int g = lane >> 2, q = lane & 3;  // MMA fragment coordinates
  // this warp's blocks: b = warp, warp + 8, ...; block index -> (I, J), I <= J
  int bI[TS::BPW], bJ[TS::BPW];
  bool act[TS::BPW];
#pragma unroll
  for (int k = 0; k < TS::BPW; ++k) {
    int blk = warp + k * TS::WARPS;
    act[k] = blk < TS::UB;
    int r = 0;
    while (act[k] && blk >= TS::NB - r) {
      blk -= TS::NB - r;
      ++r;
    }
    bI[k] = r;
    bJ[k] = r + blk;
  }
  double acc[TS::BPW][2];
#pragma unroll
  for (int k = 0; k < TS::BPW; ++k) acc[k][0] = acc[k][1] = 0.0;

  const long long total = (long long)a.N * a.H * a.W;
  const long long r0 = (long long)blockIdx.x * a.pix_per_cta;
  const long long r1 = min(total, r0 + a.pix_per_cta);
  int cur = -1;
  auto flush = [&]() {
    if (cur < 0) return;
    double* Es = a.E + (long long)cur * NTP * NTP;
#pragma unroll
    for (int k = 0; k < TS::BPW; ++k) {
      if (!act[k]) continue;
      const int row = 8 * bI[k] + g, col = 8 * bJ[k] + 2 * q;
      if (row < NTP) {
        if (col < NTP) atomicAdd(Es + row * NTP + col, acc[k][0]);
        if (col + 1 < NTP) atomicAdd(Es + row * NTP + col + 1, acc[k][1]);
      }
      acc[k][0] = acc[k][1] = 0.0;
    }
  };
  const unsigned int hw = (unsigned int)a.H * (unsigned int)a.W;
  __shared__ int pn[B];
  __shared__ int frow[B][NF], fcol[B][NF];
  __shared__ int crow[B][NC > 0 ? NC : 1], ccol[B][NC > 0 ? NC : 1];
  __shared__ int ctr[B];
  for (int e = t; e < B * 3 * (NTPX - NT - 1); e += 256) {  // padding columns stay zero
    const int j = e / (NTPX - NT - 1), c = e - j * (NTPX - NT - 1);
    xs[j][NT + 1 + c] = 0.0;
  }
  for (long long b0 = r0; b0 < r1; b0 += B) {
    const int nb = (int)min((long long)B, r1 - b0);
    __syncthreads();  // previous batch consumed
    if (t < nb) {
      const unsigned int pix = a.sorted[b0 + t];
      const unsigned int n = pix / hw, r = pix - n * hw;
      const unsigned int y = r / (unsigned int)a.W;
      pn[t] = (int)n;
      ctr[t] = (int)r;
      segs[t] = train_seg<WIDE>(a, pix);
      const int yy = (int)y, xx = (int)(r - y * (unsigned int)a.W);
#pragma unroll
      for (int d = 0; d < NF; ++d) {
        frow[t][d] = fold_idx(yy + d - RF, a.H) * a.W;
        fcol[t][d] = fold_idx(xx + d - RF, a.W);
      }
      if constexpr (NC > 0) {
#pragma unroll
        for (int d = 0; d < NC; ++d) {
          crow[t][d] = fold_idx(yy / 2 + d - RC, a.H1) * a.W1;
          ccol[t][d] = fold_idx(xx / 2 + d - RC, a.W1);
        }
      }
    }
    __syncthreads();
    const long long plane = (long long)a.H * a.W, plane1 = (long long)a.H1 * a.W1;
    for (int e = t; e < nb * 3 * NF * NF; e += 256) {
      const int j = e / (3 * NF * NF), rem = e - j * (3 * NF * NF);
      const int c = rem / (NF * NF), tap = rem - c * (NF * NF);
      const int dy = tap / NF, dx = tap - dy * NF;
      xs[3 * j + c][tap] = (double)__ldg(a.z + ((long long)pn[j] * 3 + c) * plane + frow[j][dy] + fcol[j][dx]);
    }
    if constexpr (NC > 0) {
      for (int e = t; e < nb * 3 * NC * NC; e += 256) {
        const int j = e / (3 * NC * NC), rem = e - j * (3 * NC * NC);
        const int c = rem / (NC * NC), tc = rem - c * (NC * NC);
        const int dy = tc / NC, dx = tc - dy * NC;
        xs[3 * j + c][NF * NF + tc] = (double)__ldg(a.u1 + ((long long)pn[j] * 3 + c) * plane1 + crow[j][dy] + ccol[j][dx]);
      }
    }
    for (int e = t; e < nb * 3; e += 256) {
      const int j = e / 3, c = e - 3 * j;
      xs[e][NT] = (double)__ldg(a.uc + ((long long)pn[j] * 3 + c) * plane + ctr[j]);
    }
    __syncthreads();
    // ---- runs of one segment within the batch (uniform over the CTA). The pixels are sorted by
    //      segment, so segs[] is non-decreasing: a run ends at the first larger entry (binary
    //      search; the whole batch when its last pixel is in the first pixel's segment)
    const int ns = 3 * nb;
    int pos = 0;
    while (pos < ns) {
      const int sg = segs[pos / 3];
      if (sg != cur) {
        flush();
        cur = sg;
      }
      int end;
      if (segs[nb - 1] == sg) {
        end = ns;
      } else {
        int lo = pos / 3, hi = nb - 1;  // segs[lo] == sg < segs[hi]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (segs[mid] == sg) lo = mid; else hi = mid;
        }
        end = 3 * hi;
      }
      const int full0 = (pos + 3) & ~3, full1 = end & ~3;  // 4-sample steps wholly inside the run
      auto step = [&](int k0, bool masked) {
        const int smp = k0 + q;
        const bool ok = !masked || (smp >= pos && smp < end);
        const double* xr = &xs[ok ? smp : 0][0];
#pragma unroll
        for (int k = 0; k < TS::BPW; ++k) {
          if (!act[k]) continue;  // warp-uniform
          const double av = xr[8 * bI[k] + g];
          const double bv = xr[8 * bJ[k] + g];
          dmma_884(acc[k][0], acc[k][1], ok ? av : 0.0, ok ? bv : 0.0);
        }
      };
      if (full0 >= full1) {  // a short run: every step masked
        for (int k0 = pos & ~3; k0 < end; k0 += 4) step(k0, true);
      } else {
        if ((pos & 3) != 0) step(pos & ~3, true);
        for (int k0 = full0; k0 < full1; k0 += 4) step(k0, false);
        if (end & 3) step(full1, true);
      }
      pos = end;
    }
  }
  flush();
}
}  // namespace blade
