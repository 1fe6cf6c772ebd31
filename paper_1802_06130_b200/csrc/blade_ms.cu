// Host side of the C ABI declared in include/blade_ms.h: argument validation, filterbank
// re-layout, workspace/band planning, TMA descriptors and the per-level launch sequence
// (DESIGN.md §Boundary).
//
// The launch sequence for one call:
//   down pass   k_down(l): s^l = selector(z^l) and z^{l+1} = decimate(z^l)     l = 0 .. L-2
//   up pass     k_stage(l): u^l = stage(z^l, u^{l+1}, s^l)                        l = L-2 .. 0
//               (u^{L-1} = z^{L-1});  L == 1: k_down (selector only) + k_stage (Eq. 1).
// Every call is described by a Plan: for each level the GLOBAL rows of z^l and u^l that must be
// materialised. For a full image these are all rows; for a row band (blade_ms_denoise_rows) they
// are the band's dependency cone, so the same code serves both and bands are bit-identical.
//
// Data in HBM: z^0 = the caller's fp32 input; for l >= 1, z^l is kept in
// an fp32 pair hi + lo (hi = stage input; hi + lo = the exact fp64 decimation, input of the next
// selector and decimation, l <= L-2); u^l fp32; s^l uint8.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/blade_ms.h"
#include "k_down.cuh"
#include "k_stage_ph.cuh"
#include "k_stage_tma.cuh"
#include "kernels.cuh"
#include "tables.h"

using namespace blade;

namespace {

thread_local std::string g_last_error;

blade_status fail(blade_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e__ = (expr);                                                              \
    if (e__ != cudaSuccess)                                                                \
      return fail(BLADE_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e__), __FILE__, \
                  __LINE__);                                                               \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// ------------------------------------------------------------------------------ kernel tables
// (instantiated in their own translation units, tab_*.cu, compiled in parallel; tables.h)
using namespace blade::tables;
size_t down_smem(bool hilo) { return sizeof(float) * down::WARPS * down::RING * (hilo ? 6 : 3) * 64; }

// ------------------------------------------------------------------------------ TMA encode
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    else
      cudaGetLastError();
  });
  return g_encode;
}

// 3D tiled map over a [depth][rows][W] array of `esize`-byte elements.
bool encode_3d(CUtensorMap* tm, const void* base, CUtensorMapDataType dt, int esize, int W, int rows,
               int depth, int bw, int bh, int bd, int pitch = 0) {
  auto enc = get_encode();
  if (!enc) return false;
  if (pitch <= 0) pitch = W;  // row pitch in elements (the rows of a map may be padded)
  const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)rows, (cuuint64_t)depth};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch * esize, (cuuint64_t)pitch * esize * rows};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bd};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(tm, dt, 3, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ------------------------------------------------------------------------------ row ranges
struct Range {
  int lo = 0, hi = 0;  // [lo, hi)
  int n() const { return hi - lo; }
};

int fold_host(long long i, long long n) {
  long long p = 2 * n, m = i % p;
  if (m < 0) m += p;
  return (int)(m < n ? m : p - 1 - m);
}

// Hull of {fold(i, n) : lo <= i < hi}.
Range fold_hull(long long lo, long long hi, int n) {
  if (hi <= lo) return Range{0, 0};
  if (hi - lo >= 2LL * n) return Range{0, n};
  if (lo >= 0 && hi <= n) return Range{(int)lo, (int)hi};
  int mn = n, mx = -1;
  for (long long i = lo; i < hi; ++i) {
    const int f = fold_host(i, n);
    mn = std::min(mn, f);
    mx = std::max(mx, f);
  }
  return Range{mn, mx + 1};
}

Range hull(Range a, Range b) {
  if (a.n() <= 0) return b;
  if (b.n() <= 0) return a;
  return Range{std::min(a.lo, b.lo), std::max(a.hi, b.hi)};
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

struct blade_ms {
  blade_ms_config cfg;
  int n_o, n_s, n_c, K;
  int n_stages, nt, S, PS;    // generic stage kernel bank: tap stride (odd), phase stride
  int S_tma = 0, PS_tma = 0;  // TMA stage kernel bank (tma_tap_off layout)
  int device, num_sms;
  float* d_bank = nullptr;      // [stage][phase][PS], taps in ABI order per filter (k_stage)
  float* d_bank_tma = nullptr;  // [stage][phase][PS_tma], tma_tap_off layout (k_stage_tma)
  size_t bank_bytes = 0;
  std::vector<DownParams> down;  // per stage (selector level)
  int down_slots[2] = {1, 1};    // resident k_down warps on the device (level 0 / hi-lo levels)
  // generic stage kernel
  StageVariant stage{};
  size_t stage_smem = 0;
  int stage_ctas_per_sm = 0;
  // TMA stage kernel (if the shape has one and the bank fits)
  bool has_tma = false;
  TmaVariant tma{};
  bool has_tma4 = false;  // the 4-rows-per-thread variant of the same shape (large levels)
  TmaVariant tma4{};
  // fused selector at level 0 (the 4-row TMA stage computes s^0 itself; k_down only decimates)
  bool has_fsel = false;
  size_t fsel_smem = 0;
  StageFixKernel sfix = nullptr;
  size_t tma_smem = 0;
  // profiling (blade_ms_set_profiling): event pairs around each launch
  struct ProfRec { int kind, level; cudaEvent_t e0, e1; };
  bool profiling = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  // frame-chunked schedule (blade_ms_denoise_pipelined): internal streams, fork / join events
  static constexpr int kMaxStreams = 4;
  cudaStream_t pipe[kMaxStreams] = {};
  cudaEvent_t pipe_fork = nullptr;
  cudaEvent_t pipe_join[kMaxStreams] = {};
  // serialises whole pipelined calls on this handle: the fork / join events and the internal
  // streams are handle-wide, so one call's record-then-wait pairs must not interleave with
  // another's (a re-recorded pipe_fork would let a chunk wait on the wrong caller stream)
  std::mutex pipe_mu;
  // blade_ms_denoise_host: its copy streams and chunk events, created on first use and kept (a
  // small call paid ~0.2 ms of stream / event creation and destruction per call); host_mu
  // serialises whole host calls on this handle (they are synchronous anyway)
  static constexpr int kHostChunks = 32;
  cudaStream_t host_in = nullptr, host_out = nullptr;
  cudaEvent_t host_start = nullptr;
  cudaEvent_t host_ev_in[kHostChunks] = {}, host_ev_done[kHostChunks] = {};
  std::mutex host_mu;
};

namespace {

struct Plan {
  int L = 0, N = 0;
  std::vector<int> H, W;
  std::vector<Range> z;   // rows of the z^l buffer (level 0: needed input rows)
  std::vector<Range> zc;  // rows of z^l computed by the down pass, l >= 1 (= z unless exchanged)
  std::vector<Range> u;   // rows of u^l computed (= map rows), l <= L-2 (l = 0 if L == 1)
  std::vector<Range> ub;  // rows of the u^l buffer, 1 <= l <= L-2 (= u unless exchanged)
  size_t ws_bytes = 0;
  std::vector<size_t> z32_off, zlo_off, u_off, map_off, fb_off;
  std::vector<int> map_pitch;  // entries per map row: W_l rounded up to 16 (16-B TMA rows)
  std::vector<int> pitch;      // floats per workspace plane row at level l >= 1: W_l rounded up to 4
  size_t zcopy_off = 0;        // full-image calls with W % 4 != 0: a 16-B-row copy of the input
  int zcopy_pitch = 0;         //   (written by k_down at level 0, read by the level-0 TMA stage)
  size_t ocopy_off = 0;        //   and a 16-B-row staging buffer for the level-0 output
  std::vector<unsigned int> fb_cap;
  size_t fbcnt_off = 0;
};

// Dependency cone of output rows [o0, o0+on) of the final output.
void plan_rows_cfg(const blade_ms_config& cfg, int N, int H, int W, int o0, int on, Plan& p, int map_es = 1);
void plan_layout(Plan& p, int map_es, int W, bool full_image);
void plan_rows(const blade_ms* h, int N, int H, int W, int o0, int on, Plan& p) {
  plan_rows_cfg(h->cfg, N, H, W, o0, on, p, h->K > 256 ? 2 : 1);
}
void plan_rows_cfg(const blade_ms_config& cfg, int N, int H, int W, int o0, int on, Plan& p, int map_es) {
  const int L = cfg.levels;
  p.L = L;
  p.N = N;
  p.H.assign(L, 0);
  p.W.assign(L, 0);
  p.H[0] = H;
  p.W[0] = W;
  for (int l = 1; l < L; ++l) {
    p.H[l] = (p.H[l - 1] + 1) / 2;
    p.W[l] = (p.W[l - 1] + 1) / 2;
  }
  p.z.assign(L, Range{});
  p.u.assign(L, Range{});
  const int rf = cfg.fine_size / 2;
  const int rc = cfg.coarse_size / 2;
  const int ext = std::max(rf, cfg.window_size / 2 + 1);
  p.u[0] = Range{o0, o0 + on};
  if (L == 1) {
    p.z[0] = fold_hull((long long)o0 - ext, (long long)o0 + on + ext, H);
  } else {
    for (int l = 0; l + 1 < L; ++l) {
      p.z[l] = hull(p.z[l], fold_hull((long long)p.u[l].lo - ext, (long long)p.u[l].hi + ext, p.H[l]));
      const long long clo = (long long)(p.u[l].lo / 2) - rc;
      const long long chi = (long long)((p.u[l].hi - 1) / 2) + rc + 1;
      p.u[l + 1] = fold_hull(clo, chi, p.H[l + 1]);
    }
    p.z[L - 1] = hull(p.z[L - 1], p.u[L - 1]);
    for (int l = L - 1; l >= 1; --l) {
      const long long dlo = 2LL * p.z[l].lo - 3;
      const long long dhi = 2LL * (p.z[l].hi - 1) + 4 + 1;
      p.z[l - 1] = hull(p.z[l - 1], fold_hull(dlo, dhi, p.H[l - 1]));
    }
  }
  p.zc = p.z;
  p.ub = p.u;
  plan_layout(p, map_es, W, o0 == 0 && on == H);
}

// Workspace layout of a plan whose row ranges are set (Plan::z, zc, u, ub): level planes, maps,
// fix-up lists. full_image: the call covers every row (the 16-B-row input copy is possible).
void plan_layout(Plan& p, int map_es, int W, bool full_image) {
  const int L = p.L, N = p.N, H = p.H[0];
  size_t off = 0;
  p.z32_off.assign(L, 0);
  p.zlo_off.assign(L, 0);
  p.u_off.assign(L, 0);
  p.map_off.assign(L, 0);
  p.map_pitch.assign(L, 0);
  p.pitch.assign(L, 0);
  for (int l = 0; l < L; ++l) {
    p.map_pitch[l] = (p.W[l] + 15) & ~15;
    p.pitch[l] = l == 0 ? p.W[0] : (p.W[l] + 3) & ~3;  // 16-B rows: every level >= 1 is TMA-able
  }
  // z^l hi planes, directly followed by its lo planes (levels that feed a selector): the six
  // planes of a level are one uniform-stride run (one region for a halo exchange)
  for (int l = 1; l < L; ++l) {
    const size_t planes = sizeof(float) * (size_t)N * 3 * p.z[l].n() * p.pitch[l];
    p.z32_off[l] = off;
    if (l + 1 < L) {
      p.zlo_off[l] = off + planes;
      off = align256(off + 2 * planes);
    } else {
      off = align256(off + planes);
    }
  }
  for (int l = 1; l + 1 < L; ++l) {
    p.u_off[l] = off;
    off = align256(off + sizeof(float) * (size_t)N * 3 * p.ub[l].n() * p.pitch[l]);
  }
  const int nsel = L == 1 ? 1 : L - 1;
  for (int l = 0; l < nsel; ++l) {
    p.map_off[l] = off;
    off = align256(off + (size_t)map_es * N * p.u[l].n() * p.map_pitch[l]);
  }
  p.zcopy_pitch = 0;
  if (W % 4 != 0 && full_image) {  // full image whose rows the TMA engine cannot address
    p.zcopy_pitch = (W + 3) & ~3;
    p.zcopy_off = off;
    off = align256(off + sizeof(float) * (size_t)N * 3 * H * p.zcopy_pitch);
    p.ocopy_off = off;
    off = align256(off + sizeof(float) * (size_t)N * 3 * H * p.zcopy_pitch);
  }
  // uncertified-pixel lists of the fp32 selector (DESIGN.md §6 H1): 1/64 of each level's map
  p.fb_off.assign(nsel, 0);
  p.fb_cap.assign(nsel, 0);
  for (int l = 0; l < nsel; ++l) {
    const size_t px = (size_t)N * p.u[l].n() * p.W[l];
    p.fb_cap[l] = (unsigned int)std::min<size_t>(std::max<size_t>(px / 64, 1024), 0x7fffffffu);
    p.fb_off[l] = off;
    off = align256(off + sizeof(unsigned long long) * p.fb_cap[l]);
  }
  p.fbcnt_off = off;
  off = align256(off + sizeof(unsigned int) * 16);
  p.ws_bytes = std::max<size_t>(off, 256);
}

// NEXT f3 (b): the plan of one row band whose neighbours EXCHANGE halo rows between levels
// (DESIGN.md §10c): the band owns rows own^0 = [o0, o0 + on) and own^{l+1} = [ceil(lo/2),
// ceil(hi/2)) (a partition of every level when the bands partition the image), computes only
// those (z^{l+1} by its k_down, u^l and s^l by its stage / selector), and holds hz rows of z^l
// and hu rows of u^l around them, received from the neighbours. hz covers everything a level's
// kernels read around own rows: the selector (gradient + window: ws/2 + 1), the decimation
// (2y-3 .. 2y+4: 4), the fine taps (rf) and, through z^{L-1} = u^{L-1}, the coarse taps of the
// next finer stage (floor(y/2) +- rc: rc + 1). Returns false when a level of a proper band owns
// fewer than hz rows (its halo would need rows of a non-adjacent band).
bool plan_xband(const blade_ms_config& cfg, int map_es, int H, int W, int o0, int on, Plan& p, int& hz, int& hu,
                std::vector<Range>& own) {
  const int L = cfg.levels;
  p.L = L;
  p.N = 1;
  p.H.assign(L, 0);
  p.W.assign(L, 0);
  p.H[0] = H;
  p.W[0] = W;
  for (int l = 1; l < L; ++l) {
    p.H[l] = (p.H[l - 1] + 1) / 2;
    p.W[l] = (p.W[l - 1] + 1) / 2;
  }
  const int rf = cfg.fine_size / 2, rc = L > 1 ? cfg.coarse_size / 2 : 0;
  hu = L > 1 ? rc + 1 : 0;
  hz = std::max(std::max(rf, cfg.window_size / 2 + 1), std::max(L > 1 ? 4 : 0, hu));
  own.assign(L, Range{});
  own[0] = Range{o0, o0 + on};
  for (int l = 1; l < L; ++l) own[l] = Range{(own[l - 1].lo + 1) / 2, (own[l - 1].hi + 1) / 2};
  const bool whole = o0 == 0 && on == H;
  for (int l = 0; l < L; ++l)
    if (!whole && own[l].n() < hz) return false;
  p.z.assign(L, Range{});
  p.zc.assign(L, Range{});
  p.u.assign(L, Range{});
  p.ub.assign(L, Range{});
  for (int l = 0; l < L; ++l) {
    p.z[l] = fold_hull((long long)own[l].lo - hz, (long long)own[l].hi + hz, p.H[l]);
    p.zc[l] = own[l];
  }
  const int nsel = L == 1 ? 1 : L - 1;
  for (int l = 0; l < nsel; ++l) {
    p.u[l] = own[l];
    p.ub[l] = l == 0 ? own[0] : fold_hull((long long)own[l].lo - hu, (long long)own[l].hi + hu, p.H[l]);
  }
  plan_layout(p, map_es, W, false);
  return true;
}

LevelView make_view(float* base, int H, int W, Range r, int pitch = 0) {
  LevelView v;
  v.p = base;
  v.H = H;
  v.W = W;
  v.pitch = pitch > 0 ? pitch : W;
  v.row0 = r.lo;
  v.rows = r.n();
  v.plane = (long long)r.n() * v.pitch;
  v.frame = 3 * v.plane;
  return v;
}

blade_status check_dev_ptr(const blade_ms* h, const void* p, const char* what) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(BLADE_EDEVICE, "%s: not a CUDA pointer (%s)", what, cudaGetErrorString(e));
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return fail(BLADE_EDEVICE, "%s: not device memory", what);
  if (at.device != h->device)
    return fail(BLADE_EDEVICE, "%s: on device %d, handle on device %d", what, at.device, h->device);
  return BLADE_OK;
}

bool ranges_overlap(const void* a, size_t an, const void* b, size_t bn) {
  const char* pa = (const char*)a;
  const char* pb = (const char*)b;
  return pa < pb + bn && pb < pa + an;
}

cudaEvent_t prof_event(blade_ms* h) {
  if (!h->ev_pool.empty()) {
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return e;
}

// Brackets one launch with events when profiling is on.
struct ProfScope {
  blade_ms* h;
  cudaStream_t st;
  int kind, level;
  cudaEvent_t e0 = nullptr;
  ProfScope(const blade_ms* hc, cudaStream_t s, int k, int l)
      : h(const_cast<blade_ms*>(hc)), st(s), kind(k), level(l) {
    if (h->profiling && (e0 = prof_event(h))) cudaEventRecord(e0, st);
  }
  ~ProfScope() {
    if (!e0) return;
    cudaEvent_t e1 = prof_event(h);
    if (!e1) return;
    cudaEventRecord(e1, st);
    h->prof.push_back(blade_ms::ProfRec{kind, level, e0, e1});
  }
};

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// BLADE_SYNC_DEBUG=1: synchronise after every launch and name the kernel that failed.
bool sync_debug() {
  static const bool on = [] {
    const char* e = getenv("BLADE_SYNC_DEBUG");
    return e && e[0] == '1';
  }();
  return on;
}
#define LAUNCH_CHECK(name)                                                                       \
  do {                                                                                           \
    cudaError_t e__ = cudaGetLastError();                                                        \
    if (e__ == cudaSuccess && sync_debug()) e__ = cudaStreamSynchronize(st);                     \
    if (e__ != cudaSuccess)                                                                      \
      return fail(BLADE_ECUDA, "%s (level %d): %s", name, l, cudaGetErrorString(e__));           \
  } while (0)

// BLADE_TMA_RY=2 / =4 forces the 2- / 4-row TMA stage variant on every level (A/B timing);
// default 0 = by level size.
int tma4_rows() {  // tile rows of the 4-row-thread stage variant (16: two groups; A/B builds may
                   // instantiate others, e.g. 12-row tiles in three groups: slower, r02_stage_groups)
  static const int v = [] {
    const char* e = getenv("BLADE_TMA4_ROWS");
    return e ? atoi(e) : 16;
  }();
  return v;
}
// BLADE_P2=0 keeps pair banks that fit two phases per CTA on the one-phase kernel (A/B timing)
bool p2_enabled() {
  static const bool on = [] {
    const char* e = getenv("BLADE_P2");
    return !(e && e[0] == '0');
  }();
  return on;
}
int tma_ry() {
  static const int v = [] {
    const char* e = getenv("BLADE_TMA_RY");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// Rows per thread of the TMA stage kernel for a level of width W whose computed rows span
// `span`: large levels (many tiles per SM) at least 8 tiles wide take 4, others 2 (measured: c3
// level 0 2.56 -> 2.36 ms; c3 level 1, 7.5 tiles wide, 0.718 -> 0.675 ms on the round-2 build
// (0.75 -> 0.80 in round 1, before the border fix-up was limited to the cells pixels read); the
// latency-bound small levels are slower with 8 warps per SM).
bool use_ry4(const blade_ms* h, int N, int W, int span) {
  if (!h->has_tma4 || tma_ry() == 2) return false;
  if (tma_ry() == 4) return true;
  const int tiles_x = (W + h->tma.tcols - 1) / h->tma.tcols;
  const long long tiles = (long long)N * tiles_x * ((span + h->tma.trows - 1) / h->tma.trows);
  return tiles_x >= 8 && tiles >= 8LL * h->num_sms;
}

// The fp64 fix-ups of all selector levels run as one launch after the down pass on small calls
// (launch-latency-bound: c1 63 -> 58 us warm), per level right after each k_down otherwise.
// BLADE_FIXUP_MERGE=0 / =1 forces the per-level / merged form on every call (A/B timing of the
// threshold: scripts/fixup_ab.sh); default by size.
bool fixups_merged(int nsel, long long N, long long H, long long W) {
  static const int force = [] {
    const char* e = getenv("BLADE_FIXUP_MERGE");
    return e ? atoi(e) : -1;
  }();
  if (nsel <= 1) return false;
  if (force == 0 || force == 1) return force == 1;
  return N * H * W <= (3LL << 20);  // crossover 2.07 .. 4.15 MP (profiles/r02_fixup_merge.txt)
}

// Kernel launch; with `pdl` the launch allows programmatic stream serialisation (PDL): the grid
// may be scheduled while the previous kernel in the stream drains, and its kernels call pdl_wait()
// before reading that kernel's outputs (kernels.cuh). BLADE_PDL=0 turns it off (A/B timing).
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("BLADE_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
// Small denoise calls (<= 16 Ki px) fix their uncertified pixels inside k_down (IFIX: one warp-wide
// fp64 pass per pixel, the fix-up kernel's arithmetic) instead of a fix-up launch on the critical
// path: 64 x 64 c1 38.9 -> 36.9 us, c0 20.5 -> 18.4 us; break-even at 128 x 128 and a loss above
// (512 x 512: 54 -> 59 us, the warps' serial fix-ups outlast the launch they save),
// profiles/r02_small_call_critical_path.txt. The selector diagnostic keeps the fix-up list.
// BLADE_INLINE_FIX=<max px> moves the threshold (0: never; A/B and tests).
bool inline_fixups(long long N, long long H, long long W, bool run_stages) {
  static const long long max_px = [] {
    const char* e = getenv("BLADE_INLINE_FIX");
    return e ? atoll(e) : (16LL << 10);
  }();
  return run_stages && N * H * W <= max_px;
}

// Small calls run the down pass as k_down_tile (2-D tiles, uncertified pixels fixed inline in
// fp64; bit-identical to k_down): every phase is spread over a CTA with short independent chains
// instead of k_down's ~10 dependent rows per warp, and no fix-up launch follows. FAST bucket layout,
// stage-running calls (the selector diagnostic keeps the fix-up list), level-0 rows that need no
// 16-B input copy. BLADE_DOWN_TILE=<max px> moves the size threshold (0: never; A/B and tests).
// c1 recipe, one frame, CUDA graph (profiles/r02_down_tile.txt): 256^2 49.1 -> 36.9 us, 512^2
// 53.2 -> 45.1, 768^2 63.5 -> 59.4; 1024^2 79.9 -> 84.0 (streaming k_down wins from here).
bool tile_down(const blade_ms* h, long long N, long long H, long long W, bool run_stages) {
  static const long long max_px = [] {
    const char* e = getenv("BLADE_DOWN_TILE");
    return e ? atoll(e) : (3LL << 18);  // crossover 768^2 .. 1024^2 (scripts/tile_threshold.py)
  }();
  const bool fast = h->n_o == 16 && h->n_s == 3 && h->n_c == 3;
  // (frames map to gridDim.z, tile rows to gridDim.y: both <= 65535)
  return run_stages && fast && N * H * W <= max_px && !(h->has_tma && W % 4 != 0) && N <= 65535 &&
         (H + 1) / 16 + 1 <= 65535;
}

// Shared-memory carveout of the launches of the current (small) call: consecutive kernels with
// different L1 / shared-memory splits make the SMs reconfigure between launches, which small,
// latency-bound calls feel (c1 flushed 63 -> 58 us, c0 24.6 -> 23.5 us; large batches keep the
// driver's per-kernel choice: c3's k_down1 is 4% slower with the maximal carveout).
// profiles/r02_carveout.txt. Set by CarveScope for the duration of one enqueue.
thread_local int g_carveout = -1;
struct CarveScope {
  int saved;
  explicit CarveScope(int v) : saved(g_carveout) { g_carveout = v; }
  ~CarveScope() { g_carveout = saved; }
};
int small_call_carveout(long long N, long long H, long long W) {
  static const int force = [] {  // BLADE_CARVEOUT=<percent> forces one on every call (A/B timing)
    const char* e = getenv("BLADE_CARVEOUT");
    return e ? atoi(e) : -2;
  }();
  if (force >= -1) return force;
  return N * H * W <= (4LL << 20) ? 100 : -1;
}
template <typename... KArgs, typename... Args>
cudaError_t launch(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                   Args&&... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl && pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (g_carveout >= 0) {
    at[na].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
    at[na].val.sharedMemCarveout = (unsigned)g_carveout;
    ++na;
  }
  lc.attrs = at;
  lc.numAttrs = na;
  return cudaLaunchKernelEx(&lc, fn, std::forward<Args>(args)...);
}
#define LAUNCH(name, expr)                                                                       \
  do {                                                                                           \
    cudaError_t e0__ = (expr);                                                                   \
    if (e0__ != cudaSuccess) {                                                                   \
      cudaGetLastError();                                                                        \
      return fail(BLADE_ECUDA, "%s (level %d): launch: %s", name, l, cudaGetErrorString(e0__)); \
    }                                                                                            \
    LAUNCH_CHECK(name);                                                                          \
  } while (0)

// Buffers of one cascade call for plan p (views of the workspace, or of caller-provided
// pyramid levels / maps for the diagnostics).
struct Bufs {
  std::vector<LevelView> z32;   // z^l (level 0: the input view)
  std::vector<float*> zlo;      // lo planes of z^l, 1 <= l <= L-2
  std::vector<uint8_t*> maps;   // byte addresses of the uint8 / uint16 maps
  std::vector<int> mpitch;      // entries per map row
  unsigned int* fb_cnt = nullptr;
  bool fuse0 = false;           // level 0 runs the fused-selector stage (decimation-only k_down)
};

Bufs make_bufs(const Plan& p, LevelView in_view, char* ws, void* const* maps_out, float* const* levels_out) {
  const int L = p.L;
  Bufs b;
  b.z32.resize(L);
  b.zlo.assign(L, nullptr);
  b.z32[0] = in_view;
  for (int l = 1; l < L; ++l) {
    float* base = (levels_out && levels_out[l - 1]) ? levels_out[l - 1]
                                                    : reinterpret_cast<float*>(ws + p.z32_off[l]);
    // caller-provided pyramid levels are dense (pitch W); the workspace's are padded (p.pitch);
    // the lo plane shares the hi plane's pitch
    const bool dense = levels_out && levels_out[l - 1];
    b.z32[l] = make_view(base, p.H[l], p.W[l], p.z[l], dense ? p.W[l] : p.pitch[l]);
    if (l + 1 < L) b.zlo[l] = reinterpret_cast<float*>(ws + p.zlo_off[l]);
  }
  const int nsel = L == 1 ? 1 : L - 1;
  b.maps.resize(nsel);
  b.mpitch.resize(nsel);
  for (int l = 0; l < nsel; ++l) {
    b.maps[l] = (maps_out && maps_out[l]) ? static_cast<uint8_t*>(maps_out[l]) : reinterpret_cast<uint8_t*>(ws + p.map_off[l]);
    b.mpitch[l] = (maps_out && maps_out[l]) ? p.W[l] : p.map_pitch[l];  // caller maps are dense
  }
  b.fb_cnt = reinterpret_cast<unsigned int*>(ws + p.fbcnt_off);
  return b;
}

bool use_ry4(const blade_ms* h, int N, int W, int span);
// BLADE_FUSE_SEL=1 turns the fused level-0 selector on (A/B builds; default off: measured slower,
// profiles/r02_fused_selector.txt — the stage's 8 warps per SM cannot hide the selector's
// dependent ALU chains under its shared-memory time: c3 stage0 2.36 -> 3.61 ms against k_down0
// 1.23 -> 0.56 ms)
bool fuse_sel_enabled() {
  static const bool on = [] {
    const char* e = getenv("BLADE_FUSE_SEL");
    return e && e[0] == '1';
  }();
  return on;
}
// Level-0 views of a call (the TMA stage reads the 16-B-row input copy / writes the staging output
// when the caller's rows are ragged) and whether the fused-selector stage runs there: the same
// conditions as up_level's TMA path for the 4-row variant.
struct Level0Views {
  LevelView zl, outv;
  bool ostage = false;
};
Level0Views level0_views(const blade_ms* h, const Plan& p, LevelView in_view, LevelView out_view, char* ws) {
  Level0Views v{in_view, out_view, false};
  if (h->has_tma && p.zcopy_pitch > 0) {
    v.zl = make_view(reinterpret_cast<float*>(ws + p.zcopy_off), p.H[0], p.W[0], Range{0, p.H[0]}, p.zcopy_pitch);
    v.outv = make_view(reinterpret_cast<float*>(ws + p.ocopy_off), p.H[0], p.W[0], Range{0, p.H[0]}, p.zcopy_pitch);
    v.ostage = true;
  }
  return v;
}
bool fused_level0(const blade_ms* h, const Plan& p, const Bufs& B, LevelView in_view, LevelView out_view, char* ws,
                  bool run_stages) {
  if (!h->has_fsel || !run_stages || p.L < 2 || !fuse_sel_enabled()) return false;
  const Level0Views v = level0_views(h, p, in_view, out_view, ws);
  const LevelView u1 = p.L == 2 ? B.z32[1] : make_view(reinterpret_cast<float*>(ws + p.u_off[1]), p.H[1], p.W[1], p.ub[1], p.pitch[1]);
  const int y_base = p.u[0].lo & ~1;
  return use_ry4(h, p.N, p.W[0], p.u[0].hi - y_base) && v.zl.pitch % 4 == 0 && v.outv.pitch % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(v.zl.p) & 15) == 0 && (reinterpret_cast<uintptr_t>(v.outv.p) & 15) == 0 &&
         u1.pitch % 4 == 0 && (reinterpret_cast<uintptr_t>(u1.p) & 15) == 0;
}

// Down pass at level l: k_down(l) -> s^l (rows p.u[l]) and z^{l+1} (rows p.zc[l+1] of the buffer
// p.z[l+1]); unless `fix_args` collects it for the merged launch, k_down_fixup(l) recomputes the
// (rare) pixels whose fp32 orientation is uncertified. The level's fix-up counter must be zero.
blade_status down_level(const blade_ms* h, const Plan& p, const Bufs& B, LevelView in_view, char* ws,
                        cudaStream_t st, bool run_stages, int l, std::vector<std::pair<int, DownArgs>>* fix_args,
                        bool ifix = false, bool tile = false) {
  const int L = p.L, N = p.N;
  const std::vector<LevelView>& z32 = B.z32;
  const std::vector<float*>& zlo = B.zlo;
  const std::vector<uint8_t*>& maps = B.maps;
  const std::vector<int>& mpitch = B.mpitch;
  unsigned int* fb_cnt = B.fb_cnt;
  {
    const Range U = p.u[l];
    const bool dec = L > 1;
    const Range Z1 = dec ? p.zc[l + 1] : Range{0, 0};  // rows of z^{l+1} computed
    const Range Z1b = dec ? p.z[l + 1] : Range{0, 0};  // rows of its buffer
    Range R = U;
    if (dec) R = hull(R, Range{2 * Z1.lo, 2 * Z1.hi});
    DownArgs da{};
    da.zhi = l == 0 ? in_view.p : z32[l].p;
    da.zlo = l == 0 ? nullptr : zlo[l];
    da.H = p.H[l];
    da.W = p.W[l];
    da.in_row0 = l == 0 ? in_view.row0 : p.z[l].lo;
    da.in_rows = l == 0 ? in_view.rows : p.z[l].n();
    da.in_pitch = l == 0 ? in_view.pitch : z32[l].pitch;
    da.in_plane = (long long)da.in_rows * da.in_pitch;
    da.in_frame = 3 * da.in_plane;
    da.map = maps[l];
    da.map_pitch = mpitch[l];
    da.s_r0 = U.lo;
    da.s_rn = U.n();
    da.ohi = dec ? z32[l + 1].p : nullptr;
    da.olo = (dec && l + 1 < L - 1) ? zlo[l + 1] : nullptr;
    da.H1 = dec ? p.H[l + 1] : 1;
    da.W1 = dec ? p.W[l + 1] : 1;
    da.out_pitch = dec ? z32[l + 1].pitch : 1;
    da.d_buf_row0 = Z1b.lo;
    da.d_buf_rows = Z1b.n();
    da.d_r0 = Z1.lo;
    da.d_rn = Z1.n();
    da.base = R.lo & ~1;
    const int span = R.hi - da.base;
    da.n_strips = (p.W[l] + down::STRIP - 1) / down::STRIP;
    // band height RB (even, 4..128): a task is RB + 6 input rows of one 64-column strip; pick
    // the RB that minimises (RB + 6) x ceil(tasks / resident warp slots): small images want thin
    // bands (their halo rows are cheaper than idle SMs), large batches tall ones, and no launch
    // should end with a sliver of a wave
    const long long col_tasks = (long long)N * da.n_strips;
    const double slots = (double)h->down_slots[l > 0 ? 1 : 0];
    // bands taller than 128 rows lose on c3 despite the model (1 wave of 1088-row tasks: k_down0
    // 1.28 -> 1.38 ms): a single wave cannot rebalance uneven SMs
    static const int rb_max = [] {  // BLADE_DOWN_RBMAX overrides the tallest band (A/B timing)
      const char* e = getenv("BLADE_DOWN_RBMAX");
      return e ? std::max(4, atoi(e)) & ~1 : 128;
    }();
    int RB = rb_max;
    double best = 0.0;
    for (int rb = rb_max; rb >= 4; rb -= 2) {
      const double tasks = (double)col_tasks * (double)((span + rb - 1) / rb);
      const double w = tasks / slots;
      const double cost = (rb + 6) * std::ceil(w);
      if (rb == rb_max || cost < best) {
        best = cost;
        RB = rb;
      }
    }
    RB = (RB + 1) & ~1;
    da.RB = RB;
    da.n_bands = (span + RB - 1) / RB;
    da.n_tasks = (int)(col_tasks * da.n_bands);
    da.fb_list = reinterpret_cast<unsigned long long*>(ws + p.fb_off[l]);
    da.fb_count = fb_cnt + l;
    da.fb_cap = p.fb_cap[l];
    da.N = N;
    const bool zcopy = l == 0 && run_stages && h->has_tma && p.zcopy_pitch > 0;
    da.zcopy = zcopy ? reinterpret_cast<float*>(ws + p.zcopy_off) : nullptr;
    da.copy_pitch = zcopy ? p.zcopy_pitch : 0;
    ProfScope ps(h, st, 1, l);
    const bool hilo = l > 0;
    const bool fast = h->n_o == 16 && h->n_s == 3 && h->n_c == 3;
    const bool wide = h->K > 256;
    const bool fused = l == 0 && B.fuse0;  // the level-0 stage computes s^0: decimation only
    if (tile && !fused && !zcopy && fast) {  // small call: the 2-D tile form, fixes inline
      const dim3 grid((unsigned)((p.W[l] + dtile::TX - 1) / dtile::TX), (unsigned)((span + dtile::TY - 1) / dtile::TY),
                      (unsigned)N);
      LAUNCH("k_down_tile", launch(down_tile_kernel(hilo, dec, wide), grid, dtile::THREADS, dtile::smem_bytes(hilo, dec),
                                   st, l > 0, da, h->down[l]));
      return BLADE_OK;
    }
    auto fn = fused ? dec_kernel(zcopy) : down_kernel(hilo, dec, fast, wide, zcopy, ifix);
    const unsigned grid = (unsigned)((da.n_tasks + down::WARPS - 1) / down::WARPS);
    LAUNCH("k_down", launch(fn, grid, 32 * down::WARPS, down_smem(hilo), st, l > 0, da, h->down[l]));
    if (fused || ifix) {
      // no fix-up launch: no map at this level (fused), or uncertified pixels fixed in k_down (ifix)
    } else if (fix_args) {
      fix_args->emplace_back(l, da);
    } else {
      auto fx = fixup_kernel(hilo, fast, wide);
      LAUNCH("k_down_fixup", launch(fx, 8 * h->num_sms, 128, 0, st, true, da, h->down[l]));
    }
  }
  return BLADE_OK;
}

// The merged fix-up of every selector level (small, launch-latency-bound calls): one launch per
// kFixMax levels after the down pass.
blade_status merged_fixups(const blade_ms* h, const std::vector<std::pair<int, DownArgs>>& fix_args, cudaStream_t st) {
  const int nsel = (int)fix_args.size();
  if (nsel == 0) return BLADE_OK;
  // ---- small (launch-latency-bound) calls: the fix-ups of every level in one launch per
  //      kFixMax levels after the down pass (the stages need them, the next k_down does not; on
  //      large batches the per-level fix-up right after its k_down is faster: 50 vs 70 us on c3)
  {
    const int l = nsel - 1;  // (LAUNCH's error message)
    const bool fast = h->n_o == 16 && h->n_s == 3 && h->n_c == 3;
    ProfScope ps(h, st, 3, 0);  // kind 3: the merged fix-up
    for (int l0 = 0; l0 < nsel; l0 += kFixMax) {
      FixupMulti fm{};
      fm.n = std::min(kFixMax, nsel - l0);
      for (int q = 0; q < fm.n; ++q) {
        fm.a[q] = fix_args[l0 + q].second;
        fm.prm[q] = h->down[fix_args[l0 + q].first];
      }
      LAUNCH("k_down_fixup_multi",
             launch(fixup_multi_kernel(fast, h->K > 256), h->num_sms, 128, 0, st, true, fm));  // small calls: one CTA per SM dispatches faster than 8
    }
  }
  return BLADE_OK;
}

// Up pass at level l: stage(l) -> u^l for rows p.u[l] (l = 0: into out_view; l >= 1: into the
// workspace buffer of rows p.ub[l]), reading z^l, u^{l+1} (buffer rows p.ub[l+1], or z^{L-1})
// and s^l.
blade_status up_level(const blade_ms* h, const Plan& p, const Bufs& B, LevelView out_view, char* ws,
                      cudaStream_t st, int l) {
  const int L = p.L, N = p.N;
  const std::vector<LevelView>& z32 = B.z32;
  const std::vector<uint8_t*>& maps = B.maps;
  const std::vector<int>& mpitch = B.mpitch;
  {
    const Range r = p.u[l];
    LevelView zl = z32[l];
    if (l == 0 && h->has_tma && p.zcopy_pitch > 0)  // the input copy k_down wrote (16-B rows)
      zl = make_view(reinterpret_cast<float*>(ws + p.zcopy_off), p.H[0], p.W[0], Range{0, p.H[0]}, p.zcopy_pitch);
    const bool fused = l == 0 && B.fuse0;  // this stage computes s^0 (fused selector)
    LevelView u1{};
    if (L > 1)
      u1 = (l + 1 == L - 1) ? z32[L - 1]
                            : make_view(reinterpret_cast<float*>(ws + p.u_off[l + 1]), p.H[l + 1], p.W[l + 1],
                                        p.ub[l + 1], p.pitch[l + 1]);
    LevelView outv = (l == 0) ? out_view
                              : make_view(reinterpret_cast<float*>(ws + p.u_off[l]), p.H[l], p.W[l], p.ub[l], p.pitch[l]);
    const bool ostage = l == 0 && h->has_tma && p.zcopy_pitch > 0;  // level-0 output via 16-B rows
    if (ostage)
      outv = make_view(reinterpret_cast<float*>(ws + p.ocopy_off), p.H[0], p.W[0], Range{0, p.H[0]}, p.zcopy_pitch);
    auto copy_out = [&]() {  // staged level-0 output -> the caller's dense rows
      const long long total = (long long)N * 3 * p.H[0] * p.W[0];
      const unsigned g = (unsigned)std::min<long long>((total + 255) / 256, 8LL * h->num_sms);
      return launch(k_copy_rows<>, g, 256, 0, st, true, out_view.p, out_view.pitch,
                    static_cast<const float*>(outv.p), outv.pitch, (long long)N * 3, p.H[0], p.W[0]);
    };
    const float* bank = h->d_bank + (size_t)l * h->cfg.n_filter_channels * h->cfg.n_phases * h->PS;
    const int y_base = r.lo & ~1;
    const int clamp = (l == 0 && h->cfg.clamp_output) ? 1 : 0;
    ProfScope ps(h, st, 2, l);
    // TMA path: needs 16-B aligned buffers whose row pitches are 16-B multiples
    const int map_es = h->K > 256 ? 2 : 1;
    bool use_tma = h->has_tma && zl.pitch % 4 == 0 && outv.pitch % 4 == 0 &&
                   (fused || ((mpitch[l] * map_es) % 16 == 0 && aligned16(maps[l]))) && aligned16(zl.p) &&
                   aligned16(outv.p) && (L == 1 || (u1.pitch % 4 == 0 && aligned16(u1.p)));
    CUtensorMap tmz, tmu, tmm;
    if (use_tma) {
      // box shapes of the variant that will run (the 4-row variant may use taller tiles)
      const TmaVariant& tv = (fused || use_ry4(h, N, p.W[l], r.hi - y_base)) ? h->tma4 : h->tma;
      use_tma = encode_3d(&tmz, zl.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p.W[l], zl.rows, N * 3, tv.fcb,
                          fused ? h->tma4.fsel_fr : tv.fr, 3, zl.pitch) &&
                (fused ? true
                 : h->K > 256 ? encode_3d(&tmm, maps[l], CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, p.W[l], r.n(), N, tv.tcols,
                                          tv.trows, 1, mpitch[l])
                              : encode_3d(&tmm, maps[l], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, p.W[l], r.n(), N, tv.tcols,
                                          tv.trows, 1, mpitch[l]));
      if (fused) tmm = tmz;  // unused by the fused kernel
      if (use_tma) {
        if (L > 1)
          use_tma = encode_3d(&tmu, u1.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p.W[l + 1], u1.rows, N * 3, tv.ccb,
                              tv.cr, 3, u1.pitch);
        else
          tmu = tmz;
      }
    }
    if (use_tma) {
      const TmaVariant& tv = (fused || use_ry4(h, N, p.W[l], r.hi - y_base)) ? h->tma4 : h->tma;
      StageTmaArgs a{};
      a.H = p.H[l];
      a.W = p.W[l];
      a.H1 = L > 1 ? p.H[l + 1] : 1;
      a.W1 = L > 1 ? p.W[l + 1] : 1;
      a.z_row0 = zl.row0;
      a.z_rows = zl.rows;
      a.u_row0 = u1.row0;
      a.u_rows = u1.rows;
      a.map_row0 = r.lo;
      a.map_rows = r.n();
      a.z = zl.p;
      a.u1 = u1.p;
      a.out = outv.p;
      a.out_row0 = outv.row0;
      a.out_rows = outv.rows;
      a.bank = h->d_bank_tma + (size_t)l * h->cfg.n_filter_channels * h->cfg.n_phases * h->PS_tma;
      a.K = h->K;
      a.S = h->S_tma;
      a.PS = h->PS_tma;
      a.n_phases = h->cfg.n_phases;
      a.N = N;
      a.y_base = y_base;
      a.o_r0 = r.lo;
      a.o_rn = r.n();
      a.tiles_x = (p.W[l] + tv.tcols - 1) / tv.tcols;
      a.tiles_y = (r.hi - y_base + tv.trows - 1) / tv.trows;
      a.n_tiles = N * a.tiles_x * a.tiles_y;
      a.clamp = clamp;
      a.z_pitch = zl.pitch;
      a.u_pitch = L > 1 ? u1.pitch : zl.pitch;
      a.out_pitch = outv.pitch;
      if (tv.phase_split) {  // 4 phase-CTAs (x 3 channels) or 2 row-parity CTAs per tile group,
                             // 2 workers per CTA
        const int types = tv.ch3 ? 12 : tv.ptypes;
        // one tile per worker group first: small levels spread over as many SMs as they have
        // tiles (a CTA's two groups share its SM's shared-memory bandwidth)
        const int per_type = std::max(1, std::min(h->num_sms / types, a.n_tiles));
        a.u_rgb = (L > 1 && l + 1 == L - 1) ? 1 : 0;
        if (tv.ch3) a.clamp = 0;  // clamped after the colour conversion
        LAUNCH("k_stage_ph", launch(tv.fn, types * per_type, dim3(32, 8), h->tma_smem, st, true, tmz, tmu, tmm, a));
      } else if (tv.ch3) {  // CTA b serves channel b % 3
        const int per_ch = std::max(1, std::min(h->num_sms / 3, a.n_tiles));
        a.u_rgb = (L > 1 && l + 1 == L - 1) ? 1 : 0;
        a.clamp = 0;  // clamped after the colour conversion
        LAUNCH("k_stage_tma", launch(tv.fn, 3 * per_ch, dim3(32, tv.by * tv.groups), h->tma_smem, st, true, tmz, tmu, tmm, a));
      } else if (fused) {
        // fused selector: k_down's level-0 selector arithmetic inside the stage; the uncertified
        // pixels are then recomputed (fp64 bucket + Eq. 9) by k_stage_fixup
        const DownParams& dp = h->down[0];
        a.sw0 = (float)dp.wp[0];
        a.sw1 = (float)dp.wp[1];
        a.sw2 = (float)dp.wp[2];
        a.tsR[0] = dp.tsR[0];
        a.tsR[1] = dp.tsR[1];
        a.kcR[0] = dp.kcR[0];
        a.kcR[1] = dp.kcR[1];
        a.tc_nonpos = dp.tc_nonpos;
        a.fb_list = reinterpret_cast<unsigned long long*>(ws + p.fb_off[0]);
        a.fb_count = B.fb_cnt;
        a.fb_cap = p.fb_cap[0];
        const int grid = std::min(h->num_sms, a.n_tiles);
        LAUNCH("k_stage_tma(fused selector)", launch(tv.fsel_fn, grid, dim3(32, tv.by * tv.groups), h->fsel_smem, st,
                                                     true, tmz, tmu, tmm, a));
        StageFixArgs fa{};
        fa.z = zl.p;
        fa.z_row0 = zl.row0;
        fa.z_rows = zl.rows;
        fa.z_pitch = zl.pitch;
        fa.u1 = u1.p;
        fa.u_row0 = u1.row0;
        fa.u_rows = u1.rows;
        fa.u_pitch = u1.pitch;
        fa.out = outv.p;
        fa.out_row0 = outv.row0;
        fa.out_rows = outv.rows;
        fa.out_pitch = outv.pitch;
        fa.H = p.H[0];
        fa.W = p.W[0];
        fa.H1 = p.H[1];
        fa.W1 = p.W[1];
        fa.N = N;
        fa.o_r0 = r.lo;
        fa.o_rn = r.n();
        fa.bank = bank;
        fa.S = h->S;
        fa.PS = h->PS;
        fa.n_phases = h->cfg.n_phases;
        fa.clamp = clamp;
        fa.fb_list = a.fb_list;
        fa.fb_count = a.fb_count;
        fa.fb_cap = a.fb_cap;
        LAUNCH("k_stage_fixup", launch(h->sfix, 8 * h->num_sms, 128, 0, st, true, fa, h->down[0]));
      } else {
        const int grid = std::min(h->num_sms, a.n_tiles);  // small levels: one tile per SM
        LAUNCH("k_stage_tma", launch(tv.fn, grid, dim3(32, tv.by * tv.groups), h->tma_smem, st, true, tmz, tmu, tmm, a));
      }
      if (tv.ch3 && l == 0) {  // u^0 is YCbCr planes: back to RGB in place (+ final clamp)
        const long long per_frame = (long long)r.n() * outv.pitch;
        const long long total = (long long)N * per_frame;
        const unsigned g2 = (unsigned)std::min<long long>((total + 255) / 256, 8LL * h->num_sms);
        LAUNCH("k_ycc_to_rgb", launch(k_ycc_to_rgb<>, g2, 256, 0, st, true,
                                      outv.p + (long long)(r.lo - outv.row0) * outv.pitch, outv.plane, outv.frame,
                                      per_frame, N, h->cfg.clamp_output));
      }
      if (ostage) LAUNCH("k_copy_rows", copy_out());
      return BLADE_OK;
    }
    StageArgs a{};
    a.z = zl;
    a.u1 = u1;
    a.out = outv;
    a.map = maps[l];
    a.map_row0 = r.lo;
    a.map_rows = r.n();
    a.map_pitch = mpitch[l];
    a.bank = bank;
    a.K = h->K;
    a.S = h->S;
    a.PS = h->PS;
    a.n_phases = h->cfg.n_phases;
    a.N = N;
    a.out_r0 = r.lo;
    a.out_rn = r.n();
    a.tiles_x = (p.W[l] + h->stage.tcols - 1) / h->stage.tcols;
    a.tiles_y = (r.hi - y_base + h->stage.trows - 1) / h->stage.trows;
    a.n_tiles = N * a.tiles_x * a.tiles_y;
    a.clamp = clamp;
    // CTAs come in sets of rs (row parity) x 3 (channel, CH3) specialisations
    const long long set = (long long)h->stage.rs * (h->stage.ch3 ? 3 : 1);
    long long grid = (long long)h->stage_ctas_per_sm * h->num_sms;
    grid = std::min(grid, (long long)a.n_tiles * set);
    grid = std::max<long long>(set, grid / set * set);
    a.u_rgb = (L > 1 && l + 1 == L - 1) ? 1 : 0;
    if (h->stage.ch3) a.clamp = 0;  // clamped after the colour conversion
    LAUNCH("k_stage", launch(h->stage.fn, (unsigned)grid, dim3(32, h->stage.by), h->stage_smem, st, true, a));
    if (h->stage.ch3 && l == 0) {  // u^0 is YCbCr planes: back to RGB in place (+ final clamp)
      const long long per_frame = (long long)r.n() * outv.pitch;
      const long long total = (long long)N * per_frame;
      const unsigned g2 = (unsigned)std::min<long long>((total + 255) / 256, 8LL * h->num_sms);
      LAUNCH("k_ycc_to_rgb", launch(k_ycc_to_rgb<>, g2, 256, 0, st, true,
                                    outv.p + (long long)(r.lo - outv.row0) * outv.pitch, outv.plane, outv.frame,
                                    per_frame, N, h->cfg.clamp_output));
    }
    if (ostage) LAUNCH("k_copy_rows", copy_out());
  }
  return BLADE_OK;
}

// Enqueue the cascade for plan p. in_view: level-0 input (fp32, rows >= p.z[0]); out_view: final
// output rows p.u[0]. levels_out (diagnostic) receives z^l (fp32) for l >= 1; maps_out the maps.
blade_status enqueue(const blade_ms* h, const Plan& p, LevelView in_view, LevelView out_view, char* ws,
                     cudaStream_t st, bool run_stages, void* const* maps_out, float* const* levels_out) {
  const int L = p.L, N = p.N;
  if (N == 0) return BLADE_OK;
  Bufs B = make_bufs(p, in_view, ws, maps_out, levels_out);
  B.fuse0 = !maps_out && !levels_out && fused_level0(h, p, B, in_view, out_view, ws, run_stages);
  const CarveScope carve(small_call_carveout(N, p.u[0].n(), p.W[0]));
  const int nsel = L == 1 ? 1 : L - 1;
  std::vector<std::pair<int, DownArgs>> fix_args;  // (level, args), for the merged fix-up launch
  const bool tile = !B.fuse0 && tile_down(h, N, p.H[0], p.W[0], run_stages);
  const bool ifix = !tile && inline_fixups(N, p.H[0], p.W[0], run_stages);
  const bool merge_fix = !ifix && !tile && fixups_merged(nsel, N, p.H[0], p.W[0]);
  CUDA_TRY(cudaMemsetAsync(B.fb_cnt, 0, sizeof(unsigned int) * nsel, st));
  blade_status s;
  for (int l = 0; l < nsel; ++l)
    if ((s = down_level(h, p, B, in_view, ws, st, run_stages, l, merge_fix ? &fix_args : nullptr, ifix, tile)) !=
        BLADE_OK)
      return s;
  if (merge_fix && (s = merged_fixups(h, fix_args, st)) != BLADE_OK) return s;
  if (!run_stages) return BLADE_OK;
  for (int l = nsel - 1; l >= 0; --l)
    if ((s = up_level(h, p, B, out_view, ws, st, l)) != BLADE_OK) return s;
  return BLADE_OK;
}

}  // namespace

// =============================================================================== C ABI

extern "C" {

const char* blade_ms_status_string(blade_status s) {
  switch (s) {
    case BLADE_OK: return "ok";
    case BLADE_EINVAL: return "invalid argument";
    case BLADE_ENONFINITE: return "non-finite tap or threshold";
    case BLADE_ESHAPE: return "size mismatch";
    case BLADE_EDEVICE: return "wrong device";
    case BLADE_ENOMEM: return "out of device memory";
    case BLADE_ECUDA: return "CUDA error";
    case BLADE_EUNSUPPORTED: return "unsupported configuration";
  }
  return "unknown status";
}

const char* blade_ms_last_error(void) { return g_last_error.c_str(); }

#ifdef BLADE_TRACE
// Latency probes only (BLADE_TRACE builds): kernel-kind timestamps of the k_down / k_stage_tma
// translation units, [2][16][3] (entry, griddepcontrol.wait return, exit; %globaltimer ns).
void blade_ms_trace(unsigned long long* out, int reset) {
  tables::trace_down(out, reset != 0);
  tables::trace_tma(out ? out + 48 : nullptr, reset != 0);
}
#endif

blade_status blade_ms_create(const blade_ms_config* cfg, const blade_bucket_layout* bl, const float* taps,
                             size_t n_taps, int device, blade_ms_t* out) {
  g_last_error.clear();
  if (!out) return fail(BLADE_EINVAL, "out is NULL");
  *out = nullptr;
  if (!cfg || !bl || !taps) return fail(BLADE_EINVAL, "cfg, buckets and taps must be non-NULL");
  const blade_ms_config c = *cfg;
  if (c.levels < 1 || c.levels > 12) return fail(BLADE_EINVAL, "levels must be in 1..12");
  if (c.fine_size < 1 || c.fine_size > 9 || !(c.fine_size & 1))
    return fail(BLADE_EINVAL, "fine_size must be odd in 1..9");
  if (c.levels == 1 && c.coarse_size != 0) return fail(BLADE_EINVAL, "coarse_size must be 0 when levels == 1");
  if (c.levels > 1 && (c.coarse_size < 1 || c.coarse_size > 9 || !(c.coarse_size & 1)))
    return fail(BLADE_EINVAL, "coarse_size must be odd in 1..9 when levels > 1");
  if (c.n_phases != 1 && c.n_phases != 4) return fail(BLADE_EINVAL, "n_phases must be 1 or 4");
  if (c.levels == 1 && c.n_phases != 1) return fail(BLADE_EINVAL, "n_phases must be 1 when levels == 1");
  if (c.n_filter_channels != 1 && c.n_filter_channels != 3)
    return fail(BLADE_EINVAL, "n_filter_channels must be 1 or 3");
  if (c.window_size < 1 || c.window_size > 5 || !(c.window_size & 1))
    return fail(BLADE_EINVAL, "window_size must be 1, 3 or 5");
  if (!(c.window_sigma > 0.0f) || !std::isfinite(c.window_sigma))
    return fail(BLADE_EINVAL, "window_sigma must be finite and > 0");
  if (c.clamp_output != 0 && c.clamp_output != 1) return fail(BLADE_EINVAL, "clamp_output must be 0 or 1");
  if (bl->n_orient < 1 || bl->n_strength < 1 || bl->n_coherence < 1)
    return fail(BLADE_EINVAL, "bucket counts must be >= 1");
  if (bl->n_strength - 1 > kMaxThr2 || bl->n_coherence - 1 > kMaxThr2)
    return fail(BLADE_EUNSUPPORTED, "at most %d thresholds per feature", kMaxThr2);
  const long long K = (long long)bl->n_orient * bl->n_strength * bl->n_coherence;
  if (K > 65536) return fail(BLADE_EUNSUPPORTED, "K = %lld > 65536 (uint16 bucket maps)", K);
  const bool wide = K > 256;  // uint16 maps, bank read from global memory (NEXT f2)
  if ((bl->n_strength > 1 && !bl->strength_thresholds) || (bl->n_coherence > 1 && !bl->coherence_thresholds))
    return fail(BLADE_EINVAL, "threshold arrays must be non-NULL");
  const int n_stages = std::max(c.levels - 1, 1);
  const int nf2 = c.fine_size * c.fine_size;
  const int nc2 = c.levels > 1 ? c.coarse_size * c.coarse_size : 0;
  const int nt = nf2 + nc2;
  const size_t expect = (size_t)n_stages * c.n_filter_channels * c.n_phases * K * nt;
  if (n_taps != expect)
    return fail(BLADE_ESHAPE, "n_taps = %zu, expected %zu = stages %d x channels %d x phases %d x K %lld x %d",
                n_taps, expect, n_stages, c.n_filter_channels, c.n_phases, K, nt);
  for (size_t i = 0; i < n_taps; ++i)
    if (!std::isfinite(taps[i])) return fail(BLADE_ENONFINITE, "tap %zu is not finite", i);
  auto check_thr = [&](const double* t, int cnt, const char* name) -> blade_status {
    for (int s = 0; s < n_stages; ++s)
      for (int i = 0; i < cnt; ++i) {
        const double v = t[(size_t)s * cnt + i];
        if (!std::isfinite(v)) return fail(BLADE_ENONFINITE, "%s threshold [%d][%d] not finite", name, s, i);
        if (i > 0 && !(v > t[(size_t)s * cnt + i - 1]))
          return fail(BLADE_EINVAL, "%s thresholds of stage %d not strictly ascending", name, s);
      }
    return BLADE_OK;
  };
  blade_status st;
  if ((st = check_thr(bl->strength_thresholds, bl->n_strength - 1, "strength")) != BLADE_OK) return st;
  if ((st = check_thr(bl->coherence_thresholds, bl->n_coherence - 1, "coherence")) != BLADE_OK) return st;

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
    cudaGetLastError();
    return fail(BLADE_EDEVICE, "no CUDA device");
  }
  if (device < 0 || device >= ndev) return fail(BLADE_EDEVICE, "device %d out of range (%d devices)", device, ndev);
  DeviceGuard guard(device);
  if (!guard.ok) return fail(BLADE_EDEVICE, "cudaSetDevice(%d) failed", device);

  int max_smem = 0, nsm = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  const int S = nt | 1;                      // odd tap stride (bank-conflict spread)
  const int PS = (int)((K * S + 3) & ~3LL);  // phase stride, 16-B aligned
  const int cnc = c.levels > 1 ? c.coarse_size : 0;

  // generic stage kernel: largest BY whose shared memory fits
  const int want_rs = c.levels == 1 ? 1 : 2;
  const StageVariant* best = nullptr;
  size_t best_smem = 0;
  const bool ch3 = c.n_filter_channels == 3;
  for (const auto* list : {&stage_variants(), &stage_variants_pairs(), &stage_variants_pairs2(), &stage_variants_ch3_wide()})
    for (const auto& v : *list) {
      if (v.nf != c.fine_size || v.nc != cnc || v.rs != want_rs || v.ch3 != ch3 || v.wide != wide) continue;
      const int nph_cta = c.n_phases == 4 ? (v.rs == 2 ? 2 : 4) : 1;
      const size_t bank_f = wide ? 0 : (((size_t)nph_cta * PS) + 3) / 4 * 4;
      const size_t smem = sizeof(float) * (bank_f + (size_t)v.tile_floats);
      if (smem > (size_t)max_smem) continue;
      if (!best || v.by > best->by) {
        best = &v;
        best_smem = smem;
      }
    }
  if (!best)  // no shared-bank variant fits: the bank stays in global memory (L2-resident), uint8 maps
    for (const auto& v : stage_variants_gbank()) {
      if (v.nf != c.fine_size || v.nc != cnc || v.rs != want_rs || v.ch3 != ch3 || wide) continue;
      const size_t smem = sizeof(float) * (size_t)v.tile_floats;
      if (smem > (size_t)max_smem) continue;
      best = &v;
      best_smem = smem;
    }
  if (!best)
    return fail(BLADE_EUNSUPPORTED,
                "no stage kernel for fine %d / coarse %d with K = %lld (every odd fine / coarse size 1..9 is "
                "built for shared and per-channel banks)",
                c.fine_size, c.coarse_size, K);

  blade_ms* h = new blade_ms();
  h->cfg = c;
  h->n_o = bl->n_orient;
  h->n_s = bl->n_strength;
  h->n_c = bl->n_coherence;
  h->K = (int)K;
  h->n_stages = n_stages;
  h->nt = nt;
  h->S = S;
  h->PS = PS;
  h->device = device;
  h->num_sms = nsm;
  h->stage = *best;
  h->stage_smem = best_smem;
  for (const auto* tlist : {&tma_variants(), &tma_variants_ch3_wide()})
  for (const auto& v : *tlist) {
    if (v.ch3 != ch3 || v.wide != wide || v.nf != c.fine_size || v.nc != cnc) continue;
    if (v.ry == 4) {  // 4 pixel rows per thread: 16-row tiles in two groups (BLADE_TMA4_ROWS
                      // selects another instantiated height; 20-row tiles = 10 warps per SM and
                      // 12-row tiles in three groups measured slower: profiles/r02_fused_selector.txt,
                      // profiles/r02_stage_groups.txt)
      // (the per-channel banks have the 16-row form only)
      if (tma_ry() != 2 && (v.trows == tma4_rows() || (v.trows == 16 && !(h->has_tma4 && h->tma4.trows == tma4_rows())))) {
        h->has_tma4 = true;
        h->tma4 = v;
      }
      continue;
    }
    const size_t tps = (size_t)K * v.S;  // phase stride of the TMA tap layout (multiple of 4)
    const size_t bank = wide ? 0 : ((size_t)c.n_phases * tps * 4 + 127) & ~size_t(127);
    const size_t smem = 2 * (size_t)v.stage_bytes + bank + 32;  // + 3 mbarriers
    if (smem <= (size_t)max_smem && get_encode()) {
      h->has_tma = true;
      h->tma = v;
      h->tma_smem = smem;
      h->S_tma = v.S;
      h->PS_tma = (int)tps;
    }
  }
  if (h->has_tma && h->has_tma4) {  // its tile buffers (one per group, at least two) next to the bank
    const size_t bank = wide ? 0 : ((size_t)c.n_phases * h->PS_tma * 4 + 127) & ~size_t(127);
    const size_t smem4 = (size_t)std::max(2, h->tma4.groups) * h->tma4.stage_bytes + bank + 32;
    if (smem4 <= (size_t)max_smem)
      h->tma_smem = std::max(h->tma_smem, smem4);
    else
      h->has_tma4 = false;
  }
  if (!h->has_tma && c.levels > 1 && c.n_phases == 4 && !ch3 && !wide && p2_enabled()) {
    // row-parity CTAs holding two phases each (4 consecutive pixels per thread row)
    for (const auto& v : p2_variants()) {
      if (v.nf != c.fine_size || v.nc != cnc) continue;
      const size_t tps = (size_t)K * v.S;
      const size_t smem = 2 * (size_t)v.stage_bytes + ((2 * tps * 4 + 127) & ~size_t(127)) + 32;
      if (smem <= (size_t)max_smem && get_encode()) {
        h->has_tma = true;
        h->tma = v;
        h->tma_smem = smem;
        h->S_tma = v.S;
        h->PS_tma = (int)tps;
      }
    }
  }
  if (!h->has_tma && c.levels > 1 && c.n_phases == 4) {
    for (const auto& v : ph_variants()) {
      if (v.nf != c.fine_size || v.nc != cnc || v.ch3 != ch3 || v.wide != wide) continue;
      const size_t tps = (size_t)K * v.S;
      const size_t smem = 2 * (size_t)v.stage_bytes + ((tps * 4 + 127) & ~size_t(127)) + 32;
      if (smem <= (size_t)max_smem && get_encode()) {
        h->has_tma = true;
        h->tma = v;
        h->tma_smem = smem;
        h->S_tma = v.S;
        h->PS_tma = (int)tps;
      }
    }
  }

  // ---- fused selector at level 0: the 4-row shared-bank pair stage with the
  //      configs' bucket layout and a 5 x 5 window
  if (h->has_tma && h->has_tma4 && !h->tma.phase_split && h->tma4.fsel_fn && !ch3 && !wide &&
      c.window_size == 5 && c.levels > 1 && h->n_o == 16 && h->n_s == 3 && h->n_c == 3) {
    const size_t bank = ((size_t)c.n_phases * h->PS_tma * 4 + 127) & ~size_t(127);
    const size_t smem = 2 * (size_t)h->tma4.fsel_stage_bytes + bank + 32;
    h->sfix = stage_fixup_kernel(c.fine_size, cnc);
    if (smem <= (size_t)max_smem && h->sfix) {
      h->has_fsel = true;
      h->fsel_smem = smem;
    }
  }

  // ---- selector parameters per stage (window weights fp64 -> fp32; thresholds pre-transformed)
  const int r = c.window_size / 2;
  double e[8], se = 0.0;
  for (int d = -r; d <= r; ++d) {
    e[d + r] = std::exp(-(double)(d * d) / (2.0 * (double)c.window_sigma * (double)c.window_sigma));
    se += e[d + r];
  }
  h->down.resize(n_stages);
  for (int s = 0; s < n_stages; ++s) {
    DownParams& dp = h->down[s];
    memset(&dp, 0, sizeof dp);
    for (int d = 0; d < c.window_size; ++d) dp.wp[d + 2 - r] = e[d] / se;  // offsets -r..r -> -2..2
    dp.n_o = bl->n_orient;
    dp.n_s = bl->n_strength;
    dp.n_c = bl->n_coherence;
    for (int i = 0; i < kMaxThr2; ++i) dp.ts2[i] = dp.kc2[i] = INFINITY;
    for (int i = 0; i < 2; ++i) dp.tsR[i] = dp.kcR[i] = INFINITY;
    for (int i = 0; i < bl->n_strength - 1; ++i) {
      const double t = bl->strength_thresholds[(size_t)s * (bl->n_strength - 1) + i];
      dp.ts2[i] = t <= 0.0 ? -INFINITY : (float)(t * t);  // S >= t <=> l1 >= t^2 (t > 0)
      if (i < 2) dp.tsR[i] = t <= 0.0 ? -INFINITY : (float)(8.0 * t * t);  // <=> T + R >= 8 t^2
    }
    int npos = 0;
    for (int i = 0; i < bl->n_coherence - 1; ++i) {
      const double t = bl->coherence_thresholds[(size_t)s * (bl->n_coherence - 1) + i];
      if (t <= 0.0) {
        dp.tc_nonpos += 1;
      } else {
        const double kap = 2.0 * t / (1.0 + t * t);  // C >= t <=> r >= kappa h
        if (npos < 2) dp.kcR[npos] = (float)kap;  // <=> R > kappa T (FAST selector)
        dp.kc2[npos++] = (float)(kap * kap);
      }
    }
    dp.quad_edges = (bl->n_orient % 4 == 0 && bl->n_orient <= 64) ? 1 : 0;
    for (int j = 1; dp.quad_edges && j < bl->n_orient / 4; ++j) {
      const double al = 2.0 * M_PI * j / bl->n_orient;
      dp.ecos[j - 1] = (float)std::cos(al);
      dp.esin[j - 1] = (float)std::sin(al);
    }
  }

  // ---- bank re-layout: host [stage][ch][phase][K][nt] -> device [stage][ch][phase][PS]
  // generic kernel: [K][S] rows, taps in ABI order; TMA kernel (one channel): tma_tap_off layout
  const int nch = c.n_filter_channels;
  const size_t dev_floats = (size_t)n_stages * nch * c.n_phases * PS;
  const size_t tma_floats = (size_t)n_stages * nch * c.n_phases * h->PS_tma;
  std::vector<float> relaid(dev_floats, 0.0f), relaid_tma(tma_floats, 0.0f);
  for (int s = 0; s < n_stages; ++s)
    for (int ch = 0; ch < nch; ++ch)
    for (int p = 0; p < c.n_phases; ++p)
      for (long long k = 0; k < K; ++k) {
        const float* src = taps + ((((size_t)s * nch + ch) * c.n_phases + p) * K + k) * nt;
        float* dst = relaid.data() + (((size_t)s * nch + ch) * c.n_phases + p) * PS + (size_t)k * S;
        memcpy(dst, src, sizeof(float) * nt);
        if (!h->has_tma) continue;
        float* dt = relaid_tma.data() + (((size_t)s * nch + ch) * c.n_phases + p) * h->PS_tma + (size_t)k * h->S_tma;
        for (int dy = 0; dy < c.fine_size; ++dy)
          for (int dx = 0; dx < c.fine_size; ++dx)
            dt[tma_tap_off(c.fine_size, cnc, 0, dy, dx)] = src[dy * c.fine_size + dx];
        for (int dy = 0; dy < cnc; ++dy)
          for (int dx = 0; dx < cnc; ++dx)
            dt[tma_tap_off(c.fine_size, cnc, 1, dy, dx)] = src[c.fine_size * c.fine_size + dy * cnc + dx];
      }
  h->bank_bytes = sizeof(float) * (dev_floats + tma_floats);
  if (cudaMalloc(&h->d_bank, sizeof(float) * dev_floats) != cudaSuccess ||
      (h->has_tma && cudaMalloc(&h->d_bank_tma, sizeof(float) * tma_floats) != cudaSuccess)) {
    cudaGetLastError();
    cudaFree(h->d_bank);
    delete h;
    return fail(BLADE_ENOMEM, "cudaMalloc for the bank failed");
  }
  if (h->has_tma &&
      cudaMemcpy(h->d_bank_tma, relaid_tma.data(), sizeof(float) * tma_floats, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(h->d_bank);
    cudaFree(h->d_bank_tma);
    delete h;
    return fail(BLADE_ECUDA, "bank upload failed");
  }
  cudaError_t ce = cudaMemcpy(h->d_bank, relaid.data(), sizeof(float) * dev_floats, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess)
    ce = cudaFuncSetAttribute(h->stage.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->stage_smem);
  if (ce == cudaSuccess && h->has_tma)
    ce = cudaFuncSetAttribute(h->tma.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->tma_smem);
  if (ce == cudaSuccess && h->has_tma && h->has_tma4)
    ce = cudaFuncSetAttribute(h->tma4.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->tma_smem);
  if (ce == cudaSuccess && h->has_fsel)
    ce = cudaFuncSetAttribute(h->tma4.fsel_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->fsel_smem);
  if (ce == cudaSuccess) {
    for (int hl = 0; hl < 2 && ce == cudaSuccess; ++hl)
      for (int dc = 0; dc < 2 && ce == cudaSuccess; ++dc)
        for (int sm = 0; sm < 3 && ce == cudaSuccess; ++sm)
          for (int cp = 0; cp < 2 && ce == cudaSuccess; ++cp)
            ce = cudaFuncSetAttribute(down_kernel(hl, dc, sm == 1, sm == 2, cp && !hl), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)down_smem(hl));
    for (int hl = 0; hl < 2 && ce == cudaSuccess; ++hl)
      for (int dc = 0; dc < 2 && ce == cudaSuccess; ++dc)
        for (int wd = 0; wd < 2 && ce == cudaSuccess; ++wd)
          ce = cudaFuncSetAttribute(down_tile_kernel(hl, dc, wd), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)dtile::smem_bytes(hl, dc));
  }
  for (int hl = 0; hl < 2 && ce == cudaSuccess; ++hl) {
    int oc = 0;
    ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, down_kernel(hl, true, h->n_o == 16 && h->n_s == 3 && h->n_c == 3, wide),
                                                       32 * down::WARPS, down_smem(hl));
    h->down_slots[hl] = std::max(1, oc) * down::WARPS * nsm;
  }
  int occ = 0;
  if (ce == cudaSuccess)
    ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, h->stage.fn, h->stage.threads, h->stage_smem);
  if (ce != cudaSuccess || occ < 1) {
    cudaFree(h->d_bank);
    cudaFree(h->d_bank_tma);
    delete h;
    return fail(BLADE_ECUDA, "kernel setup failed: %s (occupancy %d)", cudaGetErrorString(ce), occ);
  }
  h->stage_ctas_per_sm = occ;
  ce = cudaEventCreateWithFlags(&h->pipe_fork, cudaEventDisableTiming);
  for (int i = 0; i < blade_ms::kMaxStreams && ce == cudaSuccess; ++i) {
    ce = cudaStreamCreateWithFlags(&h->pipe[i], cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&h->pipe_join[i], cudaEventDisableTiming);
  }
  if (ce != cudaSuccess) {
    blade_ms_destroy(h);
    return fail(BLADE_ECUDA, "stream setup failed: %s", cudaGetErrorString(ce));
  }
  *out = h;
  return BLADE_OK;
}

blade_status blade_ms_set_profiling(blade_ms_t h, int32_t enable) {
  if (!h) return fail(BLADE_EINVAL, "handle is NULL");
  h->profiling = enable != 0;
  return BLADE_OK;
}

blade_status blade_ms_profile_read(blade_ms_t h, double* ms, int32_t* count) {
  if (!h || !ms || !count) return fail(BLADE_EINVAL, "NULL argument");
  DeviceGuard guard(h->device);
  for (int i = 0; i < 64; ++i) {
    ms[i] = 0.0;
    count[i] = 0;
  }
  blade_status rs = BLADE_OK;
  for (auto& r : h->prof) {
    float t = 0.0f;
    cudaError_t e = cudaEventSynchronize(r.e1);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.e0, r.e1);
    if (e != cudaSuccess && rs == BLADE_OK) rs = fail(BLADE_ECUDA, "profile read: %s", cudaGetErrorString(e));
    const int idx = r.kind * 16 + std::min(r.level, 15);
    ms[idx] += t;
    count[idx] += 1;
    h->ev_pool.push_back(r.e0);
    h->ev_pool.push_back(r.e1);
  }
  h->prof.clear();
  return rs;
}

blade_status blade_ms_destroy(blade_ms_t h) {
  if (!h) return BLADE_OK;
  DeviceGuard guard(h->device);
  for (auto& r : h->prof) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  for (int i = 0; i < blade_ms::kMaxStreams; ++i) {
    if (h->pipe[i]) cudaStreamDestroy(h->pipe[i]);
    if (h->pipe_join[i]) cudaEventDestroy(h->pipe_join[i]);
  }
  if (h->pipe_fork) cudaEventDestroy(h->pipe_fork);
  if (h->host_in) cudaStreamDestroy(h->host_in);
  if (h->host_out) cudaStreamDestroy(h->host_out);
  if (h->host_start) cudaEventDestroy(h->host_start);
  for (int i = 0; i < blade_ms::kHostChunks; ++i) {
    if (h->host_ev_in[i]) cudaEventDestroy(h->host_ev_in[i]);
    if (h->host_ev_done[i]) cudaEventDestroy(h->host_ev_done[i]);
  }
  cudaFree(h->d_bank);
  cudaFree(h->d_bank_tma);
  delete h;
  return BLADE_OK;
}

blade_status blade_ms_get_info(blade_ms_t h, blade_ms_info* info) {
  if (!h || !info) return fail(BLADE_EINVAL, "NULL argument");
  info->levels = h->cfg.levels;
  info->fine_size = h->cfg.fine_size;
  info->coarse_size = h->cfg.coarse_size;
  info->n_phases = h->cfg.n_phases;
  info->n_stages = h->n_stages;
  info->K = h->K;
  info->device = h->device;
  info->bank_bytes_device = h->bank_bytes;
  info->stage_smem_bytes = h->has_tma ? h->tma_smem : h->stage_smem;
  info->stage_phase_groups = h->has_tma ? 1 : h->stage.rs;
  return BLADE_OK;
}

static blade_status check_dims(int32_t N, int32_t H, int32_t W) {
  if (N < 0 || H < 1 || W < 1) return fail(BLADE_EINVAL, "need N >= 0, H >= 1, W >= 1 (got %d, %d, %d)", N, H, W);
  if ((long long)H * W * 3 > (1LL << 31) - 1) return fail(BLADE_EINVAL, "a frame of %d x %d exceeds 2^31 samples", H, W);
  if (N > 65535) return fail(BLADE_EINVAL, "N > 65535 frames per call");
  return BLADE_OK;
}

blade_status blade_ms_workspace_size(blade_ms_t h, int32_t N, int32_t H, int32_t W, size_t* bytes) {
  if (!h || !bytes) return fail(BLADE_EINVAL, "NULL argument");
  blade_status s = check_dims(N, H, W);
  if (s != BLADE_OK) return s;
  Plan p;
  plan_rows(h, N, H, W, 0, H, p);
  *bytes = p.ws_bytes;
  return BLADE_OK;
}

blade_status blade_ms_launch_count(blade_ms_t h, int32_t N, int32_t H, int32_t W, int32_t* count) {
  if (!h || !count) return fail(BLADE_EINVAL, "NULL argument");
  const int L = h->cfg.levels;
  // k_down + k_stage per stage level, one merged fix-up per kFixMax levels (+ the YCbCr -> RGB
  // conversion with per-channel banks, + the copy-out of a staged level-0 output)
  const int nsel = L == 1 ? 1 : L - 1;
  // fused level-0 selector (large frames): the level's fix-up is the stage fix-up (one launch
  // either way), and it leaves the merged fix-ups
  const bool fused = h->has_fsel && L > 1 && fuse_sel_enabled() && use_ry4(h, N, W, H + (H & 1));
  const int merged = fused ? nsel - 1 : nsel;
  const int fixes = tile_down(h, N, H, W, true) || inline_fixups(N, H, W, true) ? 0
                    : fixups_merged(nsel, N, H, W) ? (merged + kFixMax - 1) / kFixMax + (fused ? 1 : 0)
                                                   : nsel;
  *count = N == 0 ? 0
                  : 2 * nsel + fixes +
                        (h->cfg.n_filter_channels == 3 ? 1 : 0) + (h->has_tma && W % 4 != 0 ? 1 : 0);
  return BLADE_OK;
}

blade_status blade_ms_stage_kernel(blade_ms_t h, int32_t N, int32_t H, int32_t W, int32_t level, int32_t* kind,
                                   int32_t* rows_per_thread) {
  if (!h || !kind || !rows_per_thread) return fail(BLADE_EINVAL, "NULL argument");
  blade_status s = check_dims(N, H, W);
  if (s != BLADE_OK) return s;
  if (level < 0 || level >= h->n_stages) return fail(BLADE_EINVAL, "level %d outside 0..%d", level, h->n_stages - 1);
  Plan p;
  plan_rows(h, std::max(N, 1), H, W, 0, H, p);
  const int L = p.L, l = level;
  // level 0 reads / writes the caller's dense buffers (pitch W); levels >= 1 and the coarse inputs
  // live in the workspace with rows padded to 16 B
  const bool tma = h->has_tma;  // level 0 with W % 4 != 0 reads k_down's 16-B-row input copy
  if (!tma) {
    *kind = 0;
    *rows_per_thread = 2;
  } else if (h->tma.phase_split) {
    *kind = h->tma.ptypes == 2 ? 3 : 2;
    *rows_per_thread = 2;
  } else {
    *kind = 1;
    *rows_per_thread = use_ry4(h, N, p.W[l], p.u[l].hi - (p.u[l].lo & ~1)) ? 4 : 2;
  }
  return BLADE_OK;
}

static blade_status common_checks(blade_ms_t h, const void* in, int32_t N, void* ws, size_t ws_bytes,
                                  const Plan& p) {
  if (!h) return fail(BLADE_EINVAL, "handle is NULL");
  if (N > 0 && !in) return fail(BLADE_EINVAL, "in is NULL");
  if (N > 0 && !ws && p.ws_bytes > 0) return fail(BLADE_EINVAL, "workspace is NULL");
  if (ws_bytes < p.ws_bytes) return fail(BLADE_ESHAPE, "workspace %zu bytes < required %zu", ws_bytes, p.ws_bytes);
  blade_status s;
  if (N > 0) {
    if ((s = check_dev_ptr(h, in, "in")) != BLADE_OK) return s;
    if ((s = check_dev_ptr(h, ws, "workspace")) != BLADE_OK) return s;
    if (!aligned16(ws)) return fail(BLADE_EINVAL, "workspace must be 16-byte aligned");
  }
  return BLADE_OK;
}

blade_status blade_ms_denoise(blade_ms_t h, const float* in, float* out, int32_t N, int32_t H, int32_t W, void* ws,
                              size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (!h) return fail(BLADE_EINVAL, "handle is NULL");
  blade_status s = check_dims(N, H, W);
  if (s != BLADE_OK) return s;
  if (N == 0) return BLADE_OK;
  Plan p;
  plan_rows(h, N, H, W, 0, H, p);
  if ((s = common_checks(h, in, N, ws, ws_bytes, p)) != BLADE_OK) return s;
  if (!out) return fail(BLADE_EINVAL, "out is NULL");
  if ((s = check_dev_ptr(h, out, "out")) != BLADE_OK) return s;
  const size_t img = sizeof(float) * (size_t)N * 3 * H * W;
  if (ranges_overlap(in, img, out, img)) return fail(BLADE_EINVAL, "out overlaps in");
  if (ranges_overlap(ws, p.ws_bytes, out, img) || ranges_overlap(ws, p.ws_bytes, in, img))
    return fail(BLADE_EINVAL, "workspace overlaps in/out");
  DeviceGuard guard(h->device);
  LevelView inv = make_view(const_cast<float*>(in), H, W, Range{0, H});
  LevelView outv = make_view(out, H, W, Range{0, H});
  return enqueue(h, p, inv, outv, (char*)ws, (cudaStream_t)stream, true, nullptr, nullptr);
}

static size_t pipe_slice_bytes(const blade_ms* h, int chunk, int H, int W) {
  Plan p;
  plan_rows(h, chunk, H, W, 0, H, p);
  return align256(p.ws_bytes);
}

blade_status blade_ms_pipeline_workspace_size(blade_ms_t h, int32_t chunk, int32_t n_streams, int32_t H, int32_t W,
                                              size_t* bytes) {
  if (!h || !bytes) return fail(BLADE_EINVAL, "NULL argument");
  blade_status s = check_dims(chunk, H, W);
  if (s != BLADE_OK) return s;
  if (chunk < 1) return fail(BLADE_EINVAL, "chunk must be >= 1");
  if (n_streams < 1 || n_streams > blade_ms::kMaxStreams)
    return fail(BLADE_EINVAL, "n_streams must be in 1..%d", blade_ms::kMaxStreams);
  *bytes = (size_t)n_streams * pipe_slice_bytes(h, chunk, H, W);
  return BLADE_OK;
}

// NEXT f3: chunk i of `chunk` frames -> internal stream i % n_streams, own
// workspace slice; fork from / join into the caller's stream with events.
blade_status blade_ms_denoise_pipelined(blade_ms_t h, const float* in, float* out, int32_t N, int32_t H, int32_t W,
                                        int32_t chunk, int32_t n_streams, void* ws, size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (!h) return fail(BLADE_EINVAL, "handle is NULL");
  blade_status s = check_dims(N, H, W);
  if (s != BLADE_OK) return s;
  if (chunk < 1 || chunk > 65535) return fail(BLADE_EINVAL, "chunk must be in 1..65535");
  if (n_streams < 1 || n_streams > blade_ms::kMaxStreams)
    return fail(BLADE_EINVAL, "n_streams must be in 1..%d", blade_ms::kMaxStreams);
  if (N == 0) return BLADE_OK;
  const size_t slice = pipe_slice_bytes(h, chunk, H, W);
  Plan pneed;
  pneed.ws_bytes = (size_t)n_streams * slice;
  if ((s = common_checks(h, in, N, ws, ws_bytes, pneed)) != BLADE_OK) return s;
  if (!out) return fail(BLADE_EINVAL, "out is NULL");
  if ((s = check_dev_ptr(h, out, "out")) != BLADE_OK) return s;
  const size_t img = sizeof(float) * (size_t)N * 3 * H * W;
  if (ranges_overlap(in, img, out, img)) return fail(BLADE_EINVAL, "out overlaps in");
  if (ranges_overlap(ws, pneed.ws_bytes, out, img) || ranges_overlap(ws, pneed.ws_bytes, in, img))
    return fail(BLADE_EINVAL, "workspace overlaps in/out");
  DeviceGuard guard(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int nchunks = (N + chunk - 1) / chunk;
  const int ns = std::min(n_streams, nchunks);
  std::lock_guard<std::mutex> lock(h->pipe_mu);  // fork .. join of this call, atomically
  cudaError_t ce = cudaEventRecord(h->pipe_fork, st);
  for (int i = 0; i < ns && ce == cudaSuccess; ++i) ce = cudaStreamWaitEvent(h->pipe[i], h->pipe_fork, 0);
  if (ce != cudaSuccess) return fail(BLADE_ECUDA, "fork: %s", cudaGetErrorString(ce));
  blade_status rs = BLADE_OK;
  const size_t fr = (size_t)3 * H * W;
  for (int i = 0; i < nchunks && rs == BLADE_OK; ++i) {
    const int f0 = i * chunk, nf = std::min(chunk, N - f0);
    Plan p;
    plan_rows(h, nf, H, W, 0, H, p);
    LevelView inv = make_view(const_cast<float*>(in) + (size_t)f0 * fr, H, W, Range{0, H});
    LevelView outv = make_view(out + (size_t)f0 * fr, H, W, Range{0, H});
    rs = enqueue(h, p, inv, outv, (char*)ws + (size_t)(i % ns) * slice, h->pipe[i % ns], true, nullptr, nullptr);
  }
  // join (also after a failed enqueue, so the caller's stream never runs ahead of queued work)
  for (int i = 0; i < ns; ++i) {
    cudaError_t e = cudaEventRecord(h->pipe_join[i], h->pipe[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, h->pipe_join[i], 0);
    if (e != cudaSuccess && rs == BLADE_OK) rs = fail(BLADE_ECUDA, "join: %s", cudaGetErrorString(e));
  }
  return rs;
}

blade_status blade_ms_selector(blade_ms_t h, const float* in, int32_t N, int32_t H, int32_t W, void* const* maps,
                               void* ws, size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (!h) return fail(BLADE_EINVAL, "handle is NULL");
  blade_status s = check_dims(N, H, W);
  if (s != BLADE_OK) return s;
  if (!maps) return fail(BLADE_EINVAL, "maps_per_level is NULL");
  if (N == 0) return BLADE_OK;
  Plan p;
  plan_rows(h, N, H, W, 0, H, p);
  if ((s = common_checks(h, in, N, ws, ws_bytes, p)) != BLADE_OK) return s;
  for (int l = 0; l < h->n_stages; ++l)
    if (maps[l] && (s = check_dev_ptr(h, maps[l], "maps_per_level[l]")) != BLADE_OK) return s;
  DeviceGuard guard(h->device);
  LevelView inv = make_view(const_cast<float*>(in), H, W, Range{0, H});
  return enqueue(h, p, inv, LevelView{}, (char*)ws, (cudaStream_t)stream, false, maps, nullptr);
}

blade_status blade_ms_pyramid(blade_ms_t h, const float* in, int32_t N, int32_t H, int32_t W, float* const* levels,
                              void* ws, size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (!h) return fail(BLADE_EINVAL, "handle is NULL");
  blade_status s = check_dims(N, H, W);
  if (s != BLADE_OK) return s;
  if (!levels) return fail(BLADE_EINVAL, "levels is NULL");
  if (N == 0) return BLADE_OK;
  Plan p;
  plan_rows(h, N, H, W, 0, H, p);
  if ((s = common_checks(h, in, N, ws, ws_bytes, p)) != BLADE_OK) return s;
  for (int l = 1; l < h->cfg.levels; ++l) {
    if (!levels[l - 1]) return fail(BLADE_EINVAL, "levels[%d] is NULL", l - 1);
    if ((s = check_dev_ptr(h, levels[l - 1], "levels[l]")) != BLADE_OK) return s;
  }
  DeviceGuard guard(h->device);
  LevelView inv = make_view(const_cast<float*>(in), H, W, Range{0, H});
  return enqueue(h, p, inv, LevelView{}, (char*)ws, (cudaStream_t)stream, false, nullptr, levels);
}

blade_status blade_ms_band_rows(blade_ms_t h, int32_t H, int32_t out_row0, int32_t out_rows, int32_t* in_row0,
                                int32_t* in_rows) {
  if (!h || !in_row0 || !in_rows) return fail(BLADE_EINVAL, "NULL argument");
  if (H < 1 || out_row0 < 0 || out_rows < 1 || out_row0 + out_rows > H)
    return fail(BLADE_EINVAL, "bad band [%d, %d) of H = %d", out_row0, out_row0 + out_rows, H);
  Plan p;
  plan_rows(h, 1, H, 1, out_row0, out_rows, p);
  *in_row0 = p.z[0].lo;
  *in_rows = p.z[0].n();
  return BLADE_OK;
}

blade_status blade_ms_fallback_count(blade_ms_t h, int32_t N, int32_t H, int32_t W, const void* ws,
                                     size_t ws_bytes, uint32_t* counts) {
  if (!h || !ws || !counts) return fail(BLADE_EINVAL, "NULL argument");
  blade_status s = check_dims(N, H, W);
  if (s != BLADE_OK) return s;
  Plan p;
  plan_rows(h, N, H, W, 0, H, p);
  if (ws_bytes < p.ws_bytes) return fail(BLADE_ESHAPE, "workspace too small");
  DeviceGuard guard(h->device);
  CUDA_TRY(cudaMemcpy(counts, (const char*)ws + p.fbcnt_off, sizeof(uint32_t) * h->n_stages, cudaMemcpyDeviceToHost));
  return BLADE_OK;
}

// ------------------------------------------------------------------------------ training (NEXT f4)

static int train_nt(const blade_ms* h) {
  return h->cfg.fine_size * h->cfg.fine_size + (h->cfg.levels > 1 ? h->cfg.coarse_size * h->cfg.coarse_size : 0);
}
static const TrainVariant* train_variant(const blade_ms* h) {
  const int cnc = h->cfg.levels > 1 ? h->cfg.coarse_size : 0;
  for (const auto* list : {&train_variants(), &train_variants_pairs()})
    for (const auto& v : *list)
      if (v.nf == h->cfg.fine_size && v.nc == cnc && v.wide == (h->K > 256)) return &v;
  return nullptr;
}

struct TrainPlan {
  size_t map_off, fb_off, fbcnt_off, cnt_off, cur_off, sorted_off, bytes;
  unsigned int fb_cap;
};
static TrainPlan train_plan(const blade_ms* h, long long px) {
  TrainPlan t{};
  const int n_seg = h->cfg.n_phases * h->K;
  size_t off = 0;
  t.map_off = off;
  off = align256(off + px * (h->K > 256 ? 2 : 1));
  t.fb_cap = (unsigned int)std::min<long long>(std::max<long long>(px / 64, 1024), 0x7fffffff);
  t.fb_off = off;
  off = align256(off + sizeof(unsigned long long) * t.fb_cap);
  t.fbcnt_off = off;
  off = align256(off + 16);
  t.cnt_off = off;
  off = align256(off + sizeof(unsigned int) * n_seg);
  t.cur_off = off;
  off = align256(off + sizeof(unsigned int) * n_seg);
  t.sorted_off = off;
  off = align256(off + sizeof(unsigned int) * px);
  t.bytes = off;
  return t;
}

blade_status blade_ms_train_layout(blade_ms_t h, int32_t* nt, int32_t* ntp, int32_t* n_seg) {
  if (!h || !nt || !ntp || !n_seg) return fail(BLADE_EINVAL, "NULL argument");
  const TrainVariant* v = train_variant(h);
  if (!v) return fail(BLADE_EUNSUPPORTED, "no training kernel for this footprint / bucket layout");
  *nt = train_nt(h);
  *ntp = v->ntp;
  *n_seg = h->cfg.n_phases * h->K;
  return BLADE_OK;
}

blade_status blade_ms_train_workspace_size(blade_ms_t h, int32_t N, int32_t H, int32_t W, size_t* bytes) {
  if (!h || !bytes) return fail(BLADE_EINVAL, "NULL argument");
  blade_status s = check_dims(N, H, W);
  if (s != BLADE_OK) return s;
  *bytes = train_plan(h, (long long)N * H * W).bytes;
  return BLADE_OK;
}

blade_status blade_ms_train_accumulate(blade_ms_t h, int32_t level, const float* z, const float* u_clean,
                                       const float* u_coarse, int32_t N, int32_t H, int32_t W, double* E,
                                       uint64_t* count, void* ws, size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (!h) return fail(BLADE_EINVAL, "handle is NULL");
  blade_status s = check_dims(N, H, W);
  if (s != BLADE_OK) return s;
  if (level < 0 || level >= h->n_stages) return fail(BLADE_EINVAL, "level %d not in [0, %d)", level, h->n_stages);
  if (h->cfg.n_filter_channels != 1) return fail(BLADE_EUNSUPPORTED, "training of per-channel banks is not built");
  const TrainVariant* v = train_variant(h);
  if (!v) return fail(BLADE_EUNSUPPORTED, "no training kernel for this footprint / bucket layout");
  const int n_seg = h->cfg.n_phases * h->K;
  if (n_seg > 16384) return fail(BLADE_EUNSUPPORTED, "training supports n_phases * K <= 16384");
  const long long px = (long long)N * H * W;
  if (px >= (1LL << 32)) return fail(BLADE_EINVAL, "too many pixels for one training call");
  if (N == 0) return BLADE_OK;
  const bool multiscale = h->cfg.levels > 1;
  if (!z || !u_clean || !E || !count || !ws || (multiscale && !u_coarse))
    return fail(BLADE_EINVAL, "NULL buffer (u_coarse is required when levels > 1)");
  const TrainPlan tp = train_plan(h, px);
  if (ws_bytes < tp.bytes) return fail(BLADE_ESHAPE, "workspace %zu bytes < required %zu", ws_bytes, tp.bytes);
  if ((s = check_dev_ptr(h, z, "z")) != BLADE_OK) return s;
  if ((s = check_dev_ptr(h, u_clean, "u_clean")) != BLADE_OK) return s;
  if (multiscale && (s = check_dev_ptr(h, u_coarse, "u_coarse")) != BLADE_OK) return s;
  if ((s = check_dev_ptr(h, E, "E")) != BLADE_OK) return s;
  if ((s = check_dev_ptr(h, count, "count")) != BLADE_OK) return s;
  if ((s = check_dev_ptr(h, ws, "workspace")) != BLADE_OK) return s;
  DeviceGuard guard(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  const int l = level;
  // ---- selector on the noisy level (fp32 input, thresholds of stage `level`)
  DownArgs da{};
  da.zhi = z;
  da.zlo = nullptr;
  da.H = H;
  da.W = W;
  da.in_row0 = 0;
  da.in_rows = H;
  da.in_plane = (long long)H * W;
  da.in_frame = 3 * da.in_plane;
  da.map = w + tp.map_off;
  da.map_pitch = W;
  da.in_pitch = W;
  da.out_pitch = 1;
  da.s_r0 = 0;
  da.s_rn = H;
  da.H1 = da.W1 = 1;
  da.base = 0;
  da.n_strips = (W + down::STRIP - 1) / down::STRIP;
  const long long col_tasks = (long long)N * da.n_strips;
  const long long want_bands = std::max<long long>(1, (4LL * 16 * h->num_sms + col_tasks - 1) / col_tasks);
  int RB = (int)std::min<long long>(128, std::max<long long>(16, (H + want_bands - 1) / want_bands));
  RB = (RB + 1) & ~1;
  da.RB = RB;
  da.n_bands = (H + RB - 1) / RB;
  da.n_tasks = (int)(col_tasks * da.n_bands);
  da.fb_list = reinterpret_cast<unsigned long long*>(w + tp.fb_off);
  da.fb_count = reinterpret_cast<unsigned int*>(w + tp.fbcnt_off);
  da.fb_cap = tp.fb_cap;
  da.N = N;
  const bool fast = h->n_o == 16 && h->n_s == 3 && h->n_c == 3;
  const bool wide = h->K > 256;
  CUDA_TRY(cudaMemsetAsync(da.fb_count, 0, sizeof(unsigned int), st));
  down_kernel(false, false, fast, wide)<<<(unsigned)((da.n_tasks + down::WARPS - 1) / down::WARPS),
                                           32 * down::WARPS, down_smem(false), st>>>(da, h->down[l]);
  LAUNCH_CHECK("k_down (training selector)");
  fixup_kernel(false, fast, wide)<<<4 * h->num_sms, 128, 0, st>>>(da, h->down[l]);
  LAUNCH_CHECK("k_down_fixup (training selector)");
  // ---- counting sort of the pixels by (phase, bucket), then the segmented fp64 SYRK, per group
  //      of frames whose inputs (z, clean target, coarse input) fit in about half the L2: the
  //      sorted order scatters every segment's pixels over the group's frames, so the Gram
  //      kernel's patch gathers hit L2 only while the group stays resident (BLADE_TRAIN_GROUP =
  //      frames per group overrides; 0 = all frames in one group)
  const long long frame_bytes = (long long)H * W * 3 * 4 * 2 + (u_coarse ? (long long)((H + 1) / 2) * ((W + 1) / 2) * 12 : 0);
  static const int group_env = [] {
    const char* e = getenv("BLADE_TRAIN_GROUP");
    return e ? atoi(e) : -1;
  }();
  int fg = group_env >= 0 ? group_env : (int)std::max<long long>(1, (64LL << 20) / std::max<long long>(frame_bytes, 1));
  if (fg <= 0 || fg > N) fg = N;
  static const bool use_mma = [] {  // BLADE_TRAIN_MMA=0: the DFMA accumulation (A/B timing)
    const char* e = getenv("BLADE_TRAIN_MMA");
    return !(e && e[0] == '0');
  }();
  CUDA_TRY(cudaFuncSetAttribute(train_hist(wide), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(unsigned int) * n_seg)));
  CUDA_TRY(cudaFuncSetAttribute(train_scatter(wide), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(2 * sizeof(unsigned int) * n_seg)));
  const long long plane = (long long)H * W, plane1 = (long long)((H + 1) / 2) * ((W + 1) / 2);
  for (int f0 = 0; f0 < N; f0 += fg) {
    const int nf = std::min(fg, N - f0);
    const long long gpx = (long long)nf * H * W;
    TrainArgs ta{};
    ta.z = z + (long long)f0 * 3 * plane;
    ta.uc = u_clean + (long long)f0 * 3 * plane;
    ta.u1 = u_coarse ? u_coarse + (long long)f0 * 3 * plane1 : nullptr;
    ta.map = w + tp.map_off + (size_t)(wide ? 2 : 1) * f0 * plane;
    ta.N = nf;
    ta.H = H;
    ta.W = W;
    ta.H1 = (H + 1) / 2;
    ta.W1 = (W + 1) / 2;
    ta.n_phases = h->cfg.n_phases;
    ta.K = h->K;
    ta.n_seg = n_seg;
    ta.count = reinterpret_cast<unsigned int*>(w + tp.cnt_off);
    ta.cursor = reinterpret_cast<unsigned int*>(w + tp.cur_off);
    ta.sorted = reinterpret_cast<unsigned int*>(w + tp.sorted_off);
    ta.E = E;
    ta.count_out = reinterpret_cast<unsigned long long*>(count);
    ta.pix_per_cta = 512;
    CUDA_TRY(cudaMemsetAsync(ta.count, 0, sizeof(unsigned int) * n_seg, st));
    const unsigned g_px = (unsigned)std::min<long long>((gpx + 255) / 256, 4LL * h->num_sms);
    train_hist(wide)<<<g_px, 256, sizeof(unsigned int) * n_seg, st>>>(ta);
    LAUNCH_CHECK("k_train_hist");
    train_scan()<<<1, 1024, 0, st>>>(ta);
    LAUNCH_CHECK("k_train_scan");
    const unsigned g_sc = (unsigned)std::min<long long>((gpx + 8191) / 8192, 2LL * h->num_sms);
    train_scatter(wide)<<<g_sc, 512, 2 * sizeof(unsigned int) * n_seg, st>>>(ta);
    LAUNCH_CHECK("k_train_scatter");
    (use_mma ? v->gram : v->gram_dfma)<<<(unsigned)((gpx + ta.pix_per_cta - 1) / ta.pix_per_cta), 256, 0, st>>>(ta);
    LAUNCH_CHECK("k_train_gram");
  }
  return BLADE_OK;
}

blade_status blade_ms_train_solve(blade_ms_t h, const double* E, const uint64_t* count, double ridge,
                                  uint64_t min_count, float* taps) {
  g_last_error.clear();
  if (!h || !E || !count || !taps) return fail(BLADE_EINVAL, "NULL argument");
  const TrainVariant* v = train_variant(h);
  if (!v) return fail(BLADE_EUNSUPPORTED, "no training kernel for this footprint / bucket layout");
  if (!(ridge >= 0.0) || !std::isfinite(ridge)) return fail(BLADE_EINVAL, "ridge must be finite and >= 0");
  const int nt = train_nt(h), ntp = v->ntp, n_seg = h->cfg.n_phases * h->K, nf = h->cfg.fine_size;
  std::vector<double> A((size_t)nt * nt), b(nt);
  for (int sg = 0; sg < n_seg; ++sg) {
    float* out = taps + (size_t)sg * nt;
    const double* Es = E + (size_t)sg * ntp * ntp;
    auto e = [&](int r, int c) { return (r / 4 <= c / 4) ? Es[(size_t)r * ntp + c] : Es[(size_t)c * ntp + r]; };
    bool ok = count[sg] >= min_count && count[sg] > 0;
    if (ok) {
      double tr = 0.0;
      for (int i = 0; i < nt; ++i) tr += e(i, i);
      const double lam = ridge * tr / nt;
      for (int i = 0; i < nt; ++i) {
        for (int j = 0; j < nt; ++j) A[(size_t)i * nt + j] = e(i, j) + (i == j ? lam : 0.0);
        b[i] = e(i, nt);
      }
      // Cholesky A = L L^T (in place, lower), then two triangular solves
      for (int j = 0; j < nt && ok; ++j) {
        double d = A[(size_t)j * nt + j];
        for (int k = 0; k < j; ++k) d -= A[(size_t)j * nt + k] * A[(size_t)j * nt + k];
        if (!(d > 0.0)) {
          ok = false;
          break;
        }
        const double ljj = std::sqrt(d);
        A[(size_t)j * nt + j] = ljj;
        for (int i = j + 1; i < nt; ++i) {
          double x = A[(size_t)i * nt + j];
          for (int k = 0; k < j; ++k) x -= A[(size_t)i * nt + k] * A[(size_t)j * nt + k];
          A[(size_t)i * nt + j] = x / ljj;
        }
      }
      if (ok) {
        for (int i = 0; i < nt; ++i) {  // L y = b
          double x = b[i];
          for (int k = 0; k < i; ++k) x -= A[(size_t)i * nt + k] * b[k];
          b[i] = x / A[(size_t)i * nt + i];
        }
        for (int i = nt - 1; i >= 0; --i) {  // L^T h = y
          double x = b[i];
          for (int k = i + 1; k < nt; ++k) x -= A[(size_t)k * nt + i] * b[k];
          b[i] = x / A[(size_t)i * nt + i];
        }
        for (int i = 0; i < nt; ++i) {
          if (!std::isfinite(b[i])) ok = false;
          out[i] = (float)b[i];
        }
      }
    }
    if (!ok) {  // fallback: centred fine delta, zero coarse block [R28]
      for (int i = 0; i < nt; ++i) out[i] = 0.0f;
      out[(nf / 2) * nf + nf / 2] = 1.0f;
    }
  }
  return BLADE_OK;
}

blade_status blade_ms_band_plan(const blade_ms_config* cfg, int32_t H, int32_t out_row0, int32_t out_rows,
                                int32_t* in_row0, int32_t* in_rows) {
  if (!cfg || !in_row0 || !in_rows) return fail(BLADE_EINVAL, "NULL argument");
  if (cfg->levels < 1 || cfg->levels > 12 || cfg->fine_size < 1 || cfg->fine_size > 9 || !(cfg->fine_size & 1) ||
      (cfg->levels > 1 && (cfg->coarse_size < 1 || cfg->coarse_size > 9 || !(cfg->coarse_size & 1))) ||
      cfg->window_size < 1 || cfg->window_size > 5 || !(cfg->window_size & 1))
    return fail(BLADE_EINVAL, "bad config");
  if (H < 1 || out_row0 < 0 || out_rows < 1 || out_row0 + out_rows > H)
    return fail(BLADE_EINVAL, "bad band [%d, %d) of H = %d", out_row0, out_row0 + out_rows, H);
  Plan p;
  plan_rows_cfg(*cfg, 1, H, 1, out_row0, out_rows, p);
  *in_row0 = p.z[0].lo;
  *in_rows = p.z[0].n();
  return BLADE_OK;
}

blade_status blade_ms_band_workspace_size(blade_ms_t h, int32_t H, int32_t W, int32_t out_row0, int32_t out_rows,
                                          size_t* bytes) {
  if (!h || !bytes) return fail(BLADE_EINVAL, "NULL argument");
  if (H < 1 || W < 1 || out_row0 < 0 || out_rows < 1 || out_row0 + out_rows > H) return fail(BLADE_EINVAL, "bad band");
  Plan p;
  plan_rows(h, 1, H, W, out_row0, out_rows, p);
  *bytes = p.ws_bytes;
  return BLADE_OK;
}

blade_status blade_ms_denoise_rows(blade_ms_t h, const float* in_band, int32_t in_row0, int32_t in_rows,
                                   float* out_band, int32_t out_row0, int32_t out_rows, int32_t H, int32_t W,
                                   void* ws, size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (!h) return fail(BLADE_EINVAL, "handle is NULL");
  blade_status s = check_dims(1, H, W);
  if (s != BLADE_OK) return s;
  if (out_row0 < 0 || out_rows < 1 || out_row0 + out_rows > H)
    return fail(BLADE_EINVAL, "bad output band [%d, %d) of H = %d", out_row0, out_row0 + out_rows, H);
  if (!in_band || !out_band) return fail(BLADE_EINVAL, "NULL band pointer");
  Plan p;
  plan_rows(h, 1, H, W, out_row0, out_rows, p);
  if (in_row0 < 0 || in_rows < 1 || in_row0 > p.z[0].lo || in_row0 + in_rows < p.z[0].hi || in_row0 + in_rows > H)
    return fail(BLADE_ESHAPE, "input band [%d, %d) does not cover the needed rows [%d, %d)", in_row0,
                in_row0 + in_rows, p.z[0].lo, p.z[0].hi);
  if ((s = common_checks(h, in_band, 1, ws, ws_bytes, p)) != BLADE_OK) return s;
  if ((s = check_dev_ptr(h, out_band, "out_band")) != BLADE_OK) return s;
  if (ranges_overlap(in_band, sizeof(float) * 3 * (size_t)in_rows * W, out_band, sizeof(float) * 3 * (size_t)out_rows * W))
    return fail(BLADE_EINVAL, "out_band overlaps in_band");
  DeviceGuard guard(h->device);
  LevelView inv = make_view(const_cast<float*>(in_band), H, W, Range{in_row0, in_row0 + in_rows});
  LevelView outv = make_view(out_band, H, W, Range{out_row0, out_row0 + out_rows});
  return enqueue(h, p, inv, outv, (char*)ws, (cudaStream_t)stream, true, nullptr, nullptr);
}

static blade_status xband_layout_impl(const blade_ms_config& cfg, int map_es, int32_t H, int32_t W, int32_t o0,
                                      int32_t on, blade_xband_layout* out, Plan* plan_out) {
  if (H < 1 || W < 1 || (long long)H * W > (1LL << 31) || o0 < 0 || on < 1 || o0 + on > H)
    return fail(BLADE_EINVAL, "bad band [%d, %d) of %d x %d", o0, o0 + on, H, W);
  Plan p;
  int hz = 0, hu = 0;
  std::vector<Range> own;
  if (!plan_xband(cfg, map_es, H, W, o0, on, p, hz, hu, own))
    return fail(BLADE_EUNSUPPORTED, "band [%d, %d) owns fewer than %d rows at some level (use fewer bands or "
                "blade_ms_denoise_rows)", o0, o0 + on, hz);
  if (out) {
    std::memset(out, 0, sizeof(*out));
    const int L = p.L, nsel = L == 1 ? 1 : L - 1;
    out->levels = L;
    out->n_steps = 2 * nsel;
    out->halo_z = hz;
    out->halo_u = hu;
    for (int l = 0; l < L; ++l) {
      out->own_lo[l] = own[l].lo;
      out->own_hi[l] = own[l].hi;
    }
    out->in_row0 = p.z[0].lo;
    out->in_rows = p.z[0].n();
    out->ws_bytes = p.ws_bytes;
    // regions exchanged after each step: rows [row0, row0 + rows) of `planes` planes
    auto region = [&](size_t base, Range buf, int pitch, int planes, int row0, int rows) {
      blade_region r{};
      if (rows <= 0) return r;
      r.row0 = row0;
      r.rows = rows;
      r.pitch = pitch;
      r.planes = planes;
      r.plane_stride = (int64_t)sizeof(float) * buf.n() * pitch;
      r.offset = (int64_t)base + (int64_t)sizeof(float) * (row0 - buf.lo) * pitch;
      return r;
    };
    for (int st = 0; st < out->n_steps; ++st) {
      size_t base = 0;
      Range buf{}, mine{};
      int planes = 0, pitch = 0;
      if (L > 1 && st < nsel) {  // after down(l = st): z^{l+1} (hi, and lo when it feeds a selector)
        const int l1 = st + 1;
        base = p.z32_off[l1];
        buf = p.z[l1];
        mine = p.zc[l1];
        planes = l1 + 1 < L ? 6 : 3;
        pitch = p.pitch[l1];
      } else if (L > 1 && st >= nsel && 2 * nsel - 1 - st >= 1) {  // after up(l >= 1): u^l
        const int l = 2 * nsel - 1 - st;
        base = p.u_off[l];
        buf = p.ub[l];
        mine = p.u[l];
        planes = 3;
        pitch = p.pitch[l];
      } else {
        continue;  // nothing to exchange
      }
      const int above = mine.lo - buf.lo, below = buf.hi - mine.hi;
      out->recv[st][0] = region(base, buf, pitch, planes, buf.lo, above);
      out->send[st][0] = region(base, buf, pitch, planes, mine.lo, above);
      out->recv[st][1] = region(base, buf, pitch, planes, mine.hi, below);
      out->send[st][1] = region(base, buf, pitch, planes, mine.hi - below, below);
    }
  }
  if (plan_out) *plan_out = p;
  return BLADE_OK;
}

blade_status blade_ms_xband_layout(const blade_ms_config* cfg, int32_t K, int32_t H, int32_t W, int32_t out_row0,
                                   int32_t out_rows, blade_xband_layout* layout) {
  if (!cfg || !layout) return fail(BLADE_EINVAL, "NULL argument");
  if (cfg->levels < 1 || cfg->levels > BLADE_MAX_LEVELS || cfg->fine_size < 1 || cfg->fine_size > 9 ||
      !(cfg->fine_size & 1) ||
      (cfg->levels > 1 && (cfg->coarse_size < 1 || cfg->coarse_size > 9 || !(cfg->coarse_size & 1))) ||
      cfg->window_size < 1 || cfg->window_size > 5 || !(cfg->window_size & 1) || K < 1 || K > 65536)
    return fail(BLADE_EINVAL, "bad config");
  return xband_layout_impl(*cfg, K > 256 ? 2 : 1, H, W, out_row0, out_rows, layout, nullptr);
}

blade_status blade_ms_xband_step(blade_ms_t h, int32_t step, const float* in_band, int32_t in_row0, int32_t in_rows,
                                 float* out_band, int32_t out_row0, int32_t out_rows, int32_t H, int32_t W, void* ws,
                                 size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (!h) return fail(BLADE_EINVAL, "handle is NULL");
  blade_status s = check_dims(1, H, W);
  if (s != BLADE_OK) return s;
  Plan p;
  if ((s = xband_layout_impl(h->cfg, h->K > 256 ? 2 : 1, H, W, out_row0, out_rows, nullptr, &p)) != BLADE_OK)
    return s;
  const int L = p.L, nsel = L == 1 ? 1 : L - 1;
  if (step < 0 || step >= 2 * nsel) return fail(BLADE_EINVAL, "step %d outside 0..%d", step, 2 * nsel - 1);
  if (!in_band || !out_band) return fail(BLADE_EINVAL, "NULL band pointer");
  if (in_row0 < 0 || in_rows < 1 || in_row0 > p.z[0].lo || in_row0 + in_rows < p.z[0].hi || in_row0 + in_rows > H)
    return fail(BLADE_ESHAPE, "input band [%d, %d) does not cover the needed rows [%d, %d)", in_row0,
                in_row0 + in_rows, p.z[0].lo, p.z[0].hi);
  if ((s = common_checks(h, in_band, 1, ws, ws_bytes, p)) != BLADE_OK) return s;
  if ((s = check_dev_ptr(h, out_band, "out_band")) != BLADE_OK) return s;
  if (ranges_overlap(in_band, sizeof(float) * 3 * (size_t)in_rows * W, out_band, sizeof(float) * 3 * (size_t)out_rows * W))
    return fail(BLADE_EINVAL, "out_band overlaps in_band");
  DeviceGuard guard(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  LevelView inv = make_view(const_cast<float*>(in_band), H, W, Range{in_row0, in_row0 + in_rows});
  LevelView outv = make_view(out_band, H, W, Range{out_row0, out_row0 + out_rows});
  Bufs B = make_bufs(p, inv, (char*)ws, nullptr, nullptr);
  B.fuse0 = fused_level0(h, p, B, inv, outv, (char*)ws, true);
  if (step < nsel) {
    const int l = step;
    CUDA_TRY(cudaMemsetAsync(B.fb_cnt + l, 0, sizeof(unsigned int), st));
    return down_level(h, p, B, inv, (char*)ws, st, true, l, nullptr);
  }
  return up_level(h, p, B, outv, (char*)ws, st, 2 * nsel - 1 - step);
}

blade_status blade_ms_denoise_host(blade_ms_t h, const float* in_host, float* out_host, int32_t N, int32_t H,
                                   int32_t W, float* d_in, float* d_out, void* ws, size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (!h) return fail(BLADE_EINVAL, "handle is NULL");
  blade_status s = check_dims(N, H, W);
  if (s != BLADE_OK) return s;
  if (N == 0) return BLADE_OK;
  if (!in_host || !out_host || !d_in || !d_out) return fail(BLADE_EINVAL, "NULL buffer");
  Plan pfull;
  plan_rows(h, N, H, W, 0, H, pfull);
  if ((s = common_checks(h, d_in, N, ws, ws_bytes, pfull)) != BLADE_OK) return s;
  if ((s = check_dev_ptr(h, d_out, "d_out")) != BLADE_OK) return s;
  const size_t fbytes = sizeof(float) * 3 * (size_t)H * W;
  if (ranges_overlap(d_in, fbytes * N, d_out, fbytes * N)) return fail(BLADE_EINVAL, "d_out overlaps d_in");
  DeviceGuard guard(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  // chunked pipeline: H2D (chunk i+1) || compute (chunk i) || D2H (chunk i-1). Chunks are groups
  // of frames; a batch of fewer frames than chunks whose frames are large is cut into row bands
  // instead (blade_ms_denoise_rows' plan: each band computes its output rows from its dependency
  // cone of input rows, bit-identical to the whole frame), so one big image overlaps its copies
  // with its compute too.
  static const int max_chunks = [] {  // BLADE_E2E_CHUNKS overrides (A/B timing: 16 / 32 / 64 chunks
    const char* e = getenv("BLADE_E2E_CHUNKS");  // of a c3 batch: 34.8 / 34.6 / 35.9 ms, PCIe bound 31.7)
    return e ? std::min(blade_ms::kHostChunks, std::max(1, atoi(e))) : blade_ms::kHostChunks;
  }();
  static const int band_chunks = [] {  // BLADE_E2E_BANDS: row bands of a single large frame (0: off)
    const char* e = getenv("BLADE_E2E_BANDS");
    return e ? std::min(blade_ms::kHostChunks, std::max(0, atoi(e))) : 12;  // 8 / 12 / 16 bands: c4 e2e 3,287 / 3,591 / 3,605, c2 2,926 / 3,076 / 3,022 MP/s
  }();
  const bool banded = N == 1 && band_chunks > 1 && (long long)H * W >= (4LL << 20) && H >= 16 * band_chunks;
  const int nchunks = banded ? band_chunks : std::min<int>(N, max_chunks);
  std::lock_guard<std::mutex> lock(h->host_mu);
  cudaError_t ce = cudaSuccess;
  if (!h->host_in) ce = cudaStreamCreateWithFlags(&h->host_in, cudaStreamNonBlocking);
  if (ce == cudaSuccess && !h->host_out) ce = cudaStreamCreateWithFlags(&h->host_out, cudaStreamNonBlocking);
  if (ce == cudaSuccess && !h->host_start) ce = cudaEventCreateWithFlags(&h->host_start, cudaEventDisableTiming);
  for (int i = 0; i < nchunks && ce == cudaSuccess; ++i) {
    if (!h->host_ev_in[i]) ce = cudaEventCreateWithFlags(&h->host_ev_in[i], cudaEventDisableTiming);
    if (ce == cudaSuccess && !h->host_ev_done[i]) ce = cudaEventCreateWithFlags(&h->host_ev_done[i], cudaEventDisableTiming);
  }
  cudaStream_t s_in = h->host_in, s_out = h->host_out;
  if (ce == cudaSuccess) ce = cudaEventRecord(h->host_start, st);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(s_in, h->host_start, 0);
  if (ce != cudaSuccess) return fail(BLADE_ECUDA, "stream/event setup: %s", cudaGetErrorString(ce));
  blade_status rs = BLADE_OK;
  // rows [r0, r1) of the three planes of frame 0 between host and device
  auto copy_rows = [&](float* dst, const float* src, int r0, int r1, cudaMemcpyKind kind, cudaStream_t cs) {
    cudaError_t e = cudaSuccess;
    for (int c = 0; c < 3 && e == cudaSuccess && r1 > r0; ++c) {
      const size_t o = ((size_t)c * H + r0) * W;
      e = cudaMemcpyAsync(dst + o, src + o, sizeof(float) * (size_t)(r1 - r0) * W, kind, cs);
    }
    return e;
  };
  int f0 = 0, copied = 0;
  for (int i = 0; i < nchunks && rs == BLADE_OK; ++i) {
    Plan p;
    size_t off = 0;
    int nf = 1, r0 = 0, r1 = H;
    if (banded) {
      r0 = (int)((long long)H * i / nchunks);
      r1 = (int)((long long)H * (i + 1) / nchunks);
      plan_rows(h, 1, H, W, r0, r1 - r0, p);
      if (p.ws_bytes > ws_bytes) {
        rs = fail(BLADE_ESHAPE, "band workspace %zu bytes > %zu", p.ws_bytes, ws_bytes);
        break;
      }
      ce = copy_rows(d_in, in_host, copied, std::max(copied, p.z[0].hi), cudaMemcpyHostToDevice, s_in);
      copied = std::max(copied, p.z[0].hi);
    } else {
      nf = (N - f0) / (nchunks - i);
      off = (size_t)f0 * 3 * H * W;
      plan_rows(h, nf, H, W, 0, H, p);
      ce = cudaMemcpyAsync(d_in + off, in_host + off, fbytes * nf, cudaMemcpyHostToDevice, s_in);
    }
    if (ce == cudaSuccess) ce = cudaEventRecord(h->host_ev_in[i], s_in);
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(st, h->host_ev_in[i], 0);
    if (ce != cudaSuccess) {
      rs = fail(BLADE_ECUDA, "H2D: %s", cudaGetErrorString(ce));
      break;
    }
    LevelView inv = make_view(d_in + off, H, W, Range{0, H});
    LevelView outv = make_view(d_out + off, H, W, Range{0, H});
    rs = enqueue(h, p, inv, outv, (char*)ws, st, true, nullptr, nullptr);
    if (rs != BLADE_OK) break;
    ce = cudaEventRecord(h->host_ev_done[i], st);
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(s_out, h->host_ev_done[i], 0);
    if (ce == cudaSuccess)
      ce = banded ? copy_rows(out_host, d_out, r0, r1, cudaMemcpyDeviceToHost, s_out)
                  : cudaMemcpyAsync(out_host + off, d_out + off, fbytes * nf, cudaMemcpyDeviceToHost, s_out);
    if (ce != cudaSuccess) {
      rs = fail(BLADE_ECUDA, "D2H: %s", cudaGetErrorString(ce));
      break;
    }
    f0 += nf;
  }
  ce = cudaStreamSynchronize(s_out);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s_in);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  if (rs == BLADE_OK && ce != cudaSuccess) rs = fail(BLADE_ECUDA, "sync: %s", cudaGetErrorString(ce));
  return rs;
}

}  // extern "C"
