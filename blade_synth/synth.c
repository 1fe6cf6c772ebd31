/*
 * blade_synth — seeded synthetic INPUT generator shared by the oracle tests,
 * the CUDA parity tests and bench.py.
 *
 * This module holds none of the method's arithmetic (no gradients, tensors,
 * eigen-features, quantisation, decimation or filtering). It only produces:
 *   - piecewise-smooth RGB scenes (oriented sinusoid gratings + hard-edged
 *     disks, clipped to [0,1]) — the stand-in for the paper's Berkeley test
 *     images (§5), recipe in DESIGN.md §"Inputs";
 *   - additive noise: AWGN or the signal-dependent model of
 *     BASELINE.json configs[2] (variance = a*x + b);
 *   - seeded filterbanks (BASELINE.json configs[0]: N(0,1) taps, +4 on the
 *     centre tap, normalised to sum 1; redraw rule = DESIGN.md reading R11).
 *
 * Randomness: SplitMix64. Scene and bank parameters come from sequential
 * streams keyed by (seed, tag, index); noise is counter-based, keyed by
 * (seed, frame, channel, y, x), so any row band or frame is reproducible on
 * its own and the result is independent of the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SYNTH_PI 3.14159265358979323846

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline uint64_t key4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  return mix64(a ^ mix64(b ^ mix64(c ^ mix64(d))));
}

typedef struct { uint64_t s; } sm64;

static inline uint64_t sm_next(sm64* r) {
  r->s += 0x9E3779B97F4A7C15ULL;
  uint64_t z = r->s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* uniform in [0,1) with 53 random bits */
static inline double u01(uint64_t x) { return (double)(x >> 11) * (1.0 / 9007199254740992.0); }
/* uniform in (0,1] */
static inline double u01_open0(uint64_t x) { return ((double)(x >> 11) + 1.0) * (1.0 / 9007199254740992.0); }

static inline double sm_uniform(sm64* r, double lo, double hi) { return lo + (hi - lo) * u01(sm_next(r)); }

/* Box-Muller, cosine branch only (one normal per two uniforms). */
static inline double normal_from(uint64_t a, uint64_t b) {
  return sqrt(-2.0 * log(u01_open0(a))) * cos(2.0 * SYNTH_PI * u01(b));
}
static inline double sm_normal(sm64* r) {
  uint64_t a = sm_next(r);
  uint64_t b = sm_next(r);
  return normal_from(a, b);
}

enum { TAG_SCENE = 0x5343454EULL, TAG_NOISE = 0x4E4F4953ULL, TAG_BANK = 0x42414E4BULL };

/* counter-based standard normal for noise sample (frame, c, y, x) */
static inline double noise_normal(uint64_t seed, int64_t frame, int c, int64_t y, int64_t x) {
  uint64_t k = key4(seed ^ TAG_NOISE, (uint64_t)frame, ((uint64_t)c << 40) ^ (uint64_t)y, (uint64_t)x);
  return normal_from(mix64(k), mix64(k ^ 0xD1B54A32D192ED03ULL));
}

typedef struct {
  double ax, ay, phi, amp, col[3];
} grating_t;
typedef struct {
  double cx, cy, r, col[3];
} disk_t;

/*
 * Scene for one frame, rows [row0, row0+rows) of an H x W image (planar RGB,
 * out[c][r][x], r relative to row0). Parameters depend only on (seed, frame,
 * H, W), never on the row window.
 *   noise_kind 0: clean; 1: AWGN, std = p0; 2: var = p0*x + p1 (x = clean).
 * Returns 0 on success.
 */
int synth_scene(uint64_t seed, int64_t frame, int64_t H, int64_t W, int64_t row0, int64_t rows,
                int n_grat, int n_disk, int noise_kind, double p0, double p1, float* out) {
  if (H <= 0 || W <= 0 || rows < 0 || row0 < 0 || row0 + rows > H || n_grat < 0 || n_disk < 0) return 1;
  sm64 r = {key4(seed ^ TAG_SCENE, (uint64_t)frame, (uint64_t)H, (uint64_t)W)};
  grating_t* g = (grating_t*)malloc(sizeof(grating_t) * (size_t)(n_grat > 0 ? n_grat : 1));
  disk_t* d = (disk_t*)malloc(sizeof(disk_t) * (size_t)(n_disk > 0 ? n_disk : 1));
  if (!g || !d) { free(g); free(d); return 2; }
  for (int k = 0; k < n_grat; ++k) {
    double th = sm_uniform(&r, 0.0, SYNTH_PI);
    double f = sm_uniform(&r, 1.0 / 64.0, 1.0 / 6.0);
    g[k].phi = sm_uniform(&r, 0.0, 2.0 * SYNTH_PI);
    g[k].amp = sm_uniform(&r, 0.03, 0.12);
    for (int c = 0; c < 3; ++c) g[k].col[c] = sm_uniform(&r, -1.0, 1.0);
    g[k].ax = 2.0 * SYNTH_PI * f * cos(th);
    g[k].ay = 2.0 * SYNTH_PI * f * sin(th);
  }
  double mn = (double)(H < W ? H : W);
  for (int k = 0; k < n_disk; ++k) {
    d[k].cx = sm_uniform(&r, 0.0, (double)W);
    d[k].cy = sm_uniform(&r, 0.0, (double)H);
    d[k].r = sm_uniform(&r, 0.02, 0.15) * mn;
    for (int c = 0; c < 3; ++c) d[k].col[c] = sm_uniform(&r, 0.0, 1.0);
  }
  /* per-column sin/cos tables: sin(ax*x + ay*y + phi) = sx*cy' + cx*sy' */
  double* sx = (double*)malloc(sizeof(double) * (size_t)W * (size_t)(n_grat > 0 ? n_grat : 1) * 2);
  if (!sx) { free(g); free(d); return 2; }
  double* cxs = sx + (size_t)W * (size_t)(n_grat > 0 ? n_grat : 1);
  for (int k = 0; k < n_grat; ++k)
    for (int64_t x = 0; x < W; ++x) {
      sx[(size_t)k * W + x] = sin(g[k].ax * (double)x);
      cxs[(size_t)k * W + x] = cos(g[k].ax * (double)x);
    }
  const size_t plane = (size_t)rows * (size_t)W;
  int err = 0;
#pragma omp parallel
  {
    double* sy = (double*)malloc(sizeof(double) * (size_t)(n_grat > 0 ? n_grat : 1) * 2);
    int* act = (int*)malloc(sizeof(int) * (size_t)(n_disk > 0 ? n_disk : 1));
    if (!sy || !act) {
#pragma omp atomic write
      err = 2;
    } else {
      double* cy = sy + (n_grat > 0 ? n_grat : 1);
#pragma omp for schedule(static)
      for (int64_t rr = 0; rr < rows; ++rr) {
        const int64_t y = row0 + rr;
        for (int k = 0; k < n_grat; ++k) {
          sy[k] = sin(g[k].ay * (double)y + g[k].phi);
          cy[k] = cos(g[k].ay * (double)y + g[k].phi);
        }
        int na = 0;
        for (int k = 0; k < n_disk; ++k) {
          double dy = (double)y - d[k].cy;
          if (dy * dy <= d[k].r * d[k].r) act[na++] = k;
        }
        for (int64_t x = 0; x < W; ++x) {
          double v[3] = {0.5, 0.5, 0.5};
          for (int k = 0; k < n_grat; ++k) {
            double s = sx[(size_t)k * W + x] * cy[k] + cxs[(size_t)k * W + x] * sy[k];
            for (int c = 0; c < 3; ++c) v[c] += g[k].amp * g[k].col[c] * s;
          }
          /* disks painted in order: the last covering disk wins */
          for (int a = na - 1; a >= 0; --a) {
            const disk_t* dk = &d[act[a]];
            double dx = (double)x - dk->cx, dy = (double)y - dk->cy;
            if (dx * dx + dy * dy <= dk->r * dk->r) {
              v[0] = dk->col[0]; v[1] = dk->col[1]; v[2] = dk->col[2];
              break;
            }
          }
          for (int c = 0; c < 3; ++c) {
            double cl = v[c] < 0.0 ? 0.0 : (v[c] > 1.0 ? 1.0 : v[c]);
            double o = cl;
            if (noise_kind == 1) {
              o = cl + p0 * noise_normal(seed, frame, c, y, x);
            } else if (noise_kind == 2) {
              double var = p0 * cl + p1;
              o = cl + sqrt(var > 0.0 ? var : 0.0) * noise_normal(seed, frame, c, y, x);
            }
            out[(size_t)c * plane + (size_t)rr * W + x] = (float)o;
          }
        }
      }
    }
    free(sy);
    free(act);
  }
  free(sx);
  free(g);
  free(d);
  return err;
}

/* Plain noise plane (no scene): out[c][y][x] = std * N(0,1); used for the
 * decimation noise-factor pin. */
int synth_noise(uint64_t seed, int64_t frame, int64_t C, int64_t H, int64_t W, double std, float* out) {
  if (C <= 0 || H <= 0 || W <= 0) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t y = 0; y < H; ++y)
    for (int64_t c = 0; c < C; ++c)
      for (int64_t x = 0; x < W; ++x)
        out[((size_t)c * H + y) * W + x] = (float)(std * noise_normal(seed, frame, (int)c, y, x));
  return 0;
}

/*
 * Filterbank for one stage: taps[phase][bucket][fine nf*nf | coarse nc*nc]
 * (row-major, tap (dy,dx) at index (dy+r)*n+(dx+r)), fp32.
 * Draw rule (BASELINE.json configs[0] + DESIGN.md reading R11):
 *   fine taps then coarse taps ~ N(0,1) from the stream keyed (seed, stage);
 *   +4 on the centre tap of each block; s = sum of all taps;
 *   if redraw_below > -inf and s < redraw_below: redraw from the same stream;
 *   divide by s (joint normalisation: sum f + sum g = 1) and round to fp32.
 * `redraws` (optional) receives the number of rejected draws.
 */
int synth_bank(uint64_t seed, int stage, int n_phases, int K, int nf, int nc, double redraw_below,
               float* taps, int64_t* redraws) {
  if (n_phases <= 0 || K <= 0 || nf <= 0 || (nf & 1) == 0 || nc < 0 || (nc != 0 && (nc & 1) == 0)) return 1;
  sm64 r = {key4(seed ^ TAG_BANK, (uint64_t)stage, (uint64_t)nf, (uint64_t)nc)};
  const int nt = nf * nf + nc * nc;
  double* v = (double*)malloc(sizeof(double) * (size_t)nt);
  if (!v) return 2;
  int64_t rej = 0;
  for (int p = 0; p < n_phases; ++p)
    for (int k = 0; k < K; ++k) {
      double s;
      for (;;) {
        for (int t = 0; t < nt; ++t) v[t] = sm_normal(&r);
        v[(nf / 2) * nf + nf / 2] += 4.0;
        if (nc > 0) v[nf * nf + (nc / 2) * nc + nc / 2] += 4.0;
        s = 0.0;
        for (int t = 0; t < nt; ++t) s += v[t];
        if (s >= redraw_below && s != 0.0) break;
        ++rej;
      }
      float* o = taps + ((size_t)p * K + k) * nt;
      for (int t = 0; t < nt; ++t) o[t] = (float)(v[t] / s);
    }
  free(v);
  if (redraws) *redraws = rej;
  return 0;
}
