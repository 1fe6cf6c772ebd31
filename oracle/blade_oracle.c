/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU evaluation of the inference path of multiscale BLADE
 * (arxiv 1802.06130). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no
 * code, header, table or constant generator with the CUDA path
 * (paper_1802_06130_b200/csrc) and neither side includes the other.
 *
 * Every function follows the paper's definition step by step in its order and
 * notation; no blocking, fusion or reordering. Readings of points the paper
 * leaves open are the DESIGN.md readings R1..R24 (cited as [Rn]).
 *
 * Conventions: images are planar z[c][y][x] (row y down, column x right),
 * double precision throughout; the input fp32 samples are widened by the
 * Python wrapper before the call.
 *
 * Parallelism: OpenMP over output rows only; every output value is computed
 * by one thread from read-only inputs, so results do not depend on the thread
 * count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_PI 3.14159265358979323846

/* [R2] half-sample symmetric border, periodic with period 2n for any offset:
 * numpy.pad(mode='symmetric') / scipy.ndimage mode='reflect'. */
int64_t oracle_fold(int64_t i, int64_t n) {
  int64_t p = 2 * n;
  int64_t m = i % p;
  if (m < 0) m += p;
  return m < n ? m : p - 1 - m;
}

/* Z(c, y, x): the folded image every derived field is computed from [R2]. */
static inline double Zat(const double* z, int64_t H, int64_t W, int64_t c, int64_t y, int64_t x) {
  return z[(c * H + oracle_fold(y, H)) * W + oracle_fold(x, W)];
}

/* ------------------------------------------------------------------------
 * O1 pyramid decimation, "standard bicubic downsampling ... by factors of two"
 * (§4 Multiscale filtering) with the anti-aliased
 * Catmull-Rom (Keys a=-0.5) kernel at doubled support [R14]:
 *   z^{l+1}(c,y,x) = sum_{a=0..7} sum_{b=0..7} w_a w_b Z^l(c, 2y-3+a, 2x-3+b),
 *   w_a = k(|t_a|/2) / sum, t_a = a - 3.5, k = Keys cubic, a = -0.5.
 * Output dims ceil(H/2) x ceil(W/2).
 * ---------------------------------------------------------------------- */
static double keys_cubic(double t) {
  const double A = -0.5;
  t = fabs(t);
  if (t < 1.0) return ((A + 2.0) * t - (A + 3.0)) * t * t + 1.0;
  if (t < 2.0) return ((A * t - 5.0 * A) * t + 8.0 * A) * t - 4.0 * A;
  return 0.0;
}

void oracle_decimate_weights(double w[8]) {
  double s = 0.0;
  for (int a = 0; a < 8; ++a) {
    w[a] = keys_cubic(((double)a - 3.5) / 2.0);
    s += w[a];
  }
  for (int a = 0; a < 8; ++a) w[a] /= s;
}

void oracle_decimate(const double* z, int64_t C, int64_t H, int64_t W, double* out) {
  const int64_t H1 = (H + 1) / 2, W1 = (W + 1) / 2;
  double w[8];
  oracle_decimate_weights(w);
#pragma omp parallel for schedule(static)
  for (int64_t y = 0; y < H1; ++y)
    for (int64_t c = 0; c < C; ++c)
      for (int64_t x = 0; x < W1; ++x) {
        double acc = 0.0;
        for (int a = 0; a < 8; ++a)
          for (int b = 0; b < 8; ++b)
            acc += w[a] * w[b] * Zat(z, H, W, c, 2 * y - 3 + a, 2 * x - 3 + b);
        out[(c * H1 + y) * W1 + x] = acc;
      }
}

/* ------------------------------------------------------------------------
 * O2 structure tensor, Eq. 6 (§3 Filter selection):
 *   T_i = sum_c sum_j w_j^i [gx^2  gx gy; gx gy  gy^2]
 * [R3] gradients: central differences of the folded image,
 *   gx = (Z(c,y,x+1) - Z(c,y,x-1))/2, gy = (Z(c,y+1,x) - Z(c,y-1,x))/2;
 * [R4] window: window_size x window_size Gaussian, std window_sigma,
 *   w(dy,dx) = e(dy) e(dx) / (sum e)^2, e(d) = exp(-d^2 / (2 sigma^2)).
 * Output a = T_xx, b = T_xy, c = T_yy per pixel.
 * ---------------------------------------------------------------------- */
void oracle_tensor(const double* z, int64_t C, int64_t H, int64_t W, int ws, double wsigma,
                   double* ta, double* tb, double* tc) {
  const int r = ws / 2;
  double* e = (double*)malloc(sizeof(double) * (size_t)ws);
  double se = 0.0;
  for (int d = -r; d <= r; ++d) {
    e[d + r] = exp(-(double)(d * d) / (2.0 * wsigma * wsigma));
    se += e[d + r];
  }
#pragma omp parallel for schedule(static)
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) {
      double a = 0.0, b = 0.0, cc = 0.0;
      for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx) {
          const double wj = e[dy + r] * e[dx + r] / (se * se);
          const int64_t yj = y + dy, xj = x + dx;
          for (int64_t c = 0; c < C; ++c) {
            const double gx = (Zat(z, H, W, c, yj, xj + 1) - Zat(z, H, W, c, yj, xj - 1)) / 2.0;
            const double gy = (Zat(z, H, W, c, yj + 1, xj) - Zat(z, H, W, c, yj - 1, xj)) / 2.0;
            a += wj * gx * gx;
            b += wj * gx * gy;
            cc += wj * gy * gy;
          }
        }
      ta[y * W + x] = a;
      tb[y * W + x] = b;
      tc[y * W + x] = cc;
    }
  free(e);
}

/* ------------------------------------------------------------------------
 * Eigen-features of T = [a b; b c]:
 *   lambda_1 >= lambda_2 (closed-form 2x2), lambda_2 clamped at 0;
 *   strength  S = sqrt(lambda_1);
 *   coherence C = (sqrt l1 - sqrt l2)/(sqrt l1 + sqrt l2), 0 when l1 = 0 [R6];
 *   orientation = angle of the eigenvector of the SMALLEST eigenvalue, in
 *   [0, pi) (x right, y down); 0 when a == c and b == 0 [R5].
 * ---------------------------------------------------------------------- */
void oracle_eigen(const double* ta, const double* tb, const double* tc, int64_t n, double* theta,
                  double* strength, double* coherence) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double a = ta[i], b = tb[i], c = tc[i];
    const double half_tr = (a + c) / 2.0;
    const double r = sqrt(((a - c) / 2.0) * ((a - c) / 2.0) + b * b);
    const double l1 = half_tr + r;
    double l2 = half_tr - r;
    if (l2 < 0.0) l2 = 0.0;
    const double s1 = sqrt(l1 > 0.0 ? l1 : 0.0), s2 = sqrt(l2);
    strength[i] = s1;
    coherence[i] = l1 > 0.0 ? (s1 - s2) / (s1 + s2) : 0.0;
    double th = 0.0;
    if (!(a == c && b == 0.0)) {
      /* major eigenvector at angle 0.5*atan2(2b, a-c); minor = major + pi/2 */
      th = 0.5 * atan2(2.0 * b, a - c) + OR_PI / 2.0;
      while (th >= OR_PI) th -= OR_PI;
      while (th < 0.0) th += OR_PI;
    }
    theta[i] = th;
  }
}

/* ------------------------------------------------------------------------
 * Quantisation to a bucket s(i) (rule [R7], thresholds [R8]):
 *   o = floor(theta * n_o / pi) mod n_o;
 *   s = #{t in Ts : t <= S};  k = #{t in Tc : t <= C};
 *   bucket = (o * n_s + s) * n_c + k.
 * ---------------------------------------------------------------------- */
void oracle_quantize(const double* theta, const double* strength, const double* coherence, int64_t n,
                     int n_o, int n_s, int n_c, const double* ts, const double* tc, int32_t* bucket) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t o = (int64_t)floor(theta[i] * (double)n_o / OR_PI);
    o %= n_o;
    if (o < 0) o += n_o;
    int s = 0, k = 0;
    for (int t = 0; t < n_s - 1; ++t) s += (ts[t] <= strength[i]);
    for (int t = 0; t < n_c - 1; ++t) k += (tc[t] <= coherence[i]);
    bucket[i] = (int32_t)((o * n_s + s) * n_c + k);
  }
}

/* Selector s(i) at one level: tensor -> eigen-features -> bucket. */
int oracle_selector(const double* z, int64_t C, int64_t H, int64_t W, int ws, double wsigma, int n_o,
                    int n_s, int n_c, const double* ts, const double* tc, int32_t* bucket,
                    double* theta_out, double* strength_out, double* coherence_out) {
  const int64_t n = H * W;
  double* buf = (double*)malloc(sizeof(double) * (size_t)n * 6);
  if (!buf) return 2;
  double *a = buf, *b = buf + n, *c = buf + 2 * n, *th = buf + 3 * n, *S = buf + 4 * n, *Co = buf + 5 * n;
  oracle_tensor(z, C, H, W, ws, wsigma, a, b, c);
  oracle_eigen(a, b, c, n, th, S, Co);
  oracle_quantize(th, S, Co, n, n_o, n_s, n_c, ts, tc, bucket);
  if (theta_out) memcpy(theta_out, th, sizeof(double) * (size_t)n);
  if (strength_out) memcpy(strength_out, S, sizeof(double) * (size_t)n);
  if (coherence_out) memcpy(coherence_out, Co, sizeof(double) * (size_t)n);
  free(buf);
  return 0;
}

/* ------------------------------------------------------------------------
 * O3 one stage at level l, Eq. 9 (§4 Multiscale filtering):
 *   u^l_i = sum_{j in F_c} f^{l,s(i)}_j u^{l+1}_{i/2+j} + sum_{j in F_f} g^{l,s(i)}_j z^l_{i+j}
 * with i/2 = (floor(y/2), floor(x/2)) and the pair (f, g) indexed by the 2x2
 * output phase p = 2(y mod 2) + (x mod 2) when n_phases == 4 [R9]; one filter
 * for R, G and B [R13]; correlation orientation "z_{i+j}" (Eq. 1).
 * taps layout: [phase][bucket][ fine nf*nf | coarse nc*nc ], row-major from
 * (-r, -r) [R12]. With nc == 0 (or u1 == NULL) this is Eq. 1.
 * ---------------------------------------------------------------------- */
void oracle_stage(const double* z, int64_t C, int64_t H, int64_t W, const double* u1, int64_t H1,
                  int64_t W1, const int32_t* bucket, const double* taps, int n_phases, int K, int nf,
                  int nc, double* out) {
  const int rf = nf / 2, rc = nc / 2;
  const int64_t nt = (int64_t)nf * nf + (int64_t)nc * nc;
  (void)K;
#pragma omp parallel for schedule(static)
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) {
      const int p = n_phases == 4 ? (int)(2 * (y % 2) + (x % 2)) : 0;
      const int64_t k = bucket[y * W + x];
      const double* g = taps + ((int64_t)p * K + k) * nt;
      const double* f = g + (int64_t)nf * nf;
      for (int64_t c = 0; c < C; ++c) {
        double acc = 0.0;
        if (nc > 0 && u1 != NULL) {
          for (int dy = -rc; dy <= rc; ++dy)
            for (int dx = -rc; dx <= rc; ++dx)
              acc += f[(dy + rc) * nc + (dx + rc)] * Zat(u1, H1, W1, c, y / 2 + dy, x / 2 + dx);
        }
        for (int dy = -rf; dy <= rf; ++dy)
          for (int dx = -rf; dx <= rf; ++dx)
            acc += g[(dy + rf) * nf + (dx + rf)] * Zat(z, H, W, c, y + dy, x + dx);
        out[(c * H + y) * W + x] = acc;
      }
    }
}

/* ------------------------------------------------------------------------
 * a4 the cascade for ONE frame:
 *   z^0 = input; z^{l+1} = decimate(z^l) for l = 0..L-2;
 *   u^{L-1} = z^{L-1} (base case "u^L = z^L");
 *   for l = L-2 .. 0: s^l = selector(z^l), u^l = stage(z^l, u^{l+1}, s^l).
 *   L == 1: u^0 = Eq. 1 with the stage-0 fine taps.
 * taps: [stage][phase][bucket][nf^2 + nc^2]; ts/tc: [stage][n_s-1], [stage][n_c-1].
 * ---------------------------------------------------------------------- */
int oracle_denoise(const double* z0, int64_t H, int64_t W, int L, int nf, int nc, int n_phases, int n_o,
                   int n_s, int n_c, const double* ts, const double* tc, const double* taps, int ws,
                   double wsigma, double* out) {
  const int64_t C = 3;
  const int K = n_o * n_s * n_c;
  if (L < 1) return 1;
  double** zl = (double**)calloc((size_t)L, sizeof(double*));
  int64_t* Hl = (int64_t*)calloc((size_t)L, sizeof(int64_t));
  int64_t* Wl = (int64_t*)calloc((size_t)L, sizeof(int64_t));
  if (!zl || !Hl || !Wl) return 2;
  zl[0] = (double*)z0;
  Hl[0] = H;
  Wl[0] = W;
  for (int l = 0; l + 1 < L; ++l) {
    Hl[l + 1] = (Hl[l] + 1) / 2;
    Wl[l + 1] = (Wl[l] + 1) / 2;
    zl[l + 1] = (double*)malloc(sizeof(double) * (size_t)(C * Hl[l + 1] * Wl[l + 1]));
    oracle_decimate(zl[l], C, Hl[l], Wl[l], zl[l + 1]);
  }
  int32_t* bucket = (int32_t*)malloc(sizeof(int32_t) * (size_t)(H * W));
  const int64_t nt = (int64_t)nf * nf + (L > 1 ? (int64_t)nc * nc : 0);
  if (L == 1) {
    oracle_selector(z0, C, H, W, ws, wsigma, n_o, n_s, n_c, ts, tc, bucket, NULL, NULL, NULL);
    oracle_stage(z0, C, H, W, NULL, 0, 0, bucket, taps, n_phases, K, nf, 0, out);
  } else {
    const double* u = zl[L - 1];
    double* owned = NULL;
    for (int l = L - 2; l >= 0; --l) {
      double* ul = l == 0 ? out : (double*)malloc(sizeof(double) * (size_t)(C * Hl[l] * Wl[l]));
      oracle_selector(zl[l], C, Hl[l], Wl[l], ws, wsigma, n_o, n_s, n_c, ts + (int64_t)l * (n_s - 1),
                      tc + (int64_t)l * (n_c - 1), bucket, NULL, NULL, NULL);
      oracle_stage(zl[l], C, Hl[l], Wl[l], u, Hl[l + 1], Wl[l + 1], bucket,
                   taps + (int64_t)l * n_phases * K * nt, n_phases, K, nf, nc, ul);
      free(owned);
      owned = l == 0 ? NULL : ul;
      u = ul;
    }
  }
  free(bucket);
  for (int l = 1; l < L; ++l) free(zl[l]);
  free(zl);
  free(Hl);
  free(Wl);
  return 0;
}
