// Host-only check (nvcc, no GPU): bucket32_fast (reflection form) against the rotation form of
// the FAST selector that it replaced, on random and adversarial window sums. Certified pixels of
// both forms must get the same orientation bin; strength / coherence may differ only within the
// parity window of a threshold. Build: nvcc -std=c++17 -I paper_1802_06130_b200/csrc
//   scripts/probes/bucket_fast_check.cu -o /tmp/bfc && /tmp/bfc
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <random>

#include "k_down.cuh"

using namespace blade;

// the round-1 rotation form (k_down.cuh before the reflection rewrite), host copy
static int bucket_rot(float a, float b, float c, const float* ts2, const float* kc2, int tc_nonpos, bool& safe, int& orient) {
  const float T = a + c, Df = a - c;
  const float h = 0.125f * T;
  const float q = 0.0625f * fmaf(0.25f * Df, Df, b * b);
  const float bound = kCert * T;
  const float X = -Df, Y = -2.0f * b;
  const bool zero = Df == 0.0f && b == 0.0f;
  const bool lower = Y < 0.0f || (Y == 0.0f && X < 0.0f);
  const float X1 = lower ? -X : X, Y1 = lower ? -Y : Y;
  const bool left = X1 <= 0.0f;
  const float xr = left ? Y1 : X1, yr = left ? -X1 : Y1;
  constexpr float c1 = 0.92387953251128674f, s1 = 0.38268343236508978f, c2 = 0.70710678118654752f;
  const float e1 = fmaf(c1, yr, -s1 * xr), e2 = fmaf(c2, yr, -c2 * xr), e3 = fmaf(s1, yr, -c1 * xr);
  int o = (lower ? 8 : 0) + (left ? 4 : 0) + (e1 >= 0.0f) + (e2 >= 0.0f) + (e3 >= 0.0f);
  const float mn = fminf(fminf(fabsf(X), fabsf(Y)), fminf(fabsf(e1), fminf(fabsf(e2), fabsf(e3))));
  o = zero ? 0 : o;
  orient = o;
  safe = zero ? !(T > 0.0f) : (mn > bound);
  const float h2 = h * h;
  int s = 0, k = 0;
  for (int t = 0; t < 2; ++t) {
    const float d = ts2[t] - h;
    s += (d <= 0.0f) || (q >= d * d);
  }
  for (int t = 0; t < 2; ++t) k += (q >= kc2[t] * h2);
  k = tc_nonpos + (h > 0.0f ? k : 0);
  return (o * 3 + s) * 3 + k;
}

int main(int argc, char** argv) {
  const long iters = argc > 1 ? atol(argv[1]) : 20000000;
  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  const double tS[2] = {0.08075755089521408, 0.1473740190267563}, tC[2] = {0.07864788919687271, 0.14669400453567505};
  float ts2[2], kc2[2], tsR[2], kcR[2];
  for (int i = 0; i < 2; ++i) {
    ts2[i] = (float)(tS[i] * tS[i]);
    tsR[i] = (float)(8.0 * tS[i] * tS[i]);
    const double kap = 2.0 * tC[i] / (1.0 + tC[i] * tC[i]);
    kc2[i] = (float)(kap * kap);
    kcR[i] = (float)kap;
  }
  long n = 0, cert_both = 0, cert_rot = 0, cert_new = 0, o_mis = 0, s_mis = 0, k_mis = 0, zeros = 0;
  auto run = [&](float a, float b, float c) {
    bool sr, sn;
    int orot;
    const int br = bucket_rot(a, b, c, ts2, kc2, 0, sr, orot);
    const int bn = bucket32_fast(a, b, c, tsR, kcR, 0, sn);
    ++n;
    cert_rot += sr;
    cert_new += sn;
    if (sr && sn) {
      ++cert_both;
      if (br / 9 != bn / 9) {
        if (o_mis < 10) printf("orient mismatch a=%a b=%a c=%a rot=%d new=%d\n", a, b, c, br / 9, bn / 9);
        ++o_mis;
      }
    }
    if (sr != sn && a + c == 0.0f) ++zeros;
    s_mis += (br / 3) % 3 != (bn / 3) % 3;
    k_mis += br % 3 != bn % 3;
  };
  for (long i = 0; i < iters; ++i) {
    // a, c >= 0, b^2 <= a c (a Gram matrix); magnitudes over many decades
    const double sc = std::pow(10.0, -8.0 + 10.0 * U(rng));
    const double a = sc * U(rng), c = sc * U(rng);
    const double r = 2.0 * U(rng) - 1.0;
    const double b = r * std::sqrt(a * c);
    run((float)a, (float)b, (float)c);
    // near the bin edges: angle psi = j pi / 8 + tiny
    const double psi = (int)(16 * U(rng)) * M_PI / 8.0 + (U(rng) - 0.5) * 1e-5;
    const double R = sc * U(rng), Tt = R * (1.0 + 3.0 * U(rng));
    const double X = R * std::cos(psi), Y = R * std::sin(psi);  // X = c - a, Y = -2b
    run((float)((Tt - X) / 2), (float)(-Y / 2), (float)((Tt + X) / 2));
  }
  // exact special cases
  const float sp[] = {0.0f, 1.0f, 0.5f, 1e-30f, 3.0f};
  for (float a : sp)
    for (float c : sp)
      for (float b : {0.0f, -0.0f, 0.25f, -0.25f, 1e-31f})
        if ((double)b * b <= (double)a * c) run(a, b, c);
  printf("n=%ld certified rot=%ld new=%ld both=%ld | orient mismatches among both-certified: %ld | "
         "strength diffs %ld coherence diffs %ld | zero-trace cert diffs %ld\n",
         n, cert_rot, cert_new, cert_both, o_mis, s_mis, k_mis, zeros);
  return o_mis != 0;
}
