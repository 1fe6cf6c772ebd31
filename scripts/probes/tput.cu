// Throughput probe (B200): DFMA, FFMA, F2F.F64.F32, SHFL per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, int iters, float seed) {
  float a0 = seed + threadIdx.x, a1 = a0 * 1.1f, a2 = a0 * 1.2f, a3 = a0 * 1.3f;
  double d0 = a0, d1 = a1, d2 = a2, d3 = a3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) { d0 = fma(d0, 1.0000001, 0.5); d1 = fma(d1, 1.0000001, 0.5); d2 = fma(d2, 1.0000001, 0.5); d3 = fma(d3, 1.0000001, 0.5); }
      if (OP == 1) { a0 = fmaf(a0, 1.0001f, 0.5f); a1 = fmaf(a1, 1.0001f, 0.5f); a2 = fmaf(a2, 1.0001f, 0.5f); a3 = fmaf(a3, 1.0001f, 0.5f); }
      if (OP == 2) { d0 += (double)a0; d1 += (double)a1; d2 += (double)a2; d3 += (double)a3; a0 += 1.0f; a1 += 1.0f; a2 += 1.0f; a3 += 1.0f; }
      if (OP == 3) { a0 = __shfl_xor_sync(0xffffffff, a0, 1); a1 = __shfl_xor_sync(0xffffffff, a1, 2); a2 = __shfl_xor_sync(0xffffffff, a2, 3); a3 = __shfl_xor_sync(0xffffffff, a3, 4); }
      if (OP == 4) { a0 = (float)d0; a1 = (float)d1; a2 = (float)d2; a3 = (float)d3; d0 += 1.0; d1 += 1.0; d2 += 1.0; d3 += 1.0; }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[2 + (blockIdx.x * blockDim.x + threadIdx.x) % 64] = a0 + a1 + a2 + a3 + (float)(d0 + d1 + d2 + d3);
}
int main() {
  float* out; cudaMalloc(&out, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"DFMA", "FFMA", "F2F.F64.F32 (+FADD)", "SHFL", "F2F.F32.F64 (+DADD)"};
  for (int op = 0; op < 5; ++op) {
    int iters = 4096;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto launch = [&]() {
      switch (op) { case 0: k<0><<<sms * 4, 512>>>(out, iters, 1.f); break; case 1: k<1><<<sms * 4, 512>>>(out, iters, 1.f); break;
        case 2: k<2><<<sms * 4, 512>>>(out, iters, 1.f); break; case 3: k<3><<<sms * 4, 512>>>(out, iters, 1.f); break; case 4: k<4><<<sms * 4, 512>>>(out, iters, 1.f); break; }
    };
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 4 * 512 * iters * 16 * 4;  // lane-ops of the probed kind
    printf("%-22s %8.1f lane-ops/clk/SM at nominal %d MHz (%.3f ms)\n", names[op], ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000, ms);
  }
  return 0;
}
