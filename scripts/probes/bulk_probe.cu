// Probe: time to stage a 120 KB constant block (the 5x5-pair stage bank) into shared memory, one
// CTA per SM, the block L2-resident: one cp.async.bulk, 8 / 32 bulk copies from one thread, or
// 16-B cp.async (LDGSTS) by all 256 threads. Prints the kernel time (CUDA events, median of 20).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE, int NCH>
__global__ void __launch_bounds__(256) k(const float* __restrict__ bank, int bytes, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (MODE == 0) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
      const int ch = bytes / NCH;
      for (int c = 0; c < NCH; ++c)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + c * ch)),
                     "l"((const char*)bank + c * ch), "r"(ch), "r"(su(&bar)) : "memory");
    }
    __syncthreads();
    asm volatile("{\n\t.reg .pred P1;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su(&bar)) : "memory");
  } else {
    for (int o = threadIdx.x * 16; o < bytes; o += 256 * 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(sm + o)), "l"((const char*)bank + o) : "memory");
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }
  uint64_t t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) out[blockIdx.x] = (float)(t1 - t0) + 0.0f * reinterpret_cast<float*>(sm)[blockIdx.x % 1000];
}
template <int MODE, int NCH>
float run(const float* bank, int bytes, float* out, int grid) {
  auto f = k<MODE, NCH>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> t;
  for (int i = 0; i < 25; ++i) {
    cudaEventRecord(a); f<<<grid, 256, bytes>>>(bank, bytes, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); (void)ms;
    std::vector<float> h(grid); cudaMemcpy(h.data(), out, 4 * grid, cudaMemcpyDeviceToHost);
    if (i >= 5) t.push_back(*std::max_element(h.begin(), h.end()) / 1000.f);  // in-kernel us, slowest CTA
  }
  std::sort(t.begin(), t.end()); return t[t.size() / 2];
}
int main() {
  const int bytes = 119808;
  float *bank, *out; cudaMalloc(&bank, bytes); cudaMalloc(&out, 4096); cudaMemset(bank, 0, bytes);
  for (int grid : {1, 32, 148}) {
    printf("grid %3d: bulk x1 %.2f us | bulk x8 %.2f us | bulk x32 %.2f us | ldgsts %.2f us | empty-ish (bulk 16 KB) %.2f us\n", grid,
           run<0, 1>(bank, bytes, out, grid), run<0, 8>(bank, bytes, out, grid), run<0, 32>(bank, bytes, out, grid),
           run<1, 1>(bank, bytes, out, grid), run<0, 1>(bank, 16384, out, grid));
  }
  return 0;
}
