// Probe: per-launch cost inside a CUDA graph of 5 dependent launches of an (almost) empty
// kernel, by launch property: dynamic shared memory (0 / 200 KB), programmatic dependent launch,
// kernel parameter size (16 B / 640 B), grid (1 / 148 CTAs). Median graph replay time, us.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
struct Big { char c[640]; };
__global__ void k_small(float* o) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && o) o[blockIdx.x] += 1.f;
}
__global__ void k_big(const __grid_constant__ Big b, float* o) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && o) o[blockIdx.x] += b.c[blockIdx.x % 640];
}
template <typename F, typename... A>
void launch(F f, int grid, size_t smem, bool pdl, cudaStream_t s, A... a) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid; lc.blockDim = 256; lc.dynamicSmemBytes = smem; lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at; lc.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&lc, f, a...);
}
float time_graph(int nk, int grid, size_t smem, bool pdl, bool big, float* o) {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g; cudaGraphExec_t ge;
  Big b{};
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < nk; ++i) {
    if (big) launch(k_big, grid, smem, pdl, s, b, o); else launch(k_small, grid, smem, pdl, s, o);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t e[31]; for (auto& x : e) cudaEventCreate(&x);
  for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(e[0], s);
  for (int i = 0; i < 30; ++i) { cudaGraphLaunch(ge, s); cudaEventRecord(e[i + 1], s); }
  cudaStreamSynchronize(s);
  std::vector<float> t;
  for (int i = 0; i < 30; ++i) { float ms; cudaEventElapsedTime(&ms, e[i], e[i + 1]); t.push_back(ms * 1000.f); }
  std::sort(t.begin(), t.end());
  return t[15];
}
int main() {
  float* o; cudaMalloc(&o, 4096);
  cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int grid : {1, 148})
    for (int big : {0, 1})
      for (int pdl : {0, 1})
        for (size_t smem : {(size_t)0, (size_t)200 * 1024})
          printf("grid %3d params %s pdl %d smem %6zu: 5 launches %.2f us, 1 launch %.2f us\n", grid, big ? "640B" : " 16B", pdl, smem,
                 time_graph(5, grid, smem, pdl, big, o), time_graph(1, grid, smem, pdl, big, o));
  return 0;
}
