// Standalone probe: 3D TMA tile load (grid_constant tensormap vs global tensormap) on sm_100a.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1802_06130_b200/csrc/k_stage_tma.cuh"
using namespace blade;

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, float* out, int bw, int bh, int bd, int x0, int y0, int z0) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar, bw * bh * bd * 4);
    tma_load_3d(sm, &tm, x0, y0, z0, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  const float* s = reinterpret_cast<const float*>(sm);
  for (int i = threadIdx.x; i < bw * bh * bd; i += blockDim.x) out[i] = s[i];
}

__global__ void k_probe2(const __grid_constant__ CUtensorMap tm, float* out, int bw, int bh, int bd, int x0, int y0, int z0) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, bw * bh * bd * 4);
    tma_load_3d(sm, &tm, x0, y0, z0, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  const float* s = reinterpret_cast<const float*>(sm);
  for (int i = threadIdx.x; i < bw * bh * bd; i += blockDim.x) out[i] = s[i];
}

__global__ void k_probe_noinit_fence(const __grid_constant__ CUtensorMap tm, float* out, int bw, int bh, int bd) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, bw * bh * bd * 4);
    tma_load_3d(sm, &tm, 0, 0, 0, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  const float* s = reinterpret_cast<const float*>(sm);
  for (int i = threadIdx.x; i < bw * bh * bd; i += blockDim.x) out[i] = s[i];
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int W = 64, R = 40, D = 6;
  std::vector<float> h(W * R * D);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  const int bw = 36, bh = 12, bd = 3;
  cuuint64_t dims[3] = {W, R, D};
  cuuint64_t str[2] = {W * 4, W * 4 * R};
  cuuint32_t box[3] = {bw, bh, bd}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(k_probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  cudaFuncSetAttribute(k_probe_noinit_fence, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  k_probe_noinit_fence<<<1, 128, 65536 + 64>>>(tm, o, bw, bh, bd);
  cudaError_t e = cudaDeviceSynchronize();
  printf("probe(proxy fence) %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  {
    int cs[8][3] = {{0,0,1},{4,0,0},{2,0,0},{0,3,0},{0,-3,0},{-4,0,0},{-2,0,0},{-2,-3,1}};
    for (int i = 0; i < 8; ++i) {
      k_probe2<<<1, 128, 65536 + 64>>>(tm, o, bw, bh, bd, cs[i][0], cs[i][1], cs[i][2]);
      e = cudaDeviceSynchronize();
      printf("coords (%d,%d,%d): %s\n", cs[i][0], cs[i][1], cs[i][2], cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  }
  if (e != cudaSuccess) return 1;
  std::vector<float> got(bw * bh * bd);
  cudaMemcpy(got.data(), o, got.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  {
    k_probe<<<1, 128, 65536 + 64>>>(tm, o, bw, bh, bd, 0, 0, 0);
    cudaError_t e2 = cudaDeviceSynchronize();
    printf("probe(mbarrier_init fence, 0 coords) %s\n", cudaGetErrorString(e2));
  }
  for (int z = 0; z < bd; ++z)
    for (int y = 0; y < bh; ++y)
      for (int x = 0; x < bw; ++x) {
        int gx = x - 2, gy = y - 3, gz = z + 1;
        float ref = (gx < 0 || gy < 0 || gx >= W || gy >= R) ? 0.0f : h[(gz * R + gy) * W + gx];
        if (got[(z * bh + y) * bw + x] != ref) ++bad;
      }
  printf("bad %d of %d\n", bad, bw * bh * bd);
  return 0;
}
