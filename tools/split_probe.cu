// Cycles for 4 warps to hi/lo-split a 20 KB stage (10 float4 per thread:
// LDS.128 -> mask/sub -> STS.128) in isolation, optionally with a proxy fence.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "acct_tc.cuh"
using namespace acct;

__global__ void __launch_bounds__(128, 1) split(int iters, int fence, int nwarps, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t raw = ptx::smem_u32(sm), lo = raw + 20480;
  const int ct = threadIdx.x;
  for (int i = ct; i < 40960 / 4; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 1.0f + i;
  __syncthreads();
  long long t0 = clock64();
  if (ct < 32 * nwarps) {
    for (int it = 0; it < iters; ++it) {
      float4 r[10];
#pragma unroll
      for (int i = 0; i < 10; ++i) r[i] = ptx::lds128(raw + 16 * ((ct + 128 * i) % 1280));
#pragma unroll
      for (int i = 0; i < 10; ++i) {
        float4 v = r[i], h;
        h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
        h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
        h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
        h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
        ptx::sts128(lo + 16 * ((ct + 128 * i) % 1280), make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w));
      }
      if (fence) ptx::fence_proxy_async_smem();
      __syncwarp();
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (ct == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  long long *d, h;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(split, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  for (int fence = 0; fence < 2; ++fence)
    for (int nw : {4}) {
      split<<<148, 128, 48 * 1024>>>(1000, fence, nw, d);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("fence=%d warps=%d: %.1f cycles per 20 KB stage\n", fence, nw, h / 1000.0);
    }
  return 0;
}
