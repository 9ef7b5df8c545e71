// Cycles for 4 warps to hi/lo-split a 20 KB stage (10 float4 per thread:
// LDS.128 -> mask/sub -> STS.128), alone and while one thread keeps bulk
// copies (TMA engine, global -> shared) streaming into another region.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "acct_tc.cuh"
using namespace acct;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(160, 1) split(int iters, int tma, const float *gsrc, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[4];
  __shared__ volatile int stop;
  const uint32_t raw = ptx::smem_u32(sm), lo = raw + 20480, land = raw + 40960;
  const int ct = threadIdx.x;
  for (int i = ct; i < 40960 / 4; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 1.0f + i;
  if (ct == 0) {
    stop = 0;
    for (int b = 0; b < 4; ++b) ptx::mbar_init(&bars[b], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (ct < 128) {
    for (int it = 0; it < iters; ++it) {
      float4 r[10];
#pragma unroll
      for (int i = 0; i < 10; ++i) r[i] = ptx::lds128(raw + 16 * (ct + 128 * i));
#pragma unroll
      for (int i = 0; i < 10; ++i) {
        float4 v = r[i], h;
        h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
        h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
        h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
        h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
        ptx::sts128(lo + 16 * (ct + 128 * i), make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w));
      }
      ptx::fence_proxy_async_smem();
      asm volatile("bar.sync 1, 128;");
    }
    long long t1 = clock64();
    if (ct == 0) {
      if (blockIdx.x == 0) out[0] = t1 - t0;
      stop = 1;
    }
  } else if (ct == 128 && tma) {
    // 4 x 32 KB bulk copies in flight, refilled as they land
    const char *src = reinterpret_cast<const char *>(gsrc) + (size_t)blockIdx.x * (1 << 20);
    uint32_t phase[4] = {0, 0, 0, 0};
    long long n = 0;
    for (int b = 0; b < 4; ++b) {
      ptx::mbar_expect_tx(&bars[b], 32768);
      bulk_g2s(land + b * 32768, src + (n++ % 32) * 32768, 32768, &bars[b]);
    }
    while (!stop) {
      for (int b = 0; b < 4 && !stop; ++b) {
        ptx::mbar_wait(&bars[b], phase[b]);
        phase[b] ^= 1;
        ptx::mbar_expect_tx(&bars[b], 32768);
        bulk_g2s(land + b * 32768, src + (n++ % 32) * 32768, 32768, &bars[b]);
      }
    }
    for (int b = 0; b < 4; ++b) ptx::mbar_wait(&bars[b], phase[b]);
    if (blockIdx.x == 0) out[1] = n;
  }
  __syncthreads();
}

int main() {
  long long *d, h[2];
  float *g;
  cudaMalloc(&d, 16);
  cudaMalloc(&g, (size_t)148 << 20);
  cudaMemset(g, 0, (size_t)148 << 20);
  const int smem = 40960 + 4 * 32768 + 1024;
  cudaFuncSetAttribute(split, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int tma = 0; tma < 2; ++tma) {
    cudaMemset(d, 0, 16);
    split<<<148, 160, smem>>>(2000, tma, g, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("tma=%d: %.1f cycles per 20 KB split; TMA landed %.1f KB per split\n", tma, h[0] / 2000.0,
           h[1] * 32.0 / 2000.0);
  }
  return 0;
}
