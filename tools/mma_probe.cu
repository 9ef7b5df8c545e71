// tcgen05.mma issue-rate probe: one CTA per SM, one thread issues `iters`
// MMAs on fixed shared-memory operands (contents irrelevant), commits, waits;
// reports cycles per MMA for kind::tf32 with K-major / MN-major B and several
// N, plus kind::f16 for scale.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include \
//        -I paper_1811_03882_b200/csrc tools/mma_probe.cu -o /tmp/mma_probe -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "acct_tc.cuh"

using namespace acct;

__device__ __forceinline__ int *slot_stop() {
  __shared__ int stop;
  return &stop;
}

template <int KIND>  // 0 = tf32, 1 = f16
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  if (KIND == 0)
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a),
                 "l"(b), "r"(idesc));
  else
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a),
                 "l"(b), "r"(idesc));
}

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ volatile int g_stop;

template <int KIND>
__global__ void __launch_bounds__(256, 1) probe(int N, int b_mn, int iters, long long *out,
                                                 int noise) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<float *>(base)[i] = 0.001f * (i % 7);
  if (threadIdx.x == 0) {
    *slot_stop() = 0;
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(&slot, 256);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a_addr = ptx::smem_u32(base), b_addr = ptx::smem_u32(base + 32 * 1024);
    // A: 128 rows K-major SW128 (8 tf32 = 32 B per k step)
    const uint64_t da = ptx::smem_desc(a_addr, 16, 1024, ptx::kLayoutSW128);
    uint64_t db;
    uint32_t idesc;
    if (KIND == 0) {
      db = b_mn ? ptx::smem_desc(b_addr, 8 * 128 * 4 /*chunk*/, 512, ptx::kLayoutSW128Base32B)
                : ptx::smem_desc(b_addr, 16, 1024, ptx::kLayoutSW128);
      idesc = ptx::idesc_tf32(128, N, false, b_mn != 0);
    } else {
      db = ptx::smem_desc(b_addr, 16, 1024, ptx::kLayoutSW128);
      idesc = idesc_f16(128, N, false, false);
    }
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) mma<KIND>(tmem, da, db, idesc);
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    *reinterpret_cast<volatile int *>(slot_stop()) = 1;
  } else if (noise && warp >= 4) {
    // LSU shared-memory traffic like the hi/lo converter: read 16 B, write 16 B
    float4 *src = reinterpret_cast<float4 *>(base + 64 * 1024);
    float4 *dst = reinterpret_cast<float4 *>(base + 80 * 1024);
    const int t = threadIdx.x - 128;
    while (!*reinterpret_cast<volatile int *>(slot_stop())) {
#pragma unroll 4
      for (int v = t; v < 1024; v += 128) {
        float4 x = src[v];
        x.x += 1.0f;
        dst[v] = x;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 256);
}

int main() {
  long long *d_out, h;
  cudaMalloc(&d_out, sizeof(long long));
  const int smem = 100 * 1024;
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  for (int noise = 0; noise < 2; ++noise)
  for (int kind = 0; kind < 2; ++kind) {
    for (int b_mn = 0; b_mn < (kind == 0 ? 2 : 1); ++b_mn) {
      for (int N : {64, 128, 192, 256}) {
        for (int grid : {148}) {
          if (kind == 0) probe<0><<<grid, 256, smem>>>(N, b_mn, iters, d_out, noise);
          else probe<1><<<grid, 256, smem>>>(N, 0, iters, d_out, noise);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          cudaMemcpy(&h, d_out, sizeof h, cudaMemcpyDeviceToHost);
          const double cyc = (double)h / iters;
          const int kstep = kind == 0 ? 8 : 16;
          const double macs = 128.0 * N * kstep;
          printf("%s B=%s N=%3d grid=%3d noise=%d: %7.1f cyc/mma  %7.1f MAC/cyc/SM\n",
                 kind == 0 ? "tf32" : "f16 ", b_mn ? "MN" : "K ", N, grid, noise, cyc, macs / cyc);
        }
      }
    }
  }
  return 0;
}
