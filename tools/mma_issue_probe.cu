// tcgen05.mma issuers probe: is a narrow (N = 32/64) kind::tf32 MMA bound by
// one thread's issue rate or by the SM's tensor core?  One CTA per SM; 1 or 2
// warps each issue `iters` MMAs (A from TMEM as in the conv kernels, B K-major
// from shared memory) into their own TMEM accumulator; reports cycles per MMA
// per issuer and the SM's aggregate MMAs per 1000 cycles.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include \
//        -I paper_1811_03882_b200/csrc tools/mma_issue_probe.cu -o /tmp/mip && /tmp/mip
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "acct_tc.cuh"

using namespace acct;

__global__ void __launch_bounds__(128, 1) probe(int N, int issuers, int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<float *>(base)[i] = 0.001f * (i % 7);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (warp < issuers && lane == 0) {
    const uint64_t db = ptx::smem_desc(ptx::smem_u32(base), 16, 1024, ptx::kLayoutSW128);
    const uint32_t idesc = ptx::idesc_tf32(128, N, false, false);
    const uint32_t d = tmem + warp * 64, a = tmem + 256 + warp * 32;  // N <= 64 for 4 issuers
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) ptx::mma_tf32_ts(d, a + 8 * (i & 3), db, idesc, 1);
    ptx::mma_commit(&bar[warp]);
    ptx::mbar_wait(&bar[warp], 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[warp] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
  long long *d_out, h[4];
  cudaMalloc(&d_out, 4 * sizeof(long long));
  const int smem = 70 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  for (int N : {32, 64})
    for (int issuers : {1, 2, 3, 4}) {
      cudaMemset(d_out, 0, 4 * sizeof(long long));
      probe<<<148, 128, smem>>>(N, issuers, iters, d_out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int w = 0; w < issuers; ++w) mx = h[w] > mx ? h[w] : mx;
      printf("N=%3d issuers=%d: %6.1f cyc/mma per issuer, %6.1f MMAs per 1000 cyc per SM\n", N,
             issuers, (double)mx / iters, 1000.0 * issuers * iters / mx);
    }
  return 0;
}
