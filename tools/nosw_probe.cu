// No-swizzle K-major tf32 operands from shared memory (tcgen05.mma, both
// operands by descriptor): checks the canonical layout the row-band conv
// uses -- core matrix = 8 rows x 16 B contiguous, 8-row groups SBO apart,
// 16-B K chunks LBO apart -- including a start address shifted by whole rows
// (16 B), and times 2 issuers x N = 32 / 64.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include \
//        -I paper_1811_03882_b200/csrc tools/nosw_probe.cu -o /tmp/nsp && /tmp/nsp
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "acct_tc.cuh"

using namespace acct;

constexpr int ROWS = 160;  // A rows stored (positions); the MMA reads 128 from `shift`
constexpr int N = 32;

// A: [kq 2][ROWS][4] floats, B: [kq 2][N][4]; D[i][n] = sum_k A[shift+i][k] B[n][k]
__global__ void __launch_bounds__(128, 1) check(const float *A, const float *B, int shift,
                                                float *D) {
  __shared__ __align__(1024) float sa[2 * ROWS * 4];
  __shared__ __align__(1024) float sb[2 * N * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 2 * ROWS * 4; i += 128) sa[i] = A[i];
  for (int i = threadIdx.x; i < 2 * N * 4; i += 128) sb[i] = B[i];
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(&slot, 32);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    if (ptx::elect_one()) {
      const uint64_t da = ptx::smem_desc(ptx::smem_u32(sa) + 16 * shift, ROWS * 16, 128, 0);
      const uint64_t db = ptx::smem_desc(ptx::smem_u32(sb), N * 16, 128, 0);
      ptx::mma_tf32(tmem, da, db, ptx::idesc_tf32(128, N, false, false), 0);
      ptx::mma_commit(&bar);
    }
    __syncwarp();
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  uint32_t r[32];
  ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * warp) << 16), r);
  for (int n = 0; n < N; ++n) D[(32 * warp + lane) * N + n] = __uint_as_float(r[n]);
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 32);
}

// cycles per MMA: `issuers` warps each issue `iters` ss MMAs of 128 x n x 8
__global__ void __launch_bounds__(128, 1) rate(int n, int issuers, int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<float *>(sm)[i] = 0.001f * (i % 7);
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
  if (warp < issuers) {
    const uint32_t base = ptx::smem_u32(sm);
    const uint32_t idesc = ptx::idesc_tf32(128, n, false, false);
    const uint32_t d = tmem + warp * 128;
    __syncwarp();
    long long t0 = clock64();
    if (ptx::elect_one()) {
      for (int i = 0; i < iters; ++i) {
        const uint64_t da = ptx::smem_desc(base + 16 * (i % 9), 130 * 16, 128, 0);
        const uint64_t db = ptx::smem_desc(base + 24 * 1024 + 4096 * (i % 3), n * 16, 128, 0);
        ptx::mma_tf32(d, da, db, idesc, 1);
      }
      ptx::mma_commit(&bar[warp]);
    }
    __syncwarp();
    ptx::mbar_wait(&bar[warp], 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 4 + warp] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
  std::vector<float> A(2 * ROWS * 4), B(2 * N * 4), D(128 * N);
  srand(1);
  for (auto &v : A) v = (float)(rand() % 17 - 8);
  for (auto &v : B) v = (float)(rand() % 13 - 6);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int shift : {0, 1, 3, 17}) {
    check<<<1, 128>>>(dA, dB, shift, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("shift %d: %s\n", shift, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128; ++i)
      for (int n = 0; n < N; ++n) {
        float ref = 0;
        for (int k = 0; k < 8; ++k)
          ref += A[((k / 4) * ROWS + shift + i) * 4 + k % 4] * B[((k / 4) * N + n) * 4 + k % 4];
        if (ref != D[i * N + n] && bad++ < 3)
          printf("  shift %d D[%d][%d] = %g want %g\n", shift, i, n, D[i * N + n], ref);
      }
    printf("no-swizzle K-major, start shifted %d rows: %s\n", shift, bad ? "WRONG" : "ok");
  }
  long long *dout;
  cudaMalloc(&dout, 148 * 4 * 8);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  for (int n : {32, 64, 128})
    for (int iss : {1, 2, 4}) {
      const int iters = 2000;
      rate<<<148, 128, 48 * 1024>>>(n, iss, iters, dout);
      cudaDeviceSynchronize();
      std::vector<long long> o(148 * 4);
      cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int b = 0; b < 148; ++b)
        for (int w = 0; w < iss; ++w) mx = o[b * 4 + w] > mx ? o[b * 4 + w] : mx;
      printf("ss N=%3d issuers %d: %.1f cycles per MMA per issuer, %.1f MMAs per 1000 cycles per SM\n",
             n, iss, mx / iters, 1000.0 * iss * iters / mx);
    }
  return 0;
}
