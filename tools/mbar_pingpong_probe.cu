// mbarrier hand-off latency: two warps of one CTA ping-pong through two
// mbarriers (arrive / try_wait.parity), with and without the suspend-time
// hint, and with the second hop signalled by tcgen05.commit (no MMAs pending)
// as the conv kernels' MMA warp does.  Reports cycles per round trip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include \
//        -I paper_1811_03882_b200/csrc tools/mbar_pingpong_probe.cu -o /tmp/mpp && /tmp/mpp
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "acct_tc.cuh"

using namespace acct;

__device__ __forceinline__ void wait_plain(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(ptx::smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int MODE>  // 0 plain waits, 1 hinted waits (ptx::mbar_wait), 2 hinted + commit
__global__ void __launch_bounds__(64, 1) pingpong(int iters, long long *out) {
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_mbar_init();
  }
  if (MODE == 2 && warp == 1) ptx::tmem_alloc(&slot, 32);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (warp == 0) {
      if (lane == 0) ptx::mbar_arrive(&bar[0]);
      if (MODE == 0) wait_plain(&bar[1], i & 1); else ptx::mbar_wait(&bar[1], i & 1);
    } else {
      if (MODE == 0) wait_plain(&bar[0], i & 1); else ptx::mbar_wait(&bar[0], i & 1);
      if (MODE == 2) {
        if (ptx::elect_one()) ptx::mma_commit(&bar[1]);
        __syncwarp();
      } else if (lane == 0) {
        ptx::mbar_arrive(&bar[1]);
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  if (MODE == 2 && warp == 1) ptx::tmem_dealloc(slot, 32);
}

int main() {
  long long *d, h;
  cudaMalloc(&d, 8 * 148);
  const int iters = 20000;
  const char *names[3] = {"plain try_wait", "hinted try_wait", "hinted + tcgen05.commit"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) pingpong<0><<<1, 64>>>(iters, d);
      if (mode == 1) pingpong<1><<<1, 64>>>(iters, d);
      if (mode == 2) pingpong<2><<<1, 64>>>(iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-26s %7.1f cycles per round trip (two hand-offs)\n", names[mode], (double)h / iters);
  }
  return 0;
}
