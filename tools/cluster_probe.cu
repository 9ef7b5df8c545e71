// Cost of signalling the peer CTA of a cluster pair through an mbarrier:
// rank 1 arrives (remote, shared::cluster) once per step, rank 0 waits each
// phase; cycles per step for release vs relaxed arrives, +- proxy fence.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "acct_tc.cuh"
using namespace acct;

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1) probe(int iters, long long *out) {
  __shared__ uint64_t bar;
  __shared__ uint64_t ack;
  const uint32_t rank = ptx::cluster_rank();
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::mbar_init(&ack, 1);
    ptx::fence_mbar_init();
  }
  ptx::cluster_sync();
  const uint32_t bar0 = ptx::mapa(ptx::smem_u32(&bar), 0);
  const uint32_t ack1 = ptx::mapa(ptx::smem_u32(&ack), 1);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      if (rank == 1) {
        if (MODE == 2 || MODE == 3) ptx::fence_proxy_async_smem();
        if (MODE == 0 || MODE == 2)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar0) : "memory");
        else
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar0) : "memory");
        ptx::mbar_wait_cluster(&ack, i & 1);   // keep one phase in flight
      } else {
        ptx::mbar_wait_cluster(&bar, i & 1);
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ack1) : "memory");
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 1) out[MODE] = t1 - t0;
  ptx::cluster_sync();
}

int main() {
  long long *d, h[4];
  cudaMalloc(&d, 32);
  const int iters = 2000;
  probe<0><<<2, 64>>>(iters, d);
  probe<1><<<2, 64>>>(iters, d);
  probe<2><<<2, 64>>>(iters, d);
  probe<3><<<2, 64>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  const char *names[4] = {"release", "relaxed", "fence+release", "fence+relaxed"};
  for (int m = 0; m < 4; ++m) printf("%-14s round trip %.0f cycles\n", names[m], (double)h[m] / iters);
  return 0;
}
