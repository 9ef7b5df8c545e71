// Shared plumbing for libacct_sm100.so: error reporting, counters, launch
// geometry.  See include/acct.h for the ABI contract.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <string>

#include "acct.h"

// Pipeline-analysis knobs that SKIP work (operand build, MMAs, epilogue,
// loads -- results are then wrong) exist only in the profiling build
// (`-DACCT_PROFILING`, `python -m paper_1811_03882_b200.build --profiling`,
// used by tools/ only).  In the product library ACCT_SKIP is a constant
// false and those paths are compiled out, as are the clock64 traces of
// ACCT_TRACE (bit 64, tools/conv_trace.py).
#ifdef ACCT_PROFILING
#define ACCT_SKIP(word, bit) (((word) & (bit)) != 0)
#define ACCT_TRACE(word) (((word) & 64) != 0)
#else
#define ACCT_SKIP(word, bit) false
#define ACCT_TRACE(word) false
#endif

namespace acct {

// ---- error reporting (per host thread) ----
void set_error(const std::string &msg);
int fail(int code, const char *what);
int check_cuda(cudaError_t err, const char *what);

// ---- per-thread counters (one host thread drives one device) ----
struct Counters {
  std::atomic<int64_t> directive_execs{0}, var_transfers{0};
  std::atomic<int64_t> h2d_calls{0}, d2h_calls{0}, h2d_bytes{0}, d2h_bytes{0};
  std::atomic<int64_t> kernel_launches{0}, host_ops{0};
};
Counters &counters();

inline int note_launch(const char *what) {
  counters().kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return check_cuda(cudaGetLastError(), what);
}

// grid for a grid-stride kernel: enough CTAs to cover `work` items, capped at
// `per_sm` resident CTAs per SM over the whole chip (multiple of the SM count)
int sm_count();
inline unsigned grid_for(int64_t work, int block, int per_sm = 8) {
  int64_t need = (work + block - 1) / block;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (need > cap) need = cap;
  if (need < 1) need = 1;
  return (unsigned)need;
}

inline cudaStream_t as_stream(acct_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch.  Every kernel of the library is launched
// with programmaticStreamSerializationAllowed (so inside a CUDA graph the
// next kernel's CTAs may be scheduled, and run their prologue, while this one
// drains) and calls pdl_wait() before touching any global data a previous
// kernel produced or may still read.  On by default; ACCT_PDL=0 turns it
// off.  The dependents are released by each CTA's implicit trigger at exit:
// an explicit griddepcontrol.launch_dependents at kernel start let the next
// grid's CTAs take SM slots (shared memory, TMEM) from this grid's later
// waves -- graph replay, 16 images: yolov2-tiny 0.718 / 0.716 / 0.729 ms
// and yolov2-608 5.039 / 4.945 / 4.955 ms for early trigger / trigger at exit
// / no PDL.
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                   Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace acct

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// where a kernel may release its dependents; a no-op (the implicit trigger
// at CTA exit measured best, see above)
__device__ __forceinline__ void pdl_trigger() {}

// n / d and n % d for 0 <= n, d < 2^24 by a float reciprocal (inv_d = 1.0f /
// d, computed once) and one correction step -- the per-unit tile-index
// divisions of the persistent kernels showed in their stall samples
__device__ __forceinline__ void acct_divmod(int n, int d, float inv_d, int &q, int &r) {
  q = (int)((float)n * inv_d);
  r = n - q * d;
  if (r < 0) {
    --q;
    r += d;
  } else if (r >= d) {
    ++q;
    r -= d;
  }
}

// leaky as darknet computes it: `.1*x` is a double product rounded to float
__host__ __device__ __forceinline__ float acct_leaky_ref(float v) {
  return v < 0.0f ? (float)(0.1 * (double)v) : v;
}

// The same value without FP64 or F2F conversions (which ran the epilogues on
// the XU pipe): .1 = c1 + c2 split into floats; p = RN(v c1), its exact error
// e = fma(v, c1, -p), and RN(p + RN(fma(v, c2, e))) lands on RN(RN_double(.1 v))
// -- checked for all 2^32 inputs on the device (acct_leaky_exhaustive_check,
// tests/test_gpu_kernels.py).  |v| < 2^-100 (where p loses bits to the
// subnormal range) and |v| > 2^120 (-inf) keep the double product.
__host__ __device__ __forceinline__ float acct_leaky(float v) {
#ifdef __CUDA_ARCH__
  if (!(v < 0.0f)) return v;
  if (v > -0x1p-100f || v < -0x1p+120f) return (float)(0.1 * (double)v);
  constexpr float c1 = 0x1.99999ap-4f;                      // (float)0.1
  constexpr float c2 = (float)(0.1 - (double)0x1.99999ap-4f);  // 0.1 - c1, rounded
  const float p = __fmul_rn(v, c1);
  const float e = __fmaf_rn(v, c1, -p);
  return __fadd_rn(p, __fmaf_rn(v, c2, e));
#else
  return acct_leaky_ref(v);
#endif
}

// Epilogue form for a lane's block of values: the common path branch-free
// (five instructions, bit-identical to acct_leaky wherever
// acct_leaky_guarded is false) and, when any lane of the warp holds a guarded
// value (|v| < 2^-100 or v < -2^120, negative), acct_leaky for the whole
// block.  Predicated inline, the double-product fallback cost every value an
// F2F / DMUL issue slot.
#ifdef __CUDACC__
__device__ __forceinline__ bool acct_leaky_guarded(float v) {
  return v < -0x1p+120f || (v < 0.0f && v > -0x1p-100f);
}
__device__ __forceinline__ float acct_leaky_fast(float v) {
  constexpr float c1 = 0x1.99999ap-4f;
  constexpr float c2 = (float)(0.1 - (double)0x1.99999ap-4f);
  const float p = __fmul_rn(v, c1);
  const float e = __fmaf_rn(v, c1, -p);
  const float q = __fadd_rn(p, __fmaf_rn(v, c2, e));
  return v < 0.0f ? q : v;
}
// The guard over a block, three integer ops per value: with a = bits ^ sign,
// a negative v has a = |v| bits (>= 0 as int) and a positive one a >= 2^31
// (< 0 as int), so the unsigned min of a is the smallest |v| of the
// negatives and the signed max the largest -- against 2^-100 (0x0D800000)
// and 2^120 (0x7B800000), the exact acct_leaky_guarded ranges (-0 and
// negative NaNs take the exact path too, which handles them identically).
template <int N>
__device__ __forceinline__ bool acct_leaky_any_guarded(const float (&v)[N]) {
  uint32_t mn = 0xFFFFFFFFu;
  int32_t mx = INT32_MIN;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const uint32_t a = __float_as_uint(v[i]) ^ 0x80000000u;
    mn = min(mn, a);
    mx = max(mx, (int32_t)a);
  }
  return mn < 0x0D800000u || mx > 0x7B800000;
}
template <int N>
__device__ __forceinline__ void acct_leaky_block(float (&v)[N]) {
  const bool slow = acct_leaky_any_guarded(v);
  if (__any_sync(__activemask(), slow)) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = acct_leaky(v[i]);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = acct_leaky_fast(v[i]);
  }
}
#endif
