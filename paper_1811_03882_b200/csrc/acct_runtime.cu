// Runtime half of libacct_sm100.so: errors, counters, counted transfers, the
// gemm_nn mode dispatcher and the native schedule runner that executes a
// genome's compiled offload pattern (include/acct.h).
//
// The runner is the B200 analogue of running the emitted OpenACC program:
// `#pragma acc data` lines become counted pitched cudaMemcpy2DAsync calls at
// exactly the loops they precede (pkg/src/acctuner/emitter.py:41-84),
// `#pragma acc kernels` loops become kernel launches, every other loop runs
// natively on the host.  One stream per device; the stream is drained before
// any host loop touches host buffers, which keeps the OpenACC data-region
// ordering without extra events.

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <algorithm>
#include <vector>

#include "acct_common.cuh"

namespace acct {

static thread_local std::string g_error;

void set_error(const std::string &msg) { g_error = msg; }

int fail(int code, const char *what) {
  set_error(std::string(what) + " (code " + std::to_string(code) + ")");
  return code;
}

int check_cuda(cudaError_t err, const char *what) {
  if (err == cudaSuccess) return ACCT_OK;
  set_error(std::string(what) + ": " + cudaGetErrorName(err) + ": " + cudaGetErrorString(err));
  return (int)err;
}

// per host thread: one thread drives one device, so a run's counters are
// exactly the calling thread's
// measured slower inside the CUDA-graph replay on B200 (4.06 vs 3.91 ms per
// 16-image step), so off unless ACCT_PDL=1
bool pdl_enabled() {  // default on; ACCT_PDL=0 turns it off (tools/ comparisons)
  static const bool on = [] {
    const char *v = getenv("ACCT_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

Counters &counters() {
  static thread_local Counters c;
  return c;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

int gemm_simt(int M, int N, int K, float alpha, const float *A, int64_t lda, const float *B,
              int64_t ldb, float beta, float *C, int64_t ldc, const float *bias, int act,
              cudaStream_t s);
int gemm_tc(int M, int N, int K, float alpha, const float *A, int64_t lda, const float *B,
            int64_t ldb, float beta, float *C, int64_t ldc, const float *bias, int act,
            cudaStream_t s);
int gemm_stream(int M, int N, int K, float alpha, const float *A, int64_t lda, const float *B,
                int64_t ldb, float beta, float *C, int64_t ldc, const float *bias, int act,
                cudaStream_t s);

}  // namespace acct

using namespace acct;

extern "C" const char *acct_last_error_string(void) { return g_error.c_str(); }

extern "C" void acct_counters_get(acct_counters_t *out) {
  if (!out) return;
  Counters &c = counters();
  out->directive_execs = c.directive_execs.load();
  out->var_transfers = c.var_transfers.load();
  out->h2d_calls = c.h2d_calls.load();
  out->d2h_calls = c.d2h_calls.load();
  out->h2d_bytes = c.h2d_bytes.load();
  out->d2h_bytes = c.d2h_bytes.load();
  out->kernel_launches = c.kernel_launches.load();
  out->host_ops = c.host_ops.load();
}

extern "C" void acct_counters_reset(void) {
  Counters &c = counters();
  c.directive_execs = 0;
  c.var_transfers = 0;
  c.h2d_calls = 0;
  c.d2h_calls = 0;
  c.h2d_bytes = 0;
  c.d2h_bytes = 0;
  c.kernel_launches = 0;
  c.host_ops = 0;
}

extern "C" int acct_device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

extern "C" const char *acct_build_info(void) {
  return "libacct_sm100: sm_100a (tcgen05/TMA 3xTF32 gemm_nn, vectorized HBM kernels), CUDA "
#ifdef __CUDACC_VER_MAJOR__
      "12.x"
#endif
      ;
}

namespace {

// dense [rows][cols] -> pitched [rows][ld]; one thread per element of a row
// chunk, 2-D grid so there is no index division
__global__ void repack_kernel(const float *__restrict__ src, int64_t cols, float *__restrict__ dst,
                              int64_t ld, int64_t rows) {
  pdl_trigger();
  pdl_wait();
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cols;
         c += (int64_t)gridDim.x * blockDim.x)
      dst[r * ld + c] = __ldcs(src + r * cols + c);
}

// ACCT_A_H2D_GATHER: dense arrays laid out in one staged host range ->
// their pitched device layouts; blockIdx.z = member
struct GatherMember {
  int64_t src;   // element offset of the member in the staging range
  uint32_t *dst;
  int64_t rows, cols, ld;
};
struct GatherSet {
  int n;
  GatherMember m[12];
};
__global__ void gather_scatter_kernel(const uint32_t *__restrict__ stage, const GatherSet set) {
  pdl_trigger();
  pdl_wait();
  const GatherMember &g = set.m[blockIdx.z];
  const uint32_t *src = stage + g.src;
  for (int64_t r = blockIdx.y; r < g.rows; r += gridDim.y)
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < g.cols;
         c += (int64_t)gridDim.x * blockDim.x)
      g.dst[r * g.ld + c] = __ldcs(src + r * g.cols + c);
}

// pitched [rows][ld] -> dense [rows][cols] (the D2H half of the staging)
__global__ void pack_kernel(const float *__restrict__ src, int64_t ld, float *__restrict__ dst,
                            int64_t cols, int64_t rows) {
  pdl_trigger();
  pdl_wait();
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cols;
         c += (int64_t)gridDim.x * blockDim.x)
      dst[r * cols + c] = __ldcs(src + r * ld + c);
}

}  // namespace

extern "C" int acct_h2d_staged(void *dev, int64_t ld, const void *host, int64_t rows,
                               int64_t cols, void *stage, acct_stream_t stream) {
  if (!dev || !host || !stage || rows < 0 || cols < 0 || ld < cols)
    return fail(ACCT_EINVAL, "h2d_staged: bad arguments");
  if (rows * cols == 0) return ACCT_OK;
  const size_t bytes = (size_t)rows * cols * 4;
  cudaStream_t s = as_stream(stream);
  if (int rc = check_cuda(cudaMemcpyAsync(stage, host, bytes, cudaMemcpyHostToDevice, s),
                          "h2d_staged: copy"))
    return rc;
  Counters &c = counters();
  c.h2d_calls.fetch_add(1);
  c.h2d_bytes.fetch_add((int64_t)bytes);
  const unsigned gx = (unsigned)((cols + 255) / 256 < 64 ? (cols + 255) / 256 : 64);
  const unsigned gy = (unsigned)(rows < 1024 ? rows : 1024);
  launch(repack_kernel, dim3(gx, gy), dim3(256), 0, s, static_cast<const float *>(stage), cols,
         static_cast<float *>(dev), ld, rows);
  return note_launch("h2d_staged repack");
}

extern "C" int acct_d2h_staged(void *host, const void *dev, int64_t ld, int64_t rows,
                               int64_t cols, void *stage, acct_stream_t stream) {
  if (!dev || !host || !stage || rows < 0 || cols < 0 || ld < cols)
    return fail(ACCT_EINVAL, "d2h_staged: bad arguments");
  if (rows * cols == 0) return ACCT_OK;
  const size_t bytes = (size_t)rows * cols * 4;
  cudaStream_t s = as_stream(stream);
  const unsigned gx = (unsigned)((cols + 255) / 256 < 64 ? (cols + 255) / 256 : 64);
  const unsigned gy = (unsigned)(rows < 1024 ? rows : 1024);
  launch(pack_kernel, dim3(gx, gy), dim3(256), 0, s, static_cast<const float *>(dev), ld,
         static_cast<float *>(stage), cols, rows);
  if (int rc = note_launch("d2h_staged pack")) return rc;
  Counters &c = counters();
  c.d2h_calls.fetch_add(1);
  c.d2h_bytes.fetch_add((int64_t)bytes);
  return check_cuda(cudaMemcpyAsync(host, stage, bytes, cudaMemcpyDeviceToHost, s),
                    "d2h_staged: copy");
}

extern "C" int acct_memcpy2d(void *dst, size_t dpitch, const void *src, size_t spitch,
                             size_t row_bytes, size_t rows, int direction, acct_stream_t stream) {
  if (direction != 1 && direction != 2) return fail(ACCT_EINVAL, "memcpy2d: direction");
  if (rows == 0 || row_bytes == 0) return ACCT_OK;
  cudaMemcpyKind kind = direction == 1 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  cudaError_t err;
  if (dpitch == row_bytes && spitch == row_bytes)
    err = cudaMemcpyAsync(dst, src, row_bytes * rows, kind, as_stream(stream));
  else
    err = cudaMemcpy2DAsync(dst, dpitch, src, spitch, row_bytes, rows, kind, as_stream(stream));
  Counters &c = counters();
  if (direction == 1) {
    c.h2d_calls.fetch_add(1);
    c.h2d_bytes.fetch_add((int64_t)(row_bytes * rows));
  } else {
    c.d2h_calls.fetch_add(1);
    c.d2h_bytes.fetch_add((int64_t)(row_bytes * rows));
  }
  return check_cuda(err, "memcpy2d");
}

extern "C" int acct_gemm_nn_f32(int M, int N, int K, float alpha, const float *A, int64_t lda,
                                const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                                const float *bias, int act, int mode, acct_stream_t stream) {
  if (M < 0 || N < 0 || K < 0 || lda < K || ldb < N || ldc < N)
    return fail(ACCT_EINVAL, "gemm_nn: bad shape/pitch");
  if (act != -1 && act != ACCT_ACT_LINEAR && act != ACCT_ACT_LEAKY)
    return fail(ACCT_EINVAL, "gemm_nn: bad activation");
  if ((int64_t)M * N == 0) return ACCT_OK;
  cudaStream_t s = as_stream(stream);
  // M <= 16, or M <= 32 with K <= 64 (first conv layers, K = 27): an HBM
  // stream of B and C with < 1 flop/byte -- CUDA cores beat narrow MMA tiles
  if (mode == ACCT_GEMM_AUTO && (M <= 16 || (M <= 32 && K <= 64))) {
    int rc = gemm_stream(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
    if (rc != ACCT_ENOTSUP) return rc;
  }
  if (mode == ACCT_GEMM_TC3XTF32 || mode == ACCT_GEMM_AUTO) {
    int rc = gemm_tc(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
    if (rc != ACCT_ENOTSUP || mode == ACCT_GEMM_TC3XTF32) return rc;
  } else if (mode != ACCT_GEMM_SIMT) {
    return fail(ACCT_EINVAL, "gemm_nn: unknown mode");
  }
  return gemm_simt(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
}

// Batched gemm over `batch` images, image b's operands at base + b * stride
// (stride 0 = one shared operand, e.g. the weights).  When A is shared and B
// and C are column-interleaved ([rows][batch * s] with image b at column
// offset b * s, s >= N) the batch is ONE gemm of N' = (batch-1)*s + N
// columns -- the padding columns between images are computed and never read.
extern "C" int acct_gemm_nn_batched_f32(int M, int N, int K, float alpha, const float *A,
                                        int64_t lda, int64_t a_stride, const float *B,
                                        int64_t ldb, int64_t b_stride, float beta, float *C,
                                        int64_t ldc, int64_t c_stride, const float *bias, int act,
                                        int batch, int mode, acct_stream_t stream) {
  if (batch < 1) return fail(ACCT_EINVAL, "gemm_nn: bad batch");
  if (batch == 1)
    return acct_gemm_nn_f32(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, mode, stream);
  const int64_t span = (int64_t)(batch - 1) * b_stride + N;
  if (a_stride == 0 && b_stride == c_stride && b_stride >= N && span <= ldb && span <= ldc &&
      span < (int64_t)1 << 31)
    return acct_gemm_nn_f32(M, (int)span, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, mode,
                            stream);
  for (int b = 0; b < batch; ++b)
    if (int rc = acct_gemm_nn_f32(M, N, K, alpha, A + b * a_stride, lda, B + b * b_stride, ldb,
                                  beta, C + b * c_stride, ldc, bias, act, mode, stream))
      return rc;
  return ACCT_OK;
}

// ------------------------------------------------------------ schedule runner

namespace {

struct LoopFrame {
  int begin;
  int64_t counter, trip;
};

inline float bits_to_float(int64_t v) {
  uint32_t u = (uint32_t)v;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int device_op(const acct_action_t &a, acct_array_t *arr, int gemm_mode, cudaStream_t s) {
  const int64_t *I = a.i;
  auto D = [&](int k) { return reinterpret_cast<float *>(arr[a.a[k]].dev); };
  auto LD = [&](int k) { return arr[a.a[k]].ld_dev; };
  auto BS = [&](int k) { return arr[a.a[k]].img_stride; };  // per-image offset (0 = shared)
  const int nb = I[13] > 1 ? (int)I[13] : 1;                 // images per launch
  acct_stream_t st = reinterpret_cast<acct_stream_t>(s);
  switch ((int)I[0]) {
    case ACCT_K_FILL:
      return acct_fill_batched_f32(D(0), I[1], I[2], LD(0), BS(0), bits_to_float(I[3]), nb, st);
    case ACCT_K_COPY:
      return acct_copy_batched_f32(D(0), LD(0), BS(0), D(1), LD(1), BS(1), I[1], I[2], nb, st);
    case ACCT_K_IM2COL:
      return acct_im2col_batched_f32(D(0), LD(0), BS(0), (int)I[1], (int)I[2], (int)I[3],
                                     (int)I[4], (int)I[5], (int)I[6], D(1), LD(1), BS(1), nb, st);
    case ACCT_K_GEMM: {
      const float *bias = a.a[3] >= 0 ? D(3) : nullptr;
      return acct_gemm_nn_batched_f32((int)I[1], (int)I[2], (int)I[3], 1.0f, D(0), LD(0), BS(0),
                                      D(1), LD(1), BS(1), I[4] ? 1.0f : 0.0f, D(2), LD(2), BS(2),
                                      bias, (int)I[5], nb, gemm_mode, st);
    }
    case ACCT_K_CONV: {
      const float *bias = I[7] >= 0 ? reinterpret_cast<float *>(arr[I[7]].dev) : nullptr;
      const float beta = I[5] ? 1.0f : 0.0f;
      const int M = (int)I[4], K = 9 * (int)I[1], N = (int)(I[2] * I[3]);
      // I[8] = 1: only the last image's col is observable (col_from = nb - 1).
      // FP32 FMA from the input window (k order, the SIMT gemms' chain) for
      // M <= 16 and in SIMT mode; the
      // implicit-im2col tcgen05 swap tile (3xTF32, bit-identical to im2col +
      // the swap gemm) for the other narrow layers (M <= 64)
      const int C = (int)I[1], H = (int)I[2], W = (int)I[3], col_from = I[8] ? nb - 1 : 0;
      static const int tc_first = [] {  // experiment knob: first layers on tcgen05 too
        const char *e = getenv("ACCT_CONV_TC_FIRST");
        return e ? atoi(e) : 0;
      }();
      // FP32 window kernel for M <= 16, and for pooled first layers (c <= 4)
      // with M <= 32 (two 16-filter CTAs per tile); the unpooled M = 32 window
      // kernel ran 41.8 us/img at 608x608
      const bool simt = gemm_mode == ACCT_GEMM_SIMT ||
                        (gemm_mode == ACCT_GEMM_AUTO && !tc_first &&
                         (M <= 16 || (M <= 32 && C <= 4 && I[9] >= 0)));
      // I[9] / I[10]: a fused 2x2/2 maxpool of C into pool / idx; I[11] = 1:
      // C is then observable for the last image only
      const bool has_pool = I[9] >= 0;
      float *pool = has_pool ? reinterpret_cast<float *>(arr[I[9]].dev) : nullptr;
      int32_t *pidx = has_pool ? reinterpret_cast<int32_t *>(arr[I[10]].dev) : nullptr;
      const int64_t ldp = has_pool ? arr[I[9]].ld_dev : 0, pbs = has_pool ? arr[I[9]].img_stride : 0;
      const int64_t ldi = has_pool ? arr[I[10]].ld_dev : 0, ibs = has_pool ? arr[I[10]].img_stride : 0;
      auto fused = [&](bool with_pool) {
        float *pp = with_pool ? pool : nullptr;
        int32_t *pi = with_pool ? pidx : nullptr;
        const int c_from = (with_pool && I[11]) ? nb - 1 : 0;
        if (simt)
          return acct_conv3x3_im2col_gemm_f32(D(0), LD(0), BS(0), C, H, W, D(1), LD(1), BS(1), M,
                                              D(2), LD(2), beta, D(3), LD(3), BS(3), bias,
                                              (int)I[6], nb, col_from, pp, ldp, pbs, pi, ldi, ibs,
                                              c_from, st);
        int rc = (int)ACCT_ENOTSUP;
        if (M <= 64 || (M % 128 == 0 && M <= 256))
          rc = acct_conv3x3_tc_f32(D(0), LD(0), BS(0), C, H, W, D(1), LD(1), BS(1), M, D(2),
                                   LD(2), beta, D(3), LD(3), BS(3), bias, (int)I[6], nb, col_from,
                                   pp, ldp, pbs, pi, ldi, ibs, c_from, st);
        // wide, long-K layers (and the wide conv's misfits: 26-wide planes):
        // the CTA-pair gemm with implicit im2col, no fused pool
        if (rc == ACCT_ENOTSUP && !with_pool && M >= 256 && K > 768)
          rc = acct_conv3x3_gemm_tc_f32(D(0), LD(0), BS(0), C, H, W, D(1), LD(1), BS(1), M, D(2),
                                        LD(2), beta, D(3), LD(3), BS(3), bias, (int)I[6], nb,
                                        col_from, nullptr, 0, 0, nullptr, 0, 0, 0, st);
        return rc;
      };
      auto pool_after = [&]() {  // the maxpool the launch did not fuse
        if (!has_pool) return (int)ACCT_OK;
        return acct_maxpool_batched_f32(D(3), LD(3), BS(3), M, H, W, 2, 2, 0, H / 2, W / 2, pool,
                                        ldp, pbs, pidx, ldi, ibs, nb, st);
      };
      int rc = fused(has_pool);
      if (rc == ACCT_ENOTSUP && has_pool) {
        rc = fused(false);
        if (rc == ACCT_OK) return pool_after();
      }
      if (rc != ACCT_ENOTSUP) return rc;
      // the same ops unfused: im2col, then the gemm in the requested mode
      if (int rc2 = acct_im2col_batched_f32(D(0), LD(0), BS(0), C, H, W, 3, 1, 1, D(1), LD(1),
                                            BS(1), nb, st))
        return rc2;
      if (int rc2 = acct_gemm_nn_batched_f32(M, N, K, 1.0f, D(2), LD(2), 0, D(1), LD(1), BS(1), beta,
                                             D(3), LD(3), BS(3), bias, (int)I[6], nb, gemm_mode,
                                             st))
        return rc2;
      return pool_after();
    }
    case ACCT_K_ADD_BIAS:
      return acct_add_bias_batched_f32(D(0), LD(0), BS(0), D(1), (int)I[1], I[2], nb, st);
    case ACCT_K_LEAKY:
      return acct_activate_batched_f32(D(0), LD(0), BS(0), I[1], I[2], ACCT_ACT_LEAKY, nb, st);
    case ACCT_K_LINEAR:
      return acct_activate_batched_f32(D(0), LD(0), BS(0), I[1], I[2], ACCT_ACT_LINEAR, nb, st);
    case ACCT_K_MAXPOOL:
      return acct_maxpool_batched_f32(D(0), LD(0), BS(0), (int)I[1], (int)I[2], (int)I[3],
                                      (int)I[4], (int)I[5], (int)I[6], (int)I[7], (int)I[8], D(1),
                                      LD(1), BS(1), reinterpret_cast<int32_t *>(arr[a.a[2]].dev),
                                      LD(2), BS(2), nb, st);
  }
  return fail(ACCT_EINVAL, "schedule: unknown device op");
}

int host_op(const acct_action_t &a, acct_array_t *arr) {
  const int64_t *I = a.i;
  auto H = [&](int k) { return reinterpret_cast<float *>(arr[a.a[k]].host); };
  auto LD = [&](int k) { return arr[a.a[k]].cols; };
  int rc = ACCT_EINVAL;
  switch ((int)I[0]) {
    case ACCT_K_FILL: rc = acct_host_fill_f32(H(0), I[1], I[2], LD(0), bits_to_float(I[3])); break;
    case ACCT_K_COPY: rc = acct_host_copy_f32(H(0), LD(0), H(1), LD(1), I[1], I[2]); break;
    case ACCT_K_IM2COL:
      rc = acct_host_im2col_f32(H(0), LD(0), (int)I[1], (int)I[2], (int)I[3], (int)I[4], (int)I[5],
                                (int)I[6], H(1), LD(1));
      break;
    case ACCT_K_GEMM:
      rc = acct_host_gemm_nn_f32((int)I[1], (int)I[2], (int)I[3], 1.0f, H(0), LD(0), H(1), LD(1),
                                 H(2), LD(2));
      break;
    case ACCT_K_ADD_BIAS: rc = acct_host_add_bias_f32(H(0), LD(0), H(1), (int)I[1], I[2]); break;
    case ACCT_K_LEAKY: rc = acct_host_activate_f32(H(0), LD(0), I[1], I[2], ACCT_ACT_LEAKY); break;
    case ACCT_K_LINEAR: rc = acct_host_activate_f32(H(0), LD(0), I[1], I[2], ACCT_ACT_LINEAR); break;
    case ACCT_K_MAXPOOL:
      rc = acct_host_maxpool_f32(H(0), LD(0), (int)I[1], (int)I[2], (int)I[3], (int)I[4], (int)I[5],
                                 (int)I[6], (int)I[7], (int)I[8], H(1), LD(1),
                                 reinterpret_cast<int32_t *>(arr[a.a[2]].host), LD(2));
      break;
  }
  if (rc != ACCT_OK) return fail(rc, "schedule: host op failed");
  counters().host_ops.fetch_add(1);
  return ACCT_OK;
}

}  // namespace

namespace {

// Optional per-action device timing: an event pair around every KERNEL
// action execution, resolved after the final drain.
struct Profiler {
  float *out_ms = nullptr;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, size_t>> marks;  // (action index, first event of the pair)
  size_t used = 0;
  cudaEvent_t next() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  ~Profiler() {
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
};

int run_schedule(acct_array_t *arrays, int n_arrays, const acct_action_t *actions, int n_actions,
                 int gemm_mode, double timeout_s, acct_stream_t stream, Profiler *prof,
                 bool capturing = false);

}  // namespace

extern "C" int acct_run_schedule(acct_array_t *arrays, int n_arrays, const acct_action_t *actions,
                                 int n_actions, int gemm_mode, double timeout_s,
                                 acct_stream_t stream) {
  return run_schedule(arrays, n_arrays, actions, n_actions, gemm_mode, timeout_s, stream, nullptr);
}

extern "C" int acct_run_schedule_profiled(acct_array_t *arrays, int n_arrays,
                                          const acct_action_t *actions, int n_actions,
                                          int gemm_mode, double timeout_s, acct_stream_t stream,
                                          float *kernel_ms) {
  if (!kernel_ms) return fail(ACCT_EINVAL, "profiled schedule: null output");
  for (int k = 0; k < n_actions; ++k) kernel_ms[k] = 0.0f;
  Profiler prof;
  prof.out_ms = kernel_ms;
  int rc = run_schedule(arrays, n_arrays, actions, n_actions, gemm_mode, timeout_s, stream, &prof);
  if (rc != ACCT_OK) return rc;
  for (auto &m : prof.marks) {
    float ms = 0.0f;
    rc = check_cuda(cudaEventElapsedTime(&ms, prof.pool[m.second], prof.pool[m.second + 1]),
                    "profiled schedule: elapsed");
    if (rc) return rc;
    kernel_ms[m.first] += ms;
  }
  return ACCT_OK;
}

namespace {

// Side stream for the hoisted transfers in front of the first loop (the
// image loop): they are issued there, each followed by an event, and the
// main stream waits on an array's event only right before the first action
// that touches that array -- so layer 12's weights stream in while layers
// 0-11 compute.  One per host thread and device (thread_local).
//
// A second side stream `d` carries early copyouts (D2H actions flagged
// i[3] = 1 by the compiler: the array's final value exists once its last
// writer ran), so device->host traffic overlaps the remaining kernels and the
// host->device stream (PCIe is full duplex).  Its staged copies use their own
// scratch, `dstage`, never the arrays' shared staging buffer.
struct SideXfer {
  int device = -1;
  cudaStream_t t = nullptr, d = nullptr;
  cudaEvent_t fork = nullptr, done = nullptr, dfork = nullptr, ddone = nullptr;
  std::vector<cudaEvent_t> ev;
  void *dstage = nullptr;
  size_t dstage_bytes = 0;
  std::vector<void *> retired;
  int ensure_dstage(size_t bytes, bool capturing) {
    if (bytes <= dstage_bytes) return ACCT_OK;
    if (capturing) return fail(ACCT_ENOTSUP, "early copyout scratch grows during capture");
    // retired, not freed: a graph captured earlier may still reference it
    if (dstage) retired.push_back(dstage);
    dstage = nullptr;
    dstage_bytes = 0;
    if (int rc = check_cuda(cudaMalloc(&dstage, bytes), "early copyout scratch")) return rc;
    dstage_bytes = bytes;
    return ACCT_OK;
  }
  int ensure(int n) {
    if (!t) {
      cudaGetDevice(&device);
      if (int rc = check_cuda(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking), "side stream"))
        return rc;
      if (int rc = check_cuda(cudaStreamCreateWithFlags(&d, cudaStreamNonBlocking), "d2h stream"))
        return rc;
      cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&dfork, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ddone, cudaEventDisableTiming);
    }
    while ((int)ev.size() < n) {
      cudaEvent_t e;
      if (int rc = check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "side event"))
        return rc;
      ev.push_back(e);
    }
    return ACCT_OK;
  }
};

// one set of side streams / events / early-copyout scratch per (host thread,
// device): a GA worker thread takes whichever device is idle, and switching
// devices must neither rebuild nor leak the other device's resources
SideXfer &side_xfer() {
  static thread_local std::unordered_map<int, SideXfer> per_device;
  int dev = 0;
  cudaGetDevice(&dev);
  return per_device[dev];
}

int run_schedule(acct_array_t *arrays, int n_arrays, const acct_action_t *actions, int n_actions,
                 int gemm_mode, double timeout_s, acct_stream_t stream, Profiler *prof,
                 bool capturing) {
  cudaStream_t s = as_stream(stream);
  std::vector<LoopFrame> loops;
  bool pending = false;
  const auto t0 = std::chrono::steady_clock::now();

  // hoisted-transfer deferral: only when no host loop can touch host buffers
  // behind the side stream's back, and not under the per-kernel profiler
  bool defer = prof == nullptr;
  for (int k = 0; k < n_actions && defer; ++k)
    if (actions[k].kind == ACCT_A_HOST) defer = false;
  SideXfer *side = nullptr;
  if (defer) {
    side = &side_xfer();
    if (side->ensure(n_arrays) != ACCT_OK) defer = false;
  }
  std::vector<char> waiting(defer ? n_arrays : 0, 0);
  bool forked = false, in_prefix = true;
  auto join_all = [&]() -> int {
    if (!forked) return ACCT_OK;
    forked = false;
    std::fill(waiting.begin(), waiting.end(), 0);
    if (int rc = check_cuda(cudaEventRecord(side->done, side->t), "side join record")) return rc;
    return check_cuda(cudaStreamWaitEvent(s, side->done, 0), "side join wait");
  };
  auto need = [&](int slot) -> int {
    if (!forked || slot < 0 || slot >= n_arrays || !waiting[slot]) return ACCT_OK;
    waiting[slot] = 0;
    return check_cuda(cudaStreamWaitEvent(s, side->ev[slot], 0), "side wait");
  };

  bool dforked = false;  // early copyouts in flight on side->d
  auto join_d2h = [&]() -> int {
    if (!dforked) return ACCT_OK;
    dforked = false;
    if (int rc = check_cuda(cudaEventRecord(side->ddone, side->d), "d2h join record")) return rc;
    return check_cuda(cudaStreamWaitEvent(s, side->ddone, 0), "d2h join wait");
  };
  auto drain = [&]() -> int {
    if (int rc = join_all()) return rc;
    if (int rc = join_d2h()) return rc;
    if (!pending || capturing) return ACCT_OK;
    pending = false;
    return check_cuda(cudaStreamSynchronize(s), "schedule: stream sync");
  };
  auto check_slot = [&](int k) { return k >= 0 && k < n_arrays; };
  Counters &cnt = counters();
  int pc = 0;
  // ACCT_TRACE=1 (uncaptured runs): an event after every transfer / kernel
  // action on the stream it went to; elapsed ms from the start to stderr
  static const bool trace = getenv("ACCT_TRACE") != nullptr;
  struct Mark {
    int pc;
    char where;
    cudaEvent_t ev;
  };
  std::vector<Mark> marks;
  cudaEvent_t trace0 = nullptr;
  if (trace && !capturing && !prof) {
    cudaEventCreate(&trace0);
    cudaEventRecord(trace0, s);
  }
  auto mark = [&](int at, const acct_action_t &a) {
    if (!trace0) return;
    cudaStream_t on = s;
    char where = 'm';
    if (a.kind == ACCT_A_H2D && defer && in_prefix) on = side->t, where = 'h';
    if (a.kind == ACCT_A_D2H && a.i[3] == 1 && defer) on = side->d, where = 'd';
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, on);
    marks.push_back({at, where, e});
  };
  auto dump = [&]() {
    if (!trace0) return;
    cudaDeviceSynchronize();
    for (auto &m : marks) {
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, trace0, m.ev);
      const acct_action_t &a = actions[m.pc];
      fprintf(stderr, "trace %8.3f ms %c pc=%3d kind=%d slot=%d op=%lld\n", ms, m.where, m.pc,
              a.kind, a.a[0], (long long)a.i[0]);
      cudaEventDestroy(m.ev);
    }
    cudaEventDestroy(trace0);
  };
  while (pc < n_actions) {
    const acct_action_t &a = actions[pc];
    int rc = ACCT_OK;
    switch (a.kind) {
      case ACCT_A_LOOP_BEGIN:
        if (a.i[0] <= 0) {
          pc = (int)a.i[1] + 1;  // skip to after LOOP_END
          continue;
        }
        loops.push_back({pc, 0, a.i[0]});
        in_prefix = false;
        break;
      case ACCT_A_LOOP_END: {
        if (loops.empty()) return fail(ACCT_EINVAL, "schedule: unbalanced loop");
        LoopFrame &f = loops.back();
        if (++f.counter < f.trip) {
          pc = f.begin + 1;
          if (timeout_s > 0 && !capturing) {
            double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (el > timeout_s) {
              // no copy may still be running on a side stream when the caller
              // gets control back (it reuses the pinned buffers)
              join_all();
              join_d2h();
              cudaStreamSynchronize(s);
              return fail(ACCT_ETIMEOUT, "schedule: timeout");
            }
          }
          continue;
        }
        loops.pop_back();
        break;
      }
      case ACCT_A_DIRECTIVE: {
        const int64_t reps = a.i[2] > 1 ? a.i[2] : 1;  // executions this action stands for
        cnt.directive_execs.fetch_add(reps, std::memory_order_relaxed);
        cnt.var_transfers.fetch_add(reps * a.i[0] * (a.i[1] ? 2 : 1), std::memory_order_relaxed);
        break;
      }
      case ACCT_A_H2D:
      case ACCT_A_D2H: {
        if (!check_slot(a.a[0])) return fail(ACCT_EINVAL, "schedule: bad slot");
        acct_array_t &x = arrays[a.a[0]];
        // images [first, first + n) of the slot: device view b at dev + b * img_stride,
        // host images dense and consecutive; `reps` = transfers this action stands for
        const int64_t first = a.i[0], n = a.i[1] > 1 ? a.i[1] : 1, reps = a.i[2] > 1 ? a.i[2] : 1;
        size_t row = (size_t)x.cols * 4, dp = (size_t)x.ld_dev * 4;
        char *dev0 = static_cast<char *>(x.dev) + first * x.img_stride * 4;
        // image-major copies ([n][rows][ld]) move as one block of n * rows rows
        const bool block = n == 1 || x.img_stride == x.rows * x.ld_dev;
        const int64_t rows = block ? n * x.rows : x.rows;
        // staging only where the pitched copy is slow: H2D rows < 4 KB run at
        // 5-14 GB/s as 2-D copies vs ~50 GB/s dense (tools/xfer_probe.py);
        // D2H 2-D copies stay >= 30 GB/s down to 676-B rows, so never staged
        const bool staged = a.kind == ACCT_A_H2D && x.stage && x.ld_dev != x.cols && row < 4096;
        const int64_t h2d0 = cnt.h2d_calls.load(), d2h0 = cnt.d2h_calls.load();
        for (int64_t b = 0; b < (block ? 1 : n) && rc == ACCT_OK; ++b) {
          char *dev = dev0 + b * x.img_stride * 4;
          char *host = static_cast<char *>(x.host) + b * x.rows * x.cols * 4;
          if (a.kind == ACCT_A_H2D) {
            acct_stream_t on = stream;
            if (defer && in_prefix) {
              if (!forked) {
                if ((rc = check_cuda(cudaEventRecord(side->fork, s), "side fork record"))) return rc;
                if ((rc = check_cuda(cudaStreamWaitEvent(side->t, side->fork, 0), "side fork wait")))
                  return rc;
                forked = true;
              }
              on = reinterpret_cast<acct_stream_t>(side->t);
            } else {
              // each array owns its staging region: only this array's own
              // side-stream copy (need) can still be using it
              if ((rc = need(a.a[0]))) return rc;
            }
            rc = staged ? acct_h2d_staged(dev, x.ld_dev, host, rows, x.cols, x.stage, on)
                        : acct_memcpy2d(dev, dp, host, row, row, (size_t)rows, 1, on);
            if (rc == ACCT_OK && on != stream) {
              rc = check_cuda(cudaEventRecord(side->ev[a.a[0]], side->t), "side event record");
              waiting[a.a[0]] = 1;
            }
          } else if (a.i[3] == 1 && defer) {
            // early copyout on the d2h side stream, ordered after everything
            // issued so far on the main stream
            if ((rc = need(a.a[0]))) return rc;
            if (staged && (rc = side->ensure_dstage((size_t)rows * x.cols * 4, capturing))) return rc;
            if ((rc = check_cuda(cudaEventRecord(side->dfork, s), "d2h fork record"))) return rc;
            if ((rc = check_cuda(cudaStreamWaitEvent(side->d, side->dfork, 0), "d2h fork wait")))
              return rc;
            dforked = true;
            acct_stream_t on = reinterpret_cast<acct_stream_t>(side->d);
            rc = staged ? acct_d2h_staged(host, dev, x.ld_dev, rows, x.cols, side->dstage, on)
                        : acct_memcpy2d(host, row, dev, dp, row, (size_t)rows, 2, on);
          } else {
            if ((rc = need(a.a[0]))) return rc;
            if (staged && (rc = join_all())) return rc;
            rc = staged ? acct_d2h_staged(host, dev, x.ld_dev, rows, x.cols, x.stage, stream)
                        : acct_memcpy2d(host, row, dev, dp, row, (size_t)rows, 2, stream);
          }
        }
        // count the transfers the action stands for, not the memcpy calls it took
        if (a.kind == ACCT_A_H2D) cnt.h2d_calls.store(h2d0 + reps);
        else cnt.d2h_calls.store(d2h0 + reps);
        pending = true;
        break;
      }
      case ACCT_A_H2D_GATHER: {
        const int n = (int)a.i[0];
        if (n < 1 || n > 12 || !a.base || !a.i[13]) return fail(ACCT_EINVAL, "schedule: bad gather");
        GatherSet set{};
        set.n = n;
        char *host0 = static_cast<char *>(a.base);
        int64_t span = 0, bytes = 0, maxc = 1, maxr = 1;
        for (int k = 0; k < n; ++k) {
          const int sl = (int)a.i[1 + k];
          if (!check_slot(sl)) return fail(ACCT_EINVAL, "schedule: bad gather slot");
          acct_array_t &x = arrays[sl];
          const int64_t off = static_cast<char *>(x.host) - host0;
          if (off < 0 || off % 4) return fail(ACCT_EINVAL, "schedule: gather member outside range");
          set.m[k] = {off / 4, static_cast<uint32_t *>(x.dev), x.rows, x.cols, x.ld_dev};
          span = std::max(span, off + x.rows * x.cols * 4);
          bytes += x.rows * x.cols * 4;
          maxc = std::max(maxc, x.cols);
          maxr = std::max(maxr, x.rows);
        }
        cudaStream_t on = s;
        if (defer && in_prefix) {
          if (!forked) {
            if ((rc = check_cuda(cudaEventRecord(side->fork, s), "side fork record"))) return rc;
            if ((rc = check_cuda(cudaStreamWaitEvent(side->t, side->fork, 0), "side fork wait")))
              return rc;
            forked = true;
          }
          on = side->t;
        } else {
          for (int k = 0; k < n; ++k)
            if ((rc = need((int)a.i[1 + k]))) return rc;
        }
        void *stage = reinterpret_cast<void *>(a.i[13]);
        if ((rc = check_cuda(cudaMemcpyAsync(stage, host0, (size_t)span, cudaMemcpyHostToDevice, on),
                             "gather: copy")))
          return rc;
        const unsigned gx = (unsigned)std::min<int64_t>((maxc + 255) / 256, 64);
        const unsigned gy = (unsigned)std::min<int64_t>(maxr, 512);
        launch(gather_scatter_kernel, dim3(gx, gy, (unsigned)n), dim3(256), 0, on,
               static_cast<const uint32_t *>(stage), set);
        if ((rc = note_launch("gather scatter"))) return rc;
        cnt.h2d_calls.fetch_add(n);
        cnt.h2d_bytes.fetch_add(bytes);
        if (on != s) {
          for (int k = 0; k < n; ++k) {
            const int sl = (int)a.i[1 + k];
            if ((rc = check_cuda(cudaEventRecord(side->ev[sl], on), "gather event"))) return rc;
            waiting[sl] = 1;
          }
        }
        pending = true;
        break;
      }
      case ACCT_A_BIND: {
        if (!check_slot(a.a[0]) || a.i[0] >= (int64_t)loops.size()) return fail(ACCT_EINVAL, "schedule: bad bind");
        int64_t lv = loops[(size_t)a.i[0]].counter;
        void *p = static_cast<char *>(a.base) + lv * a.i[1];
        if (a.i[2]) arrays[a.a[0]].dev = p;
        else arrays[a.a[0]].host = p;
        break;
      }
      case ACCT_A_STORE: {
        if (!check_slot(a.a[0]) || a.i[0] >= (int64_t)loops.size()) return fail(ACCT_EINVAL, "schedule: bad store");
        rc = drain();
        if (rc) return rc;
        int64_t lv = loops[(size_t)a.i[0]].counter;
        char *dst = static_cast<char *>(a.base) + lv * a.i[1];
        if (dst != arrays[a.a[0]].host) {
          if (capturing) return fail(ACCT_ENOTSUP, "schedule capture: store_output needs a host copy");
          memcpy(dst, arrays[a.a[0]].host, (size_t)a.i[2]);
        }
        break;
      }
      case ACCT_A_KERNEL:
        for (int j = 0; j < 4 && forked; ++j)
          if ((rc = need(a.a[j]))) return rc;
        if (a.i[0] == ACCT_K_CONV && forked &&
            ((rc = need((int)a.i[7])) || (rc = need((int)a.i[9])) || (rc = need((int)a.i[10]))))
          return rc;  // bias; fused maxpool outputs
        if (prof) {
          size_t first = prof->used;
          cudaEvent_t e0 = prof->next(), e1 = prof->next();
          cudaEventRecord(e0, s);
          rc = device_op(a, arrays, gemm_mode, s);
          cudaEventRecord(e1, s);
          prof->marks.emplace_back(pc, first);
        } else {
          rc = device_op(a, arrays, gemm_mode, s);
        }
        pending = true;
        break;
      case ACCT_A_HOST:
        if (capturing) return fail(ACCT_ENOTSUP, "schedule capture: host loop in schedule");
        rc = drain();
        if (rc) return rc;
        rc = host_op(a, arrays);
        break;
      case ACCT_A_SYNC:
        rc = drain();
        break;
      /* LOOP_END timeout check above; H2D/D2H/KERNEL set `pending` */
      default:
        return fail(ACCT_EINVAL, "schedule: unknown action");
    }
    if (rc != ACCT_OK) return rc;
    if (trace0 && (a.kind == ACCT_A_H2D || a.kind == ACCT_A_D2H || a.kind == ACCT_A_KERNEL))
      mark(pc, a);
    ++pc;
  }
  const int rc = drain();  // host-only schedules never touch the CUDA runtime
  dump();
  return rc;
}

}  // namespace

// ---------------------------------------------------------------- graphs

struct acct_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  acct_counters_t delta{};
};

extern "C" int acct_schedule_capture(acct_array_t *arrays, int n_arrays,
                                     const acct_action_t *actions, int n_actions, int gemm_mode,
                                     acct_stream_t stream, acct_graph_t **out) {
  if (!out) return fail(ACCT_EINVAL, "capture: null output");
  *out = nullptr;
  for (int k = 0; k < n_actions; ++k)
    if (actions[k].kind == ACCT_A_HOST) return ACCT_ENOTSUP;
  cudaStream_t s = as_stream(stream);
  acct_counters_t before, after;
  acct_counters_get(&before);
  if (int rc = check_cuda(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal),
                          "capture: begin"))
    return rc;
  int rc = run_schedule(arrays, n_arrays, actions, n_actions, gemm_mode, 0.0, stream, nullptr,
                        /*capturing=*/true);
  cudaGraph_t graph = nullptr;
  cudaError_t end = cudaStreamEndCapture(s, &graph);
  if (rc != ACCT_OK || end != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return rc != ACCT_OK ? rc : check_cuda(end, "capture: end");
  }
  acct_counters_get(&after);
  auto *g = new acct_graph();
  g->graph = graph;
  if (int irc = check_cuda(cudaGraphInstantiate(&g->exec, graph, 0), "capture: instantiate")) {
    cudaGraphDestroy(graph);
    delete g;
    return irc;
  }
  g->delta.directive_execs = after.directive_execs - before.directive_execs;
  g->delta.var_transfers = after.var_transfers - before.var_transfers;
  g->delta.h2d_calls = after.h2d_calls - before.h2d_calls;
  g->delta.d2h_calls = after.d2h_calls - before.d2h_calls;
  g->delta.h2d_bytes = after.h2d_bytes - before.h2d_bytes;
  g->delta.d2h_bytes = after.d2h_bytes - before.d2h_bytes;
  g->delta.kernel_launches = after.kernel_launches - before.kernel_launches;
  g->delta.host_ops = 0;
  // the capture only recorded work: take its counts back out
  Counters &c = counters();
  c.directive_execs -= g->delta.directive_execs;
  c.var_transfers -= g->delta.var_transfers;
  c.h2d_calls -= g->delta.h2d_calls;
  c.d2h_calls -= g->delta.d2h_calls;
  c.h2d_bytes -= g->delta.h2d_bytes;
  c.d2h_bytes -= g->delta.d2h_bytes;
  c.kernel_launches -= g->delta.kernel_launches;
  *out = g;
  return ACCT_OK;
}

extern "C" int acct_graph_replay(acct_graph_t *g, acct_stream_t stream, int synchronize) {
  if (!g || !g->exec) return fail(ACCT_EINVAL, "replay: null graph");
  cudaStream_t s = as_stream(stream);
  if (int rc = check_cuda(cudaGraphLaunch(g->exec, s), "replay: launch")) return rc;
  Counters &c = counters();
  c.directive_execs += g->delta.directive_execs;
  c.var_transfers += g->delta.var_transfers;
  c.h2d_calls += g->delta.h2d_calls;
  c.d2h_calls += g->delta.d2h_calls;
  c.h2d_bytes += g->delta.h2d_bytes;
  c.d2h_bytes += g->delta.d2h_bytes;
  c.kernel_launches += g->delta.kernel_launches;
  if (synchronize) return check_cuda(cudaStreamSynchronize(s), "replay: sync");
  return ACCT_OK;
}

extern "C" void acct_graph_destroy(acct_graph_t *g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
}
