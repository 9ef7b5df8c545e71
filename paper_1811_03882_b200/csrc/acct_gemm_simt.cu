// gemm_nn on CUDA cores (FP32 FMA): the `mode = SIMT` path and the kernels
// for shapes the tensor-core path does not take (M < 64, or K % 4 / pitch
// misalignment that TMA cannot describe).
//
//   C[M][N] = beta*C + alpha*(A . B)  (+ bias[row]) (leaky)
//
// Two kernels:
//   * tile kernel: 128x128 CTA tile, BK = 8, 256 threads, 8x8 outputs per
//     thread, register-staged double buffering through shared memory;
//   * skinny kernel (M <= 32): one thread per output column keeps all M
//     accumulators in registers and streams B once -- the first conv layer
//     (M = 16, K = 27, N = 173056) is a pure HBM stream of B and C.
// Both accumulate each output in k order within a thread (the tile kernel
// in BK chunks), so results differ from the host i-k-j loop only by FMA
// contraction; parity is checked to the 1e-4 relative tolerance.

#include <cfloat>

#include "acct_common.cuh"

namespace {

__device__ __forceinline__ float epilogue(float acc, float alpha, float beta, const float *cptr,
                                          const float *bias, int row, int act) {
  float v = alpha * acc;
  if (beta != 0.0f) v = beta * (*cptr) + v;
  if (bias) v += __ldg(bias + row);
  if (act == ACCT_ACT_LEAKY) v = acct_leaky(v);
  return v;
}

constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8;

__global__ void __launch_bounds__(256)
gemm_tile_kernel(int M, int N, int K, float alpha, const float *__restrict__ A, int64_t lda,
                 const float *__restrict__ B, int64_t ldb, float beta, float *__restrict__ C,
                 int64_t ldc, const float *__restrict__ bias, int act) {
  pdl_trigger();
  pdl_wait();
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;

  // loaders: A tile 128x8 -> each thread 4 elems (row = tid/2, k = (tid%2)*4 ..+3)
  const int a_row = tid / 2, a_k = (tid % 2) * 4;
  // B tile 8x128 -> each thread 4 elems (k = tid/32, col = (tid%32)*4 ..+3)
  const int b_k = tid / 32, b_col = (tid % 32) * 4;

  float ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int gr = m0 + a_row, gk = k0 + a_k + e;
      ra[e] = (gr < M && gk < K) ? __ldg(A + (int64_t)gr * lda + gk) : 0.0f;
      int bk = k0 + b_k, bc = n0 + b_col + e;
      rb[e] = (bk < K && bc < N) ? __ldg(B + (int64_t)bk * ldb + bc) : 0.0f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 4; ++e) As[buf][a_k + e][a_row] = ra[e];
    *reinterpret_cast<float4 *>(&Bs[buf][b_k][b_col]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  load(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += BK) {
    const bool more = k0 + BK < K;
    if (more) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
      float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 4]);
      float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][kk][64 + ty * 4]);
      float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4]);
      float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) {
      stash(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (c >= N) continue;
      float *cp = C + (int64_t)r * ldc + c;
      *cp = epilogue(acc[i][j], alpha, beta, cp, bias, r, act);
    }
  }
}

// M <= MAXM: A (M x K) staged whole in shared memory (dynamic), one thread per
// output column.
template <int MAXM>
__global__ void __launch_bounds__(128)
gemm_skinny_kernel(int M, int N, int K, float alpha, const float *__restrict__ A, int64_t lda,
                   const float *__restrict__ B, int64_t ldb, float beta, float *__restrict__ C,
                   int64_t ldc, const float *__restrict__ bias, int act) {
  extern __shared__ float As[];  // [K][MAXM]
  pdl_trigger();
  pdl_wait();
  for (int t = threadIdx.x; t < K * MAXM; t += blockDim.x) {
    int k = t / MAXM, m = t % MAXM;
    As[t] = m < M ? A[(int64_t)m * lda + k] : 0.0f;
  }
  __syncthreads();
  for (int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; col < N;
       col += (int64_t)gridDim.x * blockDim.x) {
    float acc[MAXM];
#pragma unroll
    for (int m = 0; m < MAXM; ++m) acc[m] = 0.0f;
    const float *bp = B + col;
    for (int k = 0; k < K; ++k) {
      const float b = __ldcs(bp + (int64_t)k * ldb);
      const float4 *ak = reinterpret_cast<const float4 *>(As + k * MAXM);
#pragma unroll
      for (int q = 0; q < MAXM / 4; ++q) {
        float4 a = ak[q];
        acc[4 * q + 0] = fmaf(a.x, b, acc[4 * q + 0]);
        acc[4 * q + 1] = fmaf(a.y, b, acc[4 * q + 1]);
        acc[4 * q + 2] = fmaf(a.z, b, acc[4 * q + 2]);
        acc[4 * q + 3] = fmaf(a.w, b, acc[4 * q + 3]);
      }
    }
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
      if (m < M) {
        float *cp = C + (int64_t)m * ldc + col;
        __stcs(cp, epilogue(acc[m], alpha, beta, cp, bias, m, act));
      }
    }
  }
}

// HBM-streaming gemm for M <= MT (the first conv layers: M = 16 / 32, K <= a
// few hundred, N up to millions of pixels x images): the whole A (M x K) sits
// in shared memory as [K][MT] so each k reads MT weights as broadcast float4s,
// each thread owns 4 consecutive columns (one float4 of B per k, coalesced
// 512-B warp rows), keeps 4 x MT accumulators in registers and issues KU
// B loads before using any -- the kernel is a pure stream of B in and C out.
// Per output the k loop runs in order (as the tile kernel), so results differ
// from the host loop only by FMA contraction.
template <int MT, int KU>
__global__ void __launch_bounds__(128)
gemm_stream_kernel(int M, int N, int K, float alpha, const float *__restrict__ A, int64_t lda,
                   const float *__restrict__ B, int64_t ldb, float beta, float *__restrict__ C,
                   int64_t ldc, const float *__restrict__ bias, int act) {
  extern __shared__ float4 As4[];  // [K][MT/4]
  float *As = reinterpret_cast<float *>(As4);
  pdl_trigger();
  pdl_wait();
  for (int t = threadIdx.x; t < K * MT; t += blockDim.x) {
    const int k = t / MT, m = t - k * MT;
    As[t] = m < M ? A[(int64_t)m * lda + k] : 0.0f;
  }
  __syncthreads();
  const int nq = (N + 3) >> 2;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    const int col = q * 4;
    const bool full = col + 4 <= N;
    float acc[MT][4];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.0f;
    const float *bp = B + col;
    for (int k0 = 0; k0 < K; k0 += KU) {
      float4 b[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = k0 + u;
        if (k < K) {
          if (full) {
            b[u] = __ldcs(reinterpret_cast<const float4 *>(bp + (int64_t)k * ldb));
          } else {
            const float *r = bp + (int64_t)k * ldb;
            b[u] = make_float4(r[0], col + 1 < N ? r[1] : 0.0f, col + 2 < N ? r[2] : 0.0f, 0.0f);
          }
        } else {
          b[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        if (k0 + u >= K) break;
        const float4 *ak = As4 + (k0 + u) * (MT / 4);
#pragma unroll
        for (int g = 0; g < MT / 4; ++g) {
          const float4 a = ak[g];
          const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[4 * g + e][0] = fmaf(av[e], b[u].x, acc[4 * g + e][0]);
            acc[4 * g + e][1] = fmaf(av[e], b[u].y, acc[4 * g + e][1]);
            acc[4 * g + e][2] = fmaf(av[e], b[u].z, acc[4 * g + e][2]);
            acc[4 * g + e][3] = fmaf(av[e], b[u].w, acc[4 * g + e][3]);
          }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      if (m >= M) break;
      float *cp = C + (int64_t)m * ldc + col;
      if (full) {
        float4 cv = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (beta != 0.0f) cv = *reinterpret_cast<const float4 *>(cp);
        float4 o;
        o.x = epilogue(acc[m][0], alpha, beta, &cv.x, bias, m, act);
        o.y = epilogue(acc[m][1], alpha, beta, &cv.y, bias, m, act);
        o.z = epilogue(acc[m][2], alpha, beta, &cv.z, bias, m, act);
        o.w = epilogue(acc[m][3], alpha, beta, &cv.w, bias, m, act);
        __stcs(reinterpret_cast<float4 *>(cp), o);
      } else {
        for (int e = 0; e < 4 && col + e < N; ++e)
          cp[e] = epilogue(acc[m][e], alpha, beta, cp + e, bias, m, act);
      }
    }
  }
}

// 2 columns per thread, KU B rows (float2) in flight before any use: with
// K <= KU (layer 0: K = 27) a thread issues every load of its columns at once,
// so ~8x more bytes are in flight per SM than with 4 columns x 8 rows.
template <int MT, int KU>
__global__ void __launch_bounds__(128)
gemm_stream2_kernel(int M, int N, int K, float alpha, const float *__restrict__ A, int64_t lda,
                    const float *__restrict__ B, int64_t ldb, float beta, float *__restrict__ C,
                    int64_t ldc, const float *__restrict__ bias, int act) {
  extern __shared__ float4 As4[];  // [K][MT/4]
  float *As = reinterpret_cast<float *>(As4);
  pdl_trigger();
  pdl_wait();
  for (int t = threadIdx.x; t < K * MT; t += blockDim.x) {
    const int k = t / MT, m = t - k * MT;
    As[t] = m < M ? A[(int64_t)m * lda + k] : 0.0f;
  }
  __syncthreads();
  const int np = (N + 1) >> 1;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < np; q += gridDim.x * blockDim.x) {
    const int col = q * 2;
    const bool full = col + 2 <= N;
    float acc[MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0f;
    const float *bp = B + col;
    for (int k0 = 0; k0 < K; k0 += KU) {
      float2 b[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = k0 + u;
        if (k < K) {
          const float *r = bp + (int64_t)k * ldb;
          b[u] = full ? __ldcs(reinterpret_cast<const float2 *>(r)) : make_float2(r[0], 0.0f);
        } else {
          b[u] = make_float2(0.0f, 0.0f);
        }
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        if (k0 + u >= K) break;
        const float4 *ak = As4 + (k0 + u) * (MT / 4);
#pragma unroll
        for (int g = 0; g < MT / 4; ++g) {
          const float4 a = ak[g];
          const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[4 * g + e][0] = fmaf(av[e], b[u].x, acc[4 * g + e][0]);
            acc[4 * g + e][1] = fmaf(av[e], b[u].y, acc[4 * g + e][1]);
          }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      if (m >= M) break;
      float *cp = C + (int64_t)m * ldc + col;
      if (full) {
        float2 cv = make_float2(0.0f, 0.0f);
        if (beta != 0.0f) cv = *reinterpret_cast<const float2 *>(cp);
        float2 o;
        o.x = epilogue(acc[m][0], alpha, beta, &cv.x, bias, m, act);
        o.y = epilogue(acc[m][1], alpha, beta, &cv.y, bias, m, act);
        __stcs(reinterpret_cast<float2 *>(cp), o);
      } else {
        cp[0] = epilogue(acc[m][0], alpha, beta, cp, bias, m, act);
      }
    }
  }
}

int stream_variant() {
  static const int v = [] {
    const char *e = getenv("ACCT_STREAM");
    return e ? atoi(e) : 0;  // 0: 4 columns/thread at M <= 16, 2 at M <= 32
  }();
  return v;
}

template <int MT>
int launch_stream(int M, int N, int K, float alpha, const float *A, int64_t lda, const float *B,
                  int64_t ldb, float beta, float *C, int64_t ldc, const float *bias, int act,
                  cudaStream_t s) {
  const size_t smem = (size_t)K * MT * sizeof(float);
  // M = 32: two columns per thread (64 accumulators) keeps 4+ CTAs per SM
  constexpr int KU2 = MT <= 16 ? 32 : 8;
  if (stream_variant() == 2 || (MT > 16 && stream_variant() != 1)) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(gemm_stream2_kernel<MT, KU2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
    const int64_t np = (N + 1) / 2;
    unsigned grid = acct::grid_for(np, 128, 8);
    acct::launch(gemm_stream2_kernel<MT, KU2>, dim3(grid), dim3(128), smem, s, M, N, K, alpha, A,
                 lda, B, ldb, beta, C, ldc, bias, act);
    return acct::note_launch("gemm_stream");
  }
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(gemm_stream_kernel<MT, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const int64_t nq = (N + 3) / 4;
  const int block = 128;
  unsigned grid = acct::grid_for(nq, block, MT <= 16 ? 8 : 4);
  acct::launch(gemm_stream_kernel<MT, 8>, dim3(grid), dim3(block), smem, s, M, N, K, alpha, A, lda,
               B, ldb, beta, C, ldc, bias, act);
  return acct::note_launch("gemm_stream");
}

// im2col (3x3 / stride 1 / pad 1) fused with its gemm_nn for the narrow conv
// layers (M <= 32 filters, channels <= 64: K = 9 C <= 576 col rows; the
// first two yolov2-tiny layers).
//
// A CTA owns tiles of P = 128 x PX consecutive output pixels (flat h*w
// index; images are consecutive tile ranges).  For a tile it stages, per
// input channel, the flat input range [p0 - W - 1, p0 + P + W] (rows above,
// the tile's rows, rows below) into shared memory with 16-byte cp.async --
// out-of-plane chunks are zero, which is the conv's row padding -- double
// buffered so the next tile's loads overlap this tile's FMAs.  A thread owns
// PX pixels of one row: per channel it reads its 3 x (PX+2) window from
// shared memory (column padding masked at w = 0 / W-1), stores the 9 col
// rows of its pixels and accumulates the M x PX outputs in k order -- the FMA
// chain of every SIMT gemm over the materialised col (k ascending from 0,
// then the shared epilogue), so C is bit-identical to im2col + the SIMT gemm
// -- without re-reading col.  A is staged once per CTA as [k][m] (one
// broadcast LDS.128 per 4 filters).  Images below `col_from` skip the col
// stores (the executor passes batch-1 when only the last image's col is
// observable: dead stores of a privatised array, see executor._col_dead).
template <int PX>
struct VecOf;
template <>
struct VecOf<4> {
  using T = float4;
};
template <>
struct VecOf<2> {
  using T = float2;
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}

constexpr int CONV_THREADS = 128;

__host__ __device__ constexpr int conv_stage_floats(int px, int width) {
  return (CONV_THREADS * px + 2 * width + 5 + 3) & ~3;  // [p0-W-1 floored to 4, p0+P+W]
}

template <int MT, int PX, int MINB>
__global__ void __launch_bounds__(CONV_THREADS, MINB)
conv3x3_im2col_gemm_kernel(const float *__restrict__ im, int64_t ld_im, int64_t im_bs,
                           int channels, int height, int width, float *__restrict__ col,
                           int64_t ld_col, int64_t col_bs, int col_from, int M,
                           const float *__restrict__ A, int64_t lda, float beta,
                           float *__restrict__ C, int64_t ldc, int64_t c_bs,
                           const float *__restrict__ bias, int act, int tiles_per_img,
                           int ntiles) {
  using V = typename VecOf<PX>::T;
  constexpr int P = CONV_THREADS * PX;
  extern __shared__ float4 conv_smem[];
  const int K = channels * 9;
  const int ls = conv_stage_floats(PX, width);
  float *As = reinterpret_cast<float *>(conv_smem);  // [k][MT]
  float *sin0 = As + K * MT;                         // 2 x [channels][ls]
  const int bufsz = channels * ls;
  const int HW = height * width;
  pdl_trigger();
  pdl_wait();

  auto stage = [&](int tile, float *buf) {
    const int img = tile / tiles_per_img;
    const int p0 = (tile - img * tiles_per_img) * P;
    const int a0 = (p0 - width - 1) & ~3;  // floor to a 16-byte chunk
    const float *src = im + img * im_bs;
    const int nq = ls >> 2;
    for (int j = threadIdx.x; j < channels * nq; j += CONV_THREADS) {
      const int ci = j / nq, q = j - ci * nq;
      const int g = a0 + 4 * q;  // HW % 4 == 0: a chunk is wholly inside or outside
      float *dst = buf + ci * ls + 4 * q;
      if (g >= 0 && g < HW)
        cp_async16(dst, src + ci * ld_im + g);
      else
        *reinterpret_cast<float4 *>(dst) = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
  };

  int tile = blockIdx.x;
  if (tile < ntiles) stage(tile, sin0);
  cp_async_commit();
  for (int t = threadIdx.x; t < K * MT; t += CONV_THREADS) {
    const int k = t / MT, m = t - k * MT;
    As[t] = m < M ? A[(int64_t)m * lda + k] : 0.0f;
  }
  int buf = 0;
  for (; tile < ntiles; tile += gridDim.x) {
    const int nxt = tile + gridDim.x;
    if (nxt < ntiles) stage(nxt, sin0 + (buf ^ 1) * bufsz);
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    const int img = tile / tiles_per_img;
    const int p0 = (tile - img * tiles_per_img) * P;
    const int p = p0 + threadIdx.x * PX;
    if (p < HW) {
      const int h = p / width, w0 = p - h * width;
      const bool wcol = img >= col_from;
      float *colp = col + img * col_bs + p;
      const float *base = sin0 + buf * bufsz + (p - ((p0 - width - 1) & ~3));
      float acc[MT][PX];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int e = 0; e < PX; ++e) acc[m][e] = 0.0f;
#pragma unroll 1
      for (int ci = 0; ci < channels; ++ci) {
        const float *cb = base + ci * ls;
        float win[3][PX + 2];
#pragma unroll
        for (int kh = 0; kh < 3; ++kh) {
          const float *row = cb + (kh - 1) * width - 1;
#pragma unroll
          for (int j = 0; j < PX + 2; ++j) win[kh][j] = row[j];
          if (w0 == 0) win[kh][0] = 0.0f;
          if (w0 + PX == width) win[kh][PX + 1] = 0.0f;
        }
#pragma unroll
        for (int kh = 0; kh < 3; ++kh) {
#pragma unroll
          for (int kw = 0; kw < 3; ++kw) {
            const int k = ci * 9 + kh * 3 + kw;
            V v;
            float *vf = reinterpret_cast<float *>(&v);
#pragma unroll
            for (int e = 0; e < PX; ++e) vf[e] = win[kh][kw + e];
            if (wcol) __stcs(reinterpret_cast<V *>(colp + (int64_t)k * ld_col), v);
            const float4 *ak = reinterpret_cast<const float4 *>(As + k * MT);
#pragma unroll
            for (int m4 = 0; m4 < MT / 4; ++m4) {
              const float4 a = ak[m4];
#pragma unroll
              for (int e = 0; e < PX; ++e) {
                acc[4 * m4 + 0][e] = fmaf(a.x, vf[e], acc[4 * m4 + 0][e]);
                acc[4 * m4 + 1][e] = fmaf(a.y, vf[e], acc[4 * m4 + 1][e]);
                acc[4 * m4 + 2][e] = fmaf(a.z, vf[e], acc[4 * m4 + 2][e]);
                acc[4 * m4 + 3][e] = fmaf(a.w, vf[e], acc[4 * m4 + 3][e]);
              }
            }
          }
        }
      }
      float *cimg = C + img * c_bs + p;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (m >= M) break;
        V *cp = reinterpret_cast<V *>(cimg + (int64_t)m * ldc);
        V cv{}, o;
        if (beta != 0.0f) cv = *cp;
        const float *cvf = reinterpret_cast<const float *>(&cv);
        float *of = reinterpret_cast<float *>(&o);
#pragma unroll
        for (int e = 0; e < PX; ++e)
          of[e] = epilogue(acc[m][e], 1.0f, beta, cvf + e, bias, m, act);
        __stcs(cp, o);
      }
    }
    __syncthreads();  // this buffer is restaged two tiles later
    buf ^= 1;
  }
}

template <int MT, int PX, int MINB>
int launch_conv(int batch, cudaStream_t s, const float *im, int64_t ld_im, int64_t im_stride,
                int channels, int height, int width, float *col, int64_t ld_col,
                int64_t col_stride, int col_from, int M, const float *A, int64_t lda, float beta,
                float *C, int64_t ldc, int64_t c_stride, const float *bias, int act) {
  auto *k = conv3x3_im2col_gemm_kernel<MT, PX, MINB>;
  const size_t smem = sizeof(float) * ((size_t)channels * 9 * MT +
                                       2 * (size_t)channels * conv_stage_floats(PX, width));
  if (smem > 227 * 1024) return ACCT_ENOTSUP;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
    return acct::check_cuda(cudaGetLastError(), "conv3x3 fused: smem attribute");
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, CONV_THREADS, smem);
  if (per_sm < 1) per_sm = 1;
  const int P = CONV_THREADS * PX;
  const int64_t tpi = ((int64_t)height * width + P - 1) / P;
  const int64_t ntiles = tpi * batch;
  if (ntiles > INT32_MAX) return ACCT_ENOTSUP;
  int64_t grid = (int64_t)acct::sm_count() * per_sm;
  if (grid > ntiles) grid = ntiles;
  acct::launch(k, dim3((unsigned)grid), dim3(CONV_THREADS), smem, s, im, ld_im, im_stride,
               channels, height, width, col, ld_col, col_stride, col_from, M, A, lda, beta, C, ldc,
               c_stride, bias, act, (int)tpi, (int)ntiles);
  return ACCT_OK;
}

}  // namespace

namespace {

// The same fused conv with its 2x2/2 maxpool (first layers: M <= 16).  A
// thread owns a 2x2 pixel block -- one maxpool window -- of a 32 x 16 tile
// (16 x 8 threads), so the pool is in-thread: per filter the four finished
// values are compared in darknet's scan order (strict '>', from -FLT_MAX)
// and the argmax is the flat index into the image's C plane.  The tile's
// (16 + 2) x (32 + 2) input window per channel is staged by cp.async from a
// 16-byte aligned column x0 - 4 (rows / columns outside the image are zero),
// double-buffered across tiles.  k order and FMA chain are those of the
// window kernel (bit-identical C); C and col are stored for images >=
// c_from / col_from only.
constexpr int PT_W = 32, PT_H = 16, PT_SW = PT_W + 8, PT_SH = PT_H + 2;  // slab row 40 floats

// packed FP32 pairs (sm_100 FFMA2): two IEEE fmas per instruction, each
// rounding exactly like fmaf -- halves the issue slots of an FMA-issue-bound
// loop without changing a single result
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pack2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(f32x2 v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// BETA: beta != 0 (C += ...) -- a template flag, so the usual beta = 0 launch
// carries no per-filter C address arithmetic or predicated C loads (ncu: 26%
// of the kernel's stall samples when they were runtime-predicated)
template <bool BETA>
__global__ void __launch_bounds__(128, 4)
conv3x3_pool_kernel(const float *__restrict__ im, int64_t ld_im, int64_t im_bs, int channels,
                    int height, int width, float *__restrict__ col, int64_t ld_col,
                    int64_t col_bs, int col_from, int M, const float *__restrict__ A, int64_t lda,
                    float beta, float *__restrict__ C, int64_t ldc, int64_t c_bs,
                    const float *__restrict__ bias, int act, float *__restrict__ pool,
                    int64_t ld_pool, int64_t pool_bs, int32_t *__restrict__ pidx,
                    int64_t ld_pidx, int64_t pidx_bs, int c_from, int tiles_x, int tpi,
                    int ntiles, float inv_tpi, float inv_tiles_x) {
  constexpr int MT = 16;
  const int m_off = blockIdx.y * MT;  // this CTA's 16-filter block
  extern __shared__ float4 conv_smem[];
  const int K = channels * 9;
  float *As = reinterpret_cast<float *>(conv_smem);  // [k][MT]
  float *Bs = As + K * MT;                           // [MT] bias (0 past M)
  float *sin0 = Bs + MT;                             // 2 x [channels][PT_SH][PT_SW]
  const int bufsz = channels * PT_SH * PT_SW;
  pdl_trigger();
  pdl_wait();

  // (the integer divisions were 10% of the kernel's stall samples)
  auto tile_xy = [&](int tile, int &img, int &y0, int &x0) {
    int t, ty, tx;
    acct_divmod(tile, tpi, inv_tpi, img, t);
    acct_divmod(t, tiles_x, inv_tiles_x, ty, tx);
    y0 = ty * PT_H;
    x0 = tx * PT_W;
  };
  auto stage = [&](int tile, float *buf) {
    int img, y0, x0;
    tile_xy(tile, img, y0, x0);
    const float *src = im + img * im_bs;
    constexpr int NQ = PT_SW / 4;  // 16-byte chunks per slab row
    for (int j = threadIdx.x; j < channels * PT_SH * NQ; j += 128) {
      const int q = j % NQ, rr = (j / NQ) % PT_SH, ci = j / (NQ * PT_SH);
      const int gy = y0 - 1 + rr, gx = x0 - 4 + 4 * q;  // width % 4 == 0: whole chunks
      float *dst = buf + (ci * PT_SH + rr) * PT_SW + 4 * q;
      if (gy >= 0 && gy < height && gx >= 0 && gx < width)
        cp_async16(dst, src + ci * ld_im + (int64_t)gy * width + gx);
      else
        *reinterpret_cast<float4 *>(dst) = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
  };

  int tile = blockIdx.x;
  if (tile < ntiles) stage(tile, sin0);
  cp_async_commit();
  for (int t = threadIdx.x; t < K * MT; t += 128) {
    const int k = t / MT, m = t - k * MT;
    As[t] = m_off + m < M ? A[(int64_t)(m_off + m) * lda + k] : 0.0f;
  }
  if (threadIdx.x < MT)
    Bs[threadIdx.x] = bias && m_off + threadIdx.x < M ? bias[m_off + threadIdx.x] : 0.0f;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  int buf = 0;
  for (; tile < ntiles; tile += gridDim.x) {
    const int nxt = tile + gridDim.x;
    if (nxt < ntiles) stage(nxt, sin0 + (buf ^ 1) * bufsz);
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    int img, y0, x0;
    tile_xy(tile, img, y0, x0);
    const int y = y0 + 2 * ty, x = x0 + 2 * tx;
    if (y < height && x < width) {  // even planes: the whole 2x2 block is inside
      const bool wcol = img >= col_from && blockIdx.y == 0, wc = img >= c_from;
      const int64_t p = (int64_t)y * width + x;
      float *colp = col + img * col_bs + p;
      const float *base = sin0 + buf * bufsz + (2 * ty) * PT_SW + 2 * tx + 3;  // window (-1, -1)
      // acc2[i][e] = (filter 2i, filter 2i+1) at pixel e: one FFMA2 per pair,
      // each element the fmaf chain of the window kernel
      f32x2 acc2[MT / 2][4];
#pragma unroll
      for (int i = 0; i < MT / 2; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc2[i][e] = 0ull;
      const ulonglong2 *As2 = reinterpret_cast<const ulonglong2 *>(As);
      // the next channel's window is loaded while this one's FMAs issue
      float nwin[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) nwin[r][c] = base[r * PT_SW + c];
#pragma unroll 1
      for (int ci = 0; ci < channels; ++ci) {
        float win[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) win[r][c] = nwin[r][c];
        const float *cn = base + (ci + 1 < channels ? ci + 1 : ci) * PT_SH * PT_SW;
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) nwin[r][c] = cn[r * PT_SW + c];
#pragma unroll
        for (int kh = 0; kh < 3; ++kh) {
#pragma unroll
          for (int kw = 0; kw < 3; ++kw) {
            const int k = ci * 9 + kh * 3 + kw;
            const float v0 = win[kh][kw], v1 = win[kh][kw + 1];
            const float v2 = win[kh + 1][kw], v3 = win[kh + 1][kw + 1];
            const f32x2 vv[4] = {pack2(v0, v0), pack2(v1, v1), pack2(v2, v2), pack2(v3, v3)};
#pragma unroll
            for (int g = 0; g < MT / 4; ++g) {
              const ulonglong2 a = As2[k * (MT / 4) + g];  // filters 4g..4g+3 as two pairs
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                acc2[2 * g][e] = fma2(a.x, vv[e], acc2[2 * g][e]);
                acc2[2 * g + 1][e] = fma2(a.y, vv[e], acc2[2 * g + 1][e]);
              }
            }
          }
        }
      }
      if (!BETA && bias) {
        // + bias on the packed pairs (FADD2: the same rounding as the scalar
        // add; filters past M hold 0 + 0)
        const ulonglong2 *Bs2 = reinterpret_cast<const ulonglong2 *>(Bs);
#pragma unroll
        for (int g = 0; g < MT / 4; ++g) {
          const ulonglong2 b = Bs2[g];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc2[2 * g][e] = add2(acc2[2 * g][e], b.x);
            acc2[2 * g + 1][e] = add2(acc2[2 * g + 1][e], b.y);
          }
        }
      }
      float acc[MT][4];
#pragma unroll
      for (int i = 0; i < MT / 2; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) unpack2(acc2[i][e], acc[2 * i][e], acc[2 * i + 1][e]);
      if (wcol) {
        // the col rows of this 2x2 block, for the one image whose col is
        // observable (kept out of the FMA loop: code size, not bytes)
#pragma unroll 1
        for (int ci = 0; ci < channels; ++ci) {
          const float *cb = base + ci * PT_SH * PT_SW;
#pragma unroll
          for (int kh = 0; kh < 3; ++kh)
#pragma unroll
            for (int kw = 0; kw < 3; ++kw) {
              const int64_t k = ci * 9 + kh * 3 + kw;
              __stcs(reinterpret_cast<float2 *>(colp + k * ld_col),
                     make_float2(cb[kh * PT_SW + kw], cb[kh * PT_SW + kw + 1]));
              __stcs(reinterpret_cast<float2 *>(colp + k * ld_col + width),
                     make_float2(cb[(kh + 1) * PT_SW + kw], cb[(kh + 1) * PT_SW + kw + 1]));
            }
        }
      }
      float *cimg = C + img * c_bs + p;
      const int64_t pofs = (int64_t)(y >> 1) * (width >> 1) + (x >> 1);
      const int base_i = (int)p;
      const int plane = height * width;
      if constexpr (BETA) {
        // beta C, then bias, per filter
#pragma unroll
        for (int ml = 0; ml < MT; ++ml) {
          const int m = m_off + ml;
          if (m >= M) break;
          const float *cp = cimg + (int64_t)m * ldc;
          const float2 c0 = *reinterpret_cast<const float2 *>(cp);
          const float2 c1 = *reinterpret_cast<const float2 *>(cp + width);
          const float cv[4] = {c0.x, c0.y, c1.x, c1.y};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float v = beta * cv[e] + acc[ml][e];
            if (bias) v += Bs[ml];
            acc[ml][e] = v;
          }
        }
      }
      // Images whose C is dead (only the pool is observable): pool the raw
      // values and apply leaky to the 16 winners.  leaky is monotone, so the
      // pooled value is leaky(raw max) and darknet's first-max index equals
      // the raw scan's -- unless an earlier element's leaky rounds to the
      // same float (both <= 0 and within ~2^-22 relative) or a value is in
      // leaky's guarded ranges; then (runner-up within 2^-19 of a
      // non-positive max, a guarded winner, or an empty scan: one warp vote)
      // the exact path below runs for the warp.
      bool pooled = false;
      if (act == ACCT_ACT_LEAKY && !wc) {
        float mxv[MT];
        int ev[MT];
        bool slow = false;
#pragma unroll
        for (int ml = 0; ml < MT; ++ml) {
          // the scan from -FLT_MAX takes element 0 first unless it is not
          // above -FLT_MAX (then: exact path)
          float mx = acc[ml][0], v2 = -FLT_MAX;
          int e = 0;
#pragma unroll
          for (int i = 1; i < 4; ++i) {
            const float v = acc[ml][i];
            if (v > mx) {
              v2 = mx;
              mx = v;
              e = i;
            } else {
              v2 = fmaxf(v2, v);
            }
          }
          const float thr = mx <= 0.0f ? fmaf(mx, 0x1p-19f, mx) - 0x1p-100f : FLT_MAX;
          slow |= !(acc[ml][0] > -FLT_MAX) || (v2 < mx && v2 >= thr);
          mxv[ml] = mx;
          ev[ml] = e;
        }
        slow |= acct_leaky_any_guarded(mxv);
        if (!__any_sync(__activemask(), slow)) {
#pragma unroll
          for (int ml = 0; ml < MT; ++ml) {
            const int m = m_off + ml;
            if (m >= M) break;
            const int e = ev[ml];
            pool[img * pool_bs + (int64_t)m * ld_pool + pofs] = acct_leaky_fast(mxv[ml]);
            pidx[img * pidx_bs + (int64_t)m * ld_pidx + pofs] =
                m * plane + base_i + (e & 1) + (e >> 1) * width;
          }
          pooled = true;
        }
      }
      if (!pooled && act == ACCT_ACT_LEAKY)
        acct_leaky_block(reinterpret_cast<float(&)[MT * 4]>(acc));
#pragma unroll
      for (int ml = 0; ml < MT && !pooled; ++ml) {
        const int m = m_off + ml;  // the filter (output row)
        if (m >= M) break;
        float *cp = cimg + (int64_t)m * ldc;
        const float *o = acc[ml];
        if (wc) {
          __stcs(reinterpret_cast<float2 *>(cp), make_float2(o[0], o[1]));
          __stcs(reinterpret_cast<float2 *>(cp + width), make_float2(o[2], o[3]));
        }
        const int bi = m * plane + base_i;
        float mx = -FLT_MAX;
        int32_t kx = -1;
        if (o[0] > mx) { mx = o[0]; kx = bi; }
        if (o[1] > mx) { mx = o[1]; kx = bi + 1; }
        if (o[2] > mx) { mx = o[2]; kx = bi + width; }
        if (o[3] > mx) { mx = o[3]; kx = bi + width + 1; }
        pool[img * pool_bs + (int64_t)m * ld_pool + pofs] = mx;
        pidx[img * pidx_bs + (int64_t)m * ld_pidx + pofs] = kx;
      }
    }
    __syncthreads();  // this buffer is restaged two tiles later
    buf ^= 1;
  }
}

}  // namespace

// C = A . im2col(im) + beta C (+ bias, act) for 3x3/1/1 convolutions with
// channels <= 64 and M <= 32, also writing the col array (images >= col_from
// of the batch); batched over images
extern "C" int acct_conv3x3_im2col_gemm_f32(const float *im, int64_t ld_im, int64_t im_stride,
                                            int channels, int height, int width, float *col,
                                            int64_t ld_col, int64_t col_stride, int M,
                                            const float *A, int64_t lda, float beta, float *C,
                                            int64_t ldc, int64_t c_stride, const float *bias, int act,
                                            int batch, int col_from, float *pool, int64_t ld_pool,
                                            int64_t pool_stride, int32_t *idx, int64_t ld_idx,
                                            int64_t idx_stride, int c_from, acct_stream_t stream) {
  using namespace acct;
  if (pool) {
    // fused 2x2/2 maxpool: 2x2 pixel blocks per thread, 16 filters per CTA
    // (blockIdx.y = filter block), M <= 64
    if (!idx || M > 64 || channels < 1 || channels > 64 || (height | width) & 1 || (width & 3) ||
        col_from < 0 || c_from < 0 || batch < 1 || ld_im < (int64_t)height * width ||
        ld_col < (int64_t)height * width || ldc < (int64_t)height * width ||
        ld_pool < (int64_t)(height / 2) * (width / 2) || ld_idx < (int64_t)(height / 2) * (width / 2) ||
        (reinterpret_cast<uintptr_t>(im) | reinterpret_cast<uintptr_t>(col) |
         reinterpret_cast<uintptr_t>(C)) & 15 ||
        (ld_im | im_stride | ld_col | col_stride | ldc | c_stride) & 3)
      return fail(ACCT_ENOTSUP, "conv3x3 fused: maxpool fusion needs M <= 64, even planes");
    const size_t smem = sizeof(float) * ((size_t)channels * 9 * 16 + 16 +
                                         2 * (size_t)channels * PT_SH * PT_SW);
    if (smem > 200 * 1024) return fail(ACCT_ENOTSUP, "conv3x3 fused: slabs exceed shared memory");
    auto kern = beta != 0.0f ? conv3x3_pool_kernel<true> : conv3x3_pool_kernel<false>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int tiles_x = (width + PT_W - 1) / PT_W, tiles_y = (height + PT_H - 1) / PT_H;
    const int64_t tpi = (int64_t)tiles_x * tiles_y, ntiles = tpi * batch;
    if (ntiles >= (1 << 24)) return fail(ACCT_ENOTSUP, "conv3x3 fused: too many tiles");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem);
    if (per_sm < 1) per_sm = 1;
    const int gy = (M + 15) / 16;
    int64_t grid = ((int64_t)sm_count() * per_sm + gy - 1) / gy;
    if (grid > ntiles) grid = ntiles;
    launch(kern, dim3((unsigned)grid, (unsigned)gy), dim3(128), smem,
           as_stream(stream), im, ld_im,
           im_stride, channels, height, width, col, ld_col, col_stride, col_from, M, A, lda, beta, C,
           ldc, c_stride, bias, act, pool, ld_pool, pool_stride, idx, ld_idx, idx_stride, c_from,
           tiles_x, (int)tpi, (int)ntiles, 1.0f / (float)tpi, 1.0f / (float)tiles_x);
    return note_launch("conv3x3 im2col+gemm+maxpool");
  }
  if (channels < 1 || channels > 64 || M < 1 || M > 32 || height < 1 || width < 1 || batch < 1 ||
      col_from < 0 || (int64_t)height * width > (1 << 28) || ld_im < (int64_t)height * width ||
      ld_col < (int64_t)height * width || ldc < (int64_t)height * width)
    return fail(ACCT_ENOTSUP, "conv3x3 fused: shape not supported");
  if ((reinterpret_cast<uintptr_t>(col) | reinterpret_cast<uintptr_t>(C) |
       reinterpret_cast<uintptr_t>(im)) & 15 ||
      (ld_col | ldc | col_stride | c_stride | ld_im | im_stride | width) & 3)
    return fail(ACCT_ENOTSUP, "conv3x3 fused: needs 16-B aligned rows");
  cudaStream_t s = as_stream(stream);
  int rc;
  if (M <= 16)
    rc = launch_conv<16, 4, 4>(batch, s, im, ld_im, im_stride, channels, height, width, col,
                               ld_col, col_stride, col_from, M, A, lda, beta, C, ldc, c_stride,
                               bias, act);
  else
    rc = launch_conv<32, 2, 4>(batch, s, im, ld_im, im_stride, channels, height, width, col,
                               ld_col, col_stride, col_from, M, A, lda, beta, C, ldc, c_stride,
                               bias, act);
  if (rc == ACCT_ENOTSUP) return fail(ACCT_ENOTSUP, "conv3x3 fused: staging exceeds shared memory");
  if (rc) return rc;
  return note_launch("conv3x3 im2col+gemm");
}

namespace acct {

// M <= 16 with 16-B aligned rows: the streaming kernel (HBM-bound shapes; at
// M = 32 the 128 accumulators per thread cost more occupancy than the stream
// gains -- the tensor-core swap tile is faster there)
int gemm_stream(int M, int N, int K, float alpha, const float *A, int64_t lda, const float *B,
                int64_t ldb, float beta, float *C, int64_t ldc, const float *bias, int act,
                cudaStream_t s) {
  // M <= 16, or M <= 32 with a short K (a 3-channel first layer): beyond
  // that the 4 x 32 accumulators per thread cost more occupancy than the
  // stream gains and the tensor-core swap tile wins
  if (M < 1 || M > 32 || (M > 16 && K > 64) || N < 1 || K < 1 ||
      (int64_t)K * 32 * 4 > 200 * 1024 || (ldb % 4) ||
      (ldc % 4) || (reinterpret_cast<uintptr_t>(B) & 15) || (reinterpret_cast<uintptr_t>(C) & 15))
    return ACCT_ENOTSUP;
  if (M <= 16) return launch_stream<16>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  return launch_stream<32>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
}

int gemm_simt(int M, int N, int K, float alpha, const float *A, int64_t lda, const float *B,
              int64_t ldb, float beta, float *C, int64_t ldc, const float *bias, int act,
              cudaStream_t s) {
  if (M <= 32) {  // gemm_stream declines the shapes it does not fit
    int rc = gemm_stream(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
    if (rc != ACCT_ENOTSUP) return rc;
  }
  if (M <= 32 && (int64_t)K * 32 * 4 <= 200 * 1024) {
    const int block = 128;
    const size_t smem = (size_t)K * 32 * sizeof(float);
    const int maxm = M <= 16 ? 16 : 32;
    unsigned grid = grid_for(N, block, 4);
    if (maxm == 16) {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(gemm_skinny_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      launch(gemm_skinny_kernel<16>, dim3(grid), dim3(block), (size_t)K * 16 * sizeof(float), s, M,
             N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act);
    } else {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(gemm_skinny_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      launch(gemm_skinny_kernel<32>, dim3(grid), dim3(block), smem, s, M, N, K, alpha, A, lda, B,
             ldb, beta, C, ldc, bias, act);
    }
    return note_launch("gemm_skinny");
  }
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  launch(gemm_tile_kernel, grid, dim3(256), 0, s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias,
         act);
  return note_launch("gemm_tile");
}

}  // namespace acct
