// CPU side of an offload pattern: the Darknet loops whose gene is 0 run here,
// natively, on the host copies of the program's arrays.  Same loop order and
// arithmetic as the C-subset program (paper_1811_03882_b200/nets.py) and
// darknet's *_cpu functions, compiled with -ffp-contract=off so a host loop
// gives bit-identical results to the gcc-compiled program.
//
// Single-threaded on purpose: the CPU part of a pattern is the paper's
// single-threaded program (same operations per element, bit for bit); only
// offloaded loops go parallel.

#include <float.h>
#include <stdint.h>
#include <string.h>

#include <vector>

#include "acct.h"

extern "C" int acct_host_fill_f32(float *Y, int64_t rows, int64_t cols, int64_t ldy, float value) {
  if (rows < 0 || cols < 0 || ldy < cols) return ACCT_EINVAL;
  for (int64_t r = 0; r < rows; ++r) {
    float *y = Y + r * ldy;
    for (int64_t c = 0; c < cols; ++c) y[c] = value;
  }
  return ACCT_OK;
}

extern "C" int acct_host_copy_f32(const float *X, int64_t ldx, float *Y, int64_t ldy, int64_t rows,
                                  int64_t cols) {
  if (rows < 0 || cols < 0 || ldx < cols || ldy < cols) return ACCT_EINVAL;
  for (int64_t r = 0; r < rows; ++r) memcpy(Y + r * ldy, X + r * ldx, (size_t)cols * sizeof(float));
  return ACCT_OK;
}

extern "C" int acct_host_im2col_f32(const float *im, int64_t ld_im, int channels, int height,
                                    int width, int ksize, int stride, int pad, float *col,
                                    int64_t ld_col) {
  if (channels <= 0 || height <= 0 || width <= 0 || ksize <= 0 || stride <= 0) return ACCT_EINVAL;
  const int out_h = (height + 2 * pad - ksize) / stride + 1;
  const int out_w = (width + 2 * pad - ksize) / stride + 1;
  const int krows = channels * ksize * ksize;
  for (int c = 0; c < krows; ++c) {
    const int kw = c % ksize, kh = (c / ksize) % ksize;
    const float *src = im + (int64_t)(c / (ksize * ksize)) * ld_im;
    float *dst = col + (int64_t)c * ld_col;
    for (int h = 0; h < out_h; ++h) {
      const int row = kh + h * stride - pad;
      for (int w = 0; w < out_w; ++w) {
        const int cc = kw + w * stride - pad;
        dst[h * out_w + w] = (row < 0 || row >= height || cc < 0 || cc >= width)
                                 ? 0.0f
                                 : src[(int64_t)row * width + cc];
      }
    }
  }
  return ACCT_OK;
}

// darknet gemm_nn: i-k-j, C[i][j] += (alpha*A[i][k]) * B[k][j].  Every
// element sees exactly the program's operation sequence -- for k ascending,
// p = RN(a * b) then c = RN(c + p), no contraction -- so the result is
// bit-identical to the C loop.  The order in which ELEMENTS are updated is
// free: 4 rows x 16 columns of C stay in AVX2 registers across the whole k
// loop (one B row load and four A broadcasts per 64 multiply-adds), ~3x the
// scalar-vectorised i-k-j loop, which streamed its C row through L1 every k.
// The GA's patterns leave gemms on the host; their evaluation time is
// mostly this loop.
#if defined(__AVX2__)
#include <immintrin.h>
#endif

namespace {
#if defined(__x86_64__)
// AVX-512 body (runtime-dispatched: the build targets x86-64-v3): 4 rows x 32
// columns in 8 zmm accumulators over packed 32-column B panels -- the same
// per-element mul-then-add sequence, twice the lanes of the AVX2 body
__attribute__((target("avx512f"))) void gemm_avx512(int M4, int N32, int K, float alpha,
                                                    const float *A, int64_t lda, const float *B,
                                                    int64_t ldb, float *C, int64_t ldc) {
  std::vector<float> panel((size_t)K * 32);
  for (int j = 0; j < N32; j += 32) {
    for (int k = 0; k < K; ++k)
      memcpy(panel.data() + (size_t)k * 32, B + (int64_t)k * ldb + j, 32 * sizeof(float));
    for (int i = 0; i < M4; i += 4) {
      const float *a0 = A + (int64_t)i * lda;
      __m512 c[4][2];
      for (int r = 0; r < 4; ++r) {
        c[r][0] = _mm512_loadu_ps(C + (int64_t)(i + r) * ldc + j);
        c[r][1] = _mm512_loadu_ps(C + (int64_t)(i + r) * ldc + j + 16);
      }
      const float *b = panel.data();
      for (int k = 0; k < K; ++k, b += 32) {
        const __m512 b0 = _mm512_loadu_ps(b), b1 = _mm512_loadu_ps(b + 16);
        for (int r = 0; r < 4; ++r) {
          const __m512 a = _mm512_set1_ps(alpha * a0[(int64_t)r * lda + k]);
          c[r][0] = _mm512_add_ps(c[r][0], _mm512_mul_ps(a, b0));
          c[r][1] = _mm512_add_ps(c[r][1], _mm512_mul_ps(a, b1));
        }
      }
      for (int r = 0; r < 4; ++r) {
        _mm512_storeu_ps(C + (int64_t)(i + r) * ldc + j, c[r][0]);
        _mm512_storeu_ps(C + (int64_t)(i + r) * ldc + j + 16, c[r][1]);
      }
    }
  }
}

bool have_avx512() {
  static const bool ok = __builtin_cpu_supports("avx512f");
  return ok;
}
#endif

void gemm_rows_scalar(int i0, int i1, int j0, int N, int K, float alpha, const float *A,
                      int64_t lda, const float *B, int64_t ldb, float *C, int64_t ldc) {
  for (int i = i0; i < i1; ++i) {
    float *c = C + (int64_t)i * ldc;
    for (int k = 0; k < K; ++k) {
      const float a = alpha * A[(int64_t)i * lda + k];
      const float *b = B + (int64_t)k * ldb;
      for (int j = j0; j < N; ++j) c[j] += a * b[j];
    }
  }
}
}  // namespace

extern "C" int acct_host_gemm_nn_f32(int M, int N, int K, float alpha, const float *A, int64_t lda,
                                     const float *B, int64_t ldb, float *C, int64_t ldc) {
  if (M < 0 || N < 0 || K < 0) return ACCT_EINVAL;
#if defined(__AVX2__)
  const int M4 = M / 4 * 4, N16 = N / 16 * 16;
  int j0 = 0;
#if defined(__x86_64__)
  if (have_avx512() && M4 > 0) {
    j0 = N / 32 * 32;
    gemm_avx512(M4, j0, K, alpha, A, lda, B, ldb, C, ldc);
  }
#endif
  // column panels of 16: the panel B[0..K)[j..j+16) packed contiguously
  // (64 B per k, L2-resident) and reused by every 4-row block of C
  std::vector<float> panel((size_t)K * 16);
  for (int j = j0; j < N16; j += 16) {
    for (int k = 0; k < K; ++k)
      memcpy(panel.data() + (size_t)k * 16, B + (int64_t)k * ldb + j, 16 * sizeof(float));
    for (int i = 0; i < M4; i += 4) {
      const float *a0 = A + (int64_t)i * lda;
      __m256 c[4][2];
      for (int r = 0; r < 4; ++r) {
        c[r][0] = _mm256_loadu_ps(C + (int64_t)(i + r) * ldc + j);
        c[r][1] = _mm256_loadu_ps(C + (int64_t)(i + r) * ldc + j + 8);
      }
      const float *b = panel.data();
      for (int k = 0; k < K; ++k, b += 16) {
        const __m256 b0 = _mm256_loadu_ps(b), b1 = _mm256_loadu_ps(b + 8);
        for (int r = 0; r < 4; ++r) {
          const __m256 a = _mm256_set1_ps(alpha * a0[(int64_t)r * lda + k]);
          c[r][0] = _mm256_add_ps(c[r][0], _mm256_mul_ps(a, b0));
          c[r][1] = _mm256_add_ps(c[r][1], _mm256_mul_ps(a, b1));
        }
      }
      for (int r = 0; r < 4; ++r) {
        _mm256_storeu_ps(C + (int64_t)(i + r) * ldc + j, c[r][0]);
        _mm256_storeu_ps(C + (int64_t)(i + r) * ldc + j + 8, c[r][1]);
      }
    }
  }
  if (N16 < N) gemm_rows_scalar(0, M4, N16, N, K, alpha, A, lda, B, ldb, C, ldc);
  gemm_rows_scalar(M4, M, 0, N, K, alpha, A, lda, B, ldb, C, ldc);
#else
  gemm_rows_scalar(0, M, 0, N, K, alpha, A, lda, B, ldb, C, ldc);
#endif
  return ACCT_OK;
}

extern "C" int acct_host_add_bias_f32(float *out, int64_t ld, const float *bias, int rows,
                                      int64_t cols) {
  if (rows < 0 || cols < 0 || ld < cols) return ACCT_EINVAL;
  for (int r = 0; r < rows; ++r) {
    float *y = out + (int64_t)r * ld;
    const float b = bias[r];
    for (int64_t c = 0; c < cols; ++c) y[c] += b;
  }
  return ACCT_OK;
}

extern "C" int acct_host_activate_f32(float *X, int64_t ld, int64_t rows, int64_t cols, int act) {
  if (rows < 0 || cols < 0 || ld < cols) return ACCT_EINVAL;
  if (act == ACCT_ACT_LINEAR) return ACCT_OK;
  if (act != ACCT_ACT_LEAKY) return ACCT_EINVAL;
  for (int64_t r = 0; r < rows; ++r) {
    float *y = X + r * ld;
    for (int64_t c = 0; c < cols; ++c)
      if (y[c] < 0.0f) y[c] = (float)(0.1 * (double)y[c]);
  }
  return ACCT_OK;
}

extern "C" int acct_host_maxpool_f32(const float *in, int64_t ld_in, int channels, int height,
                                     int width, int size, int stride, int off, int out_h, int out_w,
                                     float *out, int64_t ld_out, int32_t *idx, int64_t ld_idx) {
  if (channels <= 0 || size <= 0 || stride <= 0) return ACCT_EINVAL;
  for (int c = 0; c < channels; ++c) {
    const float *src = in + (int64_t)c * ld_in;
    for (int i = 0; i < out_h; ++i) {
      for (int j = 0; j < out_w; ++j) {
        float best = -FLT_MAX;
        int32_t arg = -1;
        for (int n = 0; n < size; ++n) {
          const int r = i * stride + n - off;
          for (int m = 0; m < size; ++m) {
            const int q = j * stride + m - off;
            if (r >= 0 && r < height && q >= 0 && q < width) {
              const float v = src[(int64_t)r * width + q];
              if (v > best) {
                best = v;
                arg = c * height * width + r * width + q;
              }
            }
          }
        }
        out[(int64_t)c * ld_out + i * out_w + j] = best;
        idx[(int64_t)c * ld_idx + i * out_w + j] = arg;
      }
    }
  }
  return ACCT_OK;
}
