/*
 * TEST INFRASTRUCTURE -- the CPU oracle.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this file's
 * library; the product (paper_1811_03882_b200) never does.
 *
 * Plain-C restatement of the Darknet CPU loops the paper offloads
 * (pjreddie/darknet, src/im2col.c im2col_cpu, src/gemm.c gemm_nn,
 * src/convolutional_layer.c add_bias, src/activations.c activate_array with
 * leaky_activate / linear_activate, src/maxpool_layer.c forward_maxpool_layer,
 * src/blas.c fill_cpu / copy_cpu).  Darknet is NOT vendored in the reference
 * (/root/reference models it only as a 75-gene count: PAPER.md:169,
 * pkg/tests/fixtures/generate.py:248-309) and no version is pinned there, so
 * this restates the published algorithm of the upstream master branch; the
 * reference's own CPU path for these loops is the gcc-compiled C-subset
 * program run by its `cmd:` evaluator (pkg/src/acctuner/evaluation.py:
 * 162-196), against which tests/test_oracle.py pins these functions
 * bit-for-bit.
 *
 * Also holds the seeded synthetic-data generator shared with the program
 * harness (splitmix64 over fnv1a64(name) ^ seed*golden).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

/* darknet src/blas.c: fill_cpu(N, ALPHA, X, INCX) with INCX = 1 */
void orc_fill(float *x, long n, float alpha) {
  for (long i = 0; i < n; ++i) x[i] = alpha;
}

/* darknet src/blas.c: copy_cpu(N, X, INCX, Y, INCY) with unit strides */
void orc_copy(const float *x, float *y, long n) {
  for (long i = 0; i < n; ++i) y[i] = x[i];
}

/* darknet src/im2col.c: im2col_get_pixel + im2col_cpu */
static float get_pixel(const float *im, int height, int width, int row, int col, int channel,
                       int pad) {
  row -= pad;
  col -= pad;
  if (row < 0 || col < 0 || row >= height || col >= width) return 0;
  return im[col + width * (row + height * channel)];
}

void orc_im2col(const float *data_im, int channels, int height, int width, int ksize, int stride,
                int pad, float *data_col) {
  int height_col = (height + 2 * pad - ksize) / stride + 1;
  int width_col = (width + 2 * pad - ksize) / stride + 1;
  int channels_col = channels * ksize * ksize;
  for (int c = 0; c < channels_col; ++c) {
    int w_offset = c % ksize;
    int h_offset = (c / ksize) % ksize;
    int c_im = c / ksize / ksize;
    for (int h = 0; h < height_col; ++h) {
      for (int w = 0; w < width_col; ++w) {
        int im_row = h_offset + h * stride;
        int im_col = w_offset + w * stride;
        int col_index = (c * height_col + h) * width_col + w;
        data_col[col_index] = get_pixel(data_im, height, width, im_row, im_col, c_im, pad);
      }
    }
  }
}

/* darknet src/gemm.c: gemm_nn (C += ALPHA*A*B, i-k-j order) */
void orc_gemm_nn(int M, int N, int K, float ALPHA, const float *A, int lda, const float *B, int ldb,
                 float *C, int ldc) {
  for (int i = 0; i < M; ++i) {
    for (int k = 0; k < K; ++k) {
      float A_PART = ALPHA * A[i * lda + k];
      for (int j = 0; j < N; ++j) C[i * ldc + j] += A_PART * B[k * ldb + j];
    }
  }
}

/* darknet src/convolutional_layer.c: add_bias */
void orc_add_bias(float *output, const float *biases, int batch, int n, int size) {
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < size; ++j) output[(b * n + i) * size + j] += biases[i];
}

/* darknet src/activations.c: leaky_activate(x) = (x>0) ? x : .1*x; linear = x */
void orc_activate(float *x, long n, int leaky) {
  if (!leaky) return;
  for (long i = 0; i < n; ++i) x[i] = (x[i] > 0) ? x[i] : .1 * x[i];
}

/* darknet src/maxpool_layer.c: forward_maxpool_layer (pad = size-1 default,
 * offset = -pad/2), writing the argmax index of every output. */
void orc_maxpool(const float *input, int batch, int c, int h, int w, int size, int stride,
                 int padding, float *output, int *indexes) {
  int w_offset = -padding / 2;
  int h_offset = -padding / 2;
  int out_h = (h + padding - size) / stride + 1;
  int out_w = (w + padding - size) / stride + 1;
  for (int b = 0; b < batch; ++b) {
    for (int k = 0; k < c; ++k) {
      for (int i = 0; i < out_h; ++i) {
        for (int j = 0; j < out_w; ++j) {
          int out_index = j + out_w * (i + out_h * (k + c * b));
          float max = -FLT_MAX;
          int max_i = -1;
          for (int n = 0; n < size; ++n) {
            for (int m = 0; m < size; ++m) {
              int cur_h = h_offset + i * stride + n;
              int cur_w = w_offset + j * stride + m;
              int index = cur_w + w * (cur_h + h * (k + b * c));
              int valid = (cur_h >= 0 && cur_h < h && cur_w >= 0 && cur_w < w);
              float val = (valid != 0) ? input[index] : -FLT_MAX;
              max_i = (val > max) ? index : max_i;
              max = (val > max) ? val : max;
            }
          }
          output[out_index] = max;
          indexes[out_index] = max_i;
        }
      }
    }
  }
}

/* ---- seeded synthetic data (same recipe as paper_1811_03882_b200/nets.py) ---- */
static uint64_t fnv1a64(const char *s) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 0x100000001B3ull;
  }
  return h;
}

static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void orc_synth(const char *name, uint64_t seed, float *out, long count, float scale, long start) {
  uint64_t key = fnv1a64(name) ^ (seed * 0x9E3779B97F4A7C15ull);
  for (long i = 0; i < count; ++i) {
    uint64_t z = splitmix64(key + (uint64_t)(start + i));
    double u = (double)(z >> 40) * (1.0 / 16777216.0) - 0.5;
    out[i] = (float)u * scale;
  }
}

float orc_weight_scale(int fan_in) { return (float)sqrt(24.0 / fan_in); }
