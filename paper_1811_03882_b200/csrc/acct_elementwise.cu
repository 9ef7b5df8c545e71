// HBM-bound Darknet loops: fill_cpu, copy_cpu, add_bias, activate_array,
// im2col_cpu, forward_maxpool -- each one `#pragma acc kernels` loop of the
// C-subset CNN program (paper_1811_03882_b200/nets.py) as one sm_100a kernel.
//
// Design (B200): every kernel is a grid-stride loop over 128-bit vectors
// when the row pitch and base pointer allow it (device arrays are allocated
// with a 32-element pitch, so they always do), grid = resident CTAs per SM x
// 148 SMs, streaming stores.  No shared memory: each element is touched once
// except im2col's input (re-read k*k times, served by L1/L2).
// Results are bit-identical to the host loops: the only arithmetic is a
// float add (bias) and darknet's double-precision leaky product.

#include <float.h>

#include "acct_common.cuh"

namespace {

constexpr int kBlock = 256;

// ---- fill / copy / activation / bias: vectorized over [rows][ceil4(cols)] ----
// `vec` kernels may write up to 3 pad elements past `cols` in a row; callers
// guarantee ld >= round_up(cols, 4) for vector launches.

__global__ void fill_vec(float4 *__restrict__ y, int64_t rows, int64_t nvec, int64_t ldv,
                         float v) {
  const float4 f = make_float4(v, v, v, v);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * nvec;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / nvec, c = t - r * nvec;
    __stcs(y + r * ldv + c, f);
  }
}

__global__ void fill_scalar(float *__restrict__ y, int64_t rows, int64_t cols, int64_t ld,
                            float v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * cols;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / cols, c = t - r * cols;
    y[r * ld + c] = v;
  }
}

__global__ void copy_vec(const float4 *__restrict__ x, int64_t ldxv, float4 *__restrict__ y,
                         int64_t ldyv, int64_t rows, int64_t nvec) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * nvec;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / nvec, c = t - r * nvec;
    __stcs(y + r * ldyv + c, __ldcs(x + r * ldxv + c));
  }
}

__global__ void copy_scalar(const float *__restrict__ x, int64_t ldx, float *__restrict__ y,
                            int64_t ldy, int64_t rows, int64_t cols) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * cols;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / cols, c = t - r * cols;
    y[r * ldy + c] = x[r * ldx + c];
  }
}

__global__ void leaky_vec(float4 *__restrict__ y, int64_t rows, int64_t nvec, int64_t ldv) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * nvec;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / nvec, c = t - r * nvec;
    float4 v = __ldcs(y + r * ldv + c);
    v.x = acct_leaky(v.x);
    v.y = acct_leaky(v.y);
    v.z = acct_leaky(v.z);
    v.w = acct_leaky(v.w);
    __stcs(y + r * ldv + c, v);
  }
}

__global__ void leaky_scalar(float *__restrict__ y, int64_t rows, int64_t cols, int64_t ld) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * cols;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / cols, c = t - r * cols;
    y[r * ld + c] = acct_leaky(y[r * ld + c]);
  }
}

__global__ void bias_vec(float4 *__restrict__ y, int64_t ldv, const float *__restrict__ bias,
                         int64_t rows, int64_t nvec) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * nvec;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / nvec, c = t - r * nvec;
    const float b = __ldg(bias + r);
    float4 v = __ldcs(y + r * ldv + c);
    v.x += b;
    v.y += b;
    v.z += b;
    v.w += b;
    __stcs(y + r * ldv + c, v);
  }
}

__global__ void bias_scalar(float *__restrict__ y, int64_t ld, const float *__restrict__ bias,
                            int64_t rows, int64_t cols) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * cols;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / cols, c = t - r * cols;
    y[r * ld + c] += bias[r];
  }
}

// ---- im2col: one thread per 4 consecutive output pixels of one col row ----
// col row `c` = (channel, kh, kw); pixel p = h*ow + w.  Input reads for a
// fixed (c, h) walk one image row, so a warp's loads are contiguous (stride
// 1) and re-reads across the k*k rows of a channel hit L1/L2.
__global__ void im2col_kernel(const float *__restrict__ im, int64_t ld_im, int height, int width,
                              int ksize, int stride, int pad, int out_w, int64_t npix,
                              int64_t krows, float *__restrict__ col, int64_t ld_col, bool vec) {
  const int64_t nq = (npix + 3) / 4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < krows * nq;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / nq;
    const int64_t p0 = (t - c * nq) * 4;
    const int kw = (int)(c % ksize);
    const int kh = (int)((c / ksize) % ksize);
    const float *src = im + (c / ((int64_t)ksize * ksize)) * ld_im;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t p = p0 + e;
      float val = 0.0f;
      if (p < npix) {
        const int h = (int)(p / out_w), w = (int)(p - (int64_t)h * out_w);
        const int row = kh + h * stride - pad, cc = kw + w * stride - pad;
        if (row >= 0 && row < height && cc >= 0 && cc < width) val = __ldg(src + (int64_t)row * width + cc);
      }
      v[e] = val;
    }
    float *dst = col + c * ld_col + p0;
    if (vec) {
      __stcs(reinterpret_cast<float4 *>(dst), make_float4(v[0], v[1], v[2], v[3]));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (p0 + e < npix) dst[e] = v[e];
    }
  }
}

// ---- forward_maxpool: one thread per output pixel ----
__global__ void maxpool_kernel(const float *__restrict__ in, int64_t ld_in, int channels,
                               int height, int width, int size, int stride, int off, int out_h,
                               int out_w, float *__restrict__ out, int64_t ld_out,
                               int32_t *__restrict__ idx, int64_t ld_idx) {
  const int64_t per = (int64_t)out_h * out_w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < channels * per;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t / per);
    const int p = (int)(t - (int64_t)c * per);
    const int i = p / out_w, j = p - i * out_w;
    const float *src = in + (int64_t)c * ld_in;
    float best = -FLT_MAX;
    int32_t arg = -1;
    for (int n = 0; n < size; ++n) {
      const int r = i * stride + n - off;
      for (int m = 0; m < size; ++m) {
        const int q = j * stride + m - off;
        if (r >= 0 && r < height && q >= 0 && q < width) {
          const float v = __ldg(src + (int64_t)r * width + q);
          if (v > best) {
            best = v;
            arg = c * height * width + r * width + q;
          }
        }
      }
    }
    out[(int64_t)c * ld_out + p] = best;
    idx[(int64_t)c * ld_idx + p] = arg;
  }
}

bool vec_ok(const void *p, int64_t ld, int64_t cols) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && ld % 4 == 0 && ld >= ((cols + 3) / 4) * 4;
}

}  // namespace

using namespace acct;

extern "C" int acct_fill_f32(float *Y, int64_t rows, int64_t cols, int64_t ldy, float value,
                             acct_stream_t stream) {
  if (rows < 0 || cols < 0 || ldy < cols || (rows * cols > 0 && !Y)) return fail(ACCT_EINVAL, "fill: bad shape");
  if (rows * cols == 0) return ACCT_OK;
  cudaStream_t s = as_stream(stream);
  if (vec_ok(Y, ldy, cols)) {
    int64_t nvec = (cols + 3) / 4;
    fill_vec<<<grid_for(rows * nvec, kBlock), kBlock, 0, s>>>(reinterpret_cast<float4 *>(Y), rows, nvec, ldy / 4, value);
  } else {
    fill_scalar<<<grid_for(rows * cols, kBlock), kBlock, 0, s>>>(Y, rows, cols, ldy, value);
  }
  return note_launch("fill");
}

extern "C" int acct_copy_f32(const float *X, int64_t ldx, float *Y, int64_t ldy, int64_t rows,
                             int64_t cols, acct_stream_t stream) {
  if (rows < 0 || cols < 0 || ldx < cols || ldy < cols) return fail(ACCT_EINVAL, "copy: bad shape");
  if (rows * cols == 0) return ACCT_OK;
  cudaStream_t s = as_stream(stream);
  if (vec_ok(X, ldx, cols) && vec_ok(Y, ldy, cols)) {
    int64_t nvec = (cols + 3) / 4;
    copy_vec<<<grid_for(rows * nvec, kBlock), kBlock, 0, s>>>(
        reinterpret_cast<const float4 *>(X), ldx / 4, reinterpret_cast<float4 *>(Y), ldy / 4, rows, nvec);
  } else {
    copy_scalar<<<grid_for(rows * cols, kBlock), kBlock, 0, s>>>(X, ldx, Y, ldy, rows, cols);
  }
  return note_launch("copy");
}

extern "C" int acct_add_bias_f32(float *out, int64_t ld, const float *bias, int rows, int64_t cols,
                                 acct_stream_t stream) {
  if (rows < 0 || cols < 0 || ld < cols || !bias) return fail(ACCT_EINVAL, "add_bias: bad shape");
  if ((int64_t)rows * cols == 0) return ACCT_OK;
  cudaStream_t s = as_stream(stream);
  if (vec_ok(out, ld, cols)) {
    int64_t nvec = (cols + 3) / 4;
    bias_vec<<<grid_for(rows * nvec, kBlock), kBlock, 0, s>>>(reinterpret_cast<float4 *>(out), ld / 4, bias, rows, nvec);
  } else {
    bias_scalar<<<grid_for((int64_t)rows * cols, kBlock), kBlock, 0, s>>>(out, ld, bias, rows, cols);
  }
  return note_launch("add_bias");
}

extern "C" int acct_activate_f32(float *X, int64_t ld, int64_t rows, int64_t cols, int act,
                                 acct_stream_t stream) {
  if (rows < 0 || cols < 0 || ld < cols) return fail(ACCT_EINVAL, "activate: bad shape");
  if (act == ACCT_ACT_LINEAR || rows * cols == 0) return ACCT_OK;  // identity loop: no device work
  if (act != ACCT_ACT_LEAKY) return fail(ACCT_EINVAL, "activate: unknown activation");
  cudaStream_t s = as_stream(stream);
  if (vec_ok(X, ld, cols)) {
    int64_t nvec = (cols + 3) / 4;
    leaky_vec<<<grid_for(rows * nvec, kBlock), kBlock, 0, s>>>(reinterpret_cast<float4 *>(X), rows, nvec, ld / 4);
  } else {
    leaky_scalar<<<grid_for(rows * cols, kBlock), kBlock, 0, s>>>(X, rows, cols, ld);
  }
  return note_launch("activate");
}

extern "C" int acct_im2col_f32(const float *im, int64_t ld_im, int channels, int height, int width,
                               int ksize, int stride, int pad, float *col, int64_t ld_col,
                               acct_stream_t stream) {
  if (channels <= 0 || height <= 0 || width <= 0 || ksize <= 0 || stride <= 0 || pad < 0)
    return fail(ACCT_EINVAL, "im2col: bad geometry");
  const int out_h = (height + 2 * pad - ksize) / stride + 1;
  const int out_w = (width + 2 * pad - ksize) / stride + 1;
  const int64_t npix = (int64_t)out_h * out_w;
  const int64_t krows = (int64_t)channels * ksize * ksize;
  if (ld_im < (int64_t)height * width || ld_col < npix) return fail(ACCT_EINVAL, "im2col: pitch too small");
  const bool vec = vec_ok(col, ld_col, npix);
  const int64_t work = krows * ((npix + 3) / 4);
  im2col_kernel<<<grid_for(work, kBlock), kBlock, 0, as_stream(stream)>>>(
      im, ld_im, height, width, ksize, stride, pad, out_w, npix, krows, col, ld_col, vec);
  return note_launch("im2col");
}

extern "C" int acct_maxpool_f32(const float *in, int64_t ld_in, int channels, int height, int width,
                                int size, int stride, int off, int out_h, int out_w, float *out,
                                int64_t ld_out, int32_t *idx, int64_t ld_idx, acct_stream_t stream) {
  if (channels <= 0 || size <= 0 || stride <= 0 || out_h <= 0 || out_w <= 0 || !idx)
    return fail(ACCT_EINVAL, "maxpool: bad geometry");
  const int64_t per = (int64_t)out_h * out_w;
  if (ld_in < (int64_t)height * width || ld_out < per || ld_idx < per)
    return fail(ACCT_EINVAL, "maxpool: pitch too small");
  maxpool_kernel<<<grid_for(channels * per, kBlock), kBlock, 0, as_stream(stream)>>>(
      in, ld_in, channels, height, width, size, stride, off, out_h, out_w, out, ld_out, idx, ld_idx);
  return note_launch("maxpool");
}
