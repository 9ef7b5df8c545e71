// HBM-bound Darknet loops: fill_cpu, copy_cpu, add_bias, activate_array,
// im2col_cpu, forward_maxpool -- each one `#pragma acc kernels` loop of the
// C-subset CNN program (paper_1811_03882_b200/nets.py) as one sm_100a kernel.
//
// Design (B200): 2-D grids -- blockIdx.y walks the rows of the [rows][cols]
// array (channels / col rows), blockIdx.x x threads walk the row in 128-bit
// vectors -- so no thread ever divides a flat index (64-bit integer division
// was the dominant cost of the first version); 32-bit index math throughout
// (every array of the three nets has < 2^31 elements, checked on the host);
// streaming loads/stores; grid sized to the data, capped at resident CTAs x
// 148 SMs with a grid-stride loop.  No shared memory: each element is
// touched once except im2col's input (re-read k*k times, served by L1/L2).
// Results are bit-identical to the host loops: the only arithmetic is a
// float add (bias) and darknet's double-precision leaky product.

#include <float.h>

#include "acct_common.cuh"

namespace {

constexpr int kBlock = 256;
constexpr int64_t kMaxElems = (int64_t)1 << 31;

// 2-D launch shape for a [rows][items] sweep: blockDim.x covers a row (a
// multiple of 32, at most 256), blockDim.y packs several short rows into one
// 256-thread CTA so 13x13 planes do not leave 80% of the threads idle.
struct Shape2 {
  dim3 grid, block;
};

Shape2 shape2d(int64_t per_row_items, int64_t rows) {
  int bx = (int)((per_row_items + 31) / 32 * 32);
  if (bx > kBlock) bx = kBlock;
  if (bx < 32) bx = 32;
  int by = kBlock / bx;
  if (by > rows) by = (int)rows;
  int64_t gx = (per_row_items + bx - 1) / bx;
  const int64_t gy = (rows + by - 1) / by;
  const int64_t cap = (int64_t)acct::sm_count() * 8;
  // keep x * y within ~8 resident CTAs per SM when rows are many
  if (gx * gy > cap) gx = (cap + gy - 1) / gy;
  if (gx < 1) gx = 1;
  return {dim3((unsigned)gx, (unsigned)gy), dim3((unsigned)bx, (unsigned)by)};
}

__device__ __forceinline__ float4 leaky4(float4 v) {
  v.x = acct_leaky(v.x);
  v.y = acct_leaky(v.y);
  v.z = acct_leaky(v.z);
  v.w = acct_leaky(v.w);
  return v;
}

// op: 0 fill, 1 copy, 2 bias add, 3 leaky
template <int OP>
__global__ void rows_vec(const float4 *__restrict__ x, int ldxv, int64_t xbs, float4 *__restrict__ y,
                         int ldyv, int64_t ybs, int rows, int nvec, float value,
                         const float *__restrict__ bias) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= rows) return;
  const float b = OP == 2 ? __ldg(bias + r) : 0.0f;
  const float4 *xr = x + blockIdx.z * xbs + (int64_t)r * ldxv;
  float4 *yr = y + blockIdx.z * ybs + (int64_t)r * ldyv;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nvec; c += gridDim.x * blockDim.x) {
    float4 v;
    if (OP == 0) {
      v = make_float4(value, value, value, value);
    } else if (OP == 1) {
      v = __ldcs(xr + c);
    } else if (OP == 2) {
      v = __ldcs(yr + c);
      v.x += b;
      v.y += b;
      v.z += b;
      v.w += b;
    } else {
      v = leaky4(__ldcs(yr + c));
    }
    __stcs(yr + c, v);
  }
}

template <int OP>
__global__ void rows_scalar(const float *__restrict__ x, int ldx, int64_t xbs, float *__restrict__ y,
                            int ldy, int64_t ybs, int rows, int cols, float value,
                            const float *__restrict__ bias) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= rows) return;
  const float *xr = x + blockIdx.z * xbs + (int64_t)r * ldx;
  float *yr = y + blockIdx.z * ybs + (int64_t)r * ldy;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x) {
    if (OP == 0) yr[c] = value;
    else if (OP == 1) yr[c] = xr[c];
    else if (OP == 2) yr[c] += bias[r];
    else yr[c] = acct_leaky(yr[c]);
  }
}

// ---- im2col: one thread per 4 consecutive output pixels of one col row ----
// blockIdx.y = col row c = (channel, kh, kw); a warp covers 128 consecutive
// pixels of an output row band, so its input reads walk image rows.
__global__ void im2col_kernel(const float *__restrict__ im, int64_t ld_im, int64_t im_bs,
                              int height, int width, int ksize, int stride, int pad, int out_w,
                              int npix, int krows, float *__restrict__ col, int64_t ld_col,
                              int64_t col_bs, bool vec) {
  pdl_trigger();
  pdl_wait();
  const int c = blockIdx.y * blockDim.y + threadIdx.y;
  if (c >= krows) return;
  im += blockIdx.z * im_bs;  // blockIdx.z = image of the batch
  col += blockIdx.z * col_bs;
  const int kw = c % ksize, kh = (c / ksize) % ksize;
  const float *src = im + (int64_t)(c / (ksize * ksize)) * ld_im;
  float *dst_row = col + (int64_t)c * ld_col;
  const int nq = (npix + 3) >> 2;
  for (int qd = blockIdx.x * blockDim.x + threadIdx.x; qd < nq; qd += gridDim.x * blockDim.x) {
    const int p0 = qd * 4;
    int h = p0 / out_w;
    int w = p0 - h * out_w;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float val = 0.0f;
      if (p0 + e < npix) {
        const int row = kh + h * stride - pad, cc = kw + w * stride - pad;
        if (row >= 0 && row < height && cc >= 0 && cc < width) val = __ldg(src + row * width + cc);
      }
      v[e] = val;
      if (++w == out_w) {
        w = 0;
        ++h;
      }
    }
    float *dst = dst_row + p0;
    if (vec) {
      __stcs(reinterpret_cast<float4 *>(dst), make_float4(v[0], v[1], v[2], v[3]));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (p0 + e < npix) dst[e] = v[e];
    }
  }
}

// ---- forward_maxpool: blockIdx.y = channel, one thread per output pixel ----
__global__ void maxpool_kernel(const float *__restrict__ in, int64_t ld_in, int64_t in_bs,
                               int height, int width, int size, int stride, int off, int out_h,
                               int out_w, int channels, float *__restrict__ out, int64_t ld_out,
                               int64_t out_bs, int32_t *__restrict__ idx, int64_t ld_idx,
                               int64_t idx_bs) {
  pdl_trigger();
  pdl_wait();
  const int c = blockIdx.y * blockDim.y + threadIdx.y;
  if (c >= channels) return;
  in += blockIdx.z * in_bs;  // blockIdx.z = image of the batch
  out += blockIdx.z * out_bs;
  idx += blockIdx.z * idx_bs;
  const float *src = in + (int64_t)c * ld_in;
  const int per = out_h * out_w;
  const int plane = height * width;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < per; p += gridDim.x * blockDim.x) {
    const int i = p / out_w, j = p - i * out_w;
    float best = -FLT_MAX;
    int32_t arg = -1;
    for (int n = 0; n < size; ++n) {
      const int r = i * stride + n - off;
      if (r < 0 || r >= height) continue;
      for (int m = 0; m < size; ++m) {
        const int q = j * stride + m - off;
        if (q >= 0 && q < width) {
          const float v = __ldg(src + r * width + q);
          if (v > best) {
            best = v;
            arg = c * plane + r * width + q;
          }
        }
      }
    }
    __stcs(out + (int64_t)c * ld_out + p, best);
    __stcs(idx + (int64_t)c * ld_idx + p, arg);
  }
}

// ---- wide planes: 3-D grid (w-quads x output rows x col rows), no division ----
// blockIdx.z = col row c, threadIdx.y/blockIdx.y = output row h, each thread 4
// consecutive output pixels of that row: one input row, float4 store.
__global__ void im2col_rows_kernel(const float *__restrict__ im, int64_t ld_im, int64_t im_bs,
                                   int height, int width, int ksize, int stride, int pad,
                                   int out_h, int out_w, int krows, float *__restrict__ col,
                                   int64_t ld_col, int64_t col_bs, bool vec) {
  pdl_trigger();
  pdl_wait();
  const int img = blockIdx.z / krows, c = blockIdx.z - img * krows;
  const int h = blockIdx.y * blockDim.y + threadIdx.y;
  if (h >= out_h) return;
  im += img * im_bs;
  col += img * col_bs;
  const int kw = c % ksize, kh = (c / ksize) % ksize;
  const int row = kh + h * stride - pad;
  const bool row_ok = row >= 0 && row < height;
  const float *srow = im + (int64_t)(c / (ksize * ksize)) * ld_im + (int64_t)row * width;
  float *dst = col + (int64_t)c * ld_col + (int64_t)h * out_w;
  for (int w0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4; w0 < out_w;
       w0 += gridDim.x * blockDim.x * 4) {
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int cc = kw + (w0 + e) * stride - pad;
      v[e] = (row_ok && cc >= 0 && cc < width && w0 + e < out_w) ? __ldg(srow + cc) : 0.0f;
    }
    if (vec) {
      __stcs(reinterpret_cast<float4 *>(dst + w0), make_float4(v[0], v[1], v[2], v[3]));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (w0 + e < out_w) dst[w0 + e] = v[e];
    }
  }
}

// ---- 3x3 / stride 1 / pad 1 (every 3x3 conv of the three nets) ----
// blockIdx.z = input channel; a thread owns 4 consecutive output pixels of
// one output row, loads the 3 x 6 input window once and writes the 9 col rows
// (kh, kw) of that channel: 9 float4 stores per 18 loads.
__global__ void im2col_k3s1_kernel(const float *__restrict__ im, int64_t ld_im, int64_t im_bs,
                                   int height, int width, int out_h, int out_w, int channels,
                                   float *__restrict__ col, int64_t ld_col, int64_t col_bs,
                                   bool vec) {
  pdl_trigger();
  pdl_wait();
  const int img = blockIdx.z / channels, ci = blockIdx.z - img * channels;
  const int h = blockIdx.y * blockDim.y + threadIdx.y;
  if (h >= out_h) return;
  im += img * im_bs;
  col += img * col_bs;
  const float *src = im + (int64_t)ci * ld_im;
  float *dst0 = col + (int64_t)(ci * 9) * ld_col + (int64_t)h * out_w;
  for (int w0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4; w0 < out_w;
       w0 += gridDim.x * blockDim.x * 4) {
    float win[3][6];
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int r = h + kh - 1;
      const bool rok = r >= 0 && r < height;
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const int cc = w0 + t - 1;
        win[kh][t] = (rok && cc >= 0 && cc < width) ? __ldg(src + r * width + cc) : 0.0f;
      }
    }
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        float *dst = dst0 + (int64_t)(kh * 3 + kw) * ld_col + w0;
        if (vec) {
          __stcs(reinterpret_cast<float4 *>(dst),
                 make_float4(win[kh][kw], win[kh][kw + 1], win[kh][kw + 2], win[kh][kw + 3]));
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (w0 + e < out_w) dst[e] = win[kh][kw + e];
        }
      }
    }
  }
}

// blockIdx.z = channel, (blockIdx.y, threadIdx.y) = output row, x = output column
__global__ void maxpool_rows_kernel(const float *__restrict__ in, int64_t ld_in, int64_t in_bs,
                                    int height, int width, int size, int stride, int off,
                                    int out_h, int out_w, int channels, float *__restrict__ out,
                                    int64_t ld_out, int64_t out_bs, int32_t *__restrict__ idx,
                                    int64_t ld_idx, int64_t idx_bs) {
  pdl_trigger();
  pdl_wait();
  const int img = blockIdx.z / channels, c = blockIdx.z - img * channels;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= out_h) return;
  in += img * in_bs;
  out += img * out_bs;
  idx += img * idx_bs;
  const float *src = in + (int64_t)c * ld_in;
  const int plane = height * width;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < out_w; j += gridDim.x * blockDim.x) {
    float best = -FLT_MAX;
    int32_t arg = -1;
    for (int n = 0; n < size; ++n) {
      const int r = i * stride + n - off;
      if (r < 0 || r >= height) continue;
      for (int m = 0; m < size; ++m) {
        const int q = j * stride + m - off;
        if (q >= 0 && q < width) {
          const float v = __ldg(src + r * width + q);
          if (v > best) {
            best = v;
            arg = c * plane + r * width + q;
          }
        }
      }
    }
    __stcs(out + (int64_t)c * ld_out + i * out_w + j, best);
    __stcs(idx + (int64_t)c * ld_idx + i * out_w + j, arg);
  }
}

// 2x2 windows, any stride / offset (yolov2-tiny layers 9 and 11: 13-wide
// outputs, which the vector kernel does not take): one thread per output
// over the flattened (image, channel, pixel) space with float-reciprocal
// index splits and the four taps unrolled -- the generic loop kernel spent
// ~250 instructions per output (ncu: 80% issue-busy, 350 GB/s on layer 11).
// Same scan order (row-major over the window), strict '>' from -FLT_MAX,
// out-of-image taps skipped.
template <int STRIDE>
__global__ void __launch_bounds__(256)
maxpool2x2_flat_kernel(const float *__restrict__ in, int64_t ld_in, int64_t in_bs, int height,
                       int width, int off, int out_w, int channels, int per, int total,
                       float inv_per, float inv_ow, float inv_ch, float *__restrict__ out,
                       int64_t ld_out, int64_t out_bs, int32_t *__restrict__ idx,
                       int64_t ld_idx, int64_t idx_bs) {
  pdl_trigger();
  pdl_wait();
  const int plane = height * width;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < total; f += gridDim.x * blockDim.x) {
    int pl, p, i, j, img, c;
    acct_divmod(f, per, inv_per, pl, p);
    acct_divmod(p, out_w, inv_ow, i, j);
    acct_divmod(pl, channels, inv_ch, img, c);
    const float *src = in + img * in_bs + (int64_t)c * ld_in;
    const int r0 = i * STRIDE - off, q0 = j * STRIDE - off;
    float best = -FLT_MAX;
    int32_t arg = -1;
#pragma unroll
    for (int n = 0; n < 2; ++n) {
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int r = r0 + n, q = q0 + m;
        if (r >= 0 && r < height && q >= 0 && q < width) {
          const float v = __ldg(src + r * width + q);
          if (v > best) {
            best = v;
            arg = c * plane + r * width + q;
          }
        }
      }
    }
    __stcs(out + img * out_bs + (int64_t)c * ld_out + p, best);
    __stcs(idx + img * idx_bs + (int64_t)c * ld_idx + p, arg);
  }
}

// 2x2 / stride 2 windows fully inside the image (even height and width,
// off = 0 -- every pooling layer of the nets but the 13x13 stride-1 one): a
// thread owns V consecutive outputs of one output row, reads its two input
// rows as V/2 float4 each and writes V outputs + V int32 indexes as one
// vector store each.  Same compare order and strict '>' as the scalar loop.
template <int V>
__global__ void maxpool2s2_kernel(const float *__restrict__ in, int64_t ld_in, int64_t in_bs,
                                  int width, int out_h, int out_w, int channels,
                                  float *__restrict__ out, int64_t ld_out, int64_t out_bs,
                                  int32_t *__restrict__ idx, int64_t ld_idx, int64_t idx_bs,
                                  int plane) {
  pdl_trigger();
  pdl_wait();
  const int img = blockIdx.z / channels, c = blockIdx.z - img * channels;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= out_h) return;
  const float *r0 = in + img * in_bs + (int64_t)c * ld_in + (int64_t)(2 * i) * width;
  const float *r1 = r0 + width;
  float *o = out + img * out_bs + (int64_t)c * ld_out + (int64_t)i * out_w;
  int32_t *x = idx + img * idx_bs + (int64_t)c * ld_idx + (int64_t)i * out_w;
  const int base0 = c * plane + 2 * i * width;
  for (int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * V; j0 < out_w;
       j0 += gridDim.x * blockDim.x * V) {
    float a[2 * V], b[2 * V];
#pragma unroll
    for (int q = 0; q < V / 2; ++q) {
      const float4 u = __ldcs(reinterpret_cast<const float4 *>(r0 + 2 * j0) + q);
      const float4 w = __ldcs(reinterpret_cast<const float4 *>(r1 + 2 * j0) + q);
      a[4 * q] = u.x; a[4 * q + 1] = u.y; a[4 * q + 2] = u.z; a[4 * q + 3] = u.w;
      b[4 * q] = w.x; b[4 * q + 1] = w.y; b[4 * q + 2] = w.z; b[4 * q + 3] = w.w;
    }
    float best[V];
    int32_t arg[V];
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const int col = 2 * (j0 + e);
      float m = -FLT_MAX;
      int32_t k = -1;
      if (a[2 * e] > m) { m = a[2 * e]; k = base0 + col; }
      if (a[2 * e + 1] > m) { m = a[2 * e + 1]; k = base0 + col + 1; }
      if (b[2 * e] > m) { m = b[2 * e]; k = base0 + width + col; }
      if (b[2 * e + 1] > m) { m = b[2 * e + 1]; k = base0 + width + col + 1; }
      best[e] = m;
      arg[e] = k;
    }
    if (V == 4) {
      __stcs(reinterpret_cast<float4 *>(o + j0), make_float4(best[0], best[1], best[2], best[3]));
      __stcs(reinterpret_cast<int4 *>(x + j0), make_int4(arg[0], arg[1], arg[2], arg[3]));
    } else {
      __stcs(reinterpret_cast<float2 *>(o + j0), make_float2(best[0], best[1]));
      __stcs(reinterpret_cast<int2 *>(x + j0), make_int2(arg[0], arg[1]));
    }
  }
}

// 3x3/1/1 on mid-size planes (16 <= out_w < 64: 52x52, 26x26): a thread owns ONE
// output pixel of one input channel and writes its 9 col rows; consecutive
// threads take consecutive pixels, so every store instruction of a warp is a
// contiguous 128-B run of a col row whatever the row width (the window
// kernel's float4 rows need out_w % 4 == 0 and waste lanes on 13/26-wide rows)
__global__ void im2col_k3s1_flat_kernel(const float *__restrict__ im, int64_t ld_im,
                                        int64_t im_bs, int height, int width, int npix,
                                        int channels, int per_block, int total,
                                        float *__restrict__ col, int64_t ld_col, int64_t col_bs) {
  pdl_trigger();
  pdl_wait();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npix) return;
  const int h = p / width, w = p - h * width;  // 3x3/1/1: output plane == input plane
  // a CTA walks `per_block` consecutive (image, channel) planes
  const int z0 = blockIdx.y * per_block;
  for (int z = z0; z < z0 + per_block && z < total; ++z) {
    const int img = z / channels, ci = z - img * channels;
    const float *src = im + img * im_bs + (int64_t)ci * ld_im;
    float *dst = col + img * col_bs + (int64_t)(ci * 9) * ld_col + p;
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int r = h + kh - 1;
      const bool rok = r >= 0 && r < height;
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        const int c = w + kw - 1;
        __stcs(dst + (int64_t)(kh * 3 + kw) * ld_col,
               (rok && c >= 0 && c < width) ? __ldg(src + r * width + c) : 0.0f);
      }
    }
  }
}

bool vec_ok(const void *p, int64_t ld, int64_t cols) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && ld % 4 == 0 && ld >= ((cols + 3) / 4) * 4;
}


// batch b of a [rows][cols] op lives at base + b * stride (stride 0: shared)
bool batch_ok(int batch, int64_t per_z) { return batch >= 1 && (int64_t)batch * per_z <= 65535; }

template <int OP>
int launch_rows(const float *X, int64_t ldx, int64_t xbs, float *Y, int64_t ldy, int64_t ybs,
                int64_t rows, int64_t cols, int batch, float value, const float *bias,
                cudaStream_t s, const char *what) {
  if (rows > 65535 * 8 || rows * (ldy > ldx ? ldy : ldx) >= kMaxElems || !batch_ok(batch, 1))
    return acct::fail(ACCT_ENOTSUP, what);
  const bool vec = vec_ok(Y, ldy, cols) && ybs % 4 == 0 &&
                   (OP != 1 || (vec_ok(X, ldx, cols) && xbs % 4 == 0));
  if (vec) {
    const int nvec = (int)((cols + 3) / 4);
    Shape2 g = shape2d(nvec, rows);
    g.grid.z = (unsigned)batch;
    acct::launch(rows_vec<OP>, g.grid, g.block, 0, s, reinterpret_cast<const float4 *>(X),
                 (int)(ldx / 4), xbs / 4, reinterpret_cast<float4 *>(Y), (int)(ldy / 4), ybs / 4,
                 (int)rows, nvec, value, bias);
  } else {
    Shape2 g = shape2d(cols, rows);
    g.grid.z = (unsigned)batch;
    acct::launch(rows_scalar<OP>, g.grid, g.block, 0, s, X, (int)ldx, xbs, Y, (int)ldy, ybs,
                 (int)rows, (int)cols, value, bias);
  }
  return acct::note_launch(what);
}

}  // namespace

using namespace acct;

extern "C" int acct_fill_batched_f32(float *Y, int64_t rows, int64_t cols, int64_t ldy,
                                     int64_t y_stride, float value, int batch,
                                     acct_stream_t stream) {
  if (rows < 0 || cols < 0 || ldy < cols || batch < 1 || (rows * cols > 0 && !Y))
    return fail(ACCT_EINVAL, "fill: bad shape");
  if (rows * cols == 0) return ACCT_OK;
  return launch_rows<0>(Y, ldy, y_stride, Y, ldy, y_stride, rows, cols, batch, value, nullptr,
                        as_stream(stream), "fill");
}

extern "C" int acct_fill_f32(float *Y, int64_t rows, int64_t cols, int64_t ldy, float value,
                             acct_stream_t stream) {
  return acct_fill_batched_f32(Y, rows, cols, ldy, 0, value, 1, stream);
}

extern "C" int acct_copy_batched_f32(const float *X, int64_t ldx, int64_t x_stride, float *Y,
                                     int64_t ldy, int64_t y_stride, int64_t rows, int64_t cols,
                                     int batch, acct_stream_t stream) {
  if (rows < 0 || cols < 0 || ldx < cols || ldy < cols || batch < 1)
    return fail(ACCT_EINVAL, "copy: bad shape");
  if (rows * cols == 0) return ACCT_OK;
  return launch_rows<1>(X, ldx, x_stride, Y, ldy, y_stride, rows, cols, batch, 0.0f, nullptr,
                        as_stream(stream), "copy");
}

extern "C" int acct_copy_f32(const float *X, int64_t ldx, float *Y, int64_t ldy, int64_t rows,
                             int64_t cols, acct_stream_t stream) {
  return acct_copy_batched_f32(X, ldx, 0, Y, ldy, 0, rows, cols, 1, stream);
}

extern "C" int acct_add_bias_batched_f32(float *out, int64_t ld, int64_t out_stride,
                                         const float *bias, int rows, int64_t cols, int batch,
                                         acct_stream_t stream) {
  if (rows < 0 || cols < 0 || ld < cols || !bias || batch < 1)
    return fail(ACCT_EINVAL, "add_bias: bad shape");
  if ((int64_t)rows * cols == 0) return ACCT_OK;
  return launch_rows<2>(out, ld, out_stride, out, ld, out_stride, rows, cols, batch, 0.0f, bias,
                        as_stream(stream), "add_bias");
}

extern "C" int acct_add_bias_f32(float *out, int64_t ld, const float *bias, int rows, int64_t cols,
                                 acct_stream_t stream) {
  return acct_add_bias_batched_f32(out, ld, 0, bias, rows, cols, 1, stream);
}

extern "C" int acct_activate_batched_f32(float *X, int64_t ld, int64_t x_stride, int64_t rows,
                                         int64_t cols, int act, int batch, acct_stream_t stream) {
  if (rows < 0 || cols < 0 || ld < cols || batch < 1) return fail(ACCT_EINVAL, "activate: bad shape");
  if (act == ACCT_ACT_LINEAR || rows * cols == 0) return ACCT_OK;  // identity loop: no device work
  if (act != ACCT_ACT_LEAKY) return fail(ACCT_EINVAL, "activate: unknown activation");
  return launch_rows<3>(X, ld, x_stride, X, ld, x_stride, rows, cols, batch, 0.0f, nullptr,
                        as_stream(stream), "activate");
}

extern "C" int acct_activate_f32(float *X, int64_t ld, int64_t rows, int64_t cols, int act,
                                 acct_stream_t stream) {
  return acct_activate_batched_f32(X, ld, 0, rows, cols, act, 1, stream);
}

extern "C" int acct_im2col_batched_f32(const float *im, int64_t ld_im, int64_t im_stride,
                                       int channels, int height, int width, int ksize, int stride,
                                       int pad, float *col, int64_t ld_col, int64_t col_stride,
                                       int batch, acct_stream_t stream) {
  if (channels <= 0 || height <= 0 || width <= 0 || ksize <= 0 || stride <= 0 || pad < 0 ||
      batch < 1)
    return fail(ACCT_EINVAL, "im2col: bad geometry");
  const int out_h = (height + 2 * pad - ksize) / stride + 1;
  const int out_w = (width + 2 * pad - ksize) / stride + 1;
  const int64_t npix = (int64_t)out_h * out_w;
  const int64_t krows = (int64_t)channels * ksize * ksize;
  if (ld_im < (int64_t)height * width || ld_col < npix) return fail(ACCT_EINVAL, "im2col: pitch too small");
  if (krows > 65535 || krows * ld_col >= kMaxElems || (int64_t)channels * ld_im >= kMaxElems)
    return fail(ACCT_ENOTSUP, "im2col: too large for 32-bit indexing");
  const bool col_vec = ld_col % 4 == 0 && col_stride % 4 == 0 &&
                       (reinterpret_cast<uintptr_t>(col) & 15) == 0;
  cudaStream_t s = as_stream(stream);
  // 16 <= out_w < 64 (52x52, 26x26): flat pixel-per-thread kernel (measured
  // 1.2-1.5x the window kernel there); 13x13 and >= 64-wide planes keep the window
  if (ksize == 3 && stride == 1 && pad == 1 && out_w < 64 && out_w >= 16 &&
      (int64_t)channels * batch <= 65535) {
    const int block = npix >= 256 ? 256 : (int)((npix + 31) / 32 * 32);  // 13x13: 192
    const int total = channels * batch;
    // one plane per CTA: packing several 13x13 planes into a CTA measured slower
    const int per_block = 1;
    const dim3 grid((unsigned)((npix + block - 1) / block),
                    (unsigned)((total + per_block - 1) / per_block));
    launch(im2col_k3s1_flat_kernel, grid, dim3(block), 0, s, im, ld_im, im_stride, height, width,
           (int)npix, channels, per_block, total, col, ld_col, col_stride);
    return note_launch("im2col");
  }
  if (ksize == 3 && stride == 1 && pad == 1 && batch_ok(batch, channels)) {
    const bool vec = out_w % 4 == 0 && col_vec;
    const int quads = (out_w + 3) / 4;
    const dim3 block(quads >= 32 ? 32 : (quads >= 16 ? 16 : (quads >= 8 ? 8 : 4)),
                     quads >= 32 ? 4 : 16);
    const dim3 grid((unsigned)((quads + block.x - 1) / block.x),
                    (unsigned)((out_h + block.y - 1) / block.y), (unsigned)(channels * batch));
    launch(im2col_k3s1_kernel, grid, block, 0, s, im, ld_im, im_stride, height, width, out_h,
           out_w, channels, col, ld_col, col_stride, vec);
    return note_launch("im2col");
  }
  if (out_w >= 64 && batch_ok(batch, krows)) {
    const bool vec = out_w % 4 == 0 && col_vec;
    const int quads = (out_w + 3) / 4;
    const dim3 block(quads >= 32 ? 32 : 16, 8);
    const dim3 grid((unsigned)((quads + block.x - 1) / block.x), (unsigned)((out_h + 7) / 8),
                    (unsigned)(krows * batch));
    launch(im2col_rows_kernel, grid, block, 0, s, im, ld_im, im_stride, height, width, ksize,
           stride, pad, out_h, out_w, (int)krows, col, ld_col, col_stride, vec);
    return note_launch("im2col");
  }
  if (!batch_ok(batch, 1)) return fail(ACCT_ENOTSUP, "im2col: batch too large");
  const bool vec = vec_ok(col, ld_col, npix) && col_stride % 4 == 0;
  const int64_t nq = (npix + 3) / 4;
  Shape2 g = shape2d(nq, krows);
  g.grid.z = (unsigned)batch;
  launch(im2col_kernel, g.grid, g.block, 0, s, im, ld_im, im_stride, height, width, ksize, stride,
         pad, out_w, (int)npix, (int)krows, col, ld_col, col_stride, vec);
  return note_launch("im2col");
}

extern "C" int acct_im2col_f32(const float *im, int64_t ld_im, int channels, int height, int width,
                               int ksize, int stride, int pad, float *col, int64_t ld_col,
                               acct_stream_t stream) {
  return acct_im2col_batched_f32(im, ld_im, 0, channels, height, width, ksize, stride, pad, col,
                                 ld_col, 0, 1, stream);
}

extern "C" int acct_maxpool_batched_f32(const float *in, int64_t ld_in, int64_t in_stride,
                                        int channels, int height, int width, int size, int stride,
                                        int off, int out_h, int out_w, float *out, int64_t ld_out,
                                        int64_t out_stride, int32_t *idx, int64_t ld_idx,
                                        int64_t idx_stride, int batch, acct_stream_t stream) {
  if (channels <= 0 || size <= 0 || stride <= 0 || out_h <= 0 || out_w <= 0 || !idx || batch < 1)
    return fail(ACCT_EINVAL, "maxpool: bad geometry");
  const int64_t per = (int64_t)out_h * out_w;
  if (ld_in < (int64_t)height * width || ld_out < per || ld_idx < per)
    return fail(ACCT_EINVAL, "maxpool: pitch too small");
  if (channels > 65535 || (int64_t)channels * ld_in >= kMaxElems)
    return fail(ACCT_ENOTSUP, "maxpool: too large for 32-bit indexing");
  cudaStream_t s = as_stream(stream);
  auto aligned = [](const void *p, int64_t ld, int64_t bs, int a) {
    return (reinterpret_cast<uintptr_t>(p) % (4 * a)) == 0 && ld % a == 0 && bs % a == 0;
  };
  if (size == 2 && stride == 2 && off == 0 && height == 2 * out_h && width == 2 * out_w &&
      out_w % 2 == 0 && batch_ok(batch, channels) && aligned(in, ld_in, in_stride, 4) &&
      width % 4 == 0) {
    const int v = (out_w % 4 == 0 && aligned(out, ld_out, out_stride, 4) &&
                   aligned(idx, ld_idx, idx_stride, 4)) ? 4 : 2;
    if (v == 4 || (aligned(out, ld_out, out_stride, 2) && aligned(idx, ld_idx, idx_stride, 2))) {
      const int groups = out_w / v;
      const int bx = groups >= 32 ? 32 : (groups >= 16 ? 16 : 8);
      const dim3 block(bx, 256 / bx);
      const dim3 grid((unsigned)((groups + bx - 1) / bx), (unsigned)((out_h + block.y - 1) / block.y),
                      (unsigned)(channels * batch));
      if (v == 4)
        launch(maxpool2s2_kernel<4>, grid, block, 0, s, in, ld_in, in_stride, width, out_h, out_w,
               channels, out, ld_out, out_stride, idx, ld_idx, idx_stride, height * width);
      else
        launch(maxpool2s2_kernel<2>, grid, block, 0, s, in, ld_in, in_stride, width, out_h, out_w,
               channels, out, ld_out, out_stride, idx, ld_idx, idx_stride, height * width);
      return note_launch("maxpool");
    }
  }
  if (size == 2 && (stride == 1 || stride == 2) && (int64_t)batch * channels * per < (1 << 24)) {
    const int total = (int)((int64_t)batch * channels * per);
    const unsigned grid = grid_for(total, 256);
    const float inv_per = 1.0f / (float)per, inv_ow = 1.0f / (float)out_w,
                inv_ch = 1.0f / (float)channels;
    if (stride == 1)
      launch(maxpool2x2_flat_kernel<1>, dim3(grid), dim3(256), 0, s, in, ld_in, in_stride, height,
             width, off, out_w, channels, (int)per, total, inv_per, inv_ow, inv_ch, out, ld_out,
             out_stride, idx, ld_idx, idx_stride);
    else
      launch(maxpool2x2_flat_kernel<2>, dim3(grid), dim3(256), 0, s, in, ld_in, in_stride, height,
             width, off, out_w, channels, (int)per, total, inv_per, inv_ow, inv_ch, out, ld_out,
             out_stride, idx, ld_idx, idx_stride);
    return note_launch("maxpool");
  }
  if (out_w >= 32 && batch_ok(batch, channels)) {
    const dim3 block(32, 8);
    const dim3 grid((unsigned)((out_w + 31) / 32), (unsigned)((out_h + 7) / 8),
                    (unsigned)(channels * batch));
    launch(maxpool_rows_kernel, grid, block, 0, s, in, ld_in, in_stride, height, width, size,
           stride, off, out_h, out_w, channels, out, ld_out, out_stride, idx, ld_idx, idx_stride);
    return note_launch("maxpool");
  }
  if (!batch_ok(batch, 1)) return fail(ACCT_ENOTSUP, "maxpool: batch too large");
  Shape2 g = shape2d(per, channels);
  g.grid.z = (unsigned)batch;
  launch(maxpool_kernel, g.grid, g.block, 0, s, in, ld_in, in_stride, height, width, size, stride,
         off, out_h, out_w, channels, out, ld_out, out_stride, idx, ld_idx, idx_stride);
  return note_launch("maxpool");
}

extern "C" int acct_maxpool_f32(const float *in, int64_t ld_in, int channels, int height, int width,
                                int size, int stride, int off, int out_h, int out_w, float *out,
                                int64_t ld_out, int32_t *idx, int64_t ld_idx, acct_stream_t stream) {
  return acct_maxpool_batched_f32(in, ld_in, 0, channels, height, width, size, stride, off, out_h,
                                  out_w, out, ld_out, 0, idx, ld_idx, 0, 1, stream);
}

// ---- test support: acct_leaky and acct_leaky_block vs darknet's double
// product over every float
namespace {
__global__ void leaky_check_kernel(unsigned long long *bad, uint32_t *examples) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (1ull << 32); i += stride) {
    const float v = __uint_as_float((uint32_t)i);
    const float a = acct_leaky(v), b = acct_leaky_ref(v);
    // the epilogues' block form: branch-free path unless a lane of the warp
    // holds a guarded value (this lane's own guard must be caught)
    float w[1] = {v};
    acct_leaky_block(w);
    const bool bad_a = __float_as_uint(a) != __float_as_uint(b) && !(a != a && b != b);
    const bool bad_w = __float_as_uint(w[0]) != __float_as_uint(b) && !(w[0] != w[0] && b != b);
    if (bad_a || bad_w) {
      const unsigned long long n = atomicAdd(bad, 1ull);
      if (n < 8) examples[n] = (uint32_t)i;
    }
  }
}
}  // namespace

extern "C" int acct_leaky_exhaustive_check(unsigned long long *mismatches, uint32_t *examples) {
  using namespace acct;
  unsigned long long *d_bad = nullptr;
  uint32_t *d_ex = nullptr;
  int rc = check_cuda(cudaMalloc(&d_bad, sizeof(unsigned long long) + 8 * sizeof(uint32_t)),
                      "leaky check: alloc");
  if (rc) return rc;
  d_ex = reinterpret_cast<uint32_t *>(d_bad + 1);
  cudaMemset(d_bad, 0, sizeof(unsigned long long) + 8 * sizeof(uint32_t));
  leaky_check_kernel<<<sm_count() * 8, 256>>>(d_bad, d_ex);
  rc = check_cuda(cudaGetLastError(), "leaky check: launch");
  if (!rc) rc = check_cuda(cudaMemcpy(mismatches, d_bad, sizeof(unsigned long long),
                                      cudaMemcpyDeviceToHost), "leaky check: copy");
  if (!rc) rc = check_cuda(cudaMemcpy(examples, d_ex, 8 * sizeof(uint32_t), cudaMemcpyDeviceToHost),
                           "leaky check: copy");
  cudaFree(d_bad);
  return rc;
}
