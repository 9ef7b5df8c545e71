/*
 * acct.h -- C ABI of libacct_sm100.so, the B200 (sm_100a) execution library
 * behind the tuner's `gpu:` evaluator.
 *
 * The reference (acctuner) has no native interface: its only boundary on this
 * path is the Python callable `evaluate(bits) -> Measurement` consumed by
 * `run_ga` (pkg/src/acctuner/ga.py:170-217) and built by `build_evaluator`
 * (pkg/src/acctuner/pipeline.py:151-163); the offloaded loops themselves were
 * compiled by PGI from `#pragma acc kernels` regions.  This
 * header is what those regions become on B200: one entry point per Darknet
 * loop kind that a gene can offload, the transfer primitive the data
 * directives (`#pragma acc data copyin/copyout/copy`, pkg/src/acctuner/
 * emitter.py:41-49) execute as, the transfer counters whose contract is
 * `directive_exec_counts` (pkg/src/acctuner/transfer.py:161-165), and a
 * native runner for a compiled offload pattern.
 *
 * Conventions
 *   - plain C types only; `acct_stream_t` is a `cudaStream_t` (NULL = legacy
 *     default stream);
 *   - every int-returning call returns 0 on success or a cudaError_t / ACCT_E*
 *     code; the message is available from acct_last_error_string();
 *   - stream-ordered and asynchronous unless stated; the caller owns every
 *     device and host buffer (the library allocates only its own scratch);
 *   - 2-D arrays are row-major [rows][cols] with a row pitch `ld` in ELEMENTS
 *     (device arrays are allocated with ld rounded up to 32 so rows start on
 *     128-byte boundaries, which TMA needs); 1-D arrays are dense;
 *   - thread-safe: one host thread per device, each with its own streams.
 */
#ifndef ACCT_H
#define ACCT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *acct_stream_t;

enum {
  ACCT_OK = 0,
  ACCT_EINVAL = 1001,       /* bad argument (shape, pointer, enum) */
  ACCT_ENOTSUP = 1002,      /* shape/mode not supported by this kernel */
  ACCT_ETIMEOUT = 1003      /* schedule exceeded its wall-clock budget */
};

/* activation kinds (darknet ACTIVATION) */
enum { ACCT_ACT_LINEAR = 0, ACCT_ACT_LEAKY = 1 };

/* gemm_nn implementation modes */
enum {
  ACCT_GEMM_AUTO = 0,       /* M <= 16 (or <= 32 with K <= 64): FP32 HBM-streaming kernel; else tcgen05 3xTF32
                               where TMA applies, else SIMT FP32 */
  ACCT_GEMM_SIMT = 1,       /* FP32 FMA on CUDA cores (the recompiled-loop baseline) */
  ACCT_GEMM_TC3XTF32 = 2    /* TMA + tcgen05.mma kind::tf32, hi/lo split, TMEM accumulators */
};

/* ---------------------------------------------------------------- kernels --
 * One entry per offloadable Darknet loop.  Each replaces the body of the
 * corresponding `#pragma acc kernels` loop of the C-subset program
 * (paper_1811_03882_b200/nets.py emits those loops).                        */

/* fill_cpu: Y[r][c] = value for r < rows, c < cols */
int acct_fill_f32(float *Y, int64_t rows, int64_t cols, int64_t ldy, float value,
                  acct_stream_t stream);

/* copy_cpu: Y[r][c] = X[r][c] */
int acct_copy_f32(const float *X, int64_t ldx, float *Y, int64_t ldy, int64_t rows,
                  int64_t cols, acct_stream_t stream);

/* im2col_cpu: col[c][h*ow+w] = im[c/(k*k)][(c/k%k + h*s - pad)*width + c%k + w*s - pad]
 * or 0 outside the image; col has channels*k*k rows and oh*ow columns.      */
int acct_im2col_f32(const float *im, int64_t ld_im, int channels, int height, int width,
                    int ksize, int stride, int pad, float *col, int64_t ld_col,
                    acct_stream_t stream);

/* gemm_nn: C[M][N] = beta*C + alpha * A[M][K] . B[K][N]  (darknet gemm_nn is
 * beta = 1 after fill_cpu).  `epilogue` optionally fuses the following
 * add_bias (bias != NULL) and activation (act) of the same output array.   */
int acct_gemm_nn_f32(int M, int N, int K, float alpha, const float *A, int64_t lda,
                     const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                     const float *bias, int act, int mode, acct_stream_t stream);

/* add_bias: out[r][c] += bias[r] */
int acct_add_bias_f32(float *out, int64_t ld, const float *bias, int rows, int64_t cols,
                      acct_stream_t stream);

/* activate_array: leaky: x = x < 0 ? (float)(0.1 * (double)x) : x; linear: x */
int acct_activate_f32(float *X, int64_t ld, int64_t rows, int64_t cols, int act,
                      acct_stream_t stream);

/* forward_maxpool (batch 1): out[c][i*ow+j] = max over the size x size window
 * at (i*stride - off, j*stride - off), out-of-image = -FLT_MAX, strict '>'
 * in (n, m) order; idx = c*height*width + row*width + col of the max.      */
int acct_maxpool_f32(const float *in, int64_t ld_in, int channels, int height, int width,
                     int size, int stride, int off, int out_h, int out_w, float *out,
                     int64_t ld_out, int32_t *idx, int64_t ld_idx, acct_stream_t stream);

/* ---------------------------------------------------- image-batched forms --
 * The same loops over `batch` images in one launch: image b's operand X is at
 * X + b * x_stride (elements; 0 = one operand shared by every image, e.g. the
 * weights).  This is how the image loop `for (b ...)` (nets.py) runs when
 * every op of its body is offloaded: the loop's private arrays get one copy
 * per image and each op becomes one launch over all images.
 * The per-image arithmetic is exactly that of the single-image entries.    */
int acct_fill_batched_f32(float *Y, int64_t rows, int64_t cols, int64_t ldy, int64_t y_stride,
                          float value, int batch, acct_stream_t stream);
int acct_copy_batched_f32(const float *X, int64_t ldx, int64_t x_stride, float *Y, int64_t ldy,
                          int64_t y_stride, int64_t rows, int64_t cols, int batch,
                          acct_stream_t stream);
int acct_im2col_batched_f32(const float *im, int64_t ld_im, int64_t im_stride, int channels,
                            int height, int width, int ksize, int stride, int pad, float *col,
                            int64_t ld_col, int64_t col_stride, int batch, acct_stream_t stream);
/* one gemm of N' = (batch-1)*s + N columns when A is shared and B, C are
 * column-interleaved with the same stride s >= N; else `batch` gemms       */
int acct_gemm_nn_batched_f32(int M, int N, int K, float alpha, const float *A, int64_t lda,
                             int64_t a_stride, const float *B, int64_t ldb, int64_t b_stride,
                             float beta, float *C, int64_t ldc, int64_t c_stride,
                             const float *bias, int act, int batch, int mode,
                             acct_stream_t stream);
int acct_add_bias_batched_f32(float *out, int64_t ld, int64_t out_stride, const float *bias,
                              int rows, int64_t cols, int batch, acct_stream_t stream);
int acct_activate_batched_f32(float *X, int64_t ld, int64_t x_stride, int64_t rows, int64_t cols,
                              int act, int batch, acct_stream_t stream);
int acct_maxpool_batched_f32(const float *in, int64_t ld_in, int64_t in_stride, int channels,
                             int height, int width, int size, int stride, int off, int out_h,
                             int out_w, float *out, int64_t ld_out, int64_t out_stride,
                             int32_t *idx, int64_t ld_idx, int64_t idx_stride, int batch,
                             acct_stream_t stream);

/* im2col (3x3 / stride 1 / pad 1) fused with the gemm that consumes it, for
 * the narrow conv layers (channels <= 64, M <= 32): writes col exactly like
 * acct_im2col_batched_f32 (for images >= col_from of the batch only) and
 * C = A . col + beta C (+ bias, act) exactly like the SIMT gemms of
 * acct_gemm_nn_f32 (same FMA order: bit-identical), reading the input image
 * instead of re-reading col.  col_from = batch - 1 skips the col stores of
 * every image but the last (the executor does so when only that copy is
 * observable).  Rows of col and C (ld, strides, width) must be 16-byte
 * aligned; else ENOTSUP.
 * Both conv entries take an optional fused 2x2/2 maxpool of the (activated)
 * output: pool != NULL writes pool / idx exactly like acct_maxpool_batched_f32
 * (size 2, stride 2, offset 0; darknet's scan order and strict '>', argmax as
 * the flat index into the image's C plane), and C is then stored for images
 * >= c_from only.  ENOTSUP when the kernel cannot fuse it (odd planes; the
 * FP32 window kernel takes no pool yet). */
int acct_conv3x3_im2col_gemm_f32(const float *im, int64_t ld_im, int64_t im_stride, int channels,
                                 int height, int width, float *col, int64_t ld_col,
                                 int64_t col_stride, int M, const float *A, int64_t lda,
                                 float beta, float *C, int64_t ldc, int64_t c_stride,
                                 const float *bias, int act, int batch, int col_from,
                                 float *pool, int64_t ld_pool, int64_t pool_stride, int32_t *idx,
                                 int64_t ld_idx, int64_t idx_stride, int c_from,
                                 acct_stream_t stream);

/* The same contract on the 5th-generation tensor cores for M <= 64 filters
 * (channels <= 64): the swap-orientation 3xTF32 tile (128 pixels x 32 or 64
 * filters) whose activation operand is built from the input window in
 * shared memory -- implicit im2col -- instead of TMA-loaded col tiles.  C is
 * bit-identical to acct_im2col_batched_f32 + the GEMM_TC3XTF32 swap gemm.
 * Any input batch layout with 16-byte aligned strides (image-major or
 * column-interleaved).  ENOTSUP when the double-buffered input slabs
 * (2 x channels x ~(2W + 134) floats) exceed shared memory. */
int acct_conv3x3_tc_f32(const float *im, int64_t ld_im, int64_t im_stride, int channels,
                        int height, int width, float *col, int64_t ld_col, int64_t col_stride,
                        int M, const float *A, int64_t lda, float beta, float *C, int64_t ldc,
                        int64_t c_stride, const float *bias, int act, int batch, int col_from,
                        float *pool, int64_t ld_pool, int64_t pool_stride, int32_t *idx,
                        int64_t ld_idx, int64_t idx_stride, int c_from, acct_stream_t stream);

/* The same contract for the wide, long-K layers (M >= 256 filters, 9 x
 * channels > 768; yolov2-tiny layers 8, 10, 12, 13): the CTA-pair
 * chunked-promotion 3xTF32 gemm whose operand B -- the im2col of the input --
 * is gathered from the input planes by the kernel (implicit im2col) instead
 * of written to col by an im2col launch and read back.  Bit-identical to
 * acct_im2col_batched_f32 + the gemm; col is stored for images >= col_from.
 * C and col column-interleaved with one image pitch (c_stride ==
 * col_stride); ENOTSUP otherwise and when a maxpool is requested (pool must
 * be NULL).  Replaces the im2col + gemm_nn loop pair of
 * pkg/src/acctuner/... (SURVEY.md 8(a) CNN ops) for these layers. */
int acct_conv3x3_gemm_tc_f32(const float *im, int64_t ld_im, int64_t im_stride, int channels,
                             int height, int width, float *col, int64_t ld_col,
                             int64_t col_stride, int M, const float *A, int64_t lda, float beta,
                             float *C, int64_t ldc, int64_t c_stride, const float *bias, int act,
                             int batch, int col_from, float *pool, int64_t ld_pool,
                             int64_t pool_stride, int32_t *idx, int64_t ld_idx,
                             int64_t idx_stride, int c_from, acct_stream_t stream);

/* Test support (synchronous, allocates scratch): evaluates the kernels'
 * leaky activation against darknet's (float)(0.1 * (double)x) for all 2^32
 * float bit patterns on the current device; *mismatches = differing
 * results (NaNs of either payload count equal), examples[0..7] = the first
 * differing inputs' bits. */
int acct_leaky_exhaustive_check(unsigned long long *mismatches, uint32_t *examples);

/* ------------------------------------------------------------- transfers --
 * Direction: 1 = host->device, 2 = device->host.  Pitched 2-D copy of
 * `rows` rows of `row_bytes` bytes.  Counts calls and bytes per direction.  */
int acct_memcpy2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t row_bytes,
                  size_t rows, int direction, acct_stream_t stream);

typedef struct {
  int64_t directive_execs;   /* executions of data directives (transfer.py:161-165) */
  int64_t var_transfers;     /* sum over executions of |vars| (x2 for copy)        */
  int64_t h2d_calls, d2h_calls;
  int64_t h2d_bytes, d2h_bytes;
  int64_t kernel_launches;   /* device kernels launched by this library */
  int64_t host_ops;          /* CPU-side loop executions (genes set to 0) */
} acct_counters_t;

/* counters are per calling host thread (one thread drives one device) */
void acct_counters_get(acct_counters_t *out);
void acct_counters_reset(void);
const char *acct_last_error_string(void);

/* ------------------------------------------------------------ host loops --
 * The CPU side of a genome: the same loops run natively on host buffers when
 * their gene is 0 (dense row-major, same argument meaning as above).       */
int acct_host_fill_f32(float *Y, int64_t rows, int64_t cols, int64_t ldy, float value);
int acct_host_copy_f32(const float *X, int64_t ldx, float *Y, int64_t ldy, int64_t rows,
                       int64_t cols);
int acct_host_im2col_f32(const float *im, int64_t ld_im, int channels, int height, int width,
                         int ksize, int stride, int pad, float *col, int64_t ld_col);
int acct_host_gemm_nn_f32(int M, int N, int K, float alpha, const float *A, int64_t lda,
                          const float *B, int64_t ldb, float *C, int64_t ldc);
int acct_host_add_bias_f32(float *out, int64_t ld, const float *bias, int rows, int64_t cols);
int acct_host_activate_f32(float *X, int64_t ld, int64_t rows, int64_t cols, int act);
int acct_host_maxpool_f32(const float *in, int64_t ld_in, int channels, int height, int width,
                          int size, int stride, int off, int out_h, int out_w, float *out,
                          int64_t ld_out, int32_t *idx, int64_t ld_idx);

/* --------------------------------------------------------- schedule runner --
 * A genome's offload pattern compiled to a flat action list
 * (paper_1811_03882_b200/executor.py builds it from the transfer plan).
 * Arrays are referenced by slot index into `arrays`.                        */
enum {
  ACCT_A_LOOP_BEGIN = 1,   /* i[0]=trip count; host-side counted loop (the image loop) */
  ACCT_A_LOOP_END = 2,     /* i[0]=index of the matching LOOP_BEGIN */
  ACCT_A_DIRECTIVE = 3,    /* count directive executions: i[0]=|vars|, i[1]=is_copy,
                              i[2]=executions this action stands for (0 = 1) */
  ACCT_A_H2D = 4,          /* slot a[0]: host -> device (pitched); i[0]=first image,
                              i[1]=images (0 = 1), i[2]=transfers counted (0 = 1) */
  ACCT_A_D2H = 5,          /* slot a[0]: device -> host (pitched); same operands, plus
                              i[3] = 1: early copyout -- may run on a side stream
                              concurrently with the actions that follow (the compiler
                              places it after the array's last writer) */
  ACCT_A_BIND = 6,         /* slot a[0].host (i[2]=0) or .dev (i[2]=1) = base + loopvar(i[0]) * i[1]
                              bytes: load_input / per-image output slots */
  ACCT_A_STORE = 7,        /* memcpy(base + loopvar(i[0]) * i[1], slot a[0].host) (store_output) */
  ACCT_A_KERNEL = 8,       /* device op: i[0]=op kind, operands a[], ints i[1..];
                              i[13] = images per launch (image-batched loop, 0 = 1) */
  ACCT_A_HOST = 9,         /* host op: same encoding, runs on host buffers */
  ACCT_A_SYNC = 10,        /* drain the stream (before host ops / end) */
  ACCT_A_H2D_GATHER = 11   /* several whole-array host->device transfers as ONE copy:
                              i[0] = n (<= 12) arrays, slots i[1..n] whose host buffers
                              lie in one host range starting at `base`; i[13] = dense
                              device staging for that range; a scatter kernel then moves
                              each array into its (pitched) device layout.  Counts n
                              transfers, like n H2D actions */
};

enum {
  ACCT_K_FILL = 1, ACCT_K_COPY = 2, ACCT_K_IM2COL = 3, ACCT_K_GEMM = 4,
  ACCT_K_ADD_BIAS = 5, ACCT_K_LEAKY = 6, ACCT_K_LINEAR = 7, ACCT_K_MAXPOOL = 8,
  /* fused im2col(3x3/1/1) + gemm: slots a = (X, col, A, C); i[1..3] = c, h, w,
     i[4] = M, i[5] = beta is 1, i[6] = act, i[7] = bias slot (-1: none),
     i[8] = 1: col is written for the batch's last image only (the others are
     unobservable); i[9], i[10] = pool / idx slots of a fused 2x2/2 maxpool of
     C (-1: none), i[11] = 1: C itself is then stored for the last image only.  Device only: acct_conv3x3_im2col_gemm_f32 in SIMT mode
     and, under AUTO, for M <= 16;
     acct_conv3x3_tc_f32 otherwise (M <= 64); im2col + gemm when the fused
     kernel declines the shape */
  ACCT_K_CONV = 9
};

typedef struct {
  void *host;          /* current host buffer (dense, rows x cols x 4 bytes) */
  void *dev;           /* device buffer (rows x ld x 4 bytes) */
  int64_t rows, cols;  /* logical 2-D shape (1-D arrays: rows = 1) */
  int64_t ld_dev;      /* device row pitch in elements */
  void *stage;         /* optional dense device staging buffer owned by this array
                          (>= rows x cols x 4 bytes x images moved at once) for padded
                          arrays with rows < 4 KB: H2D is then one dense copy plus a
                          repack kernel instead of a slow short-row 2-D copy */
  int64_t img_stride;  /* image-batched schedules: elements between the private copies
                          of consecutive images (0 = one copy shared by all images).
                          [rows][B*ld] interleaved copies have img_stride = ld / B-th of
                          the pitch; image-major [B][rows][ld] copies rows * ld */
} acct_array_t;

/* H2D of a padded array through a dense staging buffer: one contiguous copy
 * (counted as one h2d call) + a repack kernel into the pitched layout.      */
int acct_h2d_staged(void *dev, int64_t ld, const void *host, int64_t rows, int64_t cols,
                    void *stage, acct_stream_t stream);
/* D2H of a padded array through the staging buffer: a pack kernel + one
 * contiguous copy (counted as one d2h call).                                */
int acct_d2h_staged(void *host, const void *dev, int64_t ld, int64_t rows, int64_t cols,
                    void *stage, acct_stream_t stream);

typedef struct {
  int32_t kind;        /* ACCT_A_* */
  int32_t a[4];        /* array slots */
  int64_t i[14];       /* integer operands */
  void *base;          /* BIND/STORE: host base pointer */
} acct_action_t;

/* Run `n` actions on `stream`.  `host_base_loop` selects which loop counter
 * BIND/STORE use.  Returns when all work is complete (synchronises the
 * stream).  `timeout_s` > 0 aborts with ACCT_ETIMEOUT between actions.     */
int acct_run_schedule(acct_array_t *arrays, int n_arrays, const acct_action_t *actions,
                      int n_actions, int gemm_mode, double timeout_s, acct_stream_t stream);

/* Same, recording a CUDA event pair around every KERNEL action on `stream`;
 * kernel_ms[k] receives the summed device milliseconds of action k over all
 * its executions (0 for non-kernel actions).  Used by bench.py's roofline. */
int acct_run_schedule_profiled(acct_array_t *arrays, int n_arrays, const acct_action_t *actions,
                               int n_actions, int gemm_mode, double timeout_s,
                               acct_stream_t stream, float *kernel_ms);

/* CUDA-graph replay of a schedule that has no host loop (every gene 1):
 * the whole action list -- every image of the loop, kernels and pitched
 * transfers -- is captured once into one graph; a replay is one
 * cudaGraphLaunch.  The counters the capture interpretation produced are
 * re-applied on every replay, so counts stay per execution.  Returns
 * ACCT_ENOTSUP (and no graph) if the schedule has host work.              */
typedef struct acct_graph acct_graph_t;
int acct_schedule_capture(acct_array_t *arrays, int n_arrays, const acct_action_t *actions,
                          int n_actions, int gemm_mode, acct_stream_t stream, acct_graph_t **out);
int acct_graph_replay(acct_graph_t *graph, acct_stream_t stream, int synchronize);
void acct_graph_destroy(acct_graph_t *graph);

/* tensor-core gemm debug word: bit 0 = store the TF32 hi part explicitly
 * (default: leave raw FP32 in shared memory, the MMA truncates); bits 1-3
 * skip the split / MMA / epilogue (timing only, results wrong; honoured only
 * by the -DACCT_PROFILING build, compiled out of the product library); bit 4
 * = record CTA 0's pipeline events; for verification and tools/ only */
void acct_tc_set_write_hi(int on);
/* copy the event trace of the last bit-4 launch: 8 x 512 int64 clock64
 * stamps (TMA issue, landed, split done, MMA in, commit, split parts) */
int acct_tc_trace(long long *out);
/* force the normal-orientation tile of the tensor-core gemm (0 = the cost
 * model; 1 = 128x192, 2/3 = 128x128 BK 16/32, 4 = 128x256, 5/6/7 = CTA pair
 * 256x192 / 256x256 / 256x128 (BK 16), 8 = pair 256x192 one accumulator,
 * 9/10 = pair 256x192 / 256x256 BK 32, 12 = pair swap tile for M <= 64,
 * 13/14 = pair 256x192 BK 16 / 256x128 BK 32 with a second accumulator for
 * the small 3xTF32 terms, 15 = pair 256x192 BK 32, second accumulator, only
 * A lo in TMEM, 16 = the same for the long-K pair launches that otherwise
 * run the stream-K chunked-promotion tile (pair 256x192 BK 32, FP32 running
 * sum every 4 k-blocks -- the default for K > 768), 17 = that tile for any
 * normal-orientation shape (the tile acct_conv3x3_gemm_tc_f32 uses);
 * tests and tools only                                                     */
void acct_tc_set_tile(int tile);
/* 1: narrow 3x3 convs with M <= 32 and channels % 8 == 0 on the row-band
 * tcgen05 kernel (shifted shared-memory operands, no im2col build) instead of
 * the im2col-operand kernel (default 0) -- tests and A/B measurements only  */
void acct_tc_set_conv_rows(int on);
/* CTA pairs of the stream-K gemm that fit on the current device at once */
int acct_tc_stream_k_pairs(void);

/* library/device facts */
int acct_device_sm_count(int device);
const char *acct_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* ACCT_H */
