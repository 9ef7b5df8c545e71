"""ctypes binding of libacct_sm100.so (include/acct.h).

The library is the product's compute path: there is no Python or CPU
fallback for an offloaded loop.  `lib()` raises `DeviceError` when the
shared object is missing or fails to load, and every wrapper raises
`DeviceError` when a call returns non-zero (the message comes from
`acct_last_error_string`).  Pointers are plain integers (e.g.
`tensor.data_ptr()`), streams are `cudaStream_t` integers
(`torch.cuda.current_stream().cuda_stream`).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import DeviceError

LIB_PATH = Path(__file__).resolve().parent / "libacct_sm100.so"

GEMM_AUTO, GEMM_SIMT, GEMM_TC3XTF32 = 0, 1, 2
ACT_NONE, ACT_LINEAR, ACT_LEAKY = -1, 0, 1

# schedule action kinds / op kinds (acct.h)
A_LOOP_BEGIN, A_LOOP_END, A_DIRECTIVE, A_H2D, A_D2H, A_BIND, A_STORE, A_KERNEL, A_HOST, A_SYNC, \
    A_H2D_GATHER = range(1, 12)
K_FILL, K_COPY, K_IM2COL, K_GEMM, K_ADD_BIAS, K_LEAKY, K_LINEAR, K_MAXPOOL, K_CONV = range(1, 10)
OP_KIND = {"fill": K_FILL, "copy": K_COPY, "im2col": K_IM2COL, "gemm": K_GEMM,
           "add_bias": K_ADD_BIAS, "leaky": K_LEAKY, "linear": K_LINEAR, "maxpool": K_MAXPOOL,
           "conv": K_CONV}

ETIMEOUT = 1003


class Counters(C.Structure):
    _fields_ = [("directive_execs", C.c_int64), ("var_transfers", C.c_int64),
                ("h2d_calls", C.c_int64), ("d2h_calls", C.c_int64),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("kernel_launches", C.c_int64), ("host_ops", C.c_int64)]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class ArraySlot(C.Structure):
    _fields_ = [("host", C.c_void_p), ("dev", C.c_void_p), ("rows", C.c_int64),
                ("cols", C.c_int64), ("ld_dev", C.c_int64), ("stage", C.c_void_p),
                ("img_stride", C.c_int64)]


class Action(C.Structure):
    _fields_ = [("kind", C.c_int32), ("a", C.c_int32 * 4), ("i", C.c_int64 * 14),
                ("base", C.c_void_p)]


_i64, _i32, _f32, _vp, _f64, _sz = C.c_int64, C.c_int, C.c_float, C.c_void_p, C.c_double, C.c_size_t

SIGNATURES = {
    "acct_fill_f32": [_vp, _i64, _i64, _i64, _f32, _vp],
    "acct_copy_f32": [_vp, _i64, _vp, _i64, _i64, _i64, _vp],
    "acct_im2col_f32": [_vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _i64, _vp],
    "acct_gemm_nn_f32": [_i32, _i32, _i32, _f32, _vp, _i64, _vp, _i64, _f32, _vp, _i64, _vp,
                         _i32, _i32, _vp],
    "acct_add_bias_f32": [_vp, _i64, _vp, _i32, _i64, _vp],
    "acct_activate_f32": [_vp, _i64, _i64, _i64, _i32, _vp],
    "acct_maxpool_f32": [_vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _i64,
                         _vp, _i64, _vp],
    "acct_memcpy2d": [_vp, _sz, _vp, _sz, _sz, _sz, _i32, _vp],
    "acct_h2d_staged": [_vp, _i64, _vp, _i64, _i64, _vp, _vp],
    "acct_d2h_staged": [_vp, _vp, _i64, _i64, _i64, _vp, _vp],
    "acct_fill_batched_f32": [_vp, _i64, _i64, _i64, _i64, _f32, _i32, _vp],
    "acct_copy_batched_f32": [_vp, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _vp],
    "acct_im2col_batched_f32": [_vp, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _i64,
                                _i64, _i32, _vp],
    "acct_gemm_nn_batched_f32": [_i32, _i32, _i32, _f32, _vp, _i64, _i64, _vp, _i64, _i64, _f32,
                                 _vp, _i64, _i64, _vp, _i32, _i32, _i32, _vp],
    "acct_conv3x3_im2col_gemm_f32": [_vp, _i64, _i64, _i32, _i32, _i32, _vp, _i64, _i64, _i32,
                                     _vp, _i64, _f32, _vp, _i64, _i64, _vp, _i32, _i32, _i32,
                                     _vp, _i64, _i64, _vp, _i64, _i64, _i32, _vp],
    "acct_conv3x3_tc_f32": [_vp, _i64, _i64, _i32, _i32, _i32, _vp, _i64, _i64, _i32, _vp, _i64,
                            _f32, _vp, _i64, _i64, _vp, _i32, _i32, _i32, _vp, _i64, _i64, _vp,
                            _i64, _i64, _i32, _vp],
    "acct_conv3x3_gemm_tc_f32": [_vp, _i64, _i64, _i32, _i32, _i32, _vp, _i64, _i64, _i32, _vp,
                                 _i64, _f32, _vp, _i64, _i64, _vp, _i32, _i32, _i32, _vp, _i64,
                                 _i64, _vp, _i64, _i64, _i32, _vp],
    "acct_add_bias_batched_f32": [_vp, _i64, _i64, _vp, _i32, _i64, _i32, _vp],
    "acct_leaky_exhaustive_check": [_vp, _vp],
    "acct_activate_batched_f32": [_vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp],
    "acct_maxpool_batched_f32": [_vp, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                 _vp, _i64, _i64, _vp, _i64, _i64, _i32, _vp],
    "acct_host_fill_f32": [_vp, _i64, _i64, _i64, _f32],
    "acct_host_copy_f32": [_vp, _i64, _vp, _i64, _i64, _i64],
    "acct_host_im2col_f32": [_vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _i64],
    "acct_host_gemm_nn_f32": [_i32, _i32, _i32, _f32, _vp, _i64, _vp, _i64, _vp, _i64],
    "acct_host_add_bias_f32": [_vp, _i64, _vp, _i32, _i64],
    "acct_host_activate_f32": [_vp, _i64, _i64, _i64, _i32],
    "acct_host_maxpool_f32": [_vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp,
                              _i64, _vp, _i64],
    "acct_run_schedule": [C.POINTER(ArraySlot), _i32, C.POINTER(Action), _i32, _i32, _f64, _vp],
    "acct_run_schedule_profiled": [C.POINTER(ArraySlot), _i32, C.POINTER(Action), _i32, _i32,
                                   _f64, _vp, C.POINTER(C.c_float)],
    "acct_device_sm_count": [_i32],
    "acct_schedule_capture": [C.POINTER(ArraySlot), _i32, C.POINTER(Action), _i32, _i32, _vp,
                              C.POINTER(C.c_void_p)],
    "acct_graph_replay": [_vp, _vp, _i32],
    "acct_tc_trace": [_vp],
    "acct_tc_stream_k_pairs": [],          # returns a count, not an error code
}
VOID_FUNCS = {"acct_counters_get": [C.POINTER(Counters)], "acct_counters_reset": [],
              "acct_graph_destroy": [_vp], "acct_tc_set_write_hi": [_i32], "acct_tc_set_tile": [_i32],
              "acct_tc_set_conv_rows": [_i32]}
ENOTSUP = 1002
STRING_FUNCS = {"acct_last_error_string": [], "acct_build_info": []}

_lock = threading.Lock()
_lib = None


def lib():
    """Load (once) and return the CDLL; raise DeviceError if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = Path(os.environ.get("ACCT_LIB", LIB_PATH))
            if not path.exists():
                raise DeviceError(f"sm_100a kernel library missing: {path} "
                                  "(build it: python -m paper_1811_03882_b200.build)")
            try:
                handle = C.CDLL(str(path))
            except OSError as exc:
                raise DeviceError(f"cannot load {path}: {exc}") from exc
            for name, args in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = C.c_int
            for name, args in VOID_FUNCS.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = None
            for name, args in STRING_FUNCS.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = C.c_char_p
            _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return sorted(list(SIGNATURES) + list(VOID_FUNCS) + list(STRING_FUNCS))


def last_error() -> str:
    return lib().acct_last_error_string().decode(errors="replace")


def check(rc: int, what: str):
    if rc != 0:
        raise DeviceError(f"{what} failed with code {rc}: {last_error()}")


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)


def counters() -> dict:
    c = Counters()
    lib().acct_counters_get(C.byref(c))
    return c.as_dict()


def reset_counters():
    lib().acct_counters_reset()


# ---- thin typed wrappers (device pointers / stream handles as ints) ----

def fill(y, rows, cols, ld, value, stream=0):
    call("acct_fill_f32", y, rows, cols, ld, value, stream)


def copy(x, ldx, y, ldy, rows, cols, stream=0):
    call("acct_copy_f32", x, ldx, y, ldy, rows, cols, stream)


def im2col(im, ld_im, channels, height, width, ksize, stride, pad, col, ld_col, stream=0):
    call("acct_im2col_f32", im, ld_im, channels, height, width, ksize, stride, pad, col, ld_col,
         stream)


def gemm_nn(M, N, K, alpha, A, lda, B, ldb, beta, Cp, ldc, bias=None, act=ACT_NONE,
            mode=GEMM_AUTO, stream=0):
    call("acct_gemm_nn_f32", M, N, K, alpha, A, lda, B, ldb, beta, Cp, ldc, bias, act, mode,
         stream)


def conv3x3_im2col_gemm(im, ld_im, im_stride, channels, height, width, col, ld_col, col_stride,
                        M, A, lda, beta, Cp, ldc, c_stride, bias=None, act=ACT_NONE, batch=1,
                        stream=0, col_from=0, pool=None):
    """pool = (pool_ptr, ld_pool, pool_stride, idx_ptr, ld_idx, idx_stride, c_from) or None"""
    pl = pool or (None, 0, 0, None, 0, 0, 0)
    call("acct_conv3x3_im2col_gemm_f32", im, ld_im, im_stride, channels, height, width, col,
         ld_col, col_stride, M, A, lda, beta, Cp, ldc, c_stride, bias, act, batch, col_from,
         *pl, stream)


def conv3x3_tc(im, ld_im, im_stride, channels, height, width, col, ld_col, col_stride, M, A, lda,
               beta, Cp, ldc, c_stride, bias=None, act=ACT_NONE, batch=1, stream=0, col_from=0,
               pool=None):
    """pool = (pool_ptr, ld_pool, pool_stride, idx_ptr, ld_idx, idx_stride, c_from) or None"""
    pl = pool or (None, 0, 0, None, 0, 0, 0)
    call("acct_conv3x3_tc_f32", im, ld_im, im_stride, channels, height, width, col, ld_col,
         col_stride, M, A, lda, beta, Cp, ldc, c_stride, bias, act, batch, col_from, *pl, stream)


def conv3x3_gemm_tc(im, ld_im, im_stride, channels, height, width, col, ld_col, col_stride, M, A,
                    lda, beta, Cp, ldc, c_stride, bias=None, act=ACT_NONE, batch=1, stream=0,
                    col_from=0):
    """Implicit-im2col CTA-pair gemm for M >= 256, 9 * channels > 768 (no pool)."""
    call("acct_conv3x3_gemm_tc_f32", im, ld_im, im_stride, channels, height, width, col, ld_col,
         col_stride, M, A, lda, beta, Cp, ldc, c_stride, bias, act, batch, col_from,
         None, 0, 0, None, 0, 0, 0, stream)


def add_bias(out, ld, bias, rows, cols, stream=0):
    call("acct_add_bias_f32", out, ld, bias, rows, cols, stream)


def activate(x, ld, rows, cols, act, stream=0):
    call("acct_activate_f32", x, ld, rows, cols, act, stream)


def maxpool(inp, ld_in, channels, height, width, size, stride, off, out_h, out_w, out, ld_out,
            idx, ld_idx, stream=0):
    call("acct_maxpool_f32", inp, ld_in, channels, height, width, size, stride, off, out_h,
         out_w, out, ld_out, idx, ld_idx, stream)
