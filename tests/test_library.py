"""The C-ABI library: loads on a CPU-only box, exports and binds every
symbol include/acct.h declares, and its host loops (the CPU side of a
genome) are bit-identical to the oracle.  No device calls here."""

from __future__ import annotations

import re

import numpy as np
import pytest

from conftest import REPO
from oracle import cprog
from paper_1811_03882_b200 import kernels as K


def header_functions() -> set[str]:
    text = (REPO / "include" / "acct.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(acct_[a-z0-9_]+)\s*\(", text))


def test_library_loads_and_exports_every_header_symbol():
    lib = K.lib()
    declared = header_functions()
    assert declared, "no functions parsed from acct.h"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(K.exported_symbols())
    assert b"sm_100a" in lib.acct_build_info()


def test_counters_roundtrip():
    K.reset_counters()
    c = K.counters()
    assert set(c) == {"directive_execs", "var_transfers", "h2d_calls", "d2h_calls",
                      "h2d_bytes", "d2h_bytes", "kernel_launches", "host_ops"}
    assert all(v == 0 for v in c.values())


@pytest.fixture(scope="module")
def orc():
    return cprog.load_oracle()


def _rand(shape, seed):
    return np.random.default_rng(seed).uniform(-1, 1, shape).astype(np.float32)


@pytest.mark.parametrize("M,N,K_", [(1, 1, 1), (5, 7, 3), (16, 169, 27), (33, 64, 40),
                                   (37, 173, 65), (64, 512, 300)])
def test_host_gemm_matches_oracle(orc, M, N, K_):
    A, B = _rand((M, K_), 1), _rand((K_, N), 2)
    C0 = _rand((M, N), 3)
    want = C0.copy()
    orc.orc_gemm_nn(M, N, K_, 1.0, A.ctypes.data, K_, B.ctypes.data, N, want.ctypes.data, N)
    got = C0.copy()
    K.check(K.lib().acct_host_gemm_nn_f32(M, N, K_, 1.0, A.ctypes.data, K_, B.ctypes.data, N,
                                          got.ctypes.data, N), "host gemm")
    assert np.array_equal(want, got)


@pytest.mark.parametrize("c,h,w,k,s,pad", [(3, 7, 5, 3, 1, 1), (2, 9, 9, 3, 2, 1),
                                            (1, 4, 4, 1, 1, 0), (4, 5, 6, 3, 1, 0)])
def test_host_im2col_matches_oracle(orc, c, h, w, k, s, pad):
    im = _rand((c, h * w), 4)
    oh, ow = (h + 2 * pad - k) // s + 1, (w + 2 * pad - k) // s + 1
    want = np.full((c * k * k, oh * ow), 7.0, dtype=np.float32)
    got = want.copy()
    orc.orc_im2col(im.ctypes.data, c, h, w, k, s, pad, want.ctypes.data)
    K.check(K.lib().acct_host_im2col_f32(im.ctypes.data, h * w, c, h, w, k, s, pad,
                                         got.ctypes.data, oh * ow), "host im2col")
    assert np.array_equal(want, got)


@pytest.mark.parametrize("c,h,w,size,stride", [(2, 6, 6, 2, 2), (3, 13, 13, 2, 1), (1, 5, 7, 3, 2)])
def test_host_maxpool_matches_oracle(orc, c, h, w, size, stride):
    x = _rand((c, h * w), 5)
    x[0, :3] = x[0, 3]  # ties
    padding = size - 1
    oh, ow = (h + padding - size) // stride + 1, (w + padding - size) // stride + 1
    wo, wi = np.empty((c, oh * ow), np.float32), np.empty((c, oh * ow), np.int32)
    go, gi = np.empty_like(wo), np.empty_like(wi)
    orc.orc_maxpool(x.ctypes.data, 1, c, h, w, size, stride, padding, wo.ctypes.data, wi.ctypes.data)
    K.check(K.lib().acct_host_maxpool_f32(x.ctypes.data, h * w, c, h, w, size, stride,
                                          padding // 2, oh, ow, go.ctypes.data, oh * ow,
                                          gi.ctypes.data, oh * ow), "host maxpool")
    assert np.array_equal(wo, go) and np.array_equal(wi, gi)


def test_host_elementwise_match_oracle(orc):
    M, N = 6, 37
    y = _rand((M, N), 6)
    bias = _rand((M,), 7)
    want, got = y.copy(), y.copy()
    orc.orc_add_bias(want.ctypes.data, bias.ctypes.data, 1, M, N)
    orc.orc_activate(want.ctypes.data, M * N, 1)
    lib = K.lib()
    K.check(lib.acct_host_add_bias_f32(got.ctypes.data, N, bias.ctypes.data, M, N), "bias")
    K.check(lib.acct_host_activate_f32(got.ctypes.data, N, M, N, K.ACT_LEAKY), "leaky")
    assert np.array_equal(want, got)
    z = np.empty_like(y)
    K.check(lib.acct_host_copy_f32(y.ctypes.data, N, z.ctypes.data, N, M, N), "copy")
    assert np.array_equal(z, y)
    K.check(lib.acct_host_fill_f32(z.ctypes.data, M, N, N, 0.0), "fill")
    assert not z.any()


def test_bad_arguments_are_reported():
    rc = K.lib().acct_host_gemm_nn_f32(-1, 1, 1, 1.0, None, 1, None, 1, None, 1)
    assert rc == 1001
