"""The implicit-im2col CTA-pair gemm (acct_conv3x3_gemm_tc_f32, B200 only).

For the wide long-K 3x3 layers the gemm's operand B is gathered from the
input planes inside the kernel instead of an im2col launch writing col and
the gemm reading it back.  The gathered values are col's, the tile / split /
stream-K decisions depend only on (M, N, K), and the MMA sequence is the
same, so C must be BIT-IDENTICAL to acct_im2col_batched_f32 + the gemm on
the same column-interleaved multi-image layout the executor uses, and the col
rows stored for the observable images (>= col_from) bit-identical to the
im2col's.  The C oracle checks the values (tolerance.py)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import cprog
from paper_1811_03882_b200 import kernels as K
from paper_1811_03882_b200 import tolerance as T

pytestmark = pytest.mark.gpu


def _pitch(n):
    from paper_1811_03882_b200.executor import _pitch as p
    return p(n)


@pytest.mark.parametrize("c,h,w,M,P", [
    (128, 26, 26, 256, 16),     # yolov2-tiny L8: 26-wide rows (no TMA plane), split-K
    (1024, 13, 13, 512, 16),    # yolov2-tiny L13
    (512, 13, 13, 1024, 4),     # yolov2-tiny L12 shape, 4 images
    (1024, 19, 19, 1024, 8),    # yolov2-608 L23 shape: >= 74 tiles -> stream-K
    (96, 9, 11, 300, 3),        # ragged: M not a multiple of 256, K tail, odd planes
    (128, 13, 13, 256, 1),      # one image
])
def test_implicit_gemm_equals_im2col_plus_gemm(cuda_device, c, h, w, M, P):
    import torch
    torch.manual_seed(c + h + M + P)
    HW, Kd = h * w, 9 * c
    ld = _pitch(HW)
    n_launch = (P - 1) * ld + HW
    lda = -(-Kd // 4) * 4
    im = torch.zeros(c, P * ld, device="cuda")
    for b in range(P):
        im[:, b * ld:b * ld + HW] = torch.rand(c, HW, device="cuda") * 2 - 1
    A = torch.zeros(M, lda, device="cuda")
    A[:, :Kd] = (torch.rand(M, Kd, device="cuda") - 0.5) * (24.0 / Kd) ** 0.5
    bias = torch.rand(M, device="cuda") - 0.5
    s = torch.cuda.current_stream().cuda_stream
    col_ref = torch.zeros(Kd, P * ld, device="cuda")
    C_ref = torch.zeros(M, P * ld, device="cuda")
    K.call("acct_im2col_batched_f32", im.data_ptr(), P * ld, ld, c, h, w, 3, 1, 1,
           col_ref.data_ptr(), P * ld, ld, P, s)
    lib = K.lib()
    lib.acct_tc_set_tile(17)            # the implicit gemm's tile: chunked-promotion pair
    try:
        K.gemm_nn(M, n_launch, Kd, 1.0, A.data_ptr(), lda, col_ref.data_ptr(), P * ld, 0.0,
                  C_ref.data_ptr(), P * ld, bias.data_ptr(), K.ACT_LEAKY, K.GEMM_AUTO, s)
    finally:
        lib.acct_tc_set_tile(0)
    for col_from in (0, P - 1):
        col = torch.full((Kd, P * ld), 7.0, device="cuda")
        C = torch.zeros(M, P * ld, device="cuda")
        K.conv3x3_gemm_tc(im.data_ptr(), P * ld, ld, c, h, w, col.data_ptr(), P * ld, ld, M,
                          A.data_ptr(), lda, 0.0, C.data_ptr(), P * ld, ld, bias.data_ptr(),
                          K.ACT_LEAKY, P, s, col_from=col_from)
        torch.cuda.synchronize()
        for b in range(P):
            sl = slice(b * ld, b * ld + HW)
            assert torch.equal(C[:, sl], C_ref[:, sl]), (b, col_from)
            if b >= col_from:
                assert torch.equal(col[:, sl], col_ref[:, sl]), (b, col_from)
            else:
                assert bool((col[:, sl] == 7.0).all()), "dead col rows must not be written"
    # values against the C oracle (last image)
    orc = cprog.load_oracle()
    b = P - 1
    x = im[:, b * ld:b * ld + HW].cpu().numpy().copy()
    colr = np.zeros((Kd, HW), np.float32)
    orc.orc_im2col(x.ctypes.data, c, h, w, 3, 1, 1, colr.ctypes.data)
    ref = np.zeros((M, HW), np.float32)
    A0 = A[:, :Kd].cpu().numpy().copy()
    orc.orc_gemm_nn(M, HW, Kd, 1.0, A0.ctypes.data, Kd, colr.ctypes.data, HW, ref.ctypes.data, HW)
    b0 = bias.cpu().numpy().copy()
    orc.orc_add_bias(ref.ctypes.data, b0.ctypes.data, 1, M, HW)
    orc.orc_activate(ref.ctypes.data, M * HW, 1)
    T.assert_within(C[:, b * ld:b * ld + HW].cpu().numpy(), ref, f"implicit gemm {c}x{h}x{w} M{M}")


def test_implicit_gemm_refuses_pool_and_short_k(cuda_device):
    import torch
    im = torch.zeros(64, 256, device="cuda")
    A = torch.zeros(256, 576, device="cuda")
    C = torch.zeros(256, 256, device="cuda")
    lib = K.lib()
    rc = lib.acct_conv3x3_gemm_tc_f32(im.data_ptr(), 256, 0, 64, 13, 13, None, 256, 0, 256,
                                      A.data_ptr(), 576, 0.0, C.data_ptr(), 256, 0, None, -1, 1,
                                      0, None, 0, 0, None, 0, 0, 0, None)
    assert rc == K.ENOTSUP                                      # K = 576 <= 768
