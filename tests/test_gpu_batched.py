"""Image-batched execution of the image loop (B200 only).

With every op of the loop body offloaded, the executor privatises the
body's arrays per image and runs P images per launch (executor
`_batch_plan`).  It must be unobservable: outputs match the oracle and the
image-at-a-time run, the transfer counters equal the planner's
(`directive_exec_counts`, pkg/src/acctuner/transfer.py:161-165) exactly, and
arrays copied out after the loop hold the last image's values.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import cprog
from paper_1811_03882_b200 import kernels as K
from paper_1811_03882_b200.executor import PatternExecutor
from paper_1811_03882_b200.nets import build_net

pytestmark = pytest.mark.gpu


def close(got, want):
    scale = max(1e-30, float(np.abs(want).max()))
    err = float(np.abs(got - want).max())
    assert err <= 1e-4 * scale, (err, scale)


@pytest.mark.parametrize("name,images,batch,expect", [
    ("micro", 2, True, 2), ("demo", 8, True, 8), ("demo", 8, 3, 2), ("demo", 6, 4, 3),
    ("yolov2-tiny", 2, True, 2)])
def test_batched_all_offload_matches_oracle(cuda_device, name, images, batch, expect):
    net = build_net(name, images=images)
    ref = cprog.reference_forward(net)["outputs"]
    ex = PatternExecutor(net, device=0, batch=batch)
    bits = "1" * len(net.ops)
    sched = ex.compile(bits)
    assert sched.batch == expect
    for _ in range(3):                       # plain run, graph capture, replay
        r = ex.run(sched)
        for key, val in sched.expected.items():
            assert r.counters[key] == val, key
        close(ex.outputs(), ref)


@pytest.mark.parametrize("name", ["micro", "demo"])
def test_batched_equals_image_at_a_time(cuda_device, name):
    net = build_net(name)
    a = PatternExecutor(net, device=0, batch=True)
    b = PatternExecutor(net, device=0, batch=False)
    bits = "1" * len(net.ops)
    sa, sb = a.compile(bits), b.compile(bits)
    assert sa.batch > 1 and sb.batch == 1
    ra, rb = a.run(sa), b.run(sb)
    assert ra.counters == {**rb.counters, "kernel_launches": ra.counters["kernel_launches"]}
    close(a.outputs(), b.outputs())
    # hoisted copyouts after the loop see the last image's arrays
    for name_ in net.arrays:
        close(a.host_array(name_), b.host_array(name_))
        close(a.device_array(name_), b.device_array(name_))


def test_partial_offload_is_not_batched(cuda_device):
    net = build_net("demo")
    ex = PatternExecutor(net, device=0)
    bits = "1" * (len(net.ops) - 1) + "0"
    assert ex.compile(bits).batch == 1


def test_batched_resident_matches_full(cuda_device):
    net = build_net("demo")
    ex = PatternExecutor(net, device=0)
    bits = "1" * len(net.ops)
    ex.run(bits)
    last = ex.device_array(net.output_name)
    r = ex.run(bits, resident=True)
    assert r.counters["h2d_calls"] == 0 and r.counters["d2h_calls"] == 0
    assert np.array_equal(ex.device_array(net.output_name), last)


def test_batched_kernel_entries_match_single(cuda_device):
    """The *_batched C-ABI entries equal a loop of single-image calls."""
    import torch
    lib = K.lib()
    P, c, h, w = 3, 4, 9, 11
    ld_im = 128
    im = torch.randn(P, c, ld_im, device="cuda")
    krows, npix = c * 9, h * w
    ldc = 128
    col_b = torch.zeros(krows, P * ldc, device="cuda")
    col_1 = torch.zeros(P, krows, ldc, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert lib.acct_im2col_batched_f32(im.data_ptr(), ld_im, c * ld_im, c, h, w, 3, 1, 1,
                                       col_b.data_ptr(), P * ldc, ldc, P, s) == 0
    for b in range(P):
        assert lib.acct_im2col_f32(im[b].data_ptr(), ld_im, c, h, w, 3, 1, 1,
                                   col_1[b].data_ptr(), ldc, s) == 0
    torch.cuda.synchronize()
    for b in range(P):
        assert torch.equal(col_b[:, b * ldc:b * ldc + npix], col_1[b][:, :npix])
    out_b = torch.zeros(c, P * 64, device="cuda")
    idx_b = torch.zeros(c, P * 64, dtype=torch.int32, device="cuda")
    out_1 = torch.zeros(P, c, 64, device="cuda")
    idx_1 = torch.zeros(P, c, 64, dtype=torch.int32, device="cuda")
    assert lib.acct_maxpool_batched_f32(im.data_ptr(), ld_im, c * ld_im, c, h, w, 2, 2, 0, 4, 5,
                                        out_b.data_ptr(), P * 64, 64, idx_b.data_ptr(), P * 64,
                                        64, P, s) == 0
    for b in range(P):
        assert lib.acct_maxpool_f32(im[b].data_ptr(), ld_im, c, h, w, 2, 2, 0, 4, 5,
                                    out_1[b].data_ptr(), 64, idx_1[b].data_ptr(), 64, s) == 0
    torch.cuda.synchronize()
    for b in range(P):
        assert torch.equal(out_b[:, b * 64:b * 64 + 20], out_1[b][:, :20])
        assert torch.equal(idx_b[:, b * 64:b * 64 + 20], idx_1[b][:, :20])
    # the vectorised 2x2/2 path (8x16 -> 4x8 per channel)
    h2, w2, ld2 = 8, 16, 128
    im2 = torch.randn(P, c, ld2, device="cuda")
    ob = torch.zeros(c, P * 32, device="cuda")
    ib = torch.zeros(c, P * 32, dtype=torch.int32, device="cuda")
    o1 = torch.zeros(P, c, 32, device="cuda")
    i1 = torch.zeros(P, c, 32, dtype=torch.int32, device="cuda")
    assert lib.acct_maxpool_batched_f32(im2.data_ptr(), ld2, c * ld2, c, h2, w2, 2, 2, 0, 4, 8,
                                        ob.data_ptr(), P * 32, 32, ib.data_ptr(), P * 32, 32, P,
                                        s) == 0
    for b in range(P):
        assert lib.acct_maxpool_f32(im2[b].data_ptr(), ld2, c, h2, w2, 2, 2, 0, 4, 8,
                                    o1[b].data_ptr(), 32, i1[b].data_ptr(), 32, s) == 0
    torch.cuda.synchronize()
    for b in range(P):
        assert torch.equal(ob[:, b * 32:b * 32 + 32], o1[b])
        assert torch.equal(ib[:, b * 32:b * 32 + 32], i1[b])


@pytest.mark.parametrize("mode", [K.GEMM_SIMT, K.GEMM_AUTO])
@pytest.mark.parametrize("name,images", [("demo", 8), ("yolov2-tiny", 2), ("micro", 4)])
def test_fused_conv_layer_is_bit_identical(cuda_device, name, images, mode):
    """The fused conv launches (im2col + gemm (+ 2x2 maxpool) in one kernel,
    col -- and a pooled output -- stored for the batch's last image only)
    leave every observable array bit-identical to the unfused schedule in
    SIMT mode (the same FMA chain), batched and resident alike; under AUTO
    (implicit-im2col tcgen05 tiles) col stays bit-exact and the output within
    the gemm tolerance; AUTO and SIMT agree within it too."""
    net = build_net(name, images=images)
    a = PatternExecutor(net, device=0, fuse=True, gemm_mode=mode)
    b = PatternExecutor(net, device=0, fuse=False, gemm_mode=mode)
    bits = "1" * len(net.ops)
    sa = a.compile(bits)
    convs = [k for k in range(sa.n_actions)
             if sa.actions[k].kind == K.A_KERNEL and sa.actions[k].i[0] == K.K_CONV]
    assert convs
    if sa.batch > 1:
        assert all(sa.actions[k].i[8] == 1 for k in convs)   # dead col stores skipped
    ra, rb = a.run(sa), b.run(bits)
    assert {k: v for k, v in ra.counters.items() if k != "kernel_launches"} == \
        {k: v for k, v in rb.counters.items() if k != "kernel_launches"}
    assert ra.counters["kernel_launches"] < rb.counters["kernel_launches"]
    if mode == K.GEMM_SIMT:
        assert np.array_equal(a.outputs(), b.outputs())
        for name_ in net.arrays:
            assert np.array_equal(a.device_array(name_), b.device_array(name_)), name_
            assert np.array_equal(a.host_array(name_), b.host_array(name_)), name_
        a.run(bits, resident=True)
        b.run(bits, resident=True)
        assert np.array_equal(a.device_array(net.output_name), b.device_array(net.output_name))
    else:
        # the tensor-core convs sum the 3xTF32 terms in their own order:
        # values within the gemm tolerance; col0 (an im2col of the input)
        # bit-exact, the later col arrays as exact as their inputs
        want = b.outputs()
        assert np.abs(a.outputs() - want).max() <= 1e-4 * np.abs(want).max()
        for name_ in net.arrays:
            if name_.startswith("col"):
                for arr_a, arr_b in ((a.device_array(name_), b.device_array(name_)),
                                     (a.host_array(name_), b.host_array(name_))):
                    if name_ == "col0":
                        assert np.array_equal(arr_a, arr_b), name_
                    else:
                        assert np.abs(arr_a - arr_b).max() <= 1e-4 * max(np.abs(arr_b).max(), 1e-30)
    c = PatternExecutor(net, device=0, fuse=True, gemm_mode=K.GEMM_SIMT + K.GEMM_AUTO - mode)
    c.run(bits)
    want = a.outputs()
    assert np.abs(c.outputs() - want).max() <= 1e-4 * np.abs(want).max()
