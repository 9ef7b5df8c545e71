"""The exact schedules bench.py times, against the reference CPU path (B200).

bench.py's legs run yolov2-tiny (BASELINE configs[1]) and yolov2-608
(configs[4]) as 16-image loops, all-offload genome, batched 16 images per
launch: the e2e leg through the public executor path (pinned host buffers,
hoisted transfers), the value leg resident in HBM (captured into a CUDA
graph).  Here the same executor configuration runs the same schedules and
is checked against what the REFERENCE's `command_evaluate` recorded for the
gcc-compiled program (tests/golden/make_cnn_golden.py):

* every image's output: the first and last image element-wise, a strided
  sample over all 16, per-image norms and sums (tolerance.py: max-relative
  1e-4, element-wise 1e-4 |ref| + 2e-5 max|ref|, normwise 1e-4);
* the last image's every array (device copies, and host copies after the
  hoisted copyouts) against the C oracle composed for that image;
* every maxpool's argmax: consistent with its own input bit for bit
  (value == input[idx]) and equal to the oracle's wherever the window's
  maximum is separated from the runner-up by more than the tolerance;
* the transfer counters against the planner's `directive_exec_counts`
  (reference `transfer.py:161-165`) and the `#pragma acc data` lines of the
  emitted source (test_transfer_counts.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import big_golden
from test_transfer_counts import pragma_counts
from oracle import cprog
from paper_1811_03882_b200 import kernels as K
from paper_1811_03882_b200 import tolerance as T
from paper_1811_03882_b200.annotate import emit_annotated
from paper_1811_03882_b200.executor import PatternExecutor
from paper_1811_03882_b200.nets import build_net
from paper_1811_03882_b200.planner import COPY, COPYOUT

pytestmark = pytest.mark.gpu

NETS = ["yolov2-tiny", "yolov2-608"]


@pytest.fixture(scope="module", params=NETS)
def bench_setup(request, cuda_device):
    name = request.param
    entry, full = big_golden(name)
    net = build_net(name, images=entry["images"])
    # exactly bench.py's executor: fuse, gemm auto, batch = all images of a step
    ex = PatternExecutor(net, device=0, fuse=True, gemm_mode=K.GEMM_AUTO, batch=True)
    last = entry["images"] - 1
    ref = cprog.reference_forward(net, image_ids=[last])
    return name, net, ex, entry, full, ref["state"]


def _pool_windows(p):
    """(oh*ow, size*size) flat input indexes of every darknet maxpool window
    (within one channel) and their validity."""
    oh, ow, size, stride, off, h, w = (p["oh"], p["ow"], p["size"], p["stride"], p["off"],
                                       p["h"], p["w"])
    i = np.arange(oh)[:, None, None, None]
    j = np.arange(ow)[None, :, None, None]
    n = np.arange(size)[None, None, :, None]
    m = np.arange(size)[None, None, None, :]
    r = i * stride + n - off
    q = j * stride + m - off
    valid = (r >= 0) & (r < h) & (q >= 0) & (q < w)
    idx = np.where(valid, r * w + q, 0)
    return idx.reshape(oh * ow, size * size), valid.reshape(oh * ow, size * size)


def check_pools(net, arrays, ref_state):
    """arrays(name) -> the last image's values of an array."""
    checked = 0
    for op in net.ops:
        if op.kind != "maxpool":
            continue
        p = op.params
        X = arrays(op.arrays["X"]).reshape(p["c"], -1)
        Y = arrays(op.arrays["Y"]).reshape(p["c"], -1)
        I = arrays(op.arrays["I"]).reshape(p["c"], -1)
        Yr = ref_state[op.arrays["Y"]].reshape(p["c"], -1)
        Ir = ref_state[op.arrays["I"]].reshape(p["c"], -1)
        Xr = ref_state[op.arrays["X"]].reshape(p["c"], -1)
        T.assert_within(Y, Yr, f"maxpool {op.arrays['Y']}")
        hw = p["h"] * p["w"]
        chan = I // hw
        assert np.array_equal(chan, np.arange(p["c"])[:, None] + 0 * chan), op.arrays["I"]
        # the argmax points at the value the pool emitted (bit for bit)
        assert np.array_equal(np.take_along_axis(X, I % hw, axis=1), Y), op.arrays["I"]
        # and is the oracle's wherever the window's winner is unambiguous
        widx, valid = _pool_windows(p)
        vals = np.where(valid[None], Xr[:, widx], -np.inf)              # (c, oh*ow, s*s)
        top2 = np.sort(vals, axis=2)[:, :, -2:]
        gap = top2[:, :, 1] - top2[:, :, 0]                     # inf for one-element windows
        scale = float(np.abs(Xr).max())
        tol = 2 * (T.REL * np.abs(top2[:, :, 1]) + T.FLOOR * scale)
        clear = gap > tol
        assert np.array_equal(I[clear], Ir[clear]), op.arrays["I"]
        checked += 1
    assert checked


def test_bench_e2e_schedule_matches_reference(bench_setup):
    name, net, ex, entry, full, ref_state = bench_setup
    bits = "1" * len(net.ops)
    sched = ex.compile(bits)
    assert sched.batch == entry["images"]                   # the 16-wide launches bench times
    # memcpy counts = the emitted `#pragma acc data` lines x loop entries
    ann = emit_annotated(ex.program, ex.tree, bits, ex.genome_map, sched.plan)
    want = pragma_counts({"source": net.source, "profile": net.profile_dict()},
                         [(ln.line_no, ln.content) for ln in ann.inserted_lines], net)
    for key, val in want.items():
        assert sched.expected[key] == val, key
    for _ in range(2):
        r = ex.run(sched)
        for key, val in sched.expected.items():
            assert r.counters[key] == val, key
        T.check_golden(ex.outputs(), entry, full)
    # every array of the last image: device copies and, for arrays the plan
    # copies out after the loop, the host copies (the output's host copy is
    # the bound output slot of each image: checked through outputs() above)
    moved_out = {v for d in sched.plan.directives if d.clause in (COPY, COPYOUT)
                 for v in d.vars} - {net.output_name}
    for a in net.arrays.values():
        if a.role in ("weight", "bias") or a.dtype != "float":
            continue
        T.assert_within(ex.device_array(a.name), ref_state[a.name], f"{name} device {a.name}")
        if a.name in moved_out:
            T.assert_within(ex.host_array(a.name), ref_state[a.name], f"{name} host {a.name}")
    check_pools(net, ex.device_array, ref_state)
    check_pools(net, lambda n: ex.host_array(n) if n in moved_out else ex.device_array(n),
                ref_state)


def test_bench_resident_schedule_matches_reference(bench_setup):
    name, net, ex, entry, full, ref_state = bench_setup
    sched = ex.compile("1" * len(net.ops), resident=True)
    assert sched.batch == entry["images"]
    for _ in range(3):                                      # plain run, graph capture, replay
        r = ex.run(sched)
        assert r.counters["h2d_calls"] == 0 and r.counters["d2h_calls"] == 0
        T.check_golden(ex.device_outputs(), entry, full)
    check_pools(net, ex.device_array, ref_state)
