"""Offload patterns executed on B200 vs the CPU oracle (B200 only).

For every tested genome: outputs of all images match the oracle within the
gemm tolerance (test_gpu_kernels.py), the all-zero genome is bit-exact,
fused and unfused execution are bit-identical, and the transfer counters
equal the counts the reference planner implies (`directive_exec_counts`,
pkg/src/acctuner/transfer.py:161-165) -- bit-exact integers.
"""

from __future__ import annotations

import random

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


def genomes(a: int, n: int, seed: int) -> list[str]:
    rng = random.Random(seed)
    out = ["1" * a, "0" * a, "10" * (a // 2) + "1" * (a % 2), "01" * (a // 2) + "0" * (a % 2)]
    while len(out) < n:
        p = rng.choice((0.2, 0.5, 0.8))
        out.append("".join("1" if rng.random() < p else "0" for _ in range(a)))
    return out


@pytest.fixture(scope="module")
def micro_ref():
    return cprog.reference_forward(build_net("micro"))["outputs"]


@pytest.mark.parametrize("name", ["micro", "demo"])
def test_patterns_match_oracle_and_counts(cuda_device, name):
    net = build_net(name)
    ref = cprog.reference_forward(net)["outputs"]
    ex = PatternExecutor(net, device=0)
    for bits in genomes(len(net.ops), 12, seed=len(name)):
        sched = ex.compile(bits)
        r = ex.run(sched)
        assert r.status == "measured"
        for key, val in sched.expected.items():
            assert r.counters[key] == val, (bits, key)
        assert r.counters["host_ops"] == sched.host_ops
        out = ex.outputs()
        if "1" not in bits:
            assert np.array_equal(out, ref)
        else:
            close(out, ref)


def test_fused_equals_unfused_bit_exact(cuda_device):
    net = build_net("micro")
    a = PatternExecutor(net, device=0, fuse=True)
    b = PatternExecutor(net, device=0, fuse=False)
    for bits in genomes(len(net.ops), 8, seed=3):
        ra, rb = a.run(bits), b.run(bits)
        assert np.array_equal(a.outputs(), b.outputs()), bits
        assert ra.counters["kernel_launches"] <= rb.counters["kernel_launches"]


@pytest.mark.parametrize("mode", [K.GEMM_SIMT, K.GEMM_AUTO])
def test_gemm_modes_agree(cuda_device, micro_ref, mode):
    net = build_net("micro")
    ex = PatternExecutor(net, device=0, gemm_mode=mode)
    ex.run("1" * len(net.ops))
    close(ex.outputs(), micro_ref)


def test_resident_schedule_matches_full_run(cuda_device):
    net = build_net("demo")
    ex = PatternExecutor(net, device=0)
    bits = "1" * len(net.ops)
    ex.run(bits)
    full_last = ex.device_array(net.output_name)
    r = ex.run(bits, resident=True)
    assert r.counters["h2d_calls"] == 0 and r.counters["d2h_calls"] == 0
    assert np.array_equal(ex.device_array(net.output_name), full_last)


def test_yolov2_tiny_all_offload_matches_oracle(cuda_device):
    net = build_net("yolov2-tiny", images=2)
    ref = cprog.reference_forward(net)["outputs"]
    ex = PatternExecutor(net, device=0)
    bits = "1" * len(net.ops)
    sched = ex.compile(bits)
    r = ex.run(sched)
    for key, val in sched.expected.items():
        assert r.counters[key] == val, key
    close(ex.outputs(), ref)
    # transfers per image: only x in and y out stay inside the image loop
    assert r.counters["h2d_bytes"] >= 2 * net.arrays["x"].nbytes


def test_timeout_is_reported_not_raised(cuda_device):
    net = build_net("demo")
    ex = PatternExecutor(net, device=0)
    r = ex.run("0" * len(net.ops), timeout_s=1e-9)
    assert r.status == "timeout"


def test_yolov2_608_all_offload_matches_oracle(cuda_device):
    """configs[4]'s deeper 608x608 net (109 genes, gemm K up to 9216): the
    batched all-offload schedule -- CTA-pair and single-SM tcgen05 tiles,
    stream and swap gemms, gathered copyins, early copyouts -- against the C
    oracle, with every host array after the hoisted copyouts."""
    net = build_net("yolov2-608", images=2)
    ref = cprog.reference_forward(net)
    ex = PatternExecutor(net, device=0)
    bits = "1" * len(net.ops)
    sched = ex.compile(bits)
    assert sched.batch == 2
    r = ex.run(sched)
    for key, val in sched.expected.items():
        assert r.counters[key] == val, key
    close(ex.outputs(), ref["outputs"])
    # arrays copied out after the loop hold the last image's values
    for name in ("out25", "col24", "pool1", "idx1"):
        want = ref["state"][name]
        got = ex.host_array(name)
        if want.dtype == np.int32:
            assert np.array_equal(got, want), name
        else:
            close(got, want)
