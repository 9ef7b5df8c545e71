"""The nvcc compile-probe oracle behind the reference's
ExternalOracle interface (reference `analysis.py:181-216`): a trial source
with one `#pragma acc kernels` line is eligible iff the loop is a Darknet op
with an sm_100a kernel whose launcher accepts the shape and whose source
builds for sm_100a.  CPU-only: nvcc cross-compiles."""

from __future__ import annotations

import json
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

from paper_1811_03882_b200 import kernel_probe as kp
from paper_1811_03882_b200 import nets
from paper_1811_03882_b200.annotate import kernels_only_annotation
from paper_1811_03882_b200.legality import (ExternalOracle, build_genome_map,
                                            check_all_parallelizable)
from paper_1811_03882_b200.loopnest import build_loop_tree, extract_accesses
from paper_1811_03882_b200.syntax import parse

GOLDEN = Path(__file__).parent / "golden"
needs_nvcc = pytest.mark.skipif(shutil.which("nvcc") is None and
                                not Path("/usr/local/cuda/bin/nvcc").exists(),
                                reason="nvcc not available")


@pytest.mark.parametrize("name", ["micro", "demo", "yolov2-tiny", "yolov2-608"])
def test_recognises_exactly_the_op_loops(name):
    net = nets.build_net(name)
    prog = parse(net.source)
    tree = build_loop_tree(prog)
    kinds = {op.loop_id: op.kind for op in net.ops}
    for lid in range(len(net.loop_trips)):
        res = kp.probe_source(kernels_only_annotation(prog, tree, lid), build=False)
        assert res.eligible == (lid in kinds), (lid, res.reason)
        if lid in kinds:
            assert res.kind == kinds[lid]
            op = next(o for o in net.ops if o.loop_id == lid)
            assert res.params == {k: v for k, v in op.params.items() if k in res.params}


def test_launch_configuration_matches_the_runtime():
    net = nets.build_net("yolov2-tiny")
    got = {}
    for op in net.ops:
        _, inst, _ = kp.launch_instance(op.kind, op.params)
        got.setdefault(op.kind, set()).add(inst)
    # single image per launch: layer 6 (M=128) keeps one SM, M >= 256 pair tiles
    assert got["gemm"] == {"gemm_stream_kernel<16, 8>", "acct::tc_gemm_kernel<32, true, 32>",
                           "acct::tc_gemm_kernel<64, true, 32>",
                           "acct::tc_gemm_kernel<192, false, 16>",
                           "acct::tc2_gemm_kernel<192, 1, 32, false>"}
    # the restated cost model picks the 256-wide pair where the C++ one does
    assert kp.gemm_tile(512, 3049, 9216) == "pair256"
    assert kp.gemm_tile(1024, 3049, 4608) == "pair192"
    assert kp.gemm_tile(128, 43249, 576) == "single192"
    assert got["im2col"] == {"im2col_k3s1_kernel", "im2col_k3s1_flat_kernel"}
    assert "maxpool2s2_kernel<4>" in got["maxpool"] and "maxpool_kernel" in got["maxpool"]


def test_rejects_foreign_and_altered_loops():
    # reference fixtures: plain loops this backend has no kernel for
    progs = {p["name"]: p for p in json.loads((GOLDEN / "reference_programs.json").read_text())}
    src = progs["stress75"]["source"]
    prog = parse(src)
    tree = build_loop_tree(prog)
    for lid in range(min(12, len(tree))):
        assert not kp.probe_source(kernels_only_annotation(prog, tree, lid), build=False).eligible
    # a gemm whose body differs from darknet's gemm_nn by one token
    net = nets.build_net("micro")
    g = next(op for op in net.ops if op.kind == "gemm")
    prog = parse(net.source)
    tree = build_loop_tree(prog)
    trial = kernels_only_annotation(prog, tree, g.loop_id)
    bad = trial.replace("[k][j * 1];", "[k][j * 1] * 2.0;", 1)
    assert bad != trial
    assert not kp.probe_source(bad, build=False).eligible
    assert not kp.probe_source("int main() { return 0; }\n", build=False).eligible


def test_shape_limits_follow_the_launcher():
    with pytest.raises(ValueError):
        kp.launch_instance("im2col", {"K": 70000, "N": 100, "ksize": 3, "stride": 1, "pad": 1,
                                      "ow": 10})
    with pytest.raises(ValueError):
        kp.launch_instance("fill", {"M": 1 << 16, "N": 1 << 16})


@needs_nvcc
def test_trial_builds_hold_the_kernel(tmp_path, monkeypatch):
    monkeypatch.setenv("ACCT_PROBE_CACHE", str(tmp_path))
    ok, note = kp.trial_build("acct_gemm_tc.cu", "acct::tc_gemm_kernel<192, false, 16>")
    assert ok and "UTCHMMA" in note
    ok, note = kp.trial_build("acct_elementwise.cu", "im2col_k3s1_kernel")
    assert ok and "im2col_k3s1_kernel" in note
    assert len(list(tmp_path.glob("*.ok"))) == 2
    ok2, _ = kp.trial_build("acct_elementwise.cu", "im2col_k3s1_kernel")  # cached
    assert ok2 and len(list(tmp_path.glob("*.ok"))) == 2


@needs_nvcc
def test_external_oracle_with_the_probe_equals_the_builtin_map(tmp_path, monkeypatch):
    """Through the reference's own ExternalOracle / check_all_parallelizable:
    the probe's genome map equals the built-in one on the demo net."""
    monkeypatch.setenv("ACCT_PROBE_CACHE", str(tmp_path))
    # the oracle runs the command from its workdir: make the package importable
    monkeypatch.setenv("PYTHONPATH", str(Path(__file__).parents[1]))
    net = nets.build_net("demo")
    prog = parse(net.source)
    tree = build_loop_tree(prog)
    acc = extract_accesses(prog)
    oracle = ExternalOracle(prog, tree,
                            f"{sys.executable} -m paper_1811_03882_b200.kernel_probe {{src}}",
                            workdir=tmp_path)
    probe = build_genome_map(check_all_parallelizable(tree, acc, oracle))
    builtin = build_genome_map(check_all_parallelizable(tree, acc))
    assert probe.loop_ids == builtin.loop_ids == tuple(op.loop_id for op in net.ops)


@needs_nvcc
def test_cli_check_with_probe_oracle(tmp_path, monkeypatch):
    """`check --oracle cmd:<config>` (reference cli.py:125,200-208) with the probe."""
    monkeypatch.setenv("ACCT_PROBE_CACHE", str(tmp_path / "cache"))
    files = nets.write_net_files("micro", tmp_path)
    conf = tmp_path / "probe.json"
    conf.write_text(json.dumps({"compile_cmd":
                                f"{sys.executable} -m paper_1811_03882_b200.kernel_probe {{src}}"}))
    out = subprocess.run([sys.executable, "-m", "paper_1811_03882_b200", "check", "--source",
                          str(files["source"]), "--oracle", f"cmd:{conf}"],
                         capture_output=True, text=True, cwd=Path(__file__).parents[1])
    assert out.returncode == 0, out.stderr[-2000:]
    report = json.loads(out.stdout)
    assert report["genome_map"] == [op.loop_id for op in nets.build_net("micro").ops]
    reasons = {v["reason"] for v in report["verdicts"] if not v["eligible"]}
    assert reasons == {"external_compile_error"}
