"""End to end through the reference-facing entry points with the gpu:
evaluator (B200 only): `tune` CLI on the demo net (BASELINE configs[0]:
pop 4 x 2 gens), the GA over a device pool, and the report's gpu section."""

from __future__ import annotations

import json

import pytest

import paper_1811_03882_b200 as at
from paper_1811_03882_b200 import cli
from paper_1811_03882_b200.nets import write_net_files

pytestmark = pytest.mark.gpu


def test_tune_cli_with_gpu_evaluator(cuda_device, tmp_path):
    paths = write_net_files("demo", tmp_path)
    code = cli.main(["tune", "--source", str(paths["source"]), "--profile",
                     str(paths["profile"]), "--evaluator", f"gpu:{paths['gpu_config']}",
                     "--pop", "4", "--gens", "2", "--seed", "1", "--out",
                     str(tmp_path / "best.c"), "--report", str(tmp_path / "report.json")])
    assert code == 0
    report = json.loads((tmp_path / "report.json").read_text())
    assert report["result"] == "ok"
    assert report["best"]["status"] == "measured" and report["best"]["seconds"] > 0
    gpu = report["gpu"]
    for key, val in gpu["expected_transfers"].items():
        assert gpu["transfers"][key] == val
    annotated = (tmp_path / "best.c").read_text()
    assert at.strip_annotations(at.AnnotatedSource(annotated, ())) is not None
    assert "#pragma acc" in annotated or set(report["best"]["genome"]) == {"0"}


def test_gpu_evaluator_rejects_foreign_source(cuda_device, tmp_path):
    paths = write_net_files("demo", tmp_path)
    program = at.parse("int main(){int i; float a[10]; for(i=0;i<10;i++){ a[i] = 1.0; }}")
    tree = at.build_loop_tree(program)
    acc = at.extract_accesses(program)
    gm = at.build_genome_map(at.check_all_parallelizable(tree, acc))
    with pytest.raises(at.ModelError):
        at.build_evaluator(f"gpu:{paths['gpu_config']}", program, tree, acc, gm, None,
                           at.GAConfig())


def test_ga_over_gpu_pool_finds_faster_than_all_cpu(cuda_device, tmp_path):
    from paper_1811_03882_b200.gpu_evaluator import GpuEvaluatorConfig, make_gpu_evaluator
    from paper_1811_03882_b200.legality import profile_from_dict
    from paper_1811_03882_b200.nets import build_net
    net = build_net("demo")
    prog = at.parse(net.source)
    tree = at.build_loop_tree(prog)
    acc = at.extract_accesses(prog)
    gm = at.build_genome_map(at.check_all_parallelizable(tree, acc))
    prof = profile_from_dict(net.profile_dict(), "demo", tree)
    ev = make_gpu_evaluator(GpuEvaluatorConfig(net="demo", devices="all"), prog, tree, acc, gm,
                            prof)
    res = at.run_ga(at.GAConfig(population=6, generations=3, rng_seed=2,
                                workers=len(ev.pool.devices)), gm, tree, ev)
    all_cpu = ev("0" * len(gm)).seconds
    assert res.best.status == "measured"
    assert res.best.seconds <= all_cpu * 1.5


def test_ga_two_workers_on_one_gpu(cuda_device):
    """Multi-device readiness on one GPU: `devices: [0, 0]` gives two
    independent executors (own buffers, stream, pinned arena), the GA's
    thread pool (`workers = 2`, reference `ga.py:210-214`) measures on both at
    once, and every measured genome's counters and outputs are right.  With
    a fitness that depends only on the genome (the measured run still happens
    on the pool), the search result is independent of the worker count."""
    import numpy as np

    from oracle import cprog
    from paper_1811_03882_b200.gpu_evaluator import GpuEvaluatorConfig, make_gpu_evaluator
    from paper_1811_03882_b200.legality import profile_from_dict
    from paper_1811_03882_b200.nets import build_net
    net = build_net("demo")
    want = cprog.reference_forward(net)["outputs"]
    prog = at.parse(net.source)
    tree = at.build_loop_tree(prog)
    acc = at.extract_accesses(prog)
    gm = at.build_genome_map(at.check_all_parallelizable(tree, acc))
    prof = profile_from_dict(net.profile_dict(), "demo", tree)
    results = {}
    for workers in (1, 2):
        ev = make_gpu_evaluator(GpuEvaluatorConfig(net="demo", devices=[0] * workers, repeats=1,
                                                   warmup=0), prog, tree, acc, gm, prof)
        pool = ev.pool
        assert len(pool.executors) == workers
        assert len({id(e) for e in pool.executors}) == workers
        pool.capture_outputs = True

        def det(bits, ev=ev):
            m = ev(bits)
            assert m.status == "measured"
            return at.Measurement(1e-3 * (1 + bits.count("0")) + 1e-6 * int(bits, 2), "measured")

        res = at.run_ga(at.GAConfig(population=8, generations=4, rng_seed=5, workers=workers),
                        gm, tree, det, at.MeasurementCache())
        assert pool.log and {e["slot"] for e in pool.log} <= set(range(workers))
        for e in pool.log:
            assert e["counters"] is not None
            for key, val in e["expected"].items():
                assert e["counters"][key] == val, (e["genome"], key)
            err = float(np.abs(e["outputs"] - want).max())
            assert err <= 1e-4 * float(np.abs(want).max()), e["genome"]
        if workers == 2:
            assert {e["slot"] for e in pool.log} == {0, 1}
        results[workers] = (res.best.genome, res.best.seconds,
                            [(h.best_seconds, h.evaluations_performed) for h in res.history],
                            res.evaluations_performed)
    assert results[1] == results[2]


def test_tune_cli_gpu_auto_on_a_layer_list_not_in_nets(cuda_device, tmp_path):
    """A program written in the templates but not one of the built-in nets
    tunes end to end through the reference CLI with `{"net": "auto"}` (the
    op manifest read off the source), and its patterns match the oracle."""
    import numpy as np

    from oracle import cprog
    from paper_1811_03882_b200.executor import PatternExecutor
    from paper_1811_03882_b200.nets import Conv, MaxPool, NetSpec, Region, net_from_source
    spec = NetSpec("custom", 3, 24, 20, (Conv(12, 3), MaxPool(2, 2), Conv(20, 3), Conv(10, 1),
                                         MaxPool(2, 1), Conv(6, 1, activation="linear"), Region()),
                   images=3)
    paths = write_net_files(spec, tmp_path, auto=True)
    code = cli.main(["tune", "--source", str(paths["source"]), "--profile",
                     str(paths["profile"]), "--evaluator", f"gpu:{paths['gpu_config']}",
                     "--pop", "6", "--gens", "3", "--seed", "2", "--gate-threshold", "1",
                     "--out", str(tmp_path / "best.c"), "--report", str(tmp_path / "report.json")])
    assert code == 0
    report = json.loads((tmp_path / "report.json").read_text())
    assert report["result"] == "ok" and report["best"]["status"] == "measured"
    gpu = report["gpu"]
    for key, val in gpu["expected_transfers"].items():
        assert gpu["transfers"][key] == val
    net = net_from_source(paths["source"].read_text(), "auto")
    want = cprog.reference_forward(net)["outputs"]
    ex = PatternExecutor(net, device=0)
    a = len(net.ops)
    for bits in (report["best"]["genome"], "1" * a, "".join("1" if k % 2 else "0" for k in range(a))):
        sched = ex.compile(bits)
        r = ex.run(sched)
        for key, val in sched.expected.items():
            assert r.counters[key] == val, (bits, key)
        scale = float(np.abs(want).max())
        assert float(np.abs(ex.outputs() - want).max()) <= 1e-4 * scale, bits
