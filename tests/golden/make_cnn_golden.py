"""Golden CNN outputs from the REFERENCE's own CPU path.

Run in the build container (needs /root/reference):

    python tests/golden/make_cnn_golden.py                         # micro, demo
    python tests/golden/make_cnn_golden.py yolov2-tiny yolov2-608  # benchmarked configs

For the demo and micro nets it writes the C-subset program and the harness
(oracle/cprog.py), then measures the all-zero genome's emitted source with
the reference's `command_evaluate` (`pkg/src/acctuner/evaluation.py:
162-196`) using a `cmd:` config whose compile_cmd is gcc -- exactly what
`acctuner tune --evaluator cmd:...` does for that genome -- and records the
outputs the run wrote: full tensors for micro, per-image checksums plus a
strided sample for demo.  tests/test_oracle.py pins the oracle against
these vectors.  For the benchmarked configurations (16-image loops of
yolov2-tiny and yolov2-608) it records per-image sums / norms / max, a
strided sample over all images and the full outputs of the first and last
image (`cnn_outputs_big.json`, `*_img*.npy`); tests/test_oracle.py pins the
oracle on those images and tests/test_gpu_bench_parity.py checks the exact
schedules bench.py times against them.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, str(REPO))

import acctuner as ref  # noqa: E402

from oracle import cprog  # noqa: E402
from paper_1811_03882_b200.nets import build_net  # noqa: E402


# the benchmarked configurations (bench.py): 16-image loops of the two big
# nets; full outputs of the listed images go to .npy files beside the JSON
BIG = {"yolov2-tiny": (16, (0, 15)), "yolov2-608": (16, (0, 15))}
BIG_STRIDE = 997


def reference_outputs(net, t: Path, timeout: float = 60.0):
    """Run the all-zero genome's emitted source through the reference's
    `command_evaluate` with a gcc `cmd:` config; returns (measurement,
    outputs)."""
    cprog.write_program(net, t)
    program = ref.parse(net.source)
    tree = ref.build_loop_tree(program)
    acc = ref.extract_accesses(program)
    gm = ref.build_genome_map(ref.check_all_parallelizable(tree, acc))
    bits = "0" * len(gm)
    plan = ref.plan_transfers(program, tree, acc, bits, gm)
    src = t / f"trial_{bits}.c"
    src.write_text(ref.emit_annotated(program, tree, bits, gm, plan).text)
    cfg = ref.CommandEvaluatorConfig(
        compile_cmd=cprog.compile_cmd(t),
        run_cmd=f"'{{bin}}' 1 '{t}/out.bin'", timeout_seconds=timeout, workdir=str(t))
    m = ref.command_evaluate(cfg, src)
    assert m.status == "measured", m
    y = np.fromfile(t / "out.bin", dtype=np.float32)
    shape = (net.spec.images,) + net.arrays[net.output_name].shape
    return m, y.reshape(shape)


def big_main(names):
    path = HERE / "cnn_outputs_big.json"
    out = json.loads(path.read_text()) if path.exists() else {}
    for name in names:
        images, full = BIG[name]
        net = build_net(name, images=images)
        with tempfile.TemporaryDirectory() as tmp:
            m, y = reference_outputs(net, Path(tmp), timeout=3600.0)
        flat = y.reshape(images, -1).astype(np.float64)
        out[name] = {"shape": list(y.shape), "seed": 1, "images": images,
                     "sha256": hashlib.sha256(y.tobytes()).hexdigest(),
                     "per_image_sum": [float(v) for v in flat.sum(1)],
                     "per_image_norm": [float(v) for v in np.linalg.norm(flat, axis=1)],
                     "per_image_absmax": [float(v) for v in np.abs(flat).max(1)],
                     "sample_stride": BIG_STRIDE,
                     "sample": [float(v) for v in y.ravel()[::BIG_STRIDE]],
                     "full_images": {str(b): f"{name}_img{b}.npy" for b in full},
                     "reference_seconds": m.seconds}
        for b in full:
            np.save(HERE / f"{name}_img{b}.npy", y[b])
        print(name, m, out[name]["sha256"][:16], flush=True)
        path.write_text(json.dumps(out, separators=(",", ":")) + "\n")


def main():
    if len(sys.argv) > 1:
        big_main([a for a in sys.argv[1:] if a in BIG])
        return
    out = {}
    for name in ("micro", "demo"):
        net = build_net(name)
        with tempfile.TemporaryDirectory() as tmp:
            t = Path(tmp)
            cprog.write_program(net, t)
            program = ref.parse(net.source)
            tree = ref.build_loop_tree(program)
            acc = ref.extract_accesses(program)
            gm = ref.build_genome_map(ref.check_all_parallelizable(tree, acc))
            bits = "0" * len(gm)
            plan = ref.plan_transfers(program, tree, acc, bits, gm)
            src = t / f"trial_{bits}.c"
            src.write_text(ref.emit_annotated(program, tree, bits, gm, plan).text)
            cfg = ref.CommandEvaluatorConfig(
                compile_cmd=cprog.compile_cmd(t),
                run_cmd=f"'{{bin}}' 1 '{t}/out.bin'", timeout_seconds=60.0, workdir=str(t))
            m = ref.command_evaluate(cfg, src)
            assert m.status == "measured", m
            y = np.fromfile(t / "out.bin", dtype=np.float32)
        shape = (net.spec.images,) + net.arrays[net.output_name].shape
        y = y.reshape(shape)
        entry = {"shape": list(shape), "seed": 1,
                 "sha256": hashlib.sha256(y.tobytes()).hexdigest(),
                 "per_image_sum": [float(np.float64(v)) for v in y.reshape(shape[0], -1).sum(1, dtype=np.float64)],
                 "sample_index": list(range(0, y.size, 97)),
                 "sample": [float(v) for v in y.ravel()[::97]]}
        if name == "micro":
            entry["full"] = [float(v) for v in y.ravel()]
        out[name] = entry
        print(name, m, entry["sha256"][:16])
    (HERE / "cnn_outputs.json").write_text(json.dumps(out, separators=(",", ":")) + "\n")


if __name__ == "__main__":
    main()
