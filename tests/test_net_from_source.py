"""Op manifests read off a program's text (`nets.net_from_source`), the basis
of the `gpu:` evaluator's `"net": "auto"` mode (CPU).

The reference's `cmd:` evaluator runs any C-subset program
(`pkg/src/acctuner/pipeline.py:136-163`); the gpu: evaluator must execute any
program written in the Darknet op templates, not only the
built-in layer lists.  The manifest recovered from the text must equal the
one the templates were written from, and programs outside the templates are
refused with the reference's ModelError (exit 14)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1811_03882_b200 as at
from oracle import cprog
from paper_1811_03882_b200.executor import PatternExecutor
from paper_1811_03882_b200.gpu_evaluator import GpuEvaluatorConfig, net_for
from paper_1811_03882_b200.nets import (Conv, MaxPool, NetSpec, ProgramError, Region, build_net,
                                        net_from_source)

CUSTOM = NetSpec("custom", 3, 24, 20, (Conv(12, 3), MaxPool(2, 2), Conv(20, 3), Conv(10, 1),
                                       MaxPool(2, 1), Conv(6, 1, activation="linear"), Region()),
                 images=3)


def manifest(net):
    return ([(o.kind, o.loop_id, o.arrays, o.params) for o in net.ops],
            {k: (v.dtype, v.shape, v.role) for k, v in net.arrays.items()},
            net.loop_trips, net.loop_parent, net.image_loop, net.input_name, net.output_name,
            net.spec.images)


@pytest.mark.parametrize("name", ["micro", "demo", "yolov2-tiny", "yolov2-608"])
def test_manifest_from_text_equals_builtin(name):
    net = build_net(name)
    assert manifest(net_from_source(net.source, name)) == manifest(net)


def test_custom_layer_list_runs_on_host_and_matches_the_c_program(tmp_path):
    net = build_net(CUSTOM)
    got = net_from_source(net.source, "auto")
    assert manifest(got) == manifest(net)
    # the derived net drives the executor: all-zero genome on the host is the
    # gcc-compiled C program bit for bit
    ex = PatternExecutor(got, device=None)
    ex.run("0" * len(got.ops))
    binary = cprog.build(got, tmp_path)
    _, want = cprog.run_outputs(got, binary)
    assert np.array_equal(ex.outputs(), want)
    assert np.array_equal(cprog.reference_forward(got)["outputs"], want)


def test_auto_config_resolves_the_tuned_program():
    net = build_net(CUSTOM)
    prog = at.parse(net.source)
    cfg = GpuEvaluatorConfig(net="auto")
    got = net_for(cfg, prog)
    assert manifest(got) == manifest(net)
    with pytest.raises(at.ModelError):
        net_for(GpuEvaluatorConfig(net="auto", images=5), prog)      # != the program's loop
    with pytest.raises(at.ModelError):
        net_for(GpuEvaluatorConfig(net="demo"), prog)                # not the demo program


@pytest.mark.parametrize("edit", [
    ("out0[i][j * 1] = 0.0;", "out0[i][j * 1] = 1.0;"),             # not a template fill
    ("load_input(x);", ""),                                           # no input call
    ("for (b = 0; b < 3; b++) {", "for (b = 0; b < 3; b += 1) {"),   # not a counted loop
])
def test_non_template_programs_are_refused(edit):
    src = build_net(CUSTOM).source
    assert edit[0] in src
    bad = src.replace(edit[0], edit[1], 1)
    with pytest.raises((ProgramError, at.ModelError)):
        net_from_source(bad)
    with pytest.raises(at.ModelError):
        try:
            prog = at.parse(bad)
        except at.ParseError as exc:
            raise at.ModelError(str(exc)) from exc
        net_for(GpuEvaluatorConfig(net="auto"), prog)
