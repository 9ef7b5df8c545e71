"""Pin the CPU oracle (oracle/) before trusting it.

* the numpy and C seeded generators agree bit for bit;
* the Darknet-restated oracle ops, composed along a net's manifest, equal
  the gcc-compiled C-subset program (the reference's `cmd:` CPU path) bit
  for bit;
* both equal the golden outputs recorded by running the REFERENCE's
  `command_evaluate` on that program (tests/golden/make_cnn_golden.py).
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import cprog
from paper_1811_03882_b200.nets import build_net, input_images, synth_values, weight_data


@pytest.fixture(scope="module")
def orc():
    return cprog.load_oracle()


def test_numpy_and_c_generators_agree(orc):
    for name, scale, start in (("x", 2.0, 0), ("w3", 0.125, 777), ("bias0", 0.2, 5)):
        want = synth_values(name, 7, 4099, scale, start)
        got = np.empty(4099, dtype=np.float32)
        orc.orc_synth(name.encode(), 7, got.ctypes.data, 4099, scale, start)
        assert np.array_equal(want, got)
    net = build_net("micro")
    w = weight_data(net, "w2", 1)
    got = np.empty(w.size, dtype=np.float32)
    orc.orc_synth(b"w2", 1, got.ctypes.data, w.size, orc.orc_weight_scale(w.shape[1]), 0)
    assert np.array_equal(w.ravel(), got)


@pytest.mark.parametrize("name", ["micro", "demo"])
def test_oracle_matches_gcc_program_and_reference_golden(name, tmp_path):
    net = build_net(name)
    binary = cprog.build(net, tmp_path)
    _, prog_out = cprog.run_outputs(net, binary)
    composed = cprog.reference_forward(net)["outputs"]
    assert np.array_equal(prog_out, composed)
    golden = json.loads((GOLDEN / "cnn_outputs.json").read_text())[name]
    assert list(prog_out.shape) == golden["shape"]
    assert hashlib.sha256(prog_out.tobytes()).hexdigest() == golden["sha256"]
    flat = prog_out.ravel()
    assert [float(v) for v in flat[::97]] == golden["sample"]
    if "full" in golden:
        assert np.array_equal(flat, np.asarray(golden["full"], dtype=np.float32))


def test_input_images_are_a_stream():
    net = build_net("demo")
    all8 = input_images(net, 1, 0, 8)
    assert np.array_equal(all8[3:5], input_images(net, 1, 3, 2))
    assert all8.dtype == np.float32 and float(np.abs(all8).max()) <= 1.0


def test_oracle_maxpool_edge_semantics(orc):
    # 2x2/1 with darknet's implicit pad: the last row/col windows hang off the
    # image; -FLT_MAX never wins a strict '>' so the in-image max is kept
    c, h, w = 2, 3, 3
    x = np.arange(c * h * w, dtype=np.float32).reshape(c, h * w) * -1.0
    out = np.empty((c, h * w), dtype=np.float32)
    idx = np.empty((c, h * w), dtype=np.int32)
    orc.orc_maxpool(x.ctypes.data, 1, c, h, w, 2, 1, 1, out.ctypes.data, idx.ctypes.data)
    # window at (2,2) only covers element 8 of each channel
    assert out[0, 8] == -8.0 and idx[0, 8] == 8
    assert out[1, 8] == -17.0 and idx[1, 8] == 17
    # ties: first maximum in (n, m) order wins
    y = np.zeros((1, 4), dtype=np.float32)
    o = np.empty((1, 4), dtype=np.float32)
    i = np.empty((1, 4), dtype=np.int32)
    orc.orc_maxpool(y.ctypes.data, 1, 1, 2, 2, 2, 2, 1, o.ctypes.data, i.ctypes.data)
    assert o[0, 0] == 0.0 and i[0, 0] == 0


@pytest.mark.parametrize("name", ["yolov2-tiny", "yolov2-608"])
def test_oracle_matches_reference_golden_of_benchmarked_nets(name):
    """The oracle composition equals, bit for bit, the outputs the reference's
    `command_evaluate` recorded for the 16-image loops bench.py times
    (tests/golden/make_cnn_golden.py): the first and last image in full and
    every sample entry that falls in them."""
    from conftest import big_golden
    entry, full = big_golden(name)
    images = entry["images"]
    net = build_net(name, images=images)
    ids = sorted(full)
    got = cprog.reference_forward(net, workers=len(ids), image_ids=ids)["outputs"]
    per = int(np.prod(entry["shape"][1:]))
    stride = entry["sample_stride"]
    for k, b in enumerate(ids):
        assert np.array_equal(got[k], full[b]), b
        lo, hi = b * per, (b + 1) * per
        first = -(-lo // stride)
        for j in range(first, -(-hi // stride)):
            assert float(got[k].ravel()[j * stride - lo]) == entry["sample"][j]
        flat = got[k].astype(np.float64).ravel()
        assert float(flat.sum()) == pytest.approx(entry["per_image_sum"][b], rel=0, abs=1e-9)
