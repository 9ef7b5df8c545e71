"""Shared test setup.

Markers: `gpu` -- needs a B200 (run with `pytest -m gpu`); everything else
runs on the CPU-only build container.
"""

from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@lru_cache(maxsize=None)
def golden_programs() -> dict:
    return {p["name"]: p for p in json.loads((GOLDEN / "reference_programs.json").read_text())}


@lru_cache(maxsize=None)
def golden_reports() -> list:
    return json.loads((GOLDEN / "reference_reports.json").read_text())


def analyze(source: str):
    import paper_1811_03882_b200 as at
    program = at.parse(source)
    return program, at.build_loop_tree(program), at.extract_accesses(program)


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@lru_cache(maxsize=None)
def big_golden(name: str):
    """(entry, {image index: full output}) of tests/golden/cnn_outputs_big.json:
    the reference CPU path's outputs for a benchmarked 16-image loop."""
    import numpy as np
    entry = json.loads((GOLDEN / "cnn_outputs_big.json").read_text())[name]
    full = {int(b): np.load(GOLDEN / f) for b, f in entry["full_images"].items()}
    return entry, full
