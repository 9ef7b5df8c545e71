"""The `gpu:<config.json>` evaluator: measure a genome by running its offload
pattern on B200.

Boundary contract (reference `pkg/src/acctuner/ga.py:170-217`,
`pipeline.py:151-163`, `evaluation.py:162-196`):

* `evaluate(bits) -> Measurement`, called only for valid uncached genomes,
  possibly concurrently from the GA's thread pool (`workers > 1`);
* status `measured` with wall-clock seconds > 0 of the program run; a run
  over `timeout_seconds` -> `Measurement(penalty, "timeout")`;
* infrastructure failures (CUDA errors, missing library) raise
  `DeviceError` -- never a penalty, as `SpawnError` in the reference.

Config file (all keys optional except `net`):

    {"net": "yolov2-tiny", "images": 16, "devices": [0, 1] | "all",
     "seed": 1, "warmup": 1, "repeats": 3, "fuse": true,
     "gemm": "auto" | "simt" | "tc", "timeout_seconds": 180,
     "penalty_seconds": 1000, "workers_per_device": 1}

`net` names a built-in program (the tuned source must then be its text:
`python -m paper_1811_03882_b200.nets <net> <dir>`), or is "auto": any
program written in the C-subset templates -- the op manifest
(kinds, shapes, operands, array roles) is read off the tuned source by
`nets.net_from_source`, which recognises every loop of the image loop as a
template op or refuses the program (ModelError, exit 14).

Multi-GPU: one `PatternExecutor` per entry of `devices` and a queue of idle
entries; a GA with `workers = len(devices)` measures one individual per
entry at a time (a device may be listed more than once).
Fitness values are gathered by the GA's order-preserving `pool.map`, so the
search stays deterministic given the measurements.  No collective is needed
(nothing crosses between GPUs).
"""

from __future__ import annotations

import json
import queue
import statistics
import threading
from dataclasses import dataclass, field
from pathlib import Path

from . import kernels as K
from .errors import ModelError
from .measure import MEASURED, TIMEOUT, Measurement
from .nets import NETS, build_net

_GEMM_MODES = {"auto": K.GEMM_AUTO, "simt": K.GEMM_SIMT, "tc": K.GEMM_TC3XTF32}


AUTO = "auto"


@dataclass
class GpuEvaluatorConfig:
    net: str = "yolov2-tiny"     # a NETS name, or "auto": the op manifest read off the tuned source
    images: int | None = None
    devices: object = field(default_factory=lambda: [0])
    seed: int = 1
    warmup: int = 1
    repeats: int = 3
    fuse: bool = True
    gemm: str = "auto"
    timeout_seconds: float = 180.0
    penalty_seconds: float = 1000.0
    # executors per listed device: the host loops of partially offloaded
    # patterns dominate an evaluation, so several concurrent evaluations per
    # GPU (one host thread each) use the host cores; their GPU work shares
    # the device, so the measured seconds include that contention
    workers_per_device: int = 1

    def __post_init__(self):
        if self.net is None:
            self.net = AUTO
        if self.net != AUTO and self.net not in NETS:
            raise ModelError(f"gpu evaluator: unknown net {self.net!r} "
                             f"(known: {sorted(NETS)}, or {AUTO!r})")
        if self.gemm not in _GEMM_MODES:
            raise ModelError(f"gpu evaluator: gemm must be one of {sorted(_GEMM_MODES)}")
        if self.repeats < 1 or self.warmup < 0:
            raise ModelError("gpu evaluator: repeats >= 1 and warmup >= 0 required")
        if self.workers_per_device < 1:
            raise ModelError("gpu evaluator: workers_per_device >= 1 required")


def load_gpu_config(path) -> GpuEvaluatorConfig:
    try:
        doc = json.loads(Path(path).read_text())
    except (OSError, json.JSONDecodeError) as exc:
        raise ModelError(f"cannot read gpu evaluator config {path}: {exc}") from exc
    if not isinstance(doc, dict):
        raise ModelError(f"gpu evaluator config {path}: expected an object")
    try:
        return GpuEvaluatorConfig(**doc)
    except TypeError as exc:
        raise ModelError(f"gpu evaluator config {path}: {exc}") from exc


def resolve_devices(spec) -> list[int]:
    import torch
    n = torch.cuda.device_count()
    if spec == "all":
        return list(range(n))
    ids = [int(d) for d in (spec if isinstance(spec, (list, tuple)) else [spec])]
    bad = [d for d in ids if d < 0 or d >= n]
    if bad or not ids:
        raise ModelError(f"gpu evaluator: devices {ids} not available ({n} visible)")
    return ids


class DevicePool:
    """One PatternExecutor per SLOT of `devices`; `measure(bits)` borrows an
    idle slot.  A device listed twice (e.g. `[0, 0]`) gets two independent
    executors -- own buffers, stream, pinned arena and schedule cache -- so
    two GA workers never share one; each executor is also guarded by its own
    lock."""

    def __init__(self, cfg: GpuEvaluatorConfig, net=None):
        from .executor import PatternExecutor
        self.cfg = cfg
        self.net = net if net is not None else build_net(cfg.net, images=cfg.images)
        self.devices = resolve_devices(cfg.devices) * cfg.workers_per_device
        self.executors = [PatternExecutor(self.net, device=d, seed=cfg.seed, fuse=cfg.fuse,
                                          gemm_mode=_GEMM_MODES[cfg.gemm]) for d in self.devices]
        self.locks = [threading.Lock() for _ in self.devices]
        self.idle: queue.Queue = queue.Queue()
        for slot in range(len(self.devices)):
            self.idle.put(slot)
        self.log_lock = threading.Lock()
        self.log: list[dict] = []
        self.capture_outputs = False   # tests: keep each measured genome's output slots

    def measure(self, bits: str) -> Measurement:
        slot = self.idle.get()
        try:
            with self.locks[slot]:
                return self._measure(slot, bits)
        finally:
            self.idle.put(slot)

    def _measure(self, slot: int, bits: str) -> Measurement:
        ex = self.executors[slot]
        sched = ex.compile(bits)
        for _ in range(self.cfg.warmup):
            r = ex.run(sched, timeout_s=self.cfg.timeout_seconds)
            if r.status == TIMEOUT:
                return self._record(bits, slot, None, r, Measurement(self.cfg.penalty_seconds, TIMEOUT))
        times = []
        last = None
        for _ in range(self.cfg.repeats):
            last = ex.run(sched, timeout_s=self.cfg.timeout_seconds)
            if last.status == TIMEOUT or last.seconds > self.cfg.timeout_seconds:
                return self._record(bits, slot, None, last,
                                    Measurement(self.cfg.penalty_seconds, TIMEOUT))
            times.append(last.seconds)
        secs = statistics.median(times)
        return self._record(bits, slot, times, last, Measurement(secs, MEASURED), sched)

    def _record(self, bits, slot, times, run, m: Measurement, sched=None) -> Measurement:
        entry = {"genome": bits, "device": self.devices[slot], "slot": slot, "times": times,
                 "counters": run.counters if run else None, "status": m.status,
                 "expected": sched.expected if sched is not None else None}
        if self.capture_outputs and sched is not None:
            entry["outputs"] = self.executors[slot].outputs()
        with self.log_lock:
            self.log.append(entry)
        return m


def net_for(cfg: GpuEvaluatorConfig, program):
    """The NetProgram the evaluator executes: a built-in net whose source
    must be the tuned program, or (net "auto") the op manifest read off the
    tuned program's text (`nets.net_from_source`)."""
    if cfg.net != AUTO:
        net = build_net(cfg.net, images=cfg.images)
        if program is not None and program.source_text != net.source:
            raise ModelError(f"gpu evaluator: the tuned source is not the {cfg.net!r} program "
                             f"(write it with `python -m paper_1811_03882_b200.nets {cfg.net} "
                             f"DIR`, or use \"net\": \"{AUTO}\")")
        return net
    if program is None:
        raise ModelError('gpu evaluator: net "auto" needs the tuned program')
    from .nets import ProgramError, net_from_source
    try:
        net = net_from_source(program.source_text, name=AUTO)
    except ProgramError as exc:
        raise ModelError(f"gpu evaluator: {exc}") from exc
    if cfg.images is not None and cfg.images != net.spec.images:
        raise ModelError(f"gpu evaluator: images {cfg.images} != the program's image loop "
                         f"trip count {net.spec.images}")
    return net


def make_gpu_evaluator(cfg: GpuEvaluatorConfig, program, tree, accesses, genome_map, profile):
    pool = DevicePool(cfg, net_for(cfg, program))

    def evaluate(bits: str) -> Measurement:
        return pool.measure(bits)

    def report_section(best_bits: str) -> dict:
        ex = pool.executors[0]
        with pool.locks[0]:
            sched = ex.compile(best_bits)
            run = ex.run(sched)
        return {"net": cfg.net, "images": ex.images, "devices": pool.devices,
                "best_seconds_rerun": run.seconds,
                "img_per_s": ex.images / run.seconds,
                "transfers": run.counters, "expected_transfers": sched.expected,
                "fused_gemm_groups": len(sched.fused_groups)}

    evaluate.pool = pool
    evaluate.report_section = report_section
    return evaluate
