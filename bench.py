#!/usr/bin/env python
"""Benchmark: the offload-pattern hot path of arXiv 1811.03882 on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--net yolov2-tiny] [--images 16]

Workload (BASELINE.json configs[1]): the yolov2-tiny 416x416 Darknet forward,
batch 1 per forward pass, written as the C-subset program of
paper_1811_03882_b200/nets.py; one STEP = one run of its image loop over
`--images` synthetic images with the all-offload genome and the planner's
hoisted transfers.

Legs printed on one JSON line (rank 0):
  value      img/s with every input image already resident in HBM (kernels
             only; CUDA events on the executor's stream; L2 flushed by a
             256 MiB write before every step), max over ranks;
  e2e        img/s through the public executor path: pinned host buffers,
             every planned H2D/D2H inside the timed region;
  roofline   dominant kernel kind from a profiled pass of the same schedule
             (CUDA event pair around every launch);
  cpu_baseline  the reference CPU path (gcc -O3 -march=native all-zero
             genome program, one process per host core, bounded sample);
  ga_search  wall seconds of the reference demo GA (pop 4 x 2 gens) with
             the gpu: evaluator;
  transfers_per_image  counted H2D/D2H calls and bytes per image.
`--impl reference` times only the reference CPU path (all host cores) on the
same metric.  Multi-GPU (torchrun): each rank runs its own image loop on its
own GPU (weak scaling, no data-path collective).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "img/s on best offload pattern; GA search wall-s; H2D/D2H transfers per image"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--net", default="yolov2-tiny")
    ap.add_argument("--images", type=int, default=16)
    ap.add_argument("--gemm", default="auto", choices=("auto", "simt", "tc"))
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--batch", type=int, default=0,
                    help="images per launch of the image loop's body (0 = all images of a "
                         "step, 1 = image at a time)")
    ap.add_argument("--no-ga", action="store_true")
    ap.add_argument("--quick", action="store_true",
                    help="main leg + demo GA only (skip yolov2-608, image-at-a-time and the "
                         "paper-scale GA)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-images", type=int, default=2, help="images per CPU process per step")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons while the timed legs run: NVML polled from a
    thread every ~2 ms (the value leg is only tens of ms long), falling back to
    `nvidia-smi -lms 100` when NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple] = []
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.nvml = (pynvml, h)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:  # noqa: BLE001 -- no NVML: use nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                                     int(get_reasons(h))))
            except Exception:  # noqa: BLE001
                break
            time.sleep(0.002)

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None:
            self.thread.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for clk, top, bits in self.samples:
            sm.append(float(clk))
            mx.append(float(top))
            reasons.update(n for n, b in self.BITS.items() if bits & b)
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


# ----------------------------------------------------------- cpu baseline
def cpu_program(net_name: str, images: int, workdir: Path):
    from oracle import cprog  # reference CPU path (test infrastructure)
    from paper_1811_03882_b200.nets import build_net
    net = build_net(net_name, images=images)
    return cprog.build(net, workdir, cflags=cprog.BASELINE_CFLAGS)


def cpu_step(binary: Path, procs: int) -> tuple[float, list]:
    """One bounded CPU step: `procs` concurrent program runs; returns the
    slowest run's timed-forward seconds and all of them."""
    from oracle import cprog
    with ThreadPoolExecutor(max_workers=procs) as pool:
        infos = list(pool.map(lambda k: cprog.run(binary, seed=1 + k), range(procs)))
    secs = [i["seconds"] for i in infos]
    return max(secs), secs


def cpu_baseline(net_name: str, images: int, steps: int = 1) -> dict:
    procs = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as tmp:
        binary = cpu_program(net_name, images, Path(tmp))
        cpu_step(binary, 1)  # warm the page cache / CPU
        worst = []
        for _ in range(steps):
            w, _ = cpu_step(binary, procs)
            worst.append(w)
        single = min(cpu_step(binary, 1)[1])
    t = statistics.median(worst)
    return {"value": procs * images / t, "unit": "img/s", "cores": procs, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{procs} concurrent processes x {images} images of the gcc -O3 "
                      f"-march=native all-zero-genome {net_name} C-subset program (the "
                      f"reference cmd: CPU path), median of {steps} step(s)",
            "single_core_img_per_s": images / single}


# -------------------------------------------------------------- reference
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as tmp:
        binary = cpu_program(args.net, args.cpu_images, Path(tmp))
        for _ in range(args.warmup):
            cpu_step(binary, procs)
        times = []
        for _ in range(args.steps):
            w, _ = cpu_step(binary, procs)
            times.append(w)
    total = sum(times)
    value = procs * args.cpu_images * args.steps / total
    from paper_1811_03882_b200.nets import NETS
    dims = f"{NETS[args.net].height}x{NETS[args.net].width}"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "img/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.net} {dims} batch 1 per forward (C-subset program, "
                               f"all-zero genome = reference CPU path)",
                   "images_per_process_step": args.cpu_images, "processes": procs},
        "cpu_baseline": {"value": value, "unit": "img/s", "cores": procs, "kind": "port",
                         "sample": f"{procs} processes x {args.cpu_images} images per step"},
        "e2e": {"value": value, "unit": "img/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ verification
def golden_entry(net_name: str, images: int, first_image: int):
    """The reference CPU path's recorded outputs for this 16-image loop
    (tests/golden/cnn_outputs_big.json + .npy, written by
    tests/golden/make_cnn_golden.py through the reference's
    `command_evaluate`), or None when this workload has no record."""
    import numpy as np
    path = REPO / "tests" / "golden" / "cnn_outputs_big.json"
    if first_image != 0 or not path.exists():
        return None
    entry = json.loads(path.read_text()).get(net_name)
    if entry is None or entry["images"] != images or entry["seed"] != 1:
        return None
    full = {int(b): np.load(path.parent / f) for b, f in entry["full_images"].items()}
    return entry, full


def verify_outputs(what: str, outputs, golden) -> dict:
    """Outputs of a timed leg against the reference's recorded outputs
    (tolerance.py).  A mismatch ends the run with a non-zero exit and no
    bench line."""
    from paper_1811_03882_b200 import tolerance
    if golden is None:
        return {"checked": False, "why": "no recorded reference outputs for this workload/shard"}
    try:
        st = tolerance.check_golden(outputs, *golden)
    except AssertionError as exc:
        sys.stderr.write(f"bench.py: {what} outputs differ from the reference CPU path: {exc}\n")
        raise SystemExit(3)
    return {"checked": True, "against": "tests/golden/cnn_outputs_big.json (reference "
            "command_evaluate of the gcc-compiled program)",
            "tolerance": {"max_rel": tolerance.REL, "floor": tolerance.FLOOR,
                          "norm_rel": tolerance.NORM},
            **{k: v for k, v in st.items() if not isinstance(v, dict)},
            "full_images": {k: {"max_rel": v["max_rel"], "norm_rel": v["norm_rel"]}
                            for k, v in st.items() if isinstance(v, dict)}}


# -------------------------------------------------------------------- ours
def ncu_traffic(shape: str):
    """dram bytes (read + write) per launch of the kernel launch with this
    gemm shape, from the committed `ncu --set full` summaries in profiles/
    (lines `shape = MxNxK` ... `dram__bytes_read.sum = X Mbyte` ...)."""
    for path in sorted((REPO / "profiles").glob("r*_ncu_full*.txt")):
        cur, rd, wr = None, None, None
        for line in path.read_text().splitlines():
            if line.startswith("shape = "):
                cur, rd, wr = line.split("=", 1)[1].strip(), None, None
            elif line.startswith("dram__bytes_read.sum = ") and cur == shape:
                rd = float(line.split()[2])
            elif line.startswith("dram__bytes_write.sum = ") and cur == shape:
                wr = float(line.split()[2])
            if rd is not None and wr is not None:
                return {"bytes": (rd + wr) * 1e6, "source": path.name}
    return None


def roofline(ex, sched, steps: int, flush, peaks: dict) -> dict:
    """Roofline of the dominant kernel launch of one resident step: its
    algorithmic flops (2MNK) or bytes over its average launch
    duration, timed live with CUDA events on the launch stream."""
    import torch
    per_action: dict[int, float] = {}
    for _ in range(steps):
        with torch.cuda.stream(ex.stream):
            flush.zero_()
        r = ex.run(sched, profile=True)
        for k, ms in enumerate(r.kernel_ms):
            if sched.actions[k].kind == 8 and ms > 0:
                per_action[k] = per_action.get(k, 0.0) + ms
    infos = {k: ex.action_op(sched, k) for k in per_action}
    per_kind_ms: dict[str, float] = {}
    per_kind_work: dict[str, dict] = {}
    for k, ms in per_action.items():
        info = infos[k]
        kind = info["kind"] + ("+epilogue" if info.get("fused") else "")
        per_kind_ms[kind] = per_kind_ms.get(kind, 0.0) + ms
        w = per_kind_work.setdefault(kind, {"flops": 0, "bytes": 0})
        w["flops"] += info["flops"] * info["executions"] * steps
        w["bytes"] += info["bytes"] * info["executions"] * steps
    total = sum(per_action.values())
    top = max(per_action, key=per_action.get)
    info = infos[top]
    launches = info["executions"] * steps
    launch_s = per_action[top] * 1e-3 / launches
    # the roofline that binds: FP32-accurate gemm (3xTF32) peaks at bf16/6; a
    # launch whose arithmetic intensity is below that ceiling's ridge point
    # (flop per HBM byte) is HBM-bound and is reported against HBM
    ridge = (peaks.get("bf16_tflops", 1.0) / 6 * 1e12) / (peaks.get("hbm_gbs", 1.0) * 1e9)
    tensor_bound = info["flops"] and info["flops"] / max(info["bytes"], 1) >= ridge
    shape = (f"{info['M']}x{info['N_launch']}x{info['K']}" if info["flops"] else None)
    if tensor_bound:
        achieved = info["flops"] / launch_s / 1e12
        peak = peaks.get("bf16_tflops")
        out = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
               "frac": achieved / peak if peak else None,
               "peak_note": "measured dense bf16 burst (MEASURED_PEAKS.json); FP32-accurate gemm "
                            "via 3xTF32 = 3 tf32 MMAs (half bf16 rate) per FP32 MAC, so its "
                            "ceiling is peak/6",
               "frac_of_3xtf32_ceiling": achieved / (peak / 6) if peak else None}
    else:
        achieved = info["bytes"] / launch_s / 1e9
        peak = peaks.get("hbm_gbs")
        out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
               "frac": achieved / peak if peak else None}
        if info["flops"]:
            out["note"] = (f"gemm below the 3xTF32 ridge ({info['flops'] / info['bytes']:.1f} "
                           f"< {ridge:.1f} flop/B): HBM-bound; {info['flops'] / launch_s / 1e12:.1f} "
                           "TFLOP/s")
        if info.get("engine") == "fp32-fma":
            # CUDA-core FP32: 148 SMs x 128 FMA/clk x 2 flop at the sampled max clock
            fma_peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
            out["fp32_fma_peak_tflops"] = fma_peak
            out["frac_of_fp32_fma_peak"] = info["flops"] / launch_s / 1e12 / fma_peak
            out["note"] = (f"FP32-FMA window kernel (fused im2col + gemm + bias + leaky + maxpool): "
                           f"{info['flops'] / launch_s / 1e12:.1f} TFLOP/s of a {fma_peak:.1f} "
                           f"TFLOP/s CUDA-core peak; issue-bound (K = {info['K']} leaves the "
                           "per-output epilogue at a third of the instructions)")
    traffic = ncu_traffic(shape) if shape else None
    name = f"{info['kind']} layer {info['layer']}" + (
        f" M{info['M']} N{info['N_launch']} K{info['K']} ({info['images']} images per launch)"
        if info["flops"] else "")
    out.update({"kernel": name, "share_of_step": per_action[top] / total if total else None,
                "launches_per_step": info["executions"],
                "algorithmic_per_launch": info["flops"] if tensor_bound else info["bytes"],
                "launch_us": launch_s * 1e6,
                "traffic": traffic["bytes"] if traffic else None,
                "traffic_source": traffic["source"] if traffic else None,
                "per_kind_ms_per_step": {k: v / steps for k, v in sorted(per_kind_ms.items())},
                "per_kind_hbm_gbs": {k: per_kind_work[k]["bytes"] / (per_kind_ms[k] * 1e-3) / 1e9
                                     for k in per_kind_ms},
                "per_kind_tflops": {k: per_kind_work[k]["flops"] / (per_kind_ms[k] * 1e-3) / 1e12
                                    for k in per_kind_ms if per_kind_work[k]["flops"]}})
    return out


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _net_program(net_name: str, images: int | None = None):
    from paper_1811_03882_b200 import (build_genome_map, build_loop_tree,
                                       check_all_parallelizable, extract_accesses, parse)
    from paper_1811_03882_b200.legality import profile_from_dict
    from paper_1811_03882_b200.nets import build_net
    net = build_net(net_name, images=images)
    prog = parse(net.source)
    tree = build_loop_tree(prog)
    acc = extract_accesses(prog)
    gm = build_genome_map(check_all_parallelizable(tree, acc))
    prof = profile_from_dict(net.profile_dict(), net_name, tree)
    return net, prog, tree, acc, gm, prof


def ga_gpu(net_name: str, images: int | None, devices, pop: int, gens: int, seed: int,
           warmup: int, repeats: int, per_device: int = 1) -> dict:
    """The GA (reference run_ga semantics, ga.py:170-282) with the gpu:
    evaluator: every individual's offload pattern executed on B200,
    `per_device` executors per GPU, workers = executors."""
    from paper_1811_03882_b200 import GAConfig, MeasurementCache, run_ga
    from paper_1811_03882_b200.gpu_evaluator import GpuEvaluatorConfig, make_gpu_evaluator
    net, prog, tree, acc, gm, prof = _net_program(net_name, images)
    cfg = GpuEvaluatorConfig(net=net_name, images=images, devices=devices, repeats=repeats,
                             warmup=warmup, workers_per_device=per_device)
    ga = GAConfig(population=pop, generations=gens, rng_seed=seed,
                  workers=len(devices) * per_device)
    t0 = time.perf_counter()
    ev = make_gpu_evaluator(cfg, prog, tree, acc, gm, prof)
    setup = time.perf_counter() - t0
    t1 = time.perf_counter()
    res = run_ga(ga, gm, tree, ev, MeasurementCache())
    wall = time.perf_counter() - t1
    a = len(gm)
    return {"config": f"{net_name} ({a} genes, {net.spec.images} image(s) per evaluation), "
                      f"pop {pop} x {gens} gens, seed {seed}, {len(devices)} GPU(s) x "
                      f"{per_device} executor(s) = workers, "
                      f"warm-up {warmup} + median of {repeats} run(s) per evaluation",
            "wall_s": wall, "setup_s": setup, "evaluations": res.evaluations_performed,
            "cache_hits": res.cache_hits, "seconds_per_evaluation": wall / max(1, res.evaluations_performed),
            "best_genome": res.best.genome, "best_seconds": res.best.seconds,
            "all_one_seconds": ev.pool.measure("1" * a).seconds,
            "all_zero_seconds": ev.pool.measure("0" * a).seconds,
            "history": [{"gen": h.generation, "best_seconds": h.best_seconds,
                         "evals": h.evaluations_performed} for h in res.history]}


def ga_reference(net_name: str, images: int | None, pop: int, gens: int, seed: int,
                 workers: int) -> dict:
    """The reference's GA CPU path: run_ga over the `cmd:` evaluator
    (pipeline.py:136-148, evaluation.py:162-196) -- each individual's
    emitted source compiled by gcc (which ignores the OpenACC pragmas, so
    every pattern runs on the CPU) and timed as a subprocess; `workers`
    concurrent evaluations on the host cores.  Bounded to `gens`
    generations; per-evaluation seconds are the comparison."""
    from oracle import cprog  # reference CPU path harness (test infrastructure)
    from paper_1811_03882_b200 import GAConfig, MeasurementCache, run_ga
    from paper_1811_03882_b200.measure import CommandEvaluatorConfig
    from paper_1811_03882_b200.tuner import make_cmd_evaluator
    net, prog, tree, acc, gm, prof = _net_program(net_name, images)
    with tempfile.TemporaryDirectory() as tmp:
        t = Path(tmp)
        cprog.write_program(net, t)
        cfg = CommandEvaluatorConfig(compile_cmd=cprog.compile_cmd(t), run_cmd="'{bin}'",
                                     timeout_seconds=600.0, workdir=str(t))
        inner = make_cmd_evaluator(cfg, prog, tree, acc, gm)
        calls, lock = [], threading.Lock()

        def ev(bits):
            t = time.perf_counter()
            m = inner(bits)
            with lock:
                calls.append((time.perf_counter() - t, m.seconds))
            return m

        t0 = time.perf_counter()
        res = run_ga(GAConfig(population=pop, generations=gens, rng_seed=seed, workers=workers,
                              timeout_seconds=600.0), gm, tree, ev, MeasurementCache())
        wall = time.perf_counter() - t0
    n = max(1, res.evaluations_performed)
    return {"config": f"{net_name} ({len(gm)} genes, {net.spec.images} image(s) per "
                      f"evaluation), pop {pop} x {gens} gen(s) (bounded), seed {seed}, "
                      f"{workers} concurrent evaluations on host cores; gcc -O2 cmd: evaluator",
            "kind": "port", "cores": workers, "cpu_model": cpu_model(),
            "wall_s": wall, "evaluations": res.evaluations_performed,
            "seconds_per_evaluation": wall / n,
            "evaluation_latency_s": statistics.median([c[0] for c in calls]) if calls else None,
            "program_run_s": statistics.median([c[1] for c in calls]) if calls else None,
            "best_seconds": res.best.seconds}


def max_over_ranks(v: float, world: int, device=None) -> float:
    """The largest of every rank's `v` (the job's time is its slowest rank's):
    all_reduce MAX over the default process group (NCCL on the GPUs, gloo on
    CPU tensors when `device` is None)."""
    if world == 1:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def weak_scaling(world: int, images: int, steps: int, local_seconds: float, device=None):
    """Weak scaling: every rank runs `images` images per step on its own GPU;
    the value is every image of every rank over the slowest rank's time.
    Returns (img/s, job seconds)."""
    total = max_over_ranks(local_seconds, world, device)
    return world * images * steps / total, total


def make_flush(torch, device):
    return torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)


def net_leg(args, net_name: str, images: int, batch, world: int, rank: int, local: int,
            flush, steps: int, warmup: int, roofline_steps: int = 3, verify: bool = True) -> dict:
    """One workload: `images`-image loop of `net_name`, all-offload genome,
    hoisted transfers.  value = kernels only with inputs resident in HBM
    (CUDA events on the executor stream, L2 flushed before every step);
    e2e = the public executor path with pinned host buffers and every planned
    transfer inside the timed region."""
    import torch

    from paper_1811_03882_b200 import kernels as K
    from paper_1811_03882_b200.executor import PatternExecutor
    from paper_1811_03882_b200.nets import build_net
    from paper_1811_03882_b200.sharding import image_shard

    gemm_mode = {"auto": K.GEMM_AUTO, "simt": K.GEMM_SIMT, "tc": K.GEMM_TC3XTF32}[args.gemm]
    net = build_net(net_name, images=images)
    # weak scaling: rank r owns images [r*images, (r+1)*images) of the stream
    shard = image_shard(world * images, world, rank)
    ex = PatternExecutor(net, device=local, fuse=not args.no_fuse, gemm_mode=gemm_mode,
                         first_image=shard.first, batch=batch)
    bits = "1" * len(net.ops)
    full = ex.compile(bits)
    res = ex.compile(bits, resident=True)

    def barrier():
        torch.cuda.synchronize(ex.device)
        if world > 1:
            torch.distributed.barrier()

    for _ in range(warmup):
        ex.run(res)
        ex.run(full)

    # ---- value: kernels only, inputs resident in HBM ----
    barrier()
    step_ms = []
    launches = 0
    for _ in range(steps):
        with torch.cuda.stream(ex.stream):
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ex.stream)
        r = ex.run(res)
        e1.record(ex.stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        launches += r.counters["kernel_launches"]
    barrier()
    value, total = weak_scaling(world, images, steps, sum(step_ms) * 1e-3, ex.device)

    # ---- e2e: public path, host buffers, transfers inside the region ----
    barrier()
    walls = []
    counters = None
    for _ in range(steps):
        with torch.cuda.stream(ex.stream):
            flush.zero_()
        torch.cuda.synchronize(ex.device)
        r = ex.run(full)
        walls.append(r.seconds)
        counters = r.counters
    barrier()
    e2e_value, e2e_total = weak_scaling(world, images, steps, sum(walls), ex.device)
    for key, val in full.expected.items():
        if counters[key] != val:
            raise SystemExit(f"transfer counter mismatch {key}: {counters[key]} != {val}")
    out = {"net": net, "ex": ex, "full": full, "res": res, "value": value, "total_s": total,
           "e2e_value": e2e_value, "e2e_total_s": e2e_total, "counters": counters,
           "launches": launches, "step_ms": step_ms, "walls": walls}
    if verify:
        # the last timed e2e step's outputs, then the resident leg's (one
        # more untimed run: the timed loop above ran the e2e schedule last)
        golden = golden_entry(net_name, images, shard.first)
        verified = {"e2e": verify_outputs(f"{net_name} e2e", ex.outputs(), golden)}
        if res.batch == images:
            ex.run(res)
            verified["value"] = verify_outputs(f"{net_name} resident", ex.device_outputs(), golden)
        out["verified"] = verified
    if rank == 0 and roofline_steps:
        peaks_path = REPO / "MEASURED_PEAKS.json"
        peaks = json.loads(peaks_path.read_text()) if peaks_path.exists() else \
            {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}
        out["roofline"] = roofline(ex, res, roofline_steps, flush, peaks)
    return out


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    flush = make_flush(torch, torch.device("cuda", local))

    # clocks are sampled from the first warm-up step to the end of the last
    # timed GPU leg (every step in between keeps the GPU busy); see ClockSampler
    clocks = ClockSampler(local).__enter__()
    main = net_leg(args, args.net, args.images, args.batch or True, world, rank, local, flush,
                   args.steps, args.warmup, roofline_steps=max(1, min(args.steps, 3)))
    extra = {}
    if world == 1 and not args.quick:
        # BASELINE configs[4]: YOLOv2-608, 16-image loop
        leg = net_leg(args, "yolov2-608", 16, True, world, rank, local, flush,
                      max(3, args.steps // 2), args.warmup, roofline_steps=1)
        extra["yolov2_608"] = leg
        # configs[1] image at a time (batch 1 per launch, graph-captured)
        extra["image_at_a_time"] = net_leg(args, args.net, args.images, 1, world, rank, local,
                                           flush, args.steps, args.warmup, roofline_steps=0)
    time.sleep(0.25)  # let the sampler log the tail of the loaded period
    clocks.__exit__(None, None, None)

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()          # rank 0 runs the GA legs on every GPU
            torch.distributed.destroy_process_group()
        return

    ex, net, counters = main["ex"], main["net"], main["counters"]
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.net, args.cpu_images, steps=3)
    devices = list(range(world))
    ga = ga_ref = ga_paper = ga_paper_ref = None
    if not args.no_ga:
        ga = ga_gpu("demo", None, devices, 4, 2, 1, 1, 3)
        ga["config"] = "BASELINE configs[0]: " + ga["config"]
        if world == 1:
            ga_ref = ga_reference("demo", None, 4, 2, 1, os.cpu_count() or 1)
        if not args.quick:
            ga_paper = ga_gpu(args.net, 1, devices, 30, 20, 1, 1, 1)
            ga_paper["config"] = "BASELINE configs[2]: " + ga_paper["config"]
            # the same search with several executors per GPU: evaluations are
            # dominated by single-threaded host loops, which then run on
            # separate host cores (GPU work of concurrent evaluations shares
            # the device, so fitness includes that contention)
            per = max(1, min(8, (os.cpu_count() or 1) // (2 * world)))
            if per > 1:
                ga_conc = ga_gpu(args.net, 1, devices, 30, 20, 1, 1, 1, per_device=per)
                ga_conc["config"] = "BASELINE configs[2], concurrent: " + ga_conc["config"]
                ga_paper["concurrent"] = ga_conc
            if world == 1:
                ga_paper_ref = ga_reference(args.net, 1, 30, 1, 1, os.cpu_count() or 1)
    if world > 1:
        torch.distributed.barrier()

    def sub(leg, cpu_images=None):
        d = {"value": leg["value"], "unit": "img/s", "ms_per_step": 1e3 * leg["total_s"] / len(leg["step_ms"]),
             "images_per_step": leg["net"].spec.images,
             "images_per_launch": leg["res"].batch,
             "e2e": {"value": leg["e2e_value"], "unit": "img/s",
                     "h2d_bytes_per_step": leg["counters"]["h2d_bytes"],
                     "d2h_bytes_per_step": leg["counters"]["d2h_bytes"]},
             "gpu_launches": leg["launches"]}
        if "roofline" in leg:
            d["roofline"] = leg["roofline"]
        if "verified" in leg:
            d["outputs_verified"] = leg["verified"]
        return d

    dims = f"{net.spec.height}x{net.spec.width}"
    line = {
        "metric": METRIC, "value": main["value"], "unit": "img/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * main["total_s"] / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.net} {dims}, batch 1 per forward pass, "
                               f"{args.images}-image loop per step, all-offload genome "
                               f"({len(net.ops)} genes) with hoisted transfers",
                   "images_per_step_per_gpu": args.images,
                   "genes": len(net.ops), "gemm": args.gemm, "fused_epilogues": not args.no_fuse,
                   "images_per_launch": main["res"].batch,
                   "l2": "flushed before every step (256 MiB write); per-step footprint "
                         f"{net.total_bytes_per_image() * args.images / 2**20:.0f} MiB",
                   "parallelism": f"images sharded, {world} GPU(s), no collective"},
        "e2e": {"value": main["e2e_value"], "unit": "img/s",
                "h2d_bytes_per_step": counters["h2d_bytes"],
                "d2h_bytes_per_step": counters["d2h_bytes"]},
        "roofline": main["roofline"],
        "cpu_baseline": cpu,
        "gpu_launches": main["launches"],
        "clocks": clocks.summary(),
        "transfers_per_image": {
            "directive_execs": counters["directive_execs"] / args.images,
            "var_transfers": counters["var_transfers"] / args.images,
            "h2d_calls": counters["h2d_calls"] / args.images,
            "d2h_calls": counters["d2h_calls"] / args.images,
            "h2d_bytes": counters["h2d_bytes"] / args.images,
            "d2h_bytes": counters["d2h_bytes"] / args.images},
        "outputs_verified": main.get("verified"),
        "ga_search": ga, "ga_search_reference": ga_ref,
        "ga_paper_scale": ga_paper, "ga_paper_scale_reference": ga_paper_ref,
        "value_step_ms": main["step_ms"], "e2e_step_s": main["walls"],
    }
    if "yolov2_608" in extra:
        leg = extra["yolov2_608"]
        d = sub(leg)
        d["config"] = "BASELINE configs[4]: yolov2-608 608x608, 16-image loop per step, " \
                      f"all-offload genome ({len(leg['net'].ops)} genes), batched 16 per launch"
        if not args.no_cpu_baseline:
            d["cpu_baseline"] = cpu_baseline("yolov2-608", 1, steps=1)
        line["yolov2_608"] = d
    if "image_at_a_time" in extra:
        d = sub(extra["image_at_a_time"])
        d["config"] = f"BASELINE configs[1] as written: {args.net}, one image per launch " \
                      "(image loop not batched), graph-captured resident leg"
        line["image_at_a_time"] = d
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse_args()
    # ACCT_* variables steer dispatch, tiles, tracing or the library path:
    # a timed run must measure the product configuration
    overrides = sorted(k for k in os.environ if k.startswith("ACCT_"))
    if overrides:
        raise SystemExit(f"bench.py: refusing to run with ACCT_* overrides set: {overrides}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
