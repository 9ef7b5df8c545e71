"""Multi-rank host logic on CPU (gloo, world_size 2): image sharding of the
offload pattern and the gather to rank 0 reproduce the single-process
result; GA individuals spread over a pool of workers keep the search
deterministic."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_03882_b200.sharding import gather_outputs, image_shard, run_image_shard


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_image_shard_partitions_the_stream():
    for total in (1, 2, 7, 16, 64):
        for world in (1, 2, 3, 8):
            shards = [image_shard(total, world, r) for r in range(world)]
            assert sum(s.count for s in shards) == total
            nxt = 0
            for s in shards:
                assert s.first == nxt
                nxt += s.count
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard, out, res = run_image_shard("micro", total, None, world, rank, device=None)
        full = gather_outputs(out, shard, total)
        if rank == 0:
            q.put((full, res.counters["host_ops"]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_sharded_image_run_matches_single_process():
    from oracle import cprog
    from paper_1811_03882_b200.nets import build_net
    total, world = 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, host_ops = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = cprog.reference_forward(build_net("micro", images=total))["outputs"]
    assert full.shape == want.shape
    assert np.array_equal(full, want)
    assert host_ops == len(build_net("micro").ops) * image_shard(total, world, 0).count


def test_ga_over_a_device_pool_is_deterministic():
    """A pool of N workers measuring individuals concurrently (the multi-GPU
    GA) gives the same search as one worker."""
    import hashlib
    import threading
    import time

    import paper_1811_03882_b200 as at
    from paper_1811_03882_b200.nets import build_net

    net = build_net("demo")
    prog = at.parse(net.source)
    tree = at.build_loop_tree(prog)
    gm = at.build_genome_map(at.check_all_parallelizable(tree, at.extract_accesses(prog)))
    lock = threading.Lock()
    busy = {"now": 0, "max": 0}

    def fake_gpu(bits):
        with lock:
            busy["now"] += 1
            busy["max"] = max(busy["max"], busy["now"])
        time.sleep(0.002)
        with lock:
            busy["now"] -= 1
        h = int(hashlib.sha256(bits.encode()).hexdigest()[:6], 16)
        return at.Measurement(0.1 + h / 1e7, "measured")

    results = []
    for workers in (1, 4):
        cfg = at.GAConfig(population=6, generations=4, rng_seed=3, workers=workers)
        r = at.run_ga(cfg, gm, tree, fake_gpu)
        results.append((r.best, [(s.best_seconds, s.mean_fitness) for s in r.history],
                        r.evaluations_performed))
    assert results[0] == results[1]
    assert busy["max"] > 1


def _bench_worker(rank, world, port, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r timed its steps at 1 + r seconds: the job took the slowest's
        value, total = bench.weak_scaling(world, 16, 10, 1.0 + rank)
        q.put((rank, value, total))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_bench_weak_scaling_arithmetic_over_ranks():
    """bench.py's value under torchrun: every rank's images over the MAX of the
    ranks' timed seconds (all_reduce over the process group), identical on
    every rank."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, value, total in got:
        assert total == 2.0
        assert value == world * 16 * 10 / 2.0
