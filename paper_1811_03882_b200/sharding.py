"""Multi-GPU sharding of the hot path.

Two independent axes, neither of which needs a data-path collective:

* GA individuals -- `gpu_evaluator.DevicePool` measures one genome per GPU
  at a time; the GA (reference `ga.py:210-214`) fans the distinct fresh
  genomes of a generation out through its order-preserving thread pool, so
  fitness gathers on the host and the search stays deterministic given the
  measurements.
* images -- one process per GPU (torchrun); rank r runs the best pattern on
  its contiguous slice of the image stream with its own copy of the hoisted
  weight transfers.  Outputs are gathered to rank 0 only when the caller asks
  (`gather_outputs`), outside any timed region.

`image_shard` is the single source of truth for which images a rank owns;
`run_image_shard` executes a rank's slice (on its GPU, or host-only for
all-zero genomes so the logic is testable on CPU with gloo).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    first: int          # first image index of the stream this rank owns
    count: int          # images this rank owns


def image_shard(total_images: int, world: int, rank: int) -> Shard:
    """Contiguous, balanced split of `total_images` over `world` ranks
    (the first `total % world` ranks get one extra image)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(total_images, world)
    first = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return Shard(rank, world, first, count)


def dist_env() -> tuple[int, int, int]:
    """(world, rank, local_rank) from torchrun's environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def run_image_shard(net_name: str, total_images: int, genome: str | None, world: int, rank: int,
                    device=None, seed: int = 1, **executor_kw):
    """Run this rank's images through the offload pattern; returns
    (shard, outputs[count, C, HW], RunResult).  device=None runs host-only
    (all-zero genome)."""
    from .executor import PatternExecutor
    from .nets import build_net
    shard = image_shard(total_images, world, rank)
    net = build_net(net_name, images=shard.count)
    ex = PatternExecutor(net, device=device, seed=seed, first_image=shard.first, **executor_kw)
    bits = genome if genome is not None else ("0" * len(net.ops) if device is None
                                              else "1" * len(net.ops))
    res = ex.run(bits)
    return shard, ex.outputs(), res


def gather_outputs(local: np.ndarray, shard: Shard, total_images: int, group=None):
    """Gather every rank's output slice to rank 0 (gloo/NCCL via
    torch.distributed; host tensors).  Returns the full (total, ...) array on
    rank 0 and None elsewhere.  Not on the timed path."""
    import torch
    import torch.distributed as dist
    world = shard.world
    if world == 1:
        return local
    per = [image_shard(total_images, world, r).count for r in range(world)]
    width = int(np.prod(local.shape[1:]))
    pad = max(per)
    buf = torch.zeros((pad, width), dtype=torch.float32)
    buf[: shard.count] = torch.from_numpy(local.reshape(shard.count, width))
    if dist.get_backend(group) == "nccl":
        buf = buf.cuda()
    bufs = [torch.zeros_like(buf) for _ in range(world)] if shard.rank == 0 else None
    dist.gather(buf, bufs, dst=0, group=group)
    if shard.rank != 0:
        return None
    parts = [b.cpu().numpy()[:n] for b, n in zip(bufs, per)]
    return np.concatenate(parts).reshape((total_images,) + local.shape[1:])
