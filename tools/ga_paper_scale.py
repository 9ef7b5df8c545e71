"""Paper-scale GA search (BASELINE configs[2]): population 30 x 20 generations
over every loop gene of a net, fitness = the gpu: evaluator (each individual's
offload pattern executed on B200), individuals spread over the given GPUs.

  python tools/ga_paper_scale.py --net yolov2-tiny --images 2 --devices all

Prints one JSON object: GA wall seconds, evaluations, cache hits, best genome
and its seconds, the all-offload and all-CPU patterns' seconds, and the
per-generation history (reference run_ga semantics, ga.py:170-282)."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1811_03882_b200 import (GAConfig, MeasurementCache, build_genome_map,  # noqa: E402
                                   build_loop_tree, check_all_parallelizable,
                                   extract_accesses, parse, run_ga)
from paper_1811_03882_b200.gpu_evaluator import (GpuEvaluatorConfig,  # noqa: E402
                                                 make_gpu_evaluator)
from paper_1811_03882_b200.legality import profile_from_dict  # noqa: E402
from paper_1811_03882_b200.nets import build_net  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="yolov2-tiny")
    ap.add_argument("--images", type=int, default=2)
    ap.add_argument("--pop", type=int, default=30)
    ap.add_argument("--gens", type=int, default=20)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--devices", default="all")
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    import torch
    devices = (list(range(torch.cuda.device_count())) if args.devices == "all"
               else [int(d) for d in args.devices.split(",")])
    net = build_net(args.net, images=args.images)
    prog = parse(net.source)
    tree = build_loop_tree(prog)
    acc = extract_accesses(prog)
    gm = build_genome_map(check_all_parallelizable(tree, acc))
    prof = profile_from_dict(net.profile_dict(), args.net, tree)
    cfg = GpuEvaluatorConfig(net=args.net, images=args.images, devices=devices,
                             repeats=args.repeats, warmup=args.warmup)
    ga = GAConfig(population=args.pop, generations=args.gens, rng_seed=args.seed,
                  workers=len(devices))
    t0 = time.perf_counter()
    ev = make_gpu_evaluator(cfg, prog, tree, acc, gm, prof)
    setup = time.perf_counter() - t0
    t1 = time.perf_counter()
    res = run_ga(ga, gm, tree, ev, MeasurementCache())
    wall = time.perf_counter() - t1
    a = len(gm)
    out = {"config": f"{args.net} {args.images} images per evaluation, pop {args.pop} x "
                     f"{args.gens} gens, seed {args.seed}, {len(devices)} GPU(s), "
                     f"warmup {args.warmup} + median of {args.repeats}",
           "genes": a, "wall_s": wall, "setup_s": setup,
           "evaluations": res.evaluations_performed, "cache_hits": res.cache_hits,
           "best_genome": res.best.genome, "best_seconds": res.best.seconds,
           "all_one_seconds": ev.pool.measure("1" * a).seconds,
           "all_zero_seconds": ev.pool.measure("0" * a).seconds,
           "history": [{"gen": h.generation, "best_seconds": h.best_seconds,
                        "evals": h.evaluations_performed} for h in res.history]}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
