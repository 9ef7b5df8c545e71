"""Run one offload pattern a few times (for ncu launch lists / captures).

    python tools/profile_pattern.py [--net yolov2-tiny] [--images 2] [--runs 2]
                                    [--resident] [--gemm auto|simt|tc]

Prints per-kind device milliseconds from the in-process event profiler
(the same numbers bench.py's roofline uses) after the last run.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1811_03882_b200 import kernels as K  # noqa: E402
from paper_1811_03882_b200.executor import PatternExecutor  # noqa: E402
from paper_1811_03882_b200.nets import build_net  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="yolov2-tiny")
    ap.add_argument("--images", type=int, default=2)
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--resident", action="store_true")
    ap.add_argument("--gemm", default="auto", choices=("auto", "simt", "tc"))
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--batch", type=int, default=0, help="images per launch (0 = all)")
    ap.add_argument("--fuse-single", action="store_true",
                    help="conv launches for one-image loops too (executor.fuse_convs_single)")
    ap.add_argument("--conv-rows", type=int, default=0,
                    help="1: narrow convs (M <= 32) on the row-band kernel (acct_tc_set_conv_rows)")
    ap.add_argument("--graph", action="store_true",
                    help="1 plain run, then graph capture + replays (ncu: skip the first run's "
                         "launches); prints device ms per replay")
    args = ap.parse_args()
    K.lib().acct_tc_set_conv_rows(args.conv_rows)
    if args.graph:
        import torch
        mode = {"auto": K.GEMM_AUTO, "simt": K.GEMM_SIMT, "tc": K.GEMM_TC3XTF32}[args.gemm]
        net = build_net(args.net, images=args.images)
        ex = PatternExecutor(net, device=0, gemm_mode=mode, fuse=not args.no_fuse,
                             batch=args.batch or True)
        ex.fuse_convs_single = args.fuse_single
        sched = ex.compile("1" * len(net.ops), resident=args.resident)
        ex.run(sched)
        for _ in range(args.runs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ex.stream)
            r = ex.run(sched)
            e1.record(ex.stream)
            e1.synchronize()
            print(f"replay: {e0.elapsed_time(e1):.3f} ms device, {r.seconds * 1e3:.3f} ms wall, "
                  f"{args.images} images, launches {r.counters['kernel_launches']}, "
                  f"graph={'yes' if sched.graph is not None else 'no'}")
        return
    mode = {"auto": K.GEMM_AUTO, "simt": K.GEMM_SIMT, "tc": K.GEMM_TC3XTF32}[args.gemm]
    net = build_net(args.net, images=args.images)
    ex = PatternExecutor(net, device=0, gemm_mode=mode, fuse=not args.no_fuse,
                             batch=args.batch or True)
    ex.fuse_convs_single = args.fuse_single
    bits = "1" * len(net.ops)
    sched = ex.compile(bits, resident=args.resident)
    for _ in range(args.runs - 1):
        ex.run(sched)
    r = ex.run(sched, profile=True)
    per = {}
    for k, ms in enumerate(r.kernel_ms):
        if sched.actions[k].kind != K.A_KERNEL:
            continue
        info = ex.action_op(sched, k)
        key = f"{info['kind']} L{info['layer']}" + (f" M{info['M']} N{info['N']} K{info['K']}"
                                                    if info["kind"] == "gemm" else "")
        per[key] = per.get(key, 0.0) + ms
    tot = sum(per.values())
    for key, ms in sorted(per.items(), key=lambda kv: -kv[1]):
        print(f"{ms / args.images * 1e3:10.1f} us/img  {100 * ms / tot:5.1f}%  {key}")
    print(f"total {tot / args.images * 1e3:.1f} us/img; wall {r.seconds * 1e3:.2f} ms "
          f"for {args.images} images; launches {r.counters['kernel_launches']}")


if __name__ == "__main__":
    main()
