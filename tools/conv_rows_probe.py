"""Time the narrow tcgen05 conv launch alone (acct_conv3x3_tc_f32) at the
yolov2 narrow-layer shapes over a batch sweep: the intercept of time vs
images is the launch's fixed cost, the slope its per-image cost.

    python tools/conv_rows_probe.py [--legacy] [--pool] [--reps 20]

(ACCT_LIB / ACCT_CONV_DBG select the profiling build and its work-skipping
bits, as for tools/profile_pattern.py.)
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1811_03882_b200 import kernels as K  # noqa: E402

SHAPES = {"tiny-L2": (16, 208, 208, 32), "tiny-L4": (32, 104, 104, 64),
          "608-L2": (32, 304, 304, 64)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--legacy", action="store_true")
    ap.add_argument("--pool", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--batches", default="1,2,4,8,16")
    ap.add_argument("--shapes", default=",".join(SHAPES))
    args = ap.parse_args()
    K.lib().acct_tc_set_conv_rows(0 if args.legacy else 1)
    s = torch.cuda.current_stream().cuda_stream
    for name in args.shapes.split(","):
        c, h, w, M = SHAPES[name]
        N = h * w
        ld = -(-N // 32) * 32
        lda = -(-9 * c // 32) * 32
        out = []
        for P in [int(b) for b in args.batches.split(",")]:
            im = torch.rand((c, P * ld), device="cuda") - 0.5
            A = (torch.rand((M, lda), device="cuda") - 0.5) * 0.1
            C = torch.zeros((M, P * ld), device="cuda")
            col = torch.zeros((9 * c, P * ld), device="cuda")
            bias = torch.rand(M, device="cuda")
            P2 = (h // 2) * (w // 2)
            ldp = -(-P2 // 32) * 32
            pool = torch.zeros((M, P * ldp), device="cuda")
            idx = torch.zeros((M, P * ldp), dtype=torch.int32, device="cuda")
            kw = {}
            if args.pool:
                kw["pool"] = (pool.data_ptr(), P * ldp, ldp, idx.data_ptr(), P * ldp, ldp, P - 1)

            def run():
                K.conv3x3_tc(im.data_ptr(), P * ld, ld, c, h, w, col.data_ptr(), P * ld, ld, M,
                             A.data_ptr(), lda, 0.0, C.data_ptr(), P * ld, ld, bias.data_ptr(),
                             K.ACT_LEAKY, P, s, col_from=P, **kw)
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / args.reps
            out.append((P, us))
        n = len(out)
        mx = sum(p for p, _ in out) / n
        my = sum(t for _, t in out) / n
        slope = sum((p - mx) * (t - my) for p, t in out) / sum((p - mx) ** 2 for p, _ in out)
        print(f"{name:8s} " + "  ".join(f"b{p}:{t:7.1f}" for p, t in out) +
              f"   fixed {my - slope * mx:6.1f} us + {slope:5.2f} us/img")


if __name__ == "__main__":
    main()
