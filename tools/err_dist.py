"""Error distribution of the benchmarked all-offload schedules against the C
oracle: max-relative (to max|ref|), normwise, and the smallest floor tau for
which |d| <= 1e-4*|ref| + tau*max|ref| holds element-wise, per gemm mode.

    python tools/err_dist.py yolov2-tiny 16
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import cprog  # noqa: E402
from paper_1811_03882_b200 import kernels as K  # noqa: E402
from paper_1811_03882_b200.executor import PatternExecutor  # noqa: E402
from paper_1811_03882_b200.nets import build_net  # noqa: E402


def stats(got, want):
    d = np.abs(got.astype(np.float64) - want.astype(np.float64))
    w = np.abs(want.astype(np.float64))
    mx = float(w.max())
    tau = float(np.max((d - 1e-4 * w) / mx))
    return {"max_rel": float(d.max() / mx),
            "norm_rel": float(np.linalg.norm(d) / np.linalg.norm(want.astype(np.float64))),
            "tau": tau, "argmax_equal": None}


name = sys.argv[1] if len(sys.argv) > 1 else "yolov2-tiny"
images = int(sys.argv[2]) if len(sys.argv) > 2 else 16
net = build_net(name, images=images)
t0 = time.time()
ref = cprog.reference_forward(net, workers=os.cpu_count() or 1)["outputs"]
out = {"net": name, "images": images, "oracle_s": time.time() - t0}
for mode_name, mode in (("auto", K.GEMM_AUTO), ("simt", K.GEMM_SIMT)):
    ex = PatternExecutor(net, device=0, gemm_mode=mode)
    bits = "1" * len(net.ops)
    sched = ex.compile(bits)
    ex.run(sched)
    st = stats(ex.outputs(), ref)
    st["batch"] = sched.batch
    per = [stats(ex.outputs()[b], ref[b])["tau"] for b in range(images)]
    st["tau_per_image_max"] = max(per)
    out[mode_name] = st
print(json.dumps(out))
