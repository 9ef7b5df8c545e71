"""End-to-end and per-array relative error of the all-offload pattern vs the
C oracle, for each gemm mode (how FP32 summation-order and 3xTF32
accumulation errors compound through a deep net)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import cprog  # noqa: E402
from paper_1811_03882_b200 import kernels as K  # noqa: E402
from paper_1811_03882_b200.executor import PatternExecutor  # noqa: E402
from paper_1811_03882_b200.nets import build_net  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "yolov2-608"
net = build_net(name, images=int(sys.argv[2]) if len(sys.argv) > 2 else 1)
ref = cprog.reference_forward(net)
for mode_name, mode in (("simt", K.GEMM_SIMT), ("auto", K.GEMM_AUTO)):
    ex = PatternExecutor(net, device=0, gemm_mode=mode)
    ex.run("1" * len(net.ops))
    out = ex.outputs()
    rel = float(np.abs(out - ref["outputs"]).max() / np.abs(ref["outputs"]).max())
    worst = []
    for a in net.arrays.values():
        if a.role in ("activation", "output") and a.dtype == "float":
            g, w = ex.host_array(a.name), ref["state"][a.name]
            worst.append((float(np.abs(g - w).max() / max(np.abs(w).max(), 1e-30)), a.name))
    worst.sort(reverse=True)
    print(f"{name} {mode_name}: output max-rel {rel:.2e}; worst arrays "
          + ", ".join(f"{n} {e:.1e}" for e, n in worst[:5]))
