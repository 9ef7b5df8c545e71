"""Wall time of the full (transfer-inclusive) all-offload schedule under
variants: CUDA graph or not, transfer reordering/early copyouts or not."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1811_03882_b200.executor import PatternExecutor  # noqa: E402
from paper_1811_03882_b200.nets import build_net  # noqa: E402

net = build_net(sys.argv[1] if len(sys.argv) > 1 else "yolov2-tiny", images=16)
bits = "1" * len(net.ops)
for graphs in (True, False):
    for overlap in (True, False):
        ex = PatternExecutor(net, device=0, graphs=graphs)
        if not overlap:
            ex._overlap_transfers = lambda acts, single_pass: acts
        sched = ex.compile(bits)
        for _ in range(3):
            ex.run(sched)
        ts = []
        for _ in range(8):
            torch.cuda.synchronize()
            ts.append(ex.run(sched).seconds)
        ts.sort()
        print(f"graphs={graphs} overlap={overlap}: median {ts[4] * 1e3:.2f} ms  min {ts[0] * 1e3:.2f} ms")
        del ex
        torch.cuda.empty_cache()
