"""Host<->device transfer rates for every array of a net: pitched 2-D copy (as
the executor issues them) vs a dense 1-D copy of the same bytes."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1811_03882_b200 import kernels as K  # noqa: E402
from paper_1811_03882_b200.executor import PatternExecutor  # noqa: E402
from paper_1811_03882_b200.nets import build_net  # noqa: E402

net = build_net(sys.argv[1] if len(sys.argv) > 1 else "yolov2-tiny", images=2)
ex = PatternExecutor(net, device=0)
s = ex.stream
tot2d = tot1d = 0.0
totb = 0
for name, spec in net.arrays.items():
    slot = ex.slots[ex.slot_of[name]]
    rows, cols, ld = slot.rows, slot.cols, slot.ld_dev
    row_b = cols * 4
    scratch = torch.empty(rows * cols, dtype=torch.float32, device="cuda")
    res = {}
    for kind in ("2d", "1d"):
        for direction in (1, 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(3):
                if kind == "2d":
                    if direction == 1:
                        K.call("acct_memcpy2d", slot.dev, ld * 4, slot.host, row_b, row_b, rows, 1, s.cuda_stream)
                    else:
                        K.call("acct_memcpy2d", slot.host, row_b, slot.dev, ld * 4, row_b, rows, 2, s.cuda_stream)
                else:
                    if direction == 1:
                        K.call("acct_memcpy2d", scratch.data_ptr(), row_b * rows, slot.host, row_b * rows, row_b * rows, 1, 1, s.cuda_stream)
                    else:
                        K.call("acct_memcpy2d", slot.host, row_b * rows, scratch.data_ptr(), row_b * rows, row_b * rows, 1, 2, s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            res[(kind, direction)] = e0.elapsed_time(e1) / 3
    b = rows * row_b
    totb += b
    tot2d += res[("2d", 1)] + res[("2d", 2)]
    tot1d += res[("1d", 1)] + res[("1d", 2)]
    if b > 1e5:
        print(f"{name:8s} {rows:5d}x{cols:6d} {b/1e6:7.2f}MB  2d H2D {b/res[('2d',1)]/1e6:6.1f} GB/s D2H {b/res[('2d',2)]/1e6:6.1f} GB/s"
              f" | 1d H2D {b/res[('1d',1)]/1e6:6.1f} D2H {b/res[('1d',2)]/1e6:6.1f}")
print(f"all arrays {totb/1e6:.1f} MB: 2d round trip {tot2d:.2f} ms, 1d round trip {tot1d:.2f} ms")
