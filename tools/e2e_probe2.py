"""e2e step time of the benchmarked 16-image yolov2-tiny schedule (median of
10 runs after 3 warm-ups) -- compare library settings (ACCT_PDL=0/1)."""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1811_03882_b200.executor import PatternExecutor  # noqa: E402
from paper_1811_03882_b200.nets import build_net  # noqa: E402

net = build_net("yolov2-tiny", images=16)
ex = PatternExecutor(net, device=0)
s = ex.compile("1" * len(net.ops))
for _ in range(3):
    ex.run(s)
t = [ex.run(s).seconds for _ in range(10)]
print(f"e2e median {statistics.median(t) * 1e3:.3f} ms, min {min(t) * 1e3:.3f} ms")
