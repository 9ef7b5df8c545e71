"""One traced (ACCT_TRACE=1) uncaptured run of the full all-offload schedule;
prints the per-action event timeline annotated with array names/bytes."""
import os
import sys
from pathlib import Path
os.environ["ACCT_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1811_03882_b200.executor import PatternExecutor  # noqa: E402
from paper_1811_03882_b200.nets import build_net  # noqa: E402

net = build_net("yolov2-tiny", images=16)
ex = PatternExecutor(net, device=0, graphs=False)
sched = ex.compile("1" * len(net.ops))
ex.run(sched)
for k in range(sched.n_actions):
    a = sched.actions[k]
    if a.kind in (4, 5):
        name = list(net.arrays)[a.a[0]]
        print(f"action {k}: {'H2D' if a.kind == 4 else 'D2H'} {name} {net.arrays[name].nbytes / 2**20:.1f} MB "
              f"imgs={a.i[1]} early={a.i[3]}", file=sys.stderr)
print("---- traced run", file=sys.stderr)
ex.run(sched)
