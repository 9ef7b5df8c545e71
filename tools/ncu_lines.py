"""Per-CUDA-source-line instruction counts and warp-stall samples from an
`ncu --set full --import-source on` report:

    ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = cur = None
inst, samp, txt = collections.Counter(), collections.Counter(), {}
stalls = collections.defaultdict(collections.Counter)
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-" or not r[0]:
        continue
    key = (cur, int(r[0]))
    inst[key] += float(r[hdr.index("Instructions Executed")] or 0)
    samp[key] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    txt[key] = r[1].strip()[:100]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stalls[key][h[6:]] += float(r[i] or 0)
            except ValueError:
                pass
ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
print(f"total warp instructions {ti:.0f}, stall samples {ts:.0f}")
print("--- by stall samples")
for k, v in sorted(samp.items(), key=lambda kv: -kv[1])[:top]:
    st = ", ".join(f"{n} {c / v * 100:.0f}%" for n, c in stalls[k].most_common(3) if c) if v else ""
    print(f"{v / ts * 100:5.1f}% samp {inst[k] / ti * 100:5.1f}% inst  {k[0]}:{k[1]}  {txt[k]}  [{st}]")
