"""profiles/rNN_ncu_full.txt from one `ncu --set full` capture of a resident
16-image step (tools/profile_pattern.py --runs 2, second run's launches):
per labelled launch, the key metrics in the `shape = ...` / `key = value`
format bench.py's ncu_traffic() reads.

    python tools/ncu_full_report.py REPORT.ncu-rep HEADER 'i:label:shape' ...

i = index of the launch in the report (its order in the step).
"""
import csv
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_full_summary import WANT  # noqa: E402


def main():
    rep, header, specs = sys.argv[1], sys.argv[2], sys.argv[3:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    print(f"# {header}")
    for spec in specs:
        i, label, shape = spec.split(":", 2)
        d = dict(zip(hdr, rows[2 + int(i)]))
        u = dict(zip(hdr, units))
        print(f"\n# ---- {label}")
        print(f"shape = {shape}")
        for k in WANT:
            if k in d:
                print(f"{k} = {d[k]} {u.get(k, '')}".rstrip())


if __name__ == "__main__":
    main()
