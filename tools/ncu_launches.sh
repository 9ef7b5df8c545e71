#!/bin/bash
# per-launch GPU time of the kernels matching $1 in one profile_pattern run:
#   tools/ncu_launches.sh REGEX NET [extra profile_pattern args]
re=$1; net=$2; shift 2
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$re" --csv \
    python tools/profile_pattern.py --net "$net" --images 16 --resident --runs 1 "$@" 2>/dev/null |
  python -c '
import csv, sys
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10 and r[0].isdigit()]
for r in rows:
    name = r[4].split("(")[0].replace("void ", "").replace("acct::", "").replace("<unnamed>::", "")
    print(f"{r[0]:>4} {name[:60]:60s} grid {r[7]:>14} {r[-1]:>10} {r[-2]}")
'
