#!/bin/bash
# Per-kernel device time of one C3 bench step (ncu, no cache flush between kernels, clocks not locked).
# Usage: bash tools/launch_list.sh [extra bench args]
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | grep -v "^==" | python -c "
import csv, sys
from collections import defaultdict
rows = list(csv.reader(sys.stdin))
h = [r for r in rows if 'Kernel Name' in r][0]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
d = defaultdict(list)
for r in rows[rows.index(h) + 1:]:
    if len(r) > vi:
        d[r[ki][:70]].append(float(r[vi].replace(',', '')) / 1e3)
tot = 0.0
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f'{sum(v) / 2:9.1f} us/step  n={len(v) / 2:4.1f}  {k}')
    tot += sum(v) / 2
print(f'{tot:9.1f} us/step total')
"
