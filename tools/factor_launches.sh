#!/bin/bash
# Per-kernel device time of the factor stage at a given config (ncu launch list of two factor calls,
# halved).  Usage (on the GPU box): bash tools/factor_launches.sh <p> <M> [N]
p=${1:-5}; M=${2:-6}; N=${3:-20000}
cat > /tmp/factor_once.py <<PY
import sys
sys.path.insert(0, "$PWD")
import numpy as np, torch
import paper_2403_12797_b200 as F
from paper_2403_12797_b200 import _device as dev
from paper_2403_12797_b200.posterior import gram_x_packed, factor_packed
rng = np.random.default_rng(0)
X = rng.uniform(-1, 1, ($N, $p)); y = np.cos(X).sum(1)
basis = F.Basis(F.ArdKernelParams.isotropic($p, 1.0, 1.0), $M)
packed = gram_x_packed(basis, dev.to_device(X), dev.to_device(y), 0.0)
torch.cuda.synchronize()
for _ in range(2):
    factor_packed(basis, packed, 0.0025, 0.0, $N)
    torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv python /tmp/factor_once.py 2>/dev/null | grep -v "^==" | python -c "
import csv, sys
from collections import defaultdict
rows = list(csv.reader(sys.stdin))
h = [r for r in rows if 'Kernel Name' in r][0]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
d = defaultdict(list)
for r in rows[rows.index(h) + 1:]:
    if len(r) > vi:
        d[r[ki][:80]].append(float(r[vi].replace(',', '')) / 1e3)
tot = 0.0
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f'{sum(v) / 2:9.1f} us/call  n={len(v) / 2:5.1f}  {k}')
    tot += sum(v) / 2
print(f'{tot:9.1f} us/call total (incl. the Gram once / 2)')
"
