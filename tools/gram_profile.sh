#!/bin/bash
# Diagnostics: build a library variant with per-warp clock64 phase counters in the fused Gram
# kernel (-DFAGP_GRAM_PROFILE) and print the split of warp time (k-loop / production / flush /
# barrier) over one C3 Gram launch.  Usage (on the GPU box): bash tools/gram_profile.sh
set -e
mkdir -p /tmp/gprof
cd paper_2403_12797_b200
for f in basis gram factor predict literal modal chol fused exact gram_tiled predict_tiled host; do
  extra=""; [ $f = fused ] && extra="-DFAGP_GRAM_PROFILE"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC $extra -I ../include -c csrc/$f.cu -o /tmp/gprof/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/gprof/libfagp_prof.so /tmp/gprof/*.o -lcudart
cd ..
FAGP_LIB_PATH=/tmp/gprof/libfagp_prof.so python - <<'PY'
import ctypes, torch, numpy as np
import paper_2403_12797_b200 as F
from paper_2403_12797_b200 import _lib
from paper_2403_12797_b200.posterior import gram_x_packed
from paper_2403_12797_b200.datagen import generate, train_seed
ds = generate(1_000_000, 3, train_seed(3), 0.05)
X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
basis = F.Basis(F.ArdKernelParams.isotropic(3, 1.0, 1.0), 10)
L = _lib.lib()
out = (ctypes.c_longlong * 4)()
rc0 = L.fagp_debug_gram_profile(out); base = list(out)
gram_x_packed(basis, X, y, 0.0); torch.cuda.synchronize()
rc1 = L.fagp_debug_gram_profile(out)
print("gram counters rc", rc0, rc1, list(out), base)
v = [a - b for a, b in zip(out, base)]
tot = max(1, sum(v))
print("gram warp-cycles share: kloop %.3f produce %.3f flush %.3f barrier %.3f  (total %.3g per warp)" % tuple([x / tot for x in v] + [tot / (148 * 16)]))
from paper_2403_12797_b200.posterior import factor_packed, predict_x_device
from paper_2403_12797_b200.datagen import test_inputs
packed = gram_x_packed(basis, X, y, 0.0)
f, st, _ = factor_packed(basis, packed, 0.0025, 0.0, 1_000_000)
Xs = torch.from_numpy(test_inputs(1_000_000, 3)).cuda()
L.fagp_debug_pred_profile(out); base = list(out)
predict_x_device(f, Xs); torch.cuda.synchronize()
L.fagp_debug_pred_profile(out)
print("predict counters", list(out), base)
v = [a - b for a, b in zip(out, base)]
tot = max(1, sum(v))
print("predict warp-cycles share: produce %.3f contract %.3f epilogue+final %.3f barrier %.3f  (total %.3g per warp)" % tuple([x / tot for x in v] + [tot / (148 * 16)]))
PY
