"""Event-timed fagp_gram_x (the hot Gram entry) for BASELINE configs: ms per launch and the
fraction of the measured FP64 DMMA peak on the modal flop count.   python tools/gram_time.py c4 c5"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2403_12797_b200 as F  # noqa: E402
from paper_2403_12797_b200 import _device as dev  # noqa: E402
from paper_2403_12797_b200.posterior import gram_x_packed  # noqa: E402

CFG = {"c2": (2, 10, 100_000), "c3": (3, 10, 1_000_000), "c4": (4, 8, 4_000_000), "c5": (5, 6, 8_000_000)}
PEAK = json.load(open(Path(__file__).resolve().parents[1] / "profiles" / "fp64_peak_r01.json"))["fp64_dmma_tflops"]
for name in sys.argv[1:] or ["c4", "c5"]:
    p, M, N = CFG[name]
    rng = np.random.default_rng(1)
    X = torch.from_numpy(rng.uniform(-1, 1, (N, p))).cuda()
    y = torch.from_numpy(rng.standard_normal(N)).cuda()
    basis = F.Basis(F.ArdKernelParams.isotropic(p, 1.0, 1.0), M)
    for _ in range(2):
        gram_x_packed(basis, X, y, 0.1)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gram_x_packed(basis, X, y, 0.1)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    L = 2 * M - 1
    fl = 2 * N * (L**p + M**p)
    print(f"{name}: gram_x {ms:.3f} ms  {fl / ms / 1e9:.2f} TF/s  frac {fl / ms / 1e9 / PEAK:.3f}", flush=True)
