"""Event-timed fagp_predict_x (the hot predict entry) at BASELINE configs: ms per launch and the
fraction of the measured FP64 DMMA peak on the modal flop count.   python tools/predict_time.py c3"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2403_12797_b200 as F  # noqa: E402
from paper_2403_12797_b200.posterior import factor_packed, gram_x_packed, predict_x_device  # noqa: E402

CFG = {"c2": (2, 10, 100_000), "c3": (3, 10, 1_000_000), "c4": (4, 8, 1_000_000), "c5": (5, 6, 2_000_000)}
PEAK = json.load(open(Path(__file__).resolve().parents[1] / "profiles" / "fp64_peak_r01.json"))["fp64_dmma_tflops"]
for name in sys.argv[1:] or ["c3"]:
    p, M, Ns = CFG[name]
    rng = np.random.default_rng(1)
    N = 20_000
    X = torch.from_numpy(rng.uniform(-1, 1, (N, p))).cuda()
    y = torch.from_numpy(np.cos(X.cpu().numpy()).sum(1)).cuda()
    Xs = torch.from_numpy(rng.uniform(-1, 1, (Ns, p))).cuda()
    basis = F.Basis(F.ArdKernelParams.isotropic(p, 1.0, 1.0), M)
    f, st, _ = factor_packed(basis, gram_x_packed(basis, X, y, 0.1), 0.0025, 0.1, N)
    for _ in range(2):
        predict_x_device(f, Xs)
    torch.cuda.synchronize()
    ts = []
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda") if os.environ.get("PT_FLUSH") else None
    for k in range(5):
        if flush is not None:  # PT_FLUSH=1: evict L2 (256 MiB write) between launches, as bench.py does
            flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        predict_x_device(f, Xs)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    mean_ms = sum(ts) / len(ts)
    L = 2 * M - 1
    fl = 2 * Ns * (L**p + M**p)
    print(f"{name}: predict_x {ms:.3f} ms  {fl / ms / 1e9:.2f} TF/s  frac {fl / ms / 1e9 / PEAK:.3f}  (mean {mean_ms:.3f} ms)", flush=True)
