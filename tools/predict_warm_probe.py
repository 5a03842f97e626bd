"""Is the predict kernel's in-step time a warm-up effect?  Times fagp_predict_x in the bench's
context after (i) an L2-flush fill, (ii) a fill then a ~1 ms single-thread spin, (iii) the full
step's factor, then (iv) a second predict right behind the in-step one.
    FAGP_PREDICT_GROUPS=1|2 python tools/predict_warm_probe.py"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2403_12797_b200.engine import PosteriorEngine  # noqa: E402
from paper_2403_12797_b200.kernels import ArdKernelParams  # noqa: E402

p, M, N, Ns = bench.CONFIGS["c3"]
Xh, yh, Xsh = bench.make_inputs("c3", 0, 1)
X, y, Xs = (torch.from_numpy(a).cuda() for a in (Xh, yh, Xsh))
eng = PosteriorEngine(ArdKernelParams.isotropic(p, 1.0, 1.0), M, N, Ns, bench.NOISE_VAR, 0.0, device=X.device)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=X.device)
for _ in range(3):
    eng.run(X, y, Xs)
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {k: [] for k in ("fill", "fill+spin", "step", "step 2nd", "gram+spin")}
for k in range(10):
    for case in ("fill", "fill+spin", "step", "gram+spin"):
        flush.fill_(float(k))
        if case == "fill+spin":
            torch.cuda._sleep(2_000_000)
        if case in ("step", "gram+spin"):
            eng.stage_gram(X, y)
            eng.stage_reduce()
            if case == "step":
                eng.stage_factor_async()
            else:
                torch.cuda._sleep(700_000)
        a, b, c = E(), E(), E()
        a.record()
        eng.stage_predict(Xs)
        b.record()
        if case == "step":
            eng.stage_predict(Xs)
        c.record()
        torch.cuda.synchronize()
        res[case].append(a.elapsed_time(b))
        if case == "step":
            res["step 2nd"].append(b.elapsed_time(c))
for kk, v in res.items():
    print(f"{kk:10s} min {min(v):.3f} mean {statistics.mean(v):.3f}")
