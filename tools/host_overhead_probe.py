"""cProfile of the host side of fagp_posterior() at a latency config (C2 by default): where the
Python time of a call goes when the GPU work is small."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2403_12797_b200 as F  # noqa: E402
from paper_2403_12797_b200.datagen import generate, test_inputs, train_seed  # noqa: E402

cfg = {"c1": (1, 10, 1000), "c2": (2, 10, 100_000)}[sys.argv[1] if len(sys.argv) > 1 else "c2"]
p, M, N = cfg
ds = generate(N, p, train_seed(p), 0.05)
Xs = test_inputs(N, p)
Xp, yp, Xsp = (torch.from_numpy(a).pin_memory() for a in (ds.X, ds.y, Xs))
model = F.GpModel(F.ArdKernelParams.isotropic(p, 1.0, 1.0), 0.0025, n_eigen=M)


class T:
    X = Xp
    y = yp


for _ in range(5):
    F.fagp_posterior(T, Xsp, model, memory_cap=None)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    F.fagp_posterior(T, Xsp, model, memory_cap=None)
torch.cuda.synchronize()
print(f"mean wall {1e3 * (time.perf_counter() - t0) / 50:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    F.fagp_posterior(T, Xsp, model, memory_cap=None)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
