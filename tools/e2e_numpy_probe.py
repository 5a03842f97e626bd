"""Where the host time of a numpy-input fagp_posterior() call goes (C3): wall time of the call and
of the staging copies into pinned memory."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2403_12797_b200 as F  # noqa: E402
import paper_2403_12797_b200.engine as E  # noqa: E402
from paper_2403_12797_b200.datagen import generate, test_inputs, train_seed  # noqa: E402

p, M, N = 3, 10, 1_000_000
ds = generate(N, p, train_seed(p), 0.05)
Xs = test_inputs(N, p)
model = F.GpModel(F.ArdKernelParams.isotropic(p, 1.0, 1.0), 0.0025, n_eigen=M)
orig = E._parallel_copy
log = []


def timed(dst, src, *a, **k):
    t0 = time.perf_counter()
    orig(dst, src, *a, **k)
    log.append((dst.nbytes, time.perf_counter() - t0))


E._parallel_copy = timed


class T:
    X = ds.X
    y = ds.y


for _ in range(3):
    F.fagp_posterior(T, Xs, model, memory_cap=None)
torch.cuda.synchronize()
for _ in range(4):
    log.clear()
    t0 = time.perf_counter()
    r = F.fagp_posterior(T, Xs, model, memory_cap=None)
    torch.cuda.synchronize()
    w = time.perf_counter() - t0
    print(f"wall {1e3 * w:.3f} ms | copies " + " ".join(f"{b / 1e6:.0f}MB:{1e3 * t:.3f}ms" for b, t in log))
