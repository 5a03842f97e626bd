"""GPU timeline of the end-to-end fagp_posterior() call at C3 (CUDA events on the copy, compute
and output streams): when each upload chunk lands, each Gram chunk / the factorisation / each
predict chunk ends, and each result D2H completes, in ms from entry."""
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
if "--numpy" in sys.argv:  # the drop-in case: plain numpy inputs, staged by the engine
    Xp, yp, Xsp = ds.X, ds.y, Xs
else:
    Xp, yp, Xsp = (torch.from_numpy(a).pin_memory() for a in (ds.X, ds.y, Xs))
model = F.GpModel(F.ArdKernelParams.isotropic(p, 1.0, 1.0), 0.0025, n_eigen=M)


class T:
    X = Xp
    y = yp


for _ in range(3):
    F.fagp_posterior(T, Xsp, model, memory_cap=None)
torch.cuda.synchronize()
E._GPU_TRACE = []
walls = []
for _ in range(6):
    t0 = time.perf_counter()
    F.fagp_posterior(T, Xsp, model, memory_cap=None)
    walls.append(1e3 * (time.perf_counter() - t0))
E_tr = E._GPU_TRACE
E._GPU_TRACE = None
for w, tr in zip(walls, E_tr):
    print(f"wall {w:.3f} ms | " + " ".join(f"{n}={t:.3f}" for n, t in tr))
