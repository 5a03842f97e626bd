"""Break down the end-to-end fagp_posterior() time at C3 (pinned host tensors in, numpy out)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2403_12797_b200 as F  # noqa: E402
from paper_2403_12797_b200.datagen import generate, test_inputs, train_seed  # noqa: E402

p, M, N = 3, 10, 1_000_000
ds = generate(N, p, train_seed(p), 0.05)
Xs = test_inputs(N, p)
Xp, yp, Xsp = (torch.from_numpy(a).pin_memory() for a in (ds.X, ds.y, Xs))
kernel = F.ArdKernelParams.isotropic(p, 1.0, 1.0)
model = F.GpModel(kernel, 0.0025, n_eigen=M)


class T:
    X = Xp
    y = yp


for _ in range(3):
    F.fagp_posterior(T, Xsp, model, memory_cap=None)
torch.cuda.synchronize()
import gc  # noqa: E402

import paper_2403_12797_b200.engine as E  # noqa: E402

E._TRACE = []
gc.callbacks.append(lambda phase, info: print(f"  [gc {phase} gen{info['generation']}]", time.perf_counter()))
for label in ("gc on", "gc off"):
    if label == "gc off":
        gc.disable()
    ts = []
    for rep in range(12):
        t0 = time.perf_counter()
        r = F.fagp_posterior(T, Xsp, model, memory_cap=None)
        t1 = time.perf_counter()
        ts.append(1e3 * (t1 - t0))
        print(f"  call {rep}: {1e3 * (t1 - t0):.2f} ms, phases", " ".join(f"{x:.2f}" for x in E._TRACE[-1]), t0)
    print(label, "api ms:", " ".join(f"{t:.2f}" for t in ts))
gc.enable()
E._TRACE = []
for rep in range(12):
    r = F.fagp_posterior(T, Xsp, model, memory_cap=None)
print("phases (upload+gram issue, factor(sync), out alloc, predict issue, d2h sync) ms:")
for t in E._TRACE:
    print("  " + " ".join(f"{x:.2f}" for x in t))
E._TRACE = None

import cProfile  # noqa: E402
import io  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
torch.cuda.synchronize()
pr.enable()
r = F.fagp_posterior(T, Xsp, model, memory_cap=None)
torch.cuda.synchronize()
pr.disable()
sio = io.StringIO()
pstats.Stats(pr, stream=sio).sort_stats("tottime").print_stats(25)
print(sio.getvalue())
