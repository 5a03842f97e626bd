"""Break down the end-to-end fagp_posterior() time at C3 (host tensors in, numpy out)."""
import time, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2403_12797_b200 as F
from paper_2403_12797_b200 import _device as dev
from paper_2403_12797_b200.engine import PosteriorEngine
from paper_2403_12797_b200.datagen import generate, test_inputs, train_seed
p, M, N = 3, 10, 1_000_000
ds = generate(N, p, train_seed(p), 0.05); Xs = test_inputs(N, p)
Xp, yp, Xsp = (torch.from_numpy(a).pin_memory() for a in (ds.X, ds.y, Xs))
kernel = F.ArdKernelParams.isotropic(p, 1.0, 1.0)
model = F.GpModel(kernel, 0.0025, n_eigen=M)
class T: X = Xp; y = yp
for _ in range(2): F.fagp_posterior(T, Xsp, model, memory_cap=None)
torch.cuda.synchronize()
def tick(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = tick(); X = dev.to_device(Xp); y = dev.to_device(yp); Xd = dev.to_device(Xsp)
    t1 = tick(); eng = PosteriorEngine(kernel, M, N, N, 0.0025, 0.0, device=X.device)
    t2 = tick(); mean, var = eng.run(X, y, Xd)
    t3 = tick(); eng.check(X, Xd, y)
    t4 = tick(); mh, vh = dev.to_host(mean), dev.to_host(var)
    t5 = tick(); r = F.fagp_posterior(T, Xsp, model, memory_cap=None)
    t6 = tick()
    print(f"h2d {1e3*(t1-t0):.2f} engine {1e3*(t2-t1):.2f} run {1e3*(t3-t2):.2f} check {1e3*(t4-t3):.2f} d2h {1e3*(t5-t4):.2f} | api total {1e3*(t6-t5):.2f} ms")

import cProfile, pstats, io
pr = cProfile.Profile()
torch.cuda.synchronize()
pr.enable()
r = F.fagp_posterior(T, Xsp, model, memory_cap=None)
torch.cuda.synchronize()
pr.disable()
sio = io.StringIO()
pstats.Stats(pr, stream=sio).sort_stats("cumulative").print_stats(30)
print(sio.getvalue())
