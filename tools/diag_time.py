"""Time the two DMMA stages at C3 without result checks (for diagnostic library builds)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2403_12797_b200 as F
from paper_2403_12797_b200.engine import PosteriorEngine
from paper_2403_12797_b200.datagen import generate, test_inputs, train_seed
p, M, N = 3, 10, 1_000_000
ds = generate(N, p, train_seed(p), 0.05); Xs = test_inputs(N, p)
X, y, Xd = (torch.from_numpy(a).cuda() for a in (ds.X, ds.y, Xs))
eng = PosteriorEngine(F.ArdKernelParams.isotropic(p, 1.0, 1.0), M, N, N, 0.0025, 0.0, device=X.device)
eng.stage_tables(X, y, Xd)
for _ in range(2):
    eng.stage_gram(); eng.stage_factor(); eng.stage_predict()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
g = pr = 0.0
for _ in range(5):
    ev[0].record(); eng.stage_gram(); ev[1].record(); eng.stage_factor(); eng.stage_predict(); ev[2].record()
    torch.cuda.synchronize()
    g += ev[0].elapsed_time(ev[1]) / 5
    pr += 0
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(); eng.stage_predict(); t1.record(); torch.cuda.synchronize(); pr += t0.elapsed_time(t1) / 5
print(f"gram {g:.3f} ms  predict {pr:.3f} ms")
