"""Time fagp_potrf (persistent vs blocked) and the factor stage pieces at m = 1000."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2403_12797_b200 import _lib, _device as dev
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
rng = np.random.default_rng(0)
B = rng.standard_normal((m, m)); A = B @ B.T + m * np.eye(m)
Ad = dev.to_device(A)
L = _lib.lib()
wsz = int(L.fagp_potrf_workspace_size(m)); ws = dev.empty((wsz // 8 + 1,)); info = dev.zeros((1,), dtype="int32")
W = torch.empty_like(Ad)
s = _lib.stream_handle()
for impl in ("persistent", "blocked", "persistent"):
    if impl == "blocked": os.environ["FAGP_POTRF"] = "blocked"
    else: os.environ.pop("FAGP_POTRF", None)
    ts = []
    for rep in range(20):
        W.copy_(Ad)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.fagp_potrf(_lib.ptr(W), m, _lib.ptr(info), _lib.ptr(ws), wsz, s), "potrf")
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    Lh = dev.to_host(W)
    err = np.abs(Lh - np.linalg.cholesky(A)).max() / np.abs(Lh).max()
    print(f"{impl:10s} m={m} median {1e3*np.median(ts):.1f} us  min {1e3*min(ts):.1f} us  err {err:.1e}")
