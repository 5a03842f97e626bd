"""H2D copy-engine throughput for the C3 train upload patterns (pinned host -> device):
one contiguous copy, 8 contiguous chunks, and the Gram pipeline's per-CTA 2-D chunks
(fagp_gram_x_upload_chunk: 148 pieces of ~20 KB (X) and ~6.7 KB (y) per chunk)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2403_12797_b200 as F  # noqa: E402
from paper_2403_12797_b200 import _lib  # noqa: E402

N, p = 1_000_000, 3
Xh = torch.randn(N, p, dtype=torch.float64).pin_memory()
yh = torch.randn(N, dtype=torch.float64).pin_memory()
Xd = torch.empty(N, p, dtype=torch.float64, device="cuda")
yd = torch.empty(N, dtype=torch.float64, device="cuda")
basis = F.Basis(F.ArdKernelParams.isotropic(p, 1.0, 1.0), 10)
L = _lib.lib()
nch = int(L.fagp_gram_x_chunks(N, basis.ref))
s = torch.cuda.Stream()
mb = (N * p + N) * 8 / 1e6


def timeit(fn, reps=10):
    ts = []
    for _ in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            fn()
            e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    return ts[len(ts) // 2]


def contiguous():
    Xd.copy_(Xh, non_blocking=True)
    yd.copy_(yh, non_blocking=True)


def chunks8():
    step = N // 8
    for k in range(8):
        a, b = k * step, (k + 1) * step
        Xd[a:b].copy_(Xh[a:b], non_blocking=True)
        yd[a:b].copy_(yh[a:b], non_blocking=True)


def pipeline2d():
    for k in range(nch):
        _lib.check(L.fagp_gram_x_upload_chunk(_lib.ptr(Xh), _lib.ptr(yh), N, basis.ref, k, _lib.ptr(Xd), _lib.ptr(yd),
                                              _lib.stream_handle(s)), "upload")


for name, fn in (("contiguous", contiguous), ("8 contiguous chunks", chunks8), (f"{nch} 2-D chunks (pipeline)", pipeline2d)):
    ms = timeit(fn)
    print(f"{name:28s} {ms:7.3f} ms  {mb / ms:6.1f} GB/s")
