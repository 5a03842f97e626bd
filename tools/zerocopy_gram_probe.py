"""fagp_gram_x reading X / y from device memory vs straight from pinned (mapped) host memory
(zero-copy loads over PCIe), C3 shape; also the H2D-then-Gram sequence for reference."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2403_12797_b200 as F  # noqa: E402
from paper_2403_12797_b200 import _device as dev  # noqa: E402
from paper_2403_12797_b200 import _lib  # noqa: E402

N, p = 1_000_000, 3
rng = np.random.default_rng(1)
Xh = torch.from_numpy(rng.uniform(-1, 1, (N, p))).pin_memory()
yh = torch.from_numpy(np.cos(Xh.numpy()).sum(1)).pin_memory()
Xd, yd = Xh.cuda(), yh.cuda()
basis = F.Basis(F.ArdKernelParams.isotropic(p, 1.0, 1.0), 10)
L = _lib.lib()
print("mapped:", L.fagp_host_mapped(Xh.data_ptr(), Xh.numel() * 8), L.fagp_host_mapped(yh.data_ptr(), yh.numel() * 8))
packed = dev.empty((int(L.fagp_gram_len(basis.ref)),))
wsz = int(L.fagp_gram_x_workspace_size(N, basis.ref))
ws = dev.empty((max(1, -(-wsz // 8)),))


def gram(X, y):
    _lib.check(L.fagp_gram_x(_lib.ptr(X), N, basis.ref, _lib.ptr(y), 0.0, _lib.ptr(packed), _lib.ptr(ws), wsz, None,
                             _lib.stream_handle()), "gram_x")


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


ref = None
gram(Xd, yd)
torch.cuda.synchronize()
ref = dev.to_host(packed).copy()
print(f"device inputs      {timed(lambda: gram(Xd, yd)):.3f} ms")
print(f"zero-copy inputs   {timed(lambda: gram(Xh, yh)):.3f} ms")
zc = dev.to_host(packed).copy()
print("bitwise equal:", np.array_equal(ref, zc))


def h2d_then_gram():
    Xd.copy_(Xh, non_blocking=True)
    yd.copy_(yh, non_blocking=True)
    gram(Xd, yd)


print(f"H2D then Gram      {timed(h2d_then_gram):.3f} ms")
