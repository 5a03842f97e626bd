"""TF/s of fagp_dgemm per large-tile configuration (FAGP_GEMM_BIG = 0, 2, 3; one process each) on the
factor's GEMM shapes.  Usage (GPU box): python tools/dgemm_cfg_probe.py"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SHAPES = [(4096, 4096, 4096, 0, 0), (4096, 4096, 4096, 1, 0), (4096, 4096, 4096, 0, 1), (7264, 7264, 512, 0, 1),
          (3888, 3888, 3888, 1, 0)]
CHILD = r'''
import sys, torch
sys.path.insert(0, "%s")
from paper_2403_12797_b200 import _lib
L = _lib.lib()
for M, N, K, ta, tb in %r:
    a = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda")
    b = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda")
    c = torch.empty((M, N), dtype=torch.float64, device="cuda")
    def run():
        _lib.check(L.fagp_dgemm(ta, tb, M, N, K, 1.0, _lib.ptr(a), a.shape[1], _lib.ptr(b), b.shape[1], 0.0,
                                _lib.ptr(c), N, _lib.stream_handle()), "dgemm")
    for _ in range(2): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"  {M}x{N}x{K} ta={ta} tb={tb}: {ms:8.3f} ms  {2.0 * M * N * K / ms / 1e9:6.2f} TF/s", flush=True)
''' % (ROOT, SHAPES)
for cfg in sys.argv[1:] or ["0", "2", "3"]:
    print(f"FAGP_GEMM_BIG={cfg}", flush=True)
    subprocess.run([sys.executable, "-c", CHILD], env={**os.environ, "FAGP_GEMM_BIG": cfg})
