"""Small invocations of the spin-synchronised and shared-memory-heavy kernels, for
compute-sanitizer (memcheck / racecheck / synccheck):

  cholinv_persistent_kernel   cooperative launch, software grid barrier with split arrive/wait,
                              tagged breakdown flag (SPD and indefinite inputs)
  fused_gram_split_kernel     the pipelined launch polling ready words set by copy-engine DMA,
                              and the plain launch
  fused_predict_split_kernel  p = 3 split predict
  (+ the rest of a small p = 3, M = 10 posterior: expand3, pair_system, ctc3, ...)
  tiled_gram_kernel / tiled_predict_kernel   output-tiled p = 4 (M = 8) and p = 5 (M = 6) paths,
                              whose m = 4096 / 7776 factors run potrf_big (persistent diagonal
                              blocks + triangular-clipped DGEMM panels), trtri and lauum
  graph                       the p = 3 step captured as a CUDA graph and replayed
  host_staging                numpy inputs through fagp_host_copy (non-temporal stores, worker pool)

Usage (on the GPU box):
  compute-sanitizer --tool memcheck  --error-exitcode 9 python tools/sanitize_cases.py [case ...]
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2403_12797_b200 as F  # noqa: E402
from paper_2403_12797_b200 import _device as dev  # noqa: E402
from paper_2403_12797_b200 import _lib  # noqa: E402


def cholinv():
    from paper_2403_12797_b200.linalg import spd_inverse

    rng = np.random.default_rng(3)
    for m in (70, 200):
        B = rng.standard_normal((m, m))
        A = B @ B.T + m * np.eye(m)
        inv, info = spd_inverse(A)
        assert info == 0 and np.abs(dev.to_host(inv) - np.linalg.inv(A)).max() < 1e-10
        U = np.eye(m) + np.tril(rng.standard_normal((m, m)), -1) / np.sqrt(m)
        for where in (5, 40, m - 1):
            d = np.ones(m)
            d[where] = -1.0
            _, info = spd_inverse((U * d) @ U.T)
            assert info == where + 1, (m, where, info)


def gram_pipelined():
    from paper_2403_12797_b200.posterior import gram_x_packed

    N = 9000
    rng = np.random.default_rng(1)
    X = rng.uniform(-1, 1, (N, 3))
    y = np.cos(X).sum(1)
    basis = F.Basis(F.ArdKernelParams.isotropic(3, 1.0, 1.0), 10)
    ref = dev.to_host(gram_x_packed(basis, dev.to_device(X), dev.to_device(y), 0.2))
    L = _lib.lib()
    nch = int(L.fagp_gram_x_chunks(N, basis.ref))
    Xh, yh = torch.from_numpy(X).pin_memory(), torch.from_numpy(y).pin_memory()
    Xd, yd = dev.empty((N, 3)), dev.empty((N,))
    ready = dev.zeros((nch,), dtype="int32")
    flags = dev.zeros((1,), dtype="int32")
    wsz = int(L.fagp_gram_x_workspace_size(N, basis.ref))
    ws = dev.empty((max(1, -(-wsz // 8)),))
    out = dev.empty((int(L.fagp_gram_len(basis.ref)),))
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    _lib.check(L.fagp_gram_x_pipelined(_lib.ptr(Xd), N, basis.ref, _lib.ptr(yd), 0.2, _lib.ptr(ready), _lib.ptr(out),
                                       _lib.ptr(ws), wsz, _lib.ptr(flags), _lib.stream_handle()), "pipelined")
    for k in reversed(range(nch)):
        _lib.check(L.fagp_gram_x_upload_chunk(_lib.ptr(Xh), _lib.ptr(yh), N, basis.ref, k, _lib.ptr(Xd), _lib.ptr(yd),
                                              _lib.stream_handle(side)), "upload")
        _lib.check(L.fagp_gram_x_signal(_lib.ptr(ready), k, _lib.stream_handle(side)), "signal")
    torch.cuda.synchronize()
    assert int(dev.to_host(flags)[0]) == 0 and np.array_equal(dev.to_host(out), ref)


def posterior():
    rng = np.random.default_rng(2)
    X = rng.uniform(-1, 1, (6000, 3))
    y = np.cos(X).sum(1)
    Xs = rng.uniform(-1, 1, (3000, 3))

    class DS:
        pass

    DS.X, DS.y = X, y
    model = F.GpModel(F.ArdKernelParams.isotropic(3, 1.0, 1.0), 0.0025, n_eigen=10)
    r = F.fagp_posterior(DS, Xs, model, memory_cap=None)
    assert np.all(np.isfinite(r.mean)) and np.all(r.var >= 0)


def _model(p, M):
    return F.GpModel(F.ArdKernelParams.isotropic(p, 1.0, 1.0), 0.0025, n_eigen=M)


def tiled():
    rng = np.random.default_rng(4)
    for p, M, N, Ns in ((4, 8, 3000, 700), (5, 6, 1500, 300)):
        X = rng.uniform(-1, 1, (N, p))
        y = np.cos(X).sum(1)
        Xs = rng.uniform(-1, 1, (Ns, p))
        r = F.fagp_posterior(F.Dataset(X, y, 0.0, 0, ((-1.0, 1.0),) * p), Xs, _model(p, M), memory_cap=None)
        assert np.all(np.isfinite(r.mean)) and np.all(r.var >= -1e-9), (p, M)


def graph():
    from paper_2403_12797_b200.engine import PosteriorEngine

    rng = np.random.default_rng(5)
    N, Ns = 5000, 2000
    X = dev.to_device(rng.uniform(-1, 1, (N, 3)))
    y = dev.to_device(np.cos(dev.to_host(X)).sum(1))
    Xs = dev.to_device(rng.uniform(-1, 1, (Ns, 3)))
    eng = PosteriorEngine(F.ArdKernelParams.isotropic(3, 1.0, 1.0), 10, N, Ns, 0.0025)
    if eng.capture(X, y, Xs) is not None:
        for _ in range(2):
            mean, var = eng.replay()
        torch.cuda.synchronize()
        assert not eng.factor_needs_retry()
        assert np.all(np.isfinite(dev.to_host(mean))) and np.all(dev.to_host(var) >= -1e-9)


def host_staging():
    from paper_2403_12797_b200 import engine

    rng = np.random.default_rng(6)
    src = rng.standard_normal(1 << 20)
    dst = torch.empty(src.shape[0], dtype=torch.float64).pin_memory()
    engine._parallel_copy(dst.numpy(), src)
    assert np.array_equal(dst.numpy(), src)


CASES = {"cholinv": cholinv, "gram_pipelined": gram_pipelined, "posterior": posterior, "tiled": tiled,
         "graph": graph, "host_staging": host_staging}

if __name__ == "__main__":
    torch.cuda.set_device(0)
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        torch.cuda.synchronize()
        print(f"{name}: ok", flush=True)
