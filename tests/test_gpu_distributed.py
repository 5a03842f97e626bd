"""Two ranks through the PRODUCT path.

Both processes run on cuda:0 (the GPU allocation is one device; NCCL needs distinct GPUs, so
the collective here is gloo on CUDA tensors -- the same torch.distributed calls the NCCL run
makes).  Each rank passes its own contiguous train / test shards; what moves between the ranks
is the product's real all-reduce payload, the packed modal [K | t] buffer (L^p + m doubles:
7,859 at p = 3, M = 10), and the gathered mean / var rows.  Checks:

  * fagp_posterior(group=) from host arrays (PosteriorEngine.run_host -> stage_reduce), from
    device tensors (PosteriorEngine.run), fit(group=) + predict, and
    fagp_posterior_sharded(gather=True): mean and var match the CPU oracle to 1e-9 (the parity
    bar) and the one-rank result to 1e-10 -- the cross-rank sum adds the Gram in another order,
    and this system (cond(A) ~ 1e8) turns that last-bit difference of G into ~1e-11 of the mean
    (measured on the B200: 1.2e-11; two blockings of the CPU oracle's Gram differ alike);
  * run-to-run bitwise at a fixed world size.
Reference: /root/reference/pkg/src/fagp/backend.py:109-130 (the row partition of the Gram).
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

P, M, N, NS = 3, 10, 60_001, 20_003
NOISE = 0.0025


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    rng = np.random.default_rng(2024)
    X = rng.uniform(-1, 1, (N, P))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    Xs = rng.uniform(-1, 1, (NS, P))
    return X, y, Xs


def _model():
    import paper_2403_12797_b200 as F

    return F.GpModel(F.ArdKernelParams.isotropic(P, 1.0, 1.0), NOISE, mean_const=0.1, n_eigen=M)


def _worker(rank, world, port, outdir):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    import paper_2403_12797_b200 as F
    from paper_2403_12797_b200 import _device as dev
    from paper_2403_12797_b200.distributed import fagp_posterior_sharded, shard_range

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = dist.group.WORLD
    X, y, Xs = _inputs()
    a, b = shard_range(N, rank, world)
    c, d = shard_range(NS, rank, world)

    class Host:
        pass

    Host.X, Host.y = X[a:b], y[a:b]

    class Dev:
        pass

    Dev.X, Dev.y = torch.from_numpy(X[a:b]).cuda(), torch.from_numpy(y[a:b]).cuda()
    model = _model()
    out = {}
    for rep in range(2):
        r = F.fagp_posterior(Host, Xs[c:d], model, memory_cap=None, group=g)
        out[f"host{rep}_mean"], out[f"host{rep}_var"] = r.mean.copy(), r.var.copy()
    r = F.fagp_posterior(Dev, torch.from_numpy(Xs[c:d]).cuda(), model, memory_cap=None, group=g,
                         return_device=True)
    out["dev_mean"], out["dev_var"] = dev.to_host(r.mean), dev.to_host(r.var)
    f = F.fit(Host, model, memory_cap=None, group=g)
    pr = F.predict(f, Xs[c:d])
    out["fit_mean"], out["fit_var"] = pr.mean, pr.var
    rs = fagp_posterior_sharded(X, y, Xs, model, group=g, gather=True, memory_cap=None)
    out["sharded_mean"], out["sharded_var"] = dev.to_host(rs.mean), dev.to_host(rs.var)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


RANK_TOL = 1e-10  # summation-order sensitivity of the posterior (see the docstring)


def _rel(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


def test_two_ranks_match_one_rank():
    import paper_2403_12797_b200 as F
    from paper_2403_12797_b200.distributed import shard_range

    import fagp_oracle as O

    X, y, Xs = _inputs()

    class Full:
        pass

    Full.X, Full.y = X, y
    ref = F.fagp_posterior(Full, Xs, _model(), memory_cap=None)
    orc = O.posterior(X, y, Xs, [1.0] * P, [1.0] * P, M, NOISE, 0.1)
    assert _rel(ref.mean, orc["mean"]) <= 1e-9 and _rel(ref.var, orc["var"]) <= 1e-9
    world = 2
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(_worker, args=(world, _free_port(), td), nprocs=world, join=True, start_method="spawn")
        outs = [dict(np.load(os.path.join(td, f"rank{r}.npz"))) for r in range(world)]
    for r, o in enumerate(outs):
        c, d = shard_range(NS, r, world)
        # bitwise run to run at a fixed world size
        assert np.array_equal(o["host0_mean"], o["host1_mean"]) and np.array_equal(o["host0_var"], o["host1_var"])
        for key in ("host0", "dev", "fit"):
            assert _rel(o[key + "_mean"], ref.mean[c:d]) <= RANK_TOL, (r, key, _rel(o[key + "_mean"], ref.mean[c:d]))
            assert _rel(o[key + "_var"], ref.var[c:d]) <= RANK_TOL, (r, key, _rel(o[key + "_var"], ref.var[c:d]))
            assert _rel(o[key + "_mean"], orc["mean"][c:d]) <= 1e-9 and _rel(o[key + "_var"], orc["var"][c:d]) <= 1e-9
        # the device-resident, host-pipelined and fit/predict routes reduce the same buffer
        assert np.array_equal(o["dev_mean"], o["host0_mean"]) and np.array_equal(o["fit_var"], o["host0_var"])
        # gathered: every rank holds the full vectors, in rank order
        assert o["sharded_mean"].shape == (NS,)
        assert _rel(o["sharded_mean"], ref.mean) <= RANK_TOL and _rel(o["sharded_var"], ref.var) <= RANK_TOL
    assert np.array_equal(outs[0]["sharded_mean"], outs[1]["sharded_mean"])
