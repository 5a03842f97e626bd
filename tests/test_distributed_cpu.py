"""CPU, world_size 2 over gloo: the sharding algebra and the collective plumbing of the
multi-GPU path (distributed.py).  Per-rank partial Grams come from the oracle here (the
CUDA kernels need a GPU); on the GPU the same host code drives fagp_gram."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2403_12797_b200.distributed import all_gather_rows, all_reduce_sum, shard_range


def test_shard_ranges_cover_rows():
    for n in (0, 1, 7, 1000, 10**6 + 3):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _packed(G, t):
    m = G.shape[0]
    ext = np.zeros((m + 1, m + 1))
    ext[:m, :m] = G
    ext[:m, m] = t
    return ext[np.triu_indices(m + 1)]


def _worker(rank, world, port, out):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import fagp_oracle as O
    from paper_2403_12797_b200.datagen import generate

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    ds = generate(3001, 2, seed=200000)
    a, b = shard_range(ds.N, rank, world)
    G, t = O.gram(ds.X[a:b], ds.y[a:b], 0.0, [1.0, 1.0], [1.0, 1.0], 6)
    packed = torch.from_numpy(_packed(G, t))
    all_reduce_sum(packed)
    mine = torch.arange(a, b, dtype=torch.float64)
    gathered = all_gather_rows(mine)
    if rank == 0:
        Gf, tf = O.gram(ds.X, ds.y, 0.0, [1.0, 1.0], [1.0, 1.0], 6)
        full = _packed(Gf, tf)
        out.put((float(np.max(np.abs(packed.numpy() - full)) / np.max(np.abs(full))),
                 bool(np.array_equal(gathered.numpy(), np.arange(ds.N, dtype=float)))))
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def test_allreduce_of_row_shards_equals_full_gram():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, gathered_ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-14
    assert gathered_ok
