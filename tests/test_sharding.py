"""Multi-rank host logic of the batch sharder on CPU (gloo, world_size 2):
the slices cover the batch exactly once, shards keyed on the global index
reproduce the single-process result bit for bit after a gather, and the
whole-job time is the MAX over ranks."""

import os
import socket

import numpy as np
import pytest

from paper_1301_0763_b200.sharding import shard_bounds


def test_shard_bounds_cover_once():
    for total in (0, 1, 7, 64, 1 << 18):
        for ws in (1, 2, 3, 4, 8):
            seen = []
            for r in range(ws):
                b0, b1 = shard_bounds(total, ws, r)
                assert 0 <= b0 <= b1 <= total
                seen.extend(range(b0, b1))
            assert seen == list(range(total))
            sizes = [shard_bounds(total, ws, r)[1] - shard_bounds(total, ws, r)[0] for r in range(ws)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, total, N, q):
    import torch
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle
    from paper_1301_0763_b200 import sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    b0, b1 = sharding.shard_bounds(total, ws, rank)
    # rows keyed on the global index (stand-in for the device generator)
    rows = np.stack([np.random.default_rng(1000 + g).standard_normal(2 * N).view(np.complex128) for g in range(b0, b1)])
    local = torch.from_numpy(oracle.cdft_rows(rows))  # the transform itself is checked elsewhere
    full = sharding.gather_rows(local, total)
    t = sharding.max_over_ranks(0.5 + rank)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, full.numpy(), t))


def test_two_rank_gloo_shard_gather_and_max():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port, total, N = _free_port(), 13, 64
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, N, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import oracle
    rows = np.stack([np.random.default_rng(1000 + g).standard_normal(2 * N).view(np.complex128) for g in range(total)])
    want = oracle.cdft_rows(rows)
    for rank, full, t in res:
        assert full.tobytes() == want.tobytes()
        assert t == 1.5
