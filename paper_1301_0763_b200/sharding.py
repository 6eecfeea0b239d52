"""Batch sharding across the GPUs of one box.

Every transform is independent (improved.py:139-150 works column by column),
so the batch is split into contiguous slices, one per rank, with NO collective
on the data path.  Ranks only meet at a barrier before/after the timed region
and in one MAX all-reduce of their elapsed times (the whole-job time).  Each
rank's inputs are keyed on the GLOBAL transform index (qft_fill_normal's
counter-based generator), so a shard is bit-identical to the same rows of a
1-GPU run.
"""

import os


def shard_bounds(total, world_size, rank):
    """[b0, b1) of rank's contiguous slice; sizes differ by at most one."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad world_size/rank")
    base, extra = divmod(total, world_size)
    b0 = rank * base + min(rank, extra)
    return b0, b0 + base + (1 if rank < extra else 0)


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value, device=None):
    """Whole-job time: MAX of a per-rank float over the default process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def transform_shard(x_local, table=None, counter=None):
    """The rank-local work: one batched transform of this rank's rows (CUDA
    tensor (rows, N)); no communication."""
    from . import improved
    return improved.cdft_rows(x_local, table=table, counter=counter)


def gather_rows(local, total, device=None):
    """Verification helper (not on the hot path): all-gather every rank's rows
    into the full (total, N) result on every rank."""
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size()
    sizes = [b1 - b0 for b0, b1 in (shard_bounds(total, ws, r) for r in range(ws))]
    n, mx = local.shape[1], max(sizes)
    pad = torch.zeros((mx, n), dtype=local.dtype, device=local.device)  # all_gather needs equal shapes
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(ws)]
    if local.dtype.is_complex:
        dist.all_gather([torch.view_as_real(b) for b in bufs], torch.view_as_real(pad))
    else:
        dist.all_gather(bufs, pad)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], 0)
