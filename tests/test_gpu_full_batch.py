"""Every BASELINE.json configuration at full size on the GPU, checked row by row
against the CPU oracle bit for bit (no sampling): config 1 (64 rows), config 2
(16384), config 3 (2048), config 4 (64) and config 5 (2^18 rows, 32 GiB in and
32 GiB out, checked in chunks).  The oracle is pinned to the reference by
tests/test_oracle.py (including rows 0-1 of each configuration's own input).
Run with -m gpu on a B200."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_config_full_batch_bitwise(torch_cuda, c):
    torch = torch_cuda
    from oracle import parity
    from paper_1301_0763_b200 import improved, workloads
    B = workloads.CONFIGS[c]["batch"]
    x = workloads.config_rows_device(c)
    y = improved.cdft_rows(x)
    torch.cuda.synchronize()
    rep = parity.check_rows(x, y)
    print(f"config {c}: {rep}")
    assert rep["rows_checked"] == B
    assert rep["mismatches"] == 0, rep


def test_config4_classical_full_batch_bitwise(torch_cuda):
    """The comparison entry point at config 4 (classical.cdft, fp64 2^20 x 64)."""
    torch = torch_cuda
    from oracle import parity
    from paper_1301_0763_b200 import classical, workloads
    x = workloads.config_rows_device(4)
    y = classical.cdft_rows(x)
    torch.cuda.synchronize()
    rep = parity.check_rows(x, y, algo="classical")
    assert rep["mismatches"] == 0, rep


@pytest.mark.parametrize("c,rows,first", [(2, 64, 0), (2, 7, 16000), (5, 5, 12345), (5, 3, (1 << 18) - 3)])
def test_device_generator_matches_numpy_twin(torch_cuda, c, rows, first):
    """qft_fill_normal == workloads.keyed_normal_rows bit for bit (any slice)."""
    from paper_1301_0763_b200 import workloads
    x = workloads.config_rows_device(c, rows, first).cpu().numpy()
    want = workloads.keyed_normal_rows(workloads.CONFIGS[c]["N"], rows, first, workloads.SEEDS[c])
    assert x.tobytes() == want.tobytes()


def test_shards_equal_single_gpu_rows(torch_cuda):
    """Batch sharding: the rows a rank generates and
    transforms for its shard equal the same rows of the 1-GPU run bit for bit."""
    from paper_1301_0763_b200 import improved, sharding, workloads
    total = 4096
    full = improved.cdft_rows(workloads.config_rows_device(5, total, 0)).cpu().numpy()
    for ws in (2, 8):
        for rank in range(ws):
            b0, b1 = sharding.shard_bounds(total, ws, rank)
            part = sharding.transform_shard(workloads.config_rows_device(5, b1 - b0, b0)).cpu().numpy()
            assert part.tobytes() == full[b0:b1].tobytes(), (ws, rank)
