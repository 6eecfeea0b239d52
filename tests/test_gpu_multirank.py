"""The bench's multi-rank path (torchrun, one process per rank, batch-sharded, no
data-path collective) executed end to end on the single GPU this pool provides:
both ranks on cuda:0 with the gloo backend for the timing reduction
(QFT_BENCH_BACKEND / QFT_BENCH_DEVICE).  Functional only -- not a scaling point."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, env_extra, timeout=900):
    env = dict(os.environ, QFT_BENCH_BACKEND="gloo", QFT_BENCH_DEVICE="0", **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py"] + args
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.gpu
def test_two_ranks_weak_config2():
    line = _torchrun(["--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e", "--config", "2"], {})
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert len(line["per_gpu"]["value"]) == 2
    # every row of both shards (each rank's 16384 rows, keyed on the global row index)
    assert line["parity"]["rows_checked"] == 2 * 16384 and line["parity"]["mismatches"] == 0
    assert line["value"] > 0 and line["ms_per_step"] == max(line["per_gpu"]["ms_per_step"])


@pytest.mark.gpu
def test_two_ranks_strong_config5_shards():
    line = _torchrun(["--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e", "--no-parity",
                      "--config", "5"], {})
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["batch_per_gpu"] == (1 << 18) // 2


@pytest.mark.gpu
def test_two_ranks_reference_arm():
    line = _torchrun(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-seconds", "0.5"],
                     {})
    assert line["impl"] == "reference" and line["value"] > 0
