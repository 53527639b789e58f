"""bench.py's N > 1 path end to end on a one-GPU box: `--gpus 2` self-launches
two ranks through torch.distributed.run; with GF2_BENCH_SHARE_GPU=1 (a
test-only switch) both ranks run on cuda:0 with gloo for the collectives
instead of NCCL. Row shards of A and C, the K-panel broadcast of B, the
max-over-ranks timing, the rank-ordered digest of the gathered C and the
sharded host pipeline all run as they would on two GPUs; the line must be
digest-verified and flagged as a code-path test, not a measurement."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_share_one_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, GF2_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
                          "--warmup", "1", "--extra", "none", "--no-cpu-baseline"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["verified_sha256"] is True
    assert "share_gpu_test" in d
    assert d["e2e"]["verified_vs_device_result"] is True
    assert d["config"]["parallelism"].startswith("rows2")


def test_bench_process_grid_share_one_gpu():
    """`--gpus 4 --grid 2x2` the same way: rank (i, j) owns C[rows_i, cols_j],
    B's column blocks are cut on grid row 0 and broadcast inside the column
    groups, rank 0 assembles the blocks and checks the cfg3 digest; the
    grid's end-to-end step (A_i gathered inside row groups, B_j's rows
    distributed over the column group) must reproduce the device result."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, GF2_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--grid", "2x2",
                          "--steps", "2", "--warmup", "1", "--extra", "none", "--no-cpu-baseline"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 4 and d["verified_sha256"] is True
    assert d["e2e"]["verified_vs_device_result"] is True
    assert d["config"]["parallelism"].startswith("grid2x2")


@pytest.mark.parametrize("nproc,grid", [(2, "rows"), (4, "2x2")])
def test_example_sharded_mul_on_one_gpu(nproc, grid):
    """examples/sharded_mul.py under torchrun, all ranks on cuda:0 over gloo:
    the row-sharded layout and a 2 x 2 process grid, every block
    Freivalds-checked against the full B."""
    import socket
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
                          os.path.join(ROOT, "examples", "sharded_mul.py"), "--size", "6144", "--grid", grid,
                          "--npanels", "3", "--backend", "gloo", "--one-gpu"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, (out.stdout + out.stderr)[-3000:]
    assert "Freivalds on every block: True" in out.stdout
