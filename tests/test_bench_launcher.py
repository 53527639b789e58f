"""bench.py's launcher on CPU: `--gpus N` is authoritative. Without torchrun
and N > 1 the script re-launches itself as N ranks (torch.distributed.run on
127.0.0.1); under torchrun WORLD_SIZE must equal N; with fewer CUDA devices
than N the GPU arm refuses instead of measuring fewer GPUs. The stub arm
(`--impl stub`) runs no GPU work: every rank reports itself over gloo."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env_extra=None, timeout=180):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, BENCH, *args], capture_output=True,
                          text=True, timeout=timeout, env=env, cwd=ROOT)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_launcher_spawns_n_ranks(n):
    p = _run(["--gpus", str(n), "--impl", "stub"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [x for x in p.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, p.stdout          # exactly one JSON line on stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "stub" and rec["n_gpus"] == n and rec["world"] == n
    assert sorted(r["rank"] for r in rec["ranks"]) == list(range(n))
    assert sorted(r["local_rank"] for r in rec["ranks"]) == list(range(n))
    assert len({r["pid"] for r in rec["ranks"]}) == n      # one process per rank


def test_world_size_must_match_gpus():
    p = _run(["--gpus", "2", "--impl", "stub"], {"WORLD_SIZE": "1", "RANK": "0",
                                                  "LOCAL_RANK": "0"})
    assert p.returncode != 0
    assert "WORLD_SIZE=1 but --gpus 2" in p.stderr
    assert p.stdout.strip() == ""


def test_gpu_arm_refuses_missing_devices():
    import torch
    have = torch.cuda.device_count()
    p = _run(["--gpus", str(max(2, have + 1))])
    assert p.returncode != 0
    assert "refusing to measure fewer GPUs" in p.stderr
    assert p.stdout.strip() == ""
    if have == 0:   # N = 1 without a device fails loudly too (no CPU fallback)
        p = _run(["--gpus", "1"])
        assert p.returncode != 0 and p.stdout.strip() == ""


def test_parse_workloads():
    sys.path.insert(0, ROOT)
    import bench
    a = bench.parse(["--workload", "cfg5"])
    assert a.workload == "cfg5" and a.extra_list == []      # cfg5 not repeated
    a = bench.parse([])
    assert a.workload == "cfg3" and a.extra_list == ["cfg5"]
    a = bench.parse(["--extra", "none"])
    assert a.extra_list == []
    assert bench.WORKLOADS["cfg5"]["kind"] == "addmul"
    assert bench.WORKLOADS["cfg5"]["digest"] == "cfg5_addmul"
    with pytest.raises(SystemExit):
        bench.parse(["--extra", "cfg9"])


def _digest_worker(rank, world, port, m, width, q):
    import hashlib

    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        import bench
        from paper_0811_1714_b200.core import words_per_row
        from paper_0811_1714_b200.sharded import shard_rows
        full = np.arange(m * width, dtype=np.uint64).reshape(m, width) * np.uint64(0x9E3779B97F4A7C15)
        r0, r1 = shard_rows(m, world, rank)

        class Out:   # a row shard with a padded pitch, like a BitMatrix
            storage = torch.from_numpy(np.pad(full[r0:r1], ((0, 0), (0, 3))).view(np.int64))

            def to_numpy(self):
                return full[r0:r1].copy()

        class G:
            pass
        G.words_per_row = staticmethod(words_per_row)
        ctx = bench.Ctx(None, G, torch.device("cpu"), world, rank, 0, True, None, None)
        got = bench.digest_rows(ctx, Out(), {"m": m, "n": width * 64})
        if rank == 0:
            q.put((got, hashlib.sha256(full.astype("<u8").tobytes()).hexdigest()))
    finally:
        dist.destroy_process_group()


def test_digest_rows_world3_gloo():
    """bench.digest_rows: rank 0 hashes the row shards in rank order (the
    sha256 of the whole matrix), each shard sent without its pitch padding."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_digest_worker, args=(r, 3, port, 200, 5, q)) for r in range(3)]
    for p in procs:
        p.start()
    got, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == want
