"""Host-side logic mirroring the reference: parameter bundles, peel rule,
shard / panel plans. CPU only."""

import numpy as np
import pytest

from paper_0811_1714_b200 import (MulParams, ParameterError, StripeSpec,
                                  default_params)
from paper_0811_1714_b200.sharded import k_panels, shard_rows


def test_mulparams_mirror():
    # test_strassen.py:21-35
    assert MulParams(cutoff=128).b_s == 64
    for kw in [dict(cutoff=32), dict(cutoff=128, t=9),
               dict(cutoff=128, b_s=256), dict(cutoff=128, k=17)]:
        with pytest.raises(ParameterError):
            MulParams(**kw)
    p = default_params()
    assert p.cutoff >= 64 and 1 <= p.b_s <= p.cutoff


def test_stripespec_mirror():
    # test_m4rm.py:21-34
    s = StripeSpec(k=6, t=8, b_s=256)
    assert (s.k, s.t, s.b_s) == (6, 8, 256)
    for kw in [dict(k=0), dict(k=17), dict(k=4, t=9), dict(k=4, t=1, b_s=0)]:
        with pytest.raises(ParameterError):
            StripeSpec(**kw)


def test_peel_split_properties():
    # test_strassen.py:50-63
    from paper_0811_1714_b200 import peel_split
    rng = np.random.default_rng(1)
    for _ in range(200):
        m, l, n = (int(x) for x in rng.integers(1, 5000, 3))
        ps = peel_split(m, l, n, 128)
        if ps.depth == 0:
            continue
        unit = 64 << ps.depth
        for x, x0 in [(ps.m, m), (ps.l, l), (ps.n, n)]:
            assert x % unit == 0 and x <= x0 < x + unit
            assert (x >> ps.depth) >= 128 and (x >> ps.depth) % 64 == 0


@pytest.mark.parametrize("m,world", [(16384, 1), (16384, 2), (16384, 8),
                                     (65536, 8), (10000, 3), (100, 8),
                                     (7, 4)])
def test_shard_rows_partition(m, world):
    spans = [shard_rows(m, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == m
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0 and a0 <= a1
    if m >= 64 * world:
        assert all(r0 % 64 == 0 for r0, _ in spans)


def test_k_panels():
    assert k_panels(0, 4) == []
    for l, p in [(16384, 4), (7001, 3), (64, 8), (65, 2), (1, 1)]:
        ps = k_panels(l, p)
        assert ps[0][0] == 0 and ps[-1][1] == l
        assert all(k0 % 64 == 0 for k0, _ in ps)
        for (a0, a1), (b0, b1) in zip(ps, ps[1:]):
            assert a1 == b0


def test_gf2m_load_errors_match_reference(golden, tmp_path):
    """core.py:455-484 messages and byte offsets (no GPU needed: the file
    is validated on the host before any upload)."""
    from paper_0811_1714_b200 import FormatError, load
    good = golden["gf2m_37x200_s5"].tobytes()
    width = 4
    dirty = bytearray(good)
    dirty[21 + (3 * width + width - 1) * 8] |= 1
    cases = {"truncated": good[:10], "magic": b"GF3M" + good[4:],
             "version": good[:4] + b"\x02" + good[5:], "length": good[:-8],
             "dirty": bytes(dirty)}
    want = dict(zip(golden["gf2m_error_names"].tolist(),
                    golden["gf2m_error_msgs"].tolist()))
    fp = tmp_path / "bad.gf2m"
    for name, data in cases.items():
        fp.write_bytes(data)
        with pytest.raises(FormatError) as exc:
            load(fp)
        assert str(exc.value) == want[name], name


def test_bench_reference_arm_contract():
    """bench.py --impl reference (CPU only): exactly one JSON line on stdout
    with the contract's keys on rank 0; other ranks print nothing and exit 0."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--size", "1024",
           "--steps", "1", "--warmup", "0"]
    out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.splitlines()
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    for k in ("metric", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "cpu_baseline", "e2e", "config"):
        assert k in d, k
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    other = subprocess.run(cmd + ["--gpus", "2"], cwd=root, capture_output=True, text=True,
                           timeout=300, env=dict(os.environ, RANK="1", WORLD_SIZE="2"))
    assert other.returncode == 0 and other.stdout == ""
