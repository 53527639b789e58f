"""Command-line front end over the device path.

    python -m paper_0811_1714_b200 gen --dims MxN --seed S --out A.gf2m
    python -m paper_0811_1714_b200 mul A.gf2m B.gf2m C.gf2m [--algo NAME]
    python -m paper_0811_1714_b200 check --dims MxLxN [--algo NAME ...]
    python -m paper_0811_1714_b200 bench [--dims MxLxN ...] [--reps R] [--out CSV]
    python -m paper_0811_1714_b200 params

Subcommands, flags, algorithm names, CSV columns and exit codes follow the
reference CLI (cli.py:65-351): algorithms cubic, m4rm, m4rm-blocked,
m4rm-t<t> (t = 1..8), strassen, auto; `check` exits 1 on a mismatch, file /
dimension errors exit 2; `bench` writes the reference's CSV header exactly
(cli.py:97-129, so gf2mat's parse_csv reads it), peak_mem_bytes being the
device memory high-water mark of the timed repetitions. Added: --engine
(m4rm | tc-i8 | tc-f8 | tc-f4) selects the Strassen leaf engine. `check`
does what the reference's does (cli.py:181-211): a host-side naive product
is the oracle (the reference's `_reference.naive_product`, restated here as
a NumPy float64 matrix product mod 2 -- the checker, never a compute path),
the device cubic product is checked against it, and every variant is
compared with the oracle and then with the cubic product.
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from . import _lib
from .core import first_difference, random
from .errors import GF2MatError, ParameterError
from .gf2m import load, save
from .m4rm import mul_m4rm, mul_m4rm_blocked, mul_m4rm_multitable
from .strassen import MulParams, default_params, mul_strassen
from .structure import mul_cubic

ALGOS = ("cubic", "m4rm", "m4rm-blocked", "m4rm-t2", "m4rm-t8", "strassen",
         "auto")
FIELDS = ("algorithm", "m", "l", "n", "k", "t", "bs", "cutoff", "reps",
          "wall_s", "mean_s", "min_s", "peak_mem_bytes")  # cli.py:97-129 BenchRecord


def _dims(text: str, parts: int):
    xs = text.lower().split("x")
    if len(xs) != parts:
        raise ParameterError(f"--dims wants {'x'.join('MLN'[:parts] if parts == 3 else 'MN')}, got {text!r}")
    try:
        vals = tuple(int(x) for x in xs)
    except ValueError:
        raise ParameterError(f"--dims wants integers, got {text!r}") from None
    if any(v < 0 for v in vals):
        raise ParameterError(f"--dims must be non-negative, got {text!r}")
    return vals


def algorithm(name: str, params: MulParams):
    """The reference's _algorithm registry (cli.py:65-94) on the device."""
    k = params.k or 8
    if name == "cubic":
        return mul_cubic
    if name == "m4rm":
        return lambda a, b: mul_m4rm(a, b, k)
    if name == "m4rm-blocked":
        return lambda a, b: mul_m4rm_blocked(a, b, k, params.b_s)
    if name.startswith("m4rm-t"):
        try:
            t = int(name[6:])
        except ValueError:
            raise ParameterError(f"unknown algorithm {name!r}") from None
        if not 1 <= t <= 8:
            raise ParameterError(f"table count in {name!r} outside 1..8")
        return lambda a, b: mul_m4rm_multitable(a, b, k, t, params.b_s)
    if name in ("strassen", "auto"):
        return lambda a, b: mul_strassen(a, b, params)
    raise ParameterError(f"unknown algorithm {name!r}")


def _params(args) -> MulParams:
    base = default_params()
    cutoff = args.cutoff if getattr(args, "cutoff", None) else base.cutoff
    bs = args.bs if getattr(args, "bs", None) else max(cutoff // 2, 1)
    k = args.k if getattr(args, "k", None) is not None else base.k
    t = args.t if getattr(args, "t", None) else base.t
    return MulParams(cutoff=cutoff, b_s=bs, k=k, t=t)


def _time(fn, a, b, reps):
    """(per-repetition seconds, peak bytes): CUDA events around each call,
    warm-up excluded (cli.py:159); the peak is the device memory high-water
    mark of the timed repetitions above what was live before them -- torch's
    allocations (matrices) plus the library's pooled workspace -- the
    device analogue of counters.peak_live_words (cli.py:161-166)."""
    import torch
    fn(a, b)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    ws0 = _lib.workspace_peak(reset=True)
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(a, b)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    peak = max(torch.cuda.max_memory_allocated() - base, 0) + max(_lib.workspace_peak() - ws0, 0)
    return times, peak


def _host_dense(m) -> np.ndarray:
    """Downloaded words -> (nrows, ncols) 0/1 array (MSB-first, core.py:405-414)."""
    w = m.to_numpy()
    if not w.size:
        return np.zeros((m.nrows, m.ncols), dtype=np.uint8)
    bits = np.unpackbits(w.astype(">u8").view(np.uint8).reshape(m.nrows, -1), axis=1)
    return bits[:, :m.ncols]


def naive_product(a, b) -> np.ndarray:
    """The check oracle (the reference's _reference.naive_product): the
    product of the downloaded operands as a float64 matrix product mod 2 --
    exact while inner dimensions stay below 2^53."""
    da, db = _host_dense(a).astype(np.float64), _host_dense(b).astype(np.float64)
    return (np.rint(da @ db).astype(np.int64) & 1).astype(np.uint8)


def _first_mismatch(m, dense):
    """First (row, col) where device matrix m differs from a 0/1 array, or None."""
    got = _host_dense(m)
    diff = np.argwhere(got != dense)
    return None if not len(diff) else (int(diff[0][0]), int(diff[0][1]))


def cmd_check(args, params) -> int:
    status = 0
    algos = args.algo or [x for x in ALGOS if x != "cubic"]
    col = max(len(x) for x in algos) + 2
    for m, l, n in args.dims:
        a, b = random(m, l, args.seed), random(l, n, args.seed + 1)
        oracle = naive_product(a, b)
        ref = mul_cubic(a, b)
        where = _first_mismatch(ref, oracle)
        if where is not None:
            print(f"{m}x{l}x{n}  cubic: FAIL at {where} (vs oracle)")
            status = 1
        cells = []
        for idx, name in enumerate(algos):
            got = algorithm(name, params)(a, b)
            if args.inject_fault and idx == 0 and m and n:
                from .core import copy_into, from_dense, to_dense, window
                d = to_dense(window(got, 0, 0, 1, 1))
                d[0, 0] ^= 1
                copy_into(window(got, 0, 0, 1, 1), from_dense(d))
            where = _first_mismatch(got, oracle)
            if where is None:
                where = first_difference(got, ref)
            if where is None:
                cells.append(f"{name}:ok".ljust(col + 3))
            else:
                cells.append(f"{name}:FAIL{where}".ljust(col + 12))
                status = 1
        print(f"{m}x{l}x{n}  " + " ".join(cells))
    print("check:", "FAIL" if status else "PASS")
    return 1 if status else 0


def cmd_bench(args, params) -> int:
    rows = []
    for m, l, n in args.dims or [(d, d, d) for d in (1024, 2048, 4096, 8192, 16384)]:
        a, b = random(m, l, args.seed), random(l, n, args.seed + 1)
        for name in args.algo or ["m4rm", "strassen"]:
            ts, peak = _time(algorithm(name, params), a, b, args.reps)
            rows.append({"algorithm": name, "m": m, "l": l, "n": n,
                         "k": params.k, "t": params.t, "bs": params.b_s,
                         "cutoff": params.cutoff, "reps": args.reps,
                         "wall_s": sum(ts), "mean_s": sum(ts) / len(ts),
                         "min_s": min(ts), "peak_mem_bytes": peak})
    print(f"engine={_lib.get_engine()}", file=sys.stderr)
    fh = open(args.out, "w", encoding="utf-8") if args.out else sys.stdout
    # the reference's emit_csv format (cli.py:117-122): floats as repr
    fh.write(",".join(FIELDS) + "\n")
    for r in rows:
        fh.write(",".join(repr(r[f]) if isinstance(r[f], float) else str(r[f]) for f in FIELDS) + "\n")
    if args.out:
        fh.close()
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_0811_1714_b200",
                                 description="GF(2) matrix multiplication on B200")
    sub = ap.add_subparsers(dest="command", required=True)

    def tuning(p):
        p.add_argument("--cutoff", type=int)
        p.add_argument("--bs", type=int)
        p.add_argument("--k", type=int)
        p.add_argument("--t", type=int)
        p.add_argument("--engine", choices=sorted(_lib.ENGINES))

    p = sub.add_parser("check")
    p.add_argument("--dims", action="append", required=True, type=lambda s: _dims(s, 3))
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--algo", action="append")
    p.add_argument("--inject-fault", action="store_true")
    tuning(p)
    p = sub.add_parser("bench")
    p.add_argument("--dims", action="append", type=lambda s: _dims(s, 3))
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--algo", action="append")
    p.add_argument("--out")
    tuning(p)
    p = sub.add_parser("gen")
    p.add_argument("--dims", required=True, type=lambda s: _dims(s, 2))
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True)
    p = sub.add_parser("mul")
    p.add_argument("a")
    p.add_argument("b")
    p.add_argument("c")
    p.add_argument("--algo")
    tuning(p)
    p = sub.add_parser("params")
    tuning(p)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        if getattr(args, "engine", None):
            _lib.set_engine(args.engine)
        if args.command == "gen":
            m, n = args.dims
            save(random(m, n, args.seed), args.out)
            return 0
        params = _params(args)
        if args.command == "check":
            return cmd_check(args, params)
        if args.command == "bench":
            return cmd_bench(args, params)
        if args.command == "mul":
            save(algorithm(args.algo or "auto", params)(load(args.a), load(args.b)), args.c)
            return 0
        for f in ("cutoff", "b_s", "k", "t"):
            print(f"{f if f != 'b_s' else 'bs'}={getattr(params, f)}")
        print(f"engine={_lib.get_engine()}")
        return 0
    except (GF2MatError, OSError) as exc:
        print(f"paper_0811_1714_b200: error: {exc}", file=sys.stderr)
        return 2
