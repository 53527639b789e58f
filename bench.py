#!/usr/bin/env python
"""Benchmark of the B200 GF(2) multiply (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--impl b200|reference|stub] [--workload cfg3|cfg5]
                    [--extra cfg5|none] [--grid rows|PRxPC|auto]

One JSON line on rank 0.

Workloads (BASELINE.json configs; seeds per SURVEY.md §8(c)):
  cfg3 (default, the shape the metric is quoted on): C = A.B over GF(2),
       A and B 16384 x 16384 splitmix64 bits (core.random seeds 31 / 32),
       Strassen-Winograd with the device default cutoff over the default
       base-case engine (tcgen05 kind::mxf4; `--engine` selects another).
  cfg5: C = C0 + A.B (addmul), A, B, C0 65536 x 65536 (seeds 51/52/53).
The line reports `--workload`; every workload named by `--extra` (default
cfg5) is measured after it with the same rules and reported under
"workloads", so one driver run covers both of north_star's shapes.

GPUs: `--gpus N` is authoritative. Under torchrun WORLD_SIZE must equal N.
Without torchrun and N > 1 the script re-launches itself as N ranks through
torch.distributed.run (one process per GPU, NCCL, NCCL_DEBUG=INFO on stderr)
and exits non-zero if fewer than N CUDA devices are visible -- it never
measures fewer GPUs than it reports. N > 1: C and A row-sharded and generated
in place, B generated on rank 0 and broadcast over NVLink (NCCL) in K-panels
inside the timed step; time = max over ranks. `--grid PRxPC|auto` lays the N
ranks out as a process grid instead (rank (i, j) owns C[rows_i, cols_j]; B's
column block j is cut on grid row 0 and broadcast inside column group j).

`--impl reference` times the reference algorithm's CPU port
(oracle/libgf2oracle.so, a C restatement of gf2mat's M4RM + Strassen-
Winograd, all host threads) on a bounded row sample of the same workload,
and beside it the stock gf2mat package (baseline/_ref, one core) on a
smaller row sample when it is installed. `--impl stub` runs no GPU work:
each rank reports itself (the launcher's CPU test).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("GF(2) matmul effective bit-ops/s (n^3) and ms/multiply at "
          "n=16384, 1/2/4/8 B200")
UNIT = "bit-ops/s"
WORKLOADS = {
    "cfg3": dict(name="cfg3", kind="product", m=16384, l=16384, n=16384,
                 seed_a=31, seed_b=32, digest="cfg3",
                 call="mul_strassen(A, B)"),
    "cfg5": dict(name="cfg5", kind="addmul", m=65536, l=65536, n=65536,
                 seed_a=51, seed_b=52, seed_c=53, digest="cfg5_addmul",
                 call="addmul(C, A, B): C = C0 + A.B (reference: "
                      "add_into(C, C, mul_strassen(A, B)))"),
}
PAPER_2008_CPU = 16384 ** 3 / 6.074   # PAPER.md:753 (M4RI, Core 2 Duo)


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference", "stub"])
    p.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    p.add_argument("--extra", default="cfg5",
                   help="comma-separated workloads measured after --workload "
                        "and reported under 'workloads' ('none' for none)")
    p.add_argument("--cutoff", type=int, default=0,
                   help="Strassen cutoff (0 = device default)")
    p.add_argument("--npanels", type=int, default=2)
    p.add_argument("--grid", default="rows",
                   help="N > 1 layout: 'rows' (north_star (e): C and A row-sharded, B "
                        "broadcast to every rank), 'PRxPC' or 'auto' (process grid: "
                        "rank (i, j) owns C[rows_i, cols_j], B's column block j is "
                        "broadcast inside column group j)")
    p.add_argument("--sharded", action="store_true",
                   help="run the multi-GPU (NCCL) step and e2e path even at "
                        "N = 1 (a world of one; for testing it on one GPU)")
    p.add_argument("--engine", default="tc-f4", choices=["m4rm", "tc-i8", "tc-f8", "tc-f4"],
                   help="product engine (results are identical)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-verify", action="store_true")
    p.add_argument("--size", type=int, default=0,
                   help="override n (debug only; the metric is n=16384)")
    args = p.parse_args(argv)
    if args.gpus < 1:
        p.error("--gpus must be >= 1")
    args.extra_list = [] if args.extra in ("", "none") else \
        [x for x in args.extra.split(",") if x != args.workload]
    for x in args.extra_list:
        if x not in WORKLOADS:
            p.error(f"--extra: unknown workload {x!r}")
    return args


def die(msg: str, code: int = 2):
    print(f"bench.py: error: {msg}", file=sys.stderr, flush=True)
    sys.exit(code)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    polled every millisecond (the device matched by PCI bus id), falling
    back to `nvidia-smi -lms 100` if NVML is unavailable. Reports the median
    and minimum SM clock under load and every throttle reason seen."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
             "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []          # (sm_mhz, set of reasons)
        self.max_mhz = None
        self.stop_flag = threading.Event()
        self.mode = None
        self.proc = None

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            nv, h = self._nvml_handle()
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}

            def loop():
                while not self.stop_flag.is_set():
                    try:
                        mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((mhz, {k for k, v in bits.items() if r & v}))
                    except Exception:
                        pass
                    time.sleep(0.001)
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
            self.mode = "nvml"
            return
        except Exception:
            pass
        try:
            fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                      "clocks_event_reasons.hw_thermal_slowdown,"
                      "clocks_event_reasons.sw_thermal_slowdown,"
                      "clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

            def read():
                for line in self.proc.stdout:
                    f = [x.strip() for x in line.split(",")]
                    if len(f) < 6:
                        continue
                    try:
                        mhz, self.max_mhz = float(f[0]), float(f[1])
                    except ValueError:
                        continue
                    self.samples.append((mhz, {n for n, v in zip(self.NAMES, f[2:6])
                                               if v.lower().startswith("active")}))
            self.t = threading.Thread(target=read, daemon=True)
            self.t.start()
            self.mode = "nvidia-smi"
        except Exception:
            self.mode = None

    def stop(self):
        if self.mode is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        if self.mode == "nvml":
            self.stop_flag.set()
            self.t.join(timeout=2)
        else:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm = sorted(x[0] for x in self.samples)
        reasons = set()
        for _, r in self.samples:
            reasons |= r
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_min_mhz": sm[0] if sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(sm), "source": self.mode}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, \
            "fallback (B200_PROFILING.md)"


def _json_file(*parts):
    try:
        with open(os.path.join(ROOT, *parts)) as fh:
            return json.load(fh)
    except Exception:
        return None


def golden_digest(key: str):
    d = _json_file("tests", "golden", "digests.json")
    return d.get(key) if d else None


def _sha(words) -> str:
    return hashlib.sha256(words.astype("<u8", copy=False).tobytes()).hexdigest()


# ------------------------------------------------------------------ CPU port
def cpu_port_sample(w, target_s=8.0, rows=None, min_total_s=10.0):
    """Time the reference algorithm's C port on a row sample A[:R] . B (plus
    the XOR of C0's rows for addmul workloads) with all host threads.
    Returns (bitops_per_s, threads, rows, mean_s, reps)."""
    import numpy as np
    from oracle import gf2_port as P
    m, l, n = w["m"], w["l"], w["n"]
    threads = len(os.sched_getaffinity(0))
    P.set_threads(threads)
    b = P.random(l, n, w["seed_b"])
    c0 = None

    def once(a):
        c = P.mul_strassen(a, b)
        if c0 is not None:
            np.bitwise_xor(c.words, c0.words, out=c.words)
        return c

    if rows is None:
        rows = min(m, 256)
        while True:
            a = P.random(rows, l, w["seed_a"])
            if w["kind"] == "addmul":
                c0 = P.random(rows, n, w["seed_c"])
            t0 = time.perf_counter()
            once(a)
            dt = time.perf_counter() - t0
            if dt * 2 > target_s or rows >= m:
                break
            rows = min(m, rows * 2)
    a = P.random(rows, l, w["seed_a"])
    if w["kind"] == "addmul":
        c0 = P.random(rows, n, w["seed_c"])
    reps, total = 0, 0.0
    while reps == 0 or total < min_total_s:
        t0 = time.perf_counter()
        once(a)
        total += time.perf_counter() - t0
        reps += 1
    dt = total / reps
    return rows * l * n / dt, threads, rows, dt, reps


def stock_reference_sample(w, rows=None, target_s=4.0):
    """The unmodified gf2mat package (installed under baseline/_ref), through
    its public API (`random`, `mul_strassen`, `add_into`) on ONE core -- it
    starts no threads -- on a row sample A[:R] . B sized to
    ~target_s. None when the package is not installed. NB: with R rows below
    the default cutoff, mul_strassen dispatches to its M4RM base case, so the
    sample times gf2mat's M4RM rate at this width (no Strassen level)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "gf2mat")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import gf2mat as R
    except Exception as exc:          # pragma: no cover - install problem
        return {"unavailable": f"import gf2mat failed: {exc}"}
    m, l, n = w["m"], w["l"], w["n"]
    b = R.random(l, n, w["seed_b"])
    rows = rows or 64
    while True:
        a = R.random(rows, l, w["seed_a"])
        c0 = R.random(rows, n, w["seed_c"]) if w["kind"] == "addmul" else None
        t0 = time.perf_counter()
        c = R.mul_strassen(a, b)
        if c0 is not None:
            R.add_into(c0, c0, c)
        dt = time.perf_counter() - t0
        if dt * 2 > target_s or rows >= m:
            break
        rows = min(m, rows * 2)
    return {"value": rows * l * n / dt, "unit": UNIT, "cores": 1,
            "kind": "reference",
            "sample": f"gf2mat {R.__version__} (baseline/_ref, stock) "
                      f"mul_strassen(A[:{rows}], B) default params"
                      + (" + add_into(C0[:rows], ...)" if c0 is not None else "")
                      + f", {rows}x{l}x{n}, {dt:.2f} s, one core"}


def run_reference(args):
    """--impl reference: the reference algorithm on the host CPU (port)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = dict(WORKLOADS[args.workload])
    if args.size:
        w.update(m=args.size, l=args.size, n=args.size)
    m, l, n = w["m"], w["l"], w["n"]
    # size the sample so that warmup + steps finish in a few minutes
    _, threads, rows, dt, _ = cpu_port_sample(w, target_s=6.0, min_total_s=0.0)
    import numpy as np
    from oracle import gf2_port as P
    b = P.random(l, n, w["seed_b"])
    a = P.random(rows, l, w["seed_a"])
    c0 = P.random(rows, n, w["seed_c"]) if w["kind"] == "addmul" else None
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        c = P.mul_strassen(a, b)
        if c0 is not None:
            np.bitwise_xor(c.words, c0.words, out=c.words)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    per = sum(times) / len(times)
    value = rows * l * n / per
    sample = (f"A[:{rows}] x B ({rows}x{l}x{n}) per step, C port of "
              f"mul_strassen default params (cutoff 2048, k auto, t 8)"
              + (" + XOR of C0's rows" if c0 is not None else ""))
    stock = stock_reference_sample(w)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3 * (m / rows), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": f"synthetic: core.random splitmix64 bits, seeds "
                f"{w['seed_a']}/{w['seed_b']}",
        "config": {"workload": f"{w['name']}: {m}x{l}x{n} GF(2) {w['call']}",
                   "m": m, "l": l, "n": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                         "kind": "port", "sample": sample},
        "stock_reference_1core": stock,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "ms_per_step extrapolated to the full m rows",
    }
    emit(line)


# ------------------------------------------------------------------ launcher
def _free_port() -> int:
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def launch_ranks(args) -> int:
    """--gpus N > 1 without torchrun: re-launch this script as N ranks (one
    process per GPU) through torch.distributed.run on 127.0.0.1. Refuses
    (exit 2) when fewer than N CUDA devices are visible."""
    if args.impl == "b200" and not os.environ.get("GF2_BENCH_SHARE_GPU"):
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            die(f"--gpus {args.gpus} but {have} CUDA device(s) are visible; "
                "refusing to measure fewer GPUs than requested")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    env = dict(os.environ)
    if args.impl == "b200":
        env.setdefault("NCCL_DEBUG", "INFO")   # rank / channel counts on stderr
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}",
          file=sys.stderr, flush=True)
    return subprocess.run(cmd, env=env, stdout=_STDOUT_FD).returncode


def run_stub(args):
    """No GPU work: every rank reports itself over gloo (launcher test)."""
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(_free_port()))
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    dist.init_process_group("gloo")
    me = {"rank": dist.get_rank(), "local_rank": int(os.environ.get("LOCAL_RANK", "0")),
          "pid": os.getpid()}
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, me)
    if dist.get_rank() == 0:
        emit({"impl": "stub", "n_gpus": args.gpus, "world": dist.get_world_size(),
              "ranks": parts})
    dist.destroy_process_group()


# ------------------------------------------------------------------ GPU arm
class Ctx:
    """Per-process state of the GPU arm."""

    def __init__(self, args, g, dev, world, rank, local, dist_on, flush, stream):
        self.args, self.g, self.dev = args, g, dev
        self.world, self.rank, self.local = world, rank, local
        self.dist_on, self.flush, self.stream = dist_on, flush, stream
        self.grid = None            # ProcessGrid when --grid is not 'rows'

    def max_over_ranks(self, ms: float, ok: bool = True):
        if not self.dist_on:
            return ms, ok
        import torch
        import torch.distributed as dist
        t = torch.tensor([ms, 0.0 if ok else 1.0], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0].item()), not bool(t[1].item())

    def barrier(self):
        import torch
        torch.cuda.synchronize()
        if self.dist_on:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()


def digest_rows(ctx, out, w):
    """sha256 of the whole matrix's raw words in row order: rank 0 hashes its
    rows, then receives every other rank's shard over NCCL in rank order."""
    g = ctx.g
    if not ctx.dist_on:
        return _sha(out.to_numpy())
    import torch
    import torch.distributed as dist
    from paper_0811_1714_b200.sharded import shard_rows
    width = g.words_per_row(w["n"])
    cuda_p2p = dist.get_backend() == "nccl"  # gloo (GF2_BENCH_SHARE_GPU) sends host tensors
    if ctx.grid is not None:
        # blocks, not row shards: rank 0 assembles the matrix on the host
        import numpy as np
        grid = ctx.grid
        full = np.zeros((w["m"], width), dtype="<u8") if ctx.rank == 0 else None
        for r in range(ctx.world):
            r0, r1, c0, c1 = grid.block_of(r, w["m"], w["n"])
            bw = g.words_per_row(c1 - c0)
            if r1 == r0 or bw == 0:
                continue
            if r == ctx.rank == 0:
                full[r0:r1, c0 // 64:c0 // 64 + bw] = out.to_numpy()
            elif r == ctx.rank:
                t = out.storage[:, :bw].contiguous()
                dist.send(t if cuda_p2p else t.cpu(), dst=0)
            elif ctx.rank == 0:
                t = torch.empty((r1 - r0, bw), dtype=torch.int64, device=ctx.dev if cuda_p2p else "cpu")
                dist.recv(t, src=r)
                full[r0:r1, c0 // 64:c0 // 64 + bw] = t.cpu().numpy().view(np.uint64)
        return hashlib.sha256(full.tobytes()).hexdigest() if ctx.rank == 0 else None
    h = hashlib.sha256() if ctx.rank == 0 else None
    for r in range(ctx.world):
        r0, r1 = shard_rows(w["m"], ctx.world, r)
        if r == ctx.rank == 0:
            h.update(out.to_numpy().astype("<u8", copy=False).tobytes())
        elif r == ctx.rank:
            t = out.storage[:, :width].contiguous()
            dist.send(t if cuda_p2p else t.cpu(), dst=0)
        elif ctx.rank == 0:
            t = torch.empty((r1 - r0, width), dtype=torch.int64, device=ctx.dev if cuda_p2p else "cpu")
            dist.recv(t, src=r)
            h.update(t.cpu().numpy().tobytes())
    return h.hexdigest() if ctx.rank == 0 else None


def _pinned(rows, width):
    import numpy as np
    import torch
    t = torch.empty((rows, width), dtype=torch.int64, pin_memory=True)
    return t, t.numpy().view(np.uint64)


def e2e_single(ctx, w, params, a, b, c0_fill, want):
    """End to end at N = 1 through the public API from pinned host buffers.
    Returns (pipelined, serial). Serial: per product, upload A and B (and
    C0 for addmul), multiply, download C. Pipelined: HostPipeline (3
    streams, 2 buffer sets; copies of neighbouring products overlap
    compute), timed from the first upload to the last download."""
    import torch
    g = ctx.g
    from paper_0811_1714_b200.pipeline import HostPipeline
    m, l, n = w["m"], w["l"], w["n"]
    addmul = w["kind"] == "addmul"
    wa, wb = g.words_per_row(l), g.words_per_row(n)
    keep = []
    ta, hav = _pinned(m, wa)
    tb, hbv = _pinned(l, wb)
    keep += [ta, tb]
    hcv = []
    for _ in range(2):
        t, v = _pinned(m, wb)
        keep.append(t)
        hcv.append(v)
    a.to_numpy(out=hav)
    b.to_numpy(out=hbv)
    hc0v = None
    if addmul:
        t, hc0v = _pinned(m, wb)
        keep.append(t)
        c0_fill().to_numpy(out=hc0v)
    h2d = int(hav.nbytes + hbv.nbytes + (hc0v.nbytes if addmul else 0))
    d2h = int(hcv[0].nbytes)

    # (1) serial
    ad, bd = g.create(m, l, ctx.dev), g.create(l, n, ctx.dev)
    cd = g.create(m, n, ctx.dev) if addmul else None

    def e2e_step():
        g.from_numpy(hav, l, out=ad, nonblocking=True)
        g.from_numpy(hbv, n, out=bd, nonblocking=True)
        if addmul:
            g.from_numpy(hc0v, n, out=cd, nonblocking=True)
            g.addmul(cd, ad, bd, params)
            cc = cd
        else:
            cc = g.mul_strassen(ad, bd, params)
        g.core._download(cc, hcv[0], nonblocking=True)
        return cc

    for _ in range(max(1, ctx.args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    ee = []
    for _ in range(ctx.args.steps):
        ctx.flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        e2e_step()
        e1.record(ctx.stream)
        ee.append((e0, e1))
    torch.cuda.synchronize()
    ser_ms = sum(x.elapsed_time(y) for x, y in ee) / ctx.args.steps
    ok = (_sha(hcv[0]) == want) if want else None
    serial = {"value": m * l * n / (ser_ms * 1e-3), "unit": UNIT,
              "ms_per_step": ser_ms, "verified_sha256": ok,
              "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    del ad, bd, cd

    # (2) pipelined
    pipe = HostPipeline(m, l, n, params, ctx.dev)
    for i in range(max(2, ctx.args.warmup)):
        pipe.submit(hav, hbv, hcv[i % 2], c_in=hc0v)
    pipe.sync()
    torch.cuda.synchronize()
    s_h2d, _, s_d2h = pipe.streams
    steps = max(ctx.args.steps, 30)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s_h2d)
    for i in range(steps):
        pipe.submit(hav, hbv, hcv[i % 2], c_in=hc0v)
    e1.record(s_d2h)
    pipe.sync()
    torch.cuda.synchronize()
    pip_ms = e0.elapsed_time(e1) / steps
    ok = all(_sha(x) == want for x in hcv) if want else None
    piped = {"value": m * l * n / (pip_ms * 1e-3), "unit": UNIT,
             "ms_per_step": pip_ms, "verified_sha256": ok, "steps": steps,
             "mode": "HostPipeline: per step H2D of A and B"
                     + (" and C0" if addmul else "")
                     + " from pinned host memory, "
                     + ("addmul" if addmul else "Strassen multiply")
                     + ", D2H of C; copies of neighbouring steps overlap "
                       "compute (3 streams); timed from the first upload to "
                       "the last download",
             "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    del pipe, keep
    return piped, serial


def e2e_sharded(ctx, w, params, a, r0, r1, c0_fill, want_rank):
    """End to end at N ranks through the public API: every product, each
    rank uploads its row shard of A (and of C0 for addmul) and its block of
    B's rows (owned_rows) from pinned host memory over its own PCIe link,
    mul_sharded(src=None) broadcasts the blocks over NVLink while the panels
    multiply, and the rank downloads its C shard. Returns (pipelined,
    serial), max over ranks; bytes are whole-job totals."""
    import torch
    g = ctx.g
    from paper_0811_1714_b200.pipeline import ShardedHostPipeline
    from paper_0811_1714_b200.sharded import mul_sharded, owned_rows
    import numpy as np

    m, l, n = w["m"], w["l"], w["n"]
    addmul = w["kind"] == "addmul"
    wa, wb = g.words_per_row(l), g.words_per_row(n)
    mr = r1 - r0
    keep = []
    ta, hav = _pinned(mr, wa)
    tb, hbv = _pinned(l, wb)
    keep += [ta, tb]
    hcv = []
    for _ in range(2):
        t, v = _pinned(mr, wb)
        keep.append(t)
        hcv.append(v)
    a.to_numpy(out=hav)
    mine = owned_rows(l, ctx.world, ctx.rank, None)
    full_b = g.random(l, n, w["seed_b"], device=ctx.dev)
    for k0, k1 in mine:
        g.window(full_b, k0, 0, k1 - k0, n).to_numpy(out=hbv[k0:k1])
    del full_b
    hc0v = None
    if addmul:
        t, hc0v = _pinned(mr, wb)
        keep.append(t)
        c0_fill().to_numpy(out=hc0v)
    h2d_rank = hav.nbytes + sum((k1 - k0) * wb * 8 for k0, k1 in mine) + \
        (hc0v.nbytes if addmul else 0)
    common = {"unit": UNIT,
              "h2d_bytes_per_step": int(m * wa * 8 + l * wb * 8 + (m * wb * 8 if addmul else 0)),
              "d2h_bytes_per_step": int(m * wb * 8),
              "h2d_bytes_per_step_rank0": int(h2d_rank),
              "d2h_bytes_per_step_rank0": int(hcv[0].nbytes)}

    # (1) serial
    ad, bd = g.create(mr, l, ctx.dev), g.create(l, n, ctx.dev)
    cd = g.create(mr, n, ctx.dev)

    def e2e_step():
        g.from_numpy(hav, l, out=ad, nonblocking=True)
        for k0, k1 in mine:
            g.from_numpy(hbv[k0:k1], n, out=g.window(bd, k0, 0, k1 - k0, n),
                         nonblocking=True)
        if addmul:
            g.from_numpy(hc0v, n, out=cd, nonblocking=True)
        mul_sharded(ad, bd, params, src=None, npanels=ctx.args.npanels, c=cd,
                    accumulate=addmul)
        g.core._download(cd, hcv[0], nonblocking=True)

    for _ in range(max(1, ctx.args.warmup)):
        e2e_step()
    ctx.barrier()
    ee = []
    for _ in range(ctx.args.steps):
        ctx.flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        e2e_step()
        e1.record(ctx.stream)
        ee.append((e0, e1))
    torch.cuda.synchronize()
    ser_ms, ser_ok = ctx.max_over_ranks(
        sum(x.elapsed_time(y) for x, y in ee) / ctx.args.steps,
        bool(np.array_equal(hcv[0], want_rank)))
    serial = dict(common, value=m * l * n / (ser_ms * 1e-3), ms_per_step=ser_ms,
                  verified_vs_device_result=ser_ok)
    del ad, bd, cd

    # (2) pipelined
    pipe = ShardedHostPipeline(mr, l, n, params, ctx.dev, npanels=ctx.args.npanels)
    for i in range(max(2, ctx.args.warmup)):
        pipe.submit(hav, hbv, hcv[i % 2], c_in=hc0v)
    pipe.sync()
    ctx.barrier()
    s_h2d, _, s_d2h = pipe.streams
    steps = max(ctx.args.steps, 30)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s_h2d)
    for i in range(steps):
        pipe.submit(hav, hbv, hcv[i % 2], c_in=hc0v)
    e1.record(s_d2h)
    pipe.sync()
    torch.cuda.synchronize()
    pip_ms, pip_ok = ctx.max_over_ranks(
        e0.elapsed_time(e1) / steps,
        all(np.array_equal(x, want_rank) for x in hcv))
    piped = dict(common, value=m * l * n / (pip_ms * 1e-3), ms_per_step=pip_ms,
                 verified_vs_device_result=pip_ok, steps=steps,
                 mode="ShardedHostPipeline: per product each rank uploads its "
                      "A rows" + (" and C0 rows" if addmul else "") + " and its "
                      "block of B's rows from pinned host memory (its own PCIe "
                      "link), mul_sharded(src=None) broadcasts the blocks over "
                      "NCCL while panels multiply, each rank downloads its C "
                      "rows; copies of neighbouring products overlap compute; "
                      "first upload to last download, max over ranks")
    del pipe, keep
    return piped, serial


def e2e_grid(ctx, w, params, a, block, c0_fill, want_rank):
    """End to end on the process grid, one product at a time: rank (i, j)
    uploads 1/pc of A's rows_i (the rest arrives inside its row group,
    gather_rows), its share of column block B_j's rows (owned_rows over the
    pr ranks of column group j) and, for addmul, its block of C0, all from
    pinned host memory; mul_sharded_grid(src_row=None) broadcasts B_j's
    pieces inside the column group while the panels multiply; the rank
    downloads its block of C. Max over ranks; bytes are whole-job totals."""
    import numpy as np
    import torch
    g, grid = ctx.g, ctx.grid
    from paper_0811_1714_b200.sharded import gather_rows, mul_sharded_grid, owned_rows, shard_rows
    m, l, n = w["m"], w["l"], w["n"]
    r0, r1, c0, c1 = block
    mr, nc = r1 - r0, c1 - c0
    addmul = w["kind"] == "addmul"
    wa, wbj = g.words_per_row(l), g.words_per_row(nc)
    keep = []
    # A_i: this rank uploads piece j of its rows, 64-row aligned
    pieces = [shard_rows(mr, grid.pc, j) for j in range(grid.pc)]
    p0, p1 = pieces[grid.j]
    ta, hav = _pinned(p1 - p0, wa)
    keep.append(ta)
    g.window(a, p0, 0, p1 - p0, l).to_numpy(out=hav)
    # B_j: this rank's rows of the column block
    mine = owned_rows(l, grid.pr, grid.i, None)
    tb, hbv = _pinned(l, wbj)
    keep.append(tb)
    full_b = g.random(l, n, w["seed_b"], device=ctx.dev)
    for k0, k1 in mine:
        g.window(full_b, k0, c0, k1 - k0, nc).to_numpy(out=hbv[k0:k1])
    del full_b
    tc, hcv = _pinned(mr, wbj)
    keep.append(tc)
    hc0v = None
    if addmul:
        t, hc0v = _pinned(mr, wbj)
        keep.append(t)
        c0_fill().to_numpy(out=hc0v)
    ad, bd, cd = g.create(mr, l, ctx.dev), g.create(l, nc, ctx.dev), g.create(mr, nc, ctx.dev)
    roots = grid.row_ranks(grid.i)

    def e2e_step():
        if p1 > p0:
            g.from_numpy(hav, l, out=g.window(ad, p0, 0, p1 - p0, l), nonblocking=True)
        if grid.pc > 1:
            gather_rows(ad.storage, pieces, roots, group=grid.row_group)
        for k0, k1 in mine:
            g.from_numpy(hbv[k0:k1], nc, out=g.window(bd, k0, 0, k1 - k0, nc), nonblocking=True)
        if addmul:
            g.from_numpy(hc0v, nc, out=cd, nonblocking=True)
        mul_sharded_grid(ad, bd, grid, params, src_row=None, npanels=ctx.args.npanels, c=cd,
                         accumulate=addmul)
        g.core._download(cd, hcv, nonblocking=True)

    for _ in range(max(1, ctx.args.warmup)):
        e2e_step()
    ctx.barrier()
    ee = []
    for _ in range(ctx.args.steps):
        ctx.flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        e2e_step()
        e1.record(ctx.stream)
        ee.append((e0, e1))
    torch.cuda.synchronize()
    ms, ok = ctx.max_over_ranks(sum(x.elapsed_time(y) for x, y in ee) / ctx.args.steps,
                                bool(np.array_equal(hcv, want_rank)))
    del ad, bd, cd, keep
    return {"unit": UNIT, "value": m * l * n / (ms * 1e-3), "ms_per_step": ms,
            "verified_vs_device_result": ok,
            "h2d_bytes_per_step": int(m * wa * 8 + l * g.words_per_row(n) * 8
                                      + (m * g.words_per_row(n) * 8 if addmul else 0)),
            "d2h_bytes_per_step": int(m * g.words_per_row(n) * 8),
            "mode": f"process grid {grid.pr}x{grid.pc}, one product at a time: each rank uploads "
                    "1/pc of A's rows_i (gathered inside the row group), its rows of column "
                    "block B_j" + (", its block of C0" if addmul else "") + " from pinned host "
                    "memory, mul_sharded_grid(src_row=None) broadcasts B_j's pieces inside the "
                    "column group while panels multiply, and downloads its block of C; max over ranks"}


def roofline_for(ctx, kern_ms, kern_ops, kern_n, steps, total_ms):
    """Roofline of the dominant kernel (the batched leaf-product launch),
    achieved from its live CUDA-event time inside the timed region."""
    args = ctx.args
    if not kern_n:
        return None
    import torch
    peaks, src = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(ctx.dev).multi_processor_count
    if args.engine == "m4rm":
        smem_peak_gbs = 128.0 * nsm * sm_max * 1e6 / 1e9   # 128 B/clk/SM crossbar
        ach = kern_ops / 64.0 / (kern_ms * 1e-3) / 1e9      # W/(8k) B, k = 8
        roof = {"bound": "smem", "kernel": "k_m4rm (batched Strassen leaves)",
                "achieved": ach, "peak": smem_peak_gbs, "unit": "GB/s",
                "frac": ach / smem_peak_gbs, "traffic": None,
                "peak_source": f"128 B/clk/SM x {nsm} SMs x {sm_max:.0f} MHz "
                               f"(sm_max_mhz from {src}); HBM bound "
                               f"{peaks.get('hbm_gbs')} GB/s never binds here"}
    else:
        # 0/1 entries through tcgen05: 2 ops per MAC
        ach = 2.0 * kern_ops / (kern_ms * 1e-3) / 1e12
        f4 = args.engine == "tc-f4"
        nominal = 9000.0 if f4 else 4500.0
        roof = {"bound": "tensor",
                "kernel": ("k_umma_f4" if f4 else "k_umma") + " (batched Strassen leaves)",
                "achieved": ach, "unit": "TFLOP/s", "traffic": None}
        mp = _json_file("profiles", "measured_peaks_lowp.json")
        key = {"tc-f4": "mxf4_tflops", "tc-i8": "i8_tops", "tc-f8": "f8_tflops"}[args.engine]
        if mp and mp.get(key):
            roof.update(peak=float(mp[key]), frac=ach / float(mp[key]),
                        peak_source=f"measured: profiles/measured_peaks_lowp.json {key} "
                                    f"({mp.get('how', '')}); nominal dense {nominal:.0f} "
                                    "TFLOP/s (B200_PROFILING.md) -> frac_of_nominal",
                        frac_of_nominal=ach / nominal)
        else:
            roof.update(peak=nominal, frac=ach / nominal,
                        peak_source=("nominal dense fp4 9 PFLOP/s" if f4 else
                                     "nominal dense fp8/int8 4.5 PFLOP/s")
                                    + " (B200_PROFILING.md; no measured low-precision peak "
                                      "in profiles/measured_peaks_lowp.json)")
    roof.update({"kernel_ms_per_step": kern_ms / steps,
                 "kernel_share_of_step": kern_ms / total_ms if ctx.world == 1 else None,
                 "kernel_bitops_per_step": kern_ops / steps,
                 "kernel_launches_per_step": kern_n / steps})
    tr = _json_file("profiles", "ncu_traffic.json")
    if tr:
        key = {"m4rm": "k_m4rm", "tc-f4": "k_umma_f4"}.get(args.engine, "k_umma")
        ent = tr.get(key)
        if isinstance(ent, dict):
            roof["traffic"] = ent.get("bytes_per_launch")
            roof["traffic_source"] = ent.get("source")
        elif ent is not None:
            roof["traffic"] = ent
            roof["traffic_source"] = "profiles/ncu_traffic.json"
    return roof


def measure(ctx, w, primary: bool):
    """Time one workload: W untimed warm-up steps, then K steps bracketed by
    CUDA events on the launching stream (L2 flushed before each; for addmul
    C is refilled with C0 before each step, outside the events), max over
    ranks; verify the timed result's sha256 against the reference digest;
    then e2e and (rank 0, N = 1) the CPU baseline."""
    import torch
    g, args = ctx.g, ctx.args
    from paper_0811_1714_b200 import _lib
    from paper_0811_1714_b200.sharded import mul_sharded, mul_sharded_grid, shard_rows

    m, l, n = w["m"], w["l"], w["n"]
    addmul = w["kind"] == "addmul"
    params = g.default_params() if not args.cutoff else \
        g.MulParams(cutoff=args.cutoff, k=8)
    grid = ctx.grid
    if grid is not None:
        (r0, r1), (c0, c1) = grid.rows(m), grid.cols(n)
    else:
        r0, r1 = shard_rows(m, ctx.world, ctx.rank) if ctx.dist_on else (0, m)
        c0, c1 = 0, n
    a = g.random(r1 - r0, l, w["seed_a"], device=ctx.dev, row_base=r0)
    c_rows = None
    if grid is not None:
        # column block B_j: an owned l x n_j matrix, filled on grid row 0 (the
        # seeded generator indexes whole rows, so the block is cut from B)
        b = g.create(l, c1 - c0, device=ctx.dev)
        if grid.i == 0:
            g.copy_into(b, g.window(g.random(l, n, w["seed_b"], device=ctx.dev), 0, c0, l, c1 - c0))
        c = g.create(r1 - r0, c1 - c0, device=ctx.dev) if addmul else None
        c_rows = g.create(r1 - r0, n, device=ctx.dev) if addmul else None
    else:
        b = g.random(l, n, w["seed_b"], device=ctx.dev) if (ctx.world == 1 or ctx.rank == 0) \
            else g.create(l, n, device=ctx.dev)
        c = g.create(r1 - r0, n, device=ctx.dev) if addmul else None

    def reset():
        if addmul and grid is not None:
            g.random_into(c_rows, w["seed_c"], row_base=r0)
            g.copy_into(c, g.window(c_rows, 0, c0, r1 - r0, c1 - c0))
        elif addmul:
            g.random_into(c, w["seed_c"], row_base=r0)
        return c

    def step():
        if grid is not None:
            return mul_sharded_grid(a, b, grid, params, src_row=0, npanels=args.npanels,
                                    c=c if addmul else None, accumulate=True)
        if not ctx.dist_on:
            if addmul:
                g.addmul(c, a, b, params)
                return c
            return g.mul_strassen(a, b, params)
        if addmul:
            return mul_sharded(a, b, params, src=0, npanels=args.npanels, c=c,
                               accumulate=True)
        return mul_sharded(a, b, params, src=0, npanels=args.npanels)

    out = None
    for _ in range(args.warmup):
        reset()
        out = None                          # let the caching allocator reuse C
        out = step()
    ctx.barrier()

    clocks = ClockSampler(ctx.local)
    clocks.start()
    _lib.timer_enable(True)
    n_launch = 0
    evs = []
    for _ in range(args.steps):
        reset()
        ctx.flush.zero_()                   # evict L2 (126 MB) between steps
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        out = None
        l0 = g.launch_count()
        e0.record(ctx.stream)
        out = step()
        e1.record(ctx.stream)
        n_launch += g.launch_count() - l0
        evs.append((e0, e1))
    while not evs[-1][1].query():           # wait without holding the GIL, so the
        time.sleep(0.0002)                  # clock sampler thread keeps sampling
    torch.cuda.synchronize()
    kern_ms, kern_ops, kern_n = _lib.timer_read()
    _lib.timer_enable(False)
    ctx.barrier()
    clk = clocks.stop()
    total_ms, _ = ctx.max_over_ranks(sum(e0.elapsed_time(e1) for e0, e1 in evs))
    ms_step = total_ms / args.steps
    bitops = float(m) * l * n
    res = {"workload": w, "params": params, "value": bitops / (ms_step * 1e-3),
           "ms_per_step": ms_step, "total_ms": total_ms, "gpu_launches": n_launch,
           "clocks": clk, "kern": (kern_ms, kern_ops, kern_n)}

    verify = not args.no_verify and not args.size
    want = golden_digest(w["digest"]) if verify else None
    res["verified_sha256"] = None
    if verify:
        got = digest_rows(ctx, out, w)
        if ctx.rank == 0:
            res["verified_sha256"] = (got == want) if want else None

    res["e2e"] = res["e2e_serial"] = None
    if not args.no_e2e:
        if grid is not None:
            want_rank = out.to_numpy()
            out = None
            res["e2e"] = res["e2e_serial"] = e2e_grid(
                ctx, w, params, a, (r0, r1, c0, c1), reset, want_rank)
        elif ctx.dist_on:
            want_rank = out.to_numpy()
            out = None
            res["e2e"], res["e2e_serial"] = e2e_sharded(
                ctx, w, params, a, r0, r1, reset, want_rank)
        else:
            out = None
            res["e2e"], res["e2e_serial"] = e2e_single(
                ctx, w, params, a, b, reset, want if verify else None)
        if res["verified_sha256"] is not None:
            for k in ("e2e", "e2e_serial"):
                e = res[k]
                ok = e.get("verified_sha256", e.get("verified_vs_device_result"))
                res["verified_sha256"] = res["verified_sha256"] and bool(ok)
    del a, b, c, c_rows, out

    res["roofline"] = roofline_for(ctx, kern_ms, kern_ops, kern_n, args.steps, total_ms) \
        if ctx.rank == 0 else None
    res["cpu_baseline"] = None
    if not args.no_cpu_baseline and ctx.world == 1:
        # primary workload: >= 10 s of CPU work; extra workloads: ~3 s
        kw = {} if primary else {"target_s": 3.0, "min_total_s": 3.0}
        v, thr, rows, dt, reps = cpu_port_sample(w, **kw)
        res["cpu_baseline"] = {
            "value": v, "unit": UNIT, "cores": thr, "kind": "port",
            "sample": f"A[:{rows}] x B ({rows}x{l}x{n})"
                      + (" + C0[:rows]" if addmul else "")
                      + f", {reps} runs, mean {dt:.2f} s ({reps * dt:.1f} s "
                        "total), C port of gf2mat mul_strassen (default "
                        f"params) on {thr} host threads"}
        stock = stock_reference_sample(w, target_s=4.0 if primary else 2.0)
        if stock:
            res["cpu_baseline"]["stock_reference_1core"] = stock
    g.release_workspace()
    return res


def _line_part(ctx, res):
    """The per-workload keys of the JSON line."""
    w, params, args = res["workload"], res["params"], ctx.args
    m, l, n = w["m"], w["l"], w["n"]
    return {
        "value": res["value"], "unit": UNIT, "ms_per_step": res["ms_per_step"],
        "config": {"workload": f"{w['name']}: {w['call']}, A {m}x{l}, B {l}x{n}, "
                               f"Strassen-Winograd (cutoff {params.cutoff}) over "
                               f"the {args.engine} base case",
                   "m": m, "l": l, "n": n, "cutoff": params.cutoff,
                   "seeds": [w["seed_a"], w["seed_b"]] + ([w["seed_c"]] if "seed_c" in w else []),
                   "parallelism": "single" if not ctx.dist_on else
                   (f"grid{ctx.grid.pr}x{ctx.grid.pc} + NCCL broadcast of B's column blocks "
                    f"inside column groups ({args.npanels} panels)" if ctx.grid is not None else
                    f"rows{ctx.world} + NCCL broadcast of B ({args.npanels} panels)"),
                   "l2": "flushed between timed steps (512 MiB write)"
                         + ("; C refilled with C0 before each step, outside the "
                            "timed events" if w["kind"] == "addmul" else "")},
        "data": "synthetic: core.random splitmix64 Bernoulli(0.5) bits, seeds "
                + "/".join(str(s) for s in [w["seed_a"], w["seed_b"]]
                           + ([w["seed_c"]] if "seed_c" in w else [])),
        "verified_sha256": res["verified_sha256"],
        "digest_key": w["digest"],
        "gpu_launches": res["gpu_launches"],
        "gpu_launches_per_step": res["gpu_launches"] / args.steps,
        "clocks": res["clocks"],
        "roofline": res["roofline"],
        "cpu_baseline": res["cpu_baseline"],
        "e2e": res["e2e"],
        "e2e_serial": res["e2e_serial"],
    }


def run_b200(args):
    import torch
    import torch.distributed as dist
    import paper_0811_1714_b200 as g

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # GF2_BENCH_SHARE_GPU=1 (tests only): every rank on cuda:0 with gloo for
    # the collectives, to run the N > 1 code path on a one-GPU box; the
    # numbers it prints are not a measurement and the line says so
    share = bool(os.environ.get("GF2_BENCH_SHARE_GPU"))
    if share:
        local = 0
    ndev = torch.cuda.device_count()
    if local >= ndev:
        die(f"rank {rank}: LOCAL_RANK {local} but {ndev} CUDA device(s) visible")
    torch.cuda.set_device(local)
    dist_on = world > 1 or args.sharded
    if dist_on:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if dist.get_world_size() != args.gpus and not (args.sharded and world == 1):
            die(f"process group has {dist.get_world_size()} ranks, --gpus {args.gpus}")
    dev = torch.device("cuda", local)
    g.set_engine(args.engine)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    ctx = Ctx(args, g, dev, world, rank, local, dist_on, flush,
              torch.cuda.current_stream())

    w = dict(WORKLOADS[args.workload])
    if args.size:
        w.update(m=args.size, l=args.size, n=args.size)
    if dist_on and world > 1 and args.grid != "rows":
        from paper_0811_1714_b200.sharded import ProcessGrid, choose_grid
        if args.grid == "auto":
            pr, pc = choose_grid(world, w["m"], w["n"])
        else:
            try:
                pr, pc = (int(x) for x in args.grid.lower().split("x"))
            except ValueError:
                die(f"--grid {args.grid!r}: expected rows, auto or PRxPC")
        if pr * pc != world:
            die(f"--grid {pr}x{pc} does not cover {world} ranks")
        if pc > 1:                      # PR x 1 is the row-sharded layout
            ctx.grid = ProcessGrid(world, rank, pr, pc, make_groups=True)
    main_res = measure(ctx, w, primary=True)
    extra = {}
    if not args.size:
        for name in args.extra_list:
            extra[name] = measure(ctx, dict(WORKLOADS[name]), primary=False)

    if rank == 0:
        peaks, _ = measured_peaks()
        line = {"metric": METRIC, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u64",
                "engine": args.engine}
        line.update(_line_part(ctx, main_res))
        if share:
            line["share_gpu_test"] = "all ranks on cuda:0 over gloo: a code-path test, not a measurement"
        line["compute"] = {
            "tc-f4": "GF(2) words as u64 (XOR additions); leaf products as "
                     "e2m1 nibbles x e2m1 -> f32 (tcgen05 kind::mxf4, exact "
                     "integer sums), parity of the f32 sum",
            "tc-i8": "u64 words; leaf products as u8 x u8 -> s32 (kind::i8), parity",
            "tc-f8": "u64 words; leaf products as e4m3 x e4m3 -> f32 (kind::f8f6f4), parity",
            "m4rm": "u64 words throughout (XOR of 128-bit Gray-table rows)"}[args.engine]
        m, n = w["m"], w["n"]
        line["hbm_roofline_ms"] = 3.0 * m * g.words_per_row(n) * 8 / \
            (float(peaks.get("hbm_gbs", 6650)) * 1e9) * 1e3
        line["vs_paper_2008_cpu"] = main_res["value"] / PAPER_2008_CPU
        if extra:
            line["workloads"] = {k: _line_part(ctx, r) for k, r in extra.items()}
        emit(line)
    if dist_on:
        dist.destroy_process_group()


_STDOUT_FD = None


def _quiet_stdout():
    """Point fd 1 at stderr for the run (NCCL / torch print banners such as
    "NCCL version ..." to stdout) and keep the real stdout for the one JSON
    line the driver parses."""
    global _STDOUT_FD
    if _STDOUT_FD is None:
        sys.stdout.flush()
        _STDOUT_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line: dict) -> None:
    text = json.dumps(line) + "\n"
    if _STDOUT_FD is None:
        print(text, end="", flush=True)
    else:
        sys.stdout.flush()
        os.write(_STDOUT_FD, text.encode())


def main():
    args = parse()
    _quiet_stdout()
    in_torchrun = "WORLD_SIZE" in os.environ
    if args.impl == "reference" and not in_torchrun:
        run_reference(args)                 # CPU only: no ranks to launch
        return
    if not in_torchrun and args.gpus > 1:
        sys.exit(launch_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        die(f"WORLD_SIZE={world} but --gpus {args.gpus}: the ranks must "
            "match the GPU count the line reports")
    if args.impl == "stub":
        run_stub(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
