#!/usr/bin/env python
"""Benchmark of the B200 GF(2) multiply (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One JSON line on rank 0. Workload (BASELINE.json configs[2], the shape the
metric is quoted on): C = A.B over GF(2), A and B 16384 x 16384 seeded
splitmix64 bits (core.random seeds 31 / 32), Strassen-Winograd with the
device default cutoff over the default base-case engine (tcgen05
kind::mxf4; `--engine` selects another). N = 1: one GPU multiplies. N > 1
(torchrun): C and A row-sharded, B broadcast from rank 0 over NVLink (NCCL)
in K-panels inside the timed step.

`--impl reference` times the reference algorithm's CPU port
(oracle/libgf2oracle.so, a C restatement of gf2mat's M4RM + Strassen-
Winograd, all host threads) on a bounded row sample of the same workload.
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
WORKLOAD = dict(name="cfg3", m=16384, l=16384, n=16384, seed_a=31, seed_b=32)
PAPER_2008_CPU = 16384 ** 3 / 6.074   # PAPER.md:753 (M4RI, Core 2 Duo)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--cutoff", type=int, default=0,
                   help="Strassen cutoff (0 = device default)")
    p.add_argument("--npanels", type=int, default=2)
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
    return p.parse_args()


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


def golden_digest(key: str):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "digests.json")) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


# ------------------------------------------------------------------ CPU port
def cpu_port_sample(m, l, n, seed_a, seed_b, target_s=8.0, rows=None,
                    min_total_s=10.0):
    """Time the reference algorithm's C port on a row sample A[:R] . B with
    all host threads. Returns (bitops_per_s, threads, rows, mean_s, reps)."""
    from oracle import gf2_port as P
    threads = len(os.sched_getaffinity(0))
    P.set_threads(threads)
    b = P.random(l, n, seed_b)
    if rows is None:
        rows = min(m, 256)
        while True:
            a = P.random(rows, l, seed_a)
            t0 = time.perf_counter()
            P.mul_strassen(a, b)
            dt = time.perf_counter() - t0
            if dt * 2 > target_s or rows >= m:
                break
            rows = min(m, rows * 2)
    a = P.random(rows, l, seed_a)
    # repeat the sample until at least min_total_s of CPU work is timed and
    # report the mean (one full 16384^3 product is ~2 s on 16 threads)
    reps, total = 0, 0.0
    while reps == 0 or total < min_total_s:
        t0 = time.perf_counter()
        P.mul_strassen(a, b)
        total += time.perf_counter() - t0
        reps += 1
    dt = total / reps
    ops = rows * l * n
    return ops / dt, threads, rows, dt, reps


def run_reference(args):
    """--impl reference: the reference algorithm on the host CPU (port)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = dict(WORKLOAD)
    if args.size:
        w.update(m=args.size, l=args.size, n=args.size)
    m, l, n = w["m"], w["l"], w["n"]
    # size the sample so that warmup + steps finish in a few minutes
    _, threads, rows, dt, _ = cpu_port_sample(m, l, n, w["seed_a"], w["seed_b"],
                                              target_s=6.0, min_total_s=0.0)
    times = []
    from oracle import gf2_port as P
    b = P.random(l, n, w["seed_b"])
    a = P.random(rows, l, w["seed_a"])
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        P.mul_strassen(a, b)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    per = sum(times) / len(times)
    value = rows * l * n / per
    sample = (f"A[:{rows}] x B ({rows}x{l}x{n}) per step, C port of "
              f"mul_strassen default params (cutoff 2048, k auto, t 8)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3 * (m / rows), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: core.random splitmix64 bits, seeds 31/32",
        "config": {"workload": f"{w['name']}: {m}x{l}x{n} GF(2) multiply",
                   "m": m, "l": l, "n": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "ms_per_step extrapolated to the full m rows",
    }
    emit(line)


# ------------------------------------------------------------------ GPU arm
def _free_port() -> int:
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def e2e_sharded(args, g, dev, stream, flush, a, r0, r1, w, params, world,
                rank, c_dev):
    """End to end at N ranks through the public API: every product, each
    rank uploads its row shard of A and its block of B's rows (owned_rows)
    from pinned host memory over its own PCIe link, mul_sharded(src=None)
    broadcasts the blocks over NVLink while the panels multiply, and the
    rank downloads its C shard. Returns (pipelined, serial): the pipelined
    figure runs ShardedHostPipeline (copies of neighbouring products overlap
    compute, as HostPipeline at N = 1), timed from the first upload to the
    last download; both max over ranks; bytes are whole-job totals."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_0811_1714_b200.pipeline import ShardedHostPipeline
    from paper_0811_1714_b200.sharded import mul_sharded, owned_rows

    m, l, n = w["m"], w["l"], w["n"]
    wa, wb = g.words_per_row(l), g.words_per_row(n)
    mr = r1 - r0
    ha = torch.empty((mr, wa), dtype=torch.int64, pin_memory=True)
    hb = torch.empty((l, wb), dtype=torch.int64, pin_memory=True)
    hcs = [torch.empty((mr, wb), dtype=torch.int64, pin_memory=True)
           for _ in range(2)]
    hav, hbv = ha.numpy().view(np.uint64), hb.numpy().view(np.uint64)
    hcv = [x.numpy().view(np.uint64) for x in hcs]
    a.to_numpy(out=hav)
    mine = owned_rows(l, world, rank, None)
    full_b = g.random(l, n, w["seed_b"], device=dev)
    for k0, k1 in mine:
        g.window(full_b, k0, 0, k1 - k0, n).to_numpy(out=hbv[k0:k1])
    del full_b
    want = c_dev.to_numpy()                   # this rank's digest-checked C
    bitops = float(m) * l * n
    h2d_rank = hav.nbytes + sum((k1 - k0) * wb * 8 for k0, k1 in mine)
    common = {"unit": UNIT, "h2d_bytes_per_step": int(m * wa * 8 + l * wb * 8),
              "d2h_bytes_per_step": int(m * wb * 8),
              "h2d_bytes_per_step_rank0": int(h2d_rank),
              "d2h_bytes_per_step_rank0": int(hcv[0].nbytes)}

    def max_over_ranks(ms, ok):
        t = torch.tensor([ms, 0.0 if ok else 1.0], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0].item()), not bool(t[1].item())

    # (1) serial: upload, multiply, download, one product at a time
    ad, bd = g.create(mr, l, dev), g.create(l, n, dev)

    def e2e_step():
        g.from_numpy(hav, l, out=ad, nonblocking=True)
        for k0, k1 in mine:
            g.from_numpy(hbv[k0:k1], n, out=g.window(bd, k0, 0, k1 - k0, n),
                         nonblocking=True)
        cc = mul_sharded(ad, bd, params, src=None, npanels=args.npanels)
        g.core._download(cc, hcv[0], nonblocking=True)
        return cc

    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    ee = []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        ee.append((e0, e1))
    torch.cuda.synchronize()
    ser_ms, ser_ok = max_over_ranks(
        sum(x.elapsed_time(y) for x, y in ee) / args.steps,
        bool(np.array_equal(hcv[0], want)))
    serial = dict(common, value=bitops / (ser_ms * 1e-3), ms_per_step=ser_ms,
                  verified_vs_device_result=ser_ok)
    del ad, bd

    # (2) pipelined
    pipe = ShardedHostPipeline(mr, l, n, params, dev, npanels=args.npanels)
    for i in range(max(2, args.warmup)):
        pipe.submit(hav, hbv, hcv[i % 2])
    pipe.sync()
    torch.cuda.synchronize()
    dist.barrier()
    h2d, _, d2h = pipe.streams
    steps = max(args.steps, 30)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(h2d)
    for i in range(steps):
        pipe.submit(hav, hbv, hcv[i % 2])
    e1.record(d2h)
    pipe.sync()
    torch.cuda.synchronize()
    pip_ms, pip_ok = max_over_ranks(
        e0.elapsed_time(e1) / steps,
        all(np.array_equal(x, want) for x in hcv))
    piped = dict(common, value=bitops / (pip_ms * 1e-3), ms_per_step=pip_ms,
                 verified_vs_device_result=pip_ok, steps=steps,
                 mode="ShardedHostPipeline: per product each rank uploads its "
                      "A rows and its block of B's rows from pinned host "
                      "memory (its own PCIe link), mul_sharded(src=None) "
                      "broadcasts the blocks over NCCL while panels multiply, "
                      "each rank downloads its C rows; copies of neighbouring "
                      "products overlap compute; first upload to last "
                      "download, max over ranks")
    return piped, serial


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
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import paper_0811_1714_b200 as g
    from paper_0811_1714_b200 import _lib
    from paper_0811_1714_b200.sharded import mul_sharded, shard_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist_on = world > 1 or args.sharded
    if dist_on:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    g.set_engine(args.engine)
    w = dict(WORKLOAD)
    if args.size:
        w.update(m=args.size, l=args.size, n=args.size)
    m, l, n = w["m"], w["l"], w["n"]
    params = g.default_params() if not args.cutoff else \
        g.MulParams(cutoff=args.cutoff, k=8)
    r0, r1 = shard_rows(m, world, rank) if dist_on else (0, m)
    a = g.random(r1 - r0, l, w["seed_a"], device=dev, row_base=r0)
    b = g.random(l, n, w["seed_b"], device=dev) if (world == 1 or rank == 0) \
        else g.create(l, n, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step():
        if not dist_on:
            return g.mul_strassen(a, b, params)
        return mul_sharded(a, b, params, src=0, npanels=args.npanels)

    stream = torch.cuda.current_stream()
    c = None
    for _ in range(args.warmup):
        c = None                           # let the caching allocator reuse C
        c = step()
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    _lib.timer_enable(True)
    n_launch0 = g.launch_count()
    evs = []
    for _ in range(args.steps):
        flush.zero_()                      # evict L2 (126 MB) between steps
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        c = None
        e0.record(stream)
        c = step()
        e1.record(stream)
        evs.append((e0, e1))
    while not evs[-1][1].query():          # wait without holding the GIL, so the
        time.sleep(0.0002)                 # clock sampler thread keeps sampling
    torch.cuda.synchronize()
    n_launch = g.launch_count() - n_launch0
    kern_ms, kern_ops, kern_n = _lib.timer_read()
    _lib.timer_enable(False)
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    if dist_on:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    bitops = float(m) * l * n
    value = bitops / (ms_step * 1e-3)

    # ---- verification of the timed result (sha256 of the raw words)
    verified = None
    if not args.no_verify and not args.size:
        words = c.to_numpy()
        if dist_on:
            parts = [None] * world
            dist.all_gather_object(parts, words)
            words = None
            if rank == 0:
                import numpy as np
                words = np.concatenate(parts, axis=0)
        if rank == 0:
            want = golden_digest(w["name"])
            got = hashlib.sha256(words.astype("<u8").tobytes()).hexdigest()
            verified = (got == want) if want else None

    # ---- end to end through the public API with pinned host buffers
    e2e = e2e_serial = None
    if not args.no_e2e and dist_on:
        e2e, e2e_serial = e2e_sharded(args, g, dev, stream, flush, a, r0, r1,
                                      w, params, world, rank, c)
    if not args.no_e2e and not dist_on:
        import numpy as np
        from paper_0811_1714_b200.pipeline import HostPipeline
        wa, wb = g.words_per_row(l), g.words_per_row(n)
        ha = torch.empty((m, wa), dtype=torch.int64, pin_memory=True)
        hb = torch.empty((l, wb), dtype=torch.int64, pin_memory=True)
        hcs = [torch.empty((m, wb), dtype=torch.int64, pin_memory=True)
               for _ in range(2)]
        hav, hbv = ha.numpy().view(np.uint64), hb.numpy().view(np.uint64)
        hcv = [x.numpy().view(np.uint64) for x in hcs]
        a.to_numpy(out=hav)
        b.to_numpy(out=hbv)
        want = golden_digest(w["name"]) if not args.size else None

        # (1) serial: upload, multiply, download, one product at a time
        ad, bd = g.create(m, l, dev), g.create(l, n, dev)

        def e2e_step():
            g.from_numpy(hav, l, out=ad, nonblocking=True)
            g.from_numpy(hbv, n, out=bd, nonblocking=True)
            cc = g.mul_strassen(ad, bd, params)
            g.core._download(cc, hcv[0], nonblocking=True)
            return cc

        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize()
        ee = []
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            ee.append((e0, e1))
        torch.cuda.synchronize()
        ser_ms = sum(x.elapsed_time(y) for x, y in ee) / args.steps
        ok = hashlib.sha256(hcv[0].astype("<u8").tobytes()).hexdigest() == want
        e2e_serial = {"value": bitops / (ser_ms * 1e-3), "unit": UNIT,
                      "ms_per_step": ser_ms, "verified_sha256": ok if want else None,
                      "h2d_bytes_per_step": int(hav.nbytes + hbv.nbytes),
                      "d2h_bytes_per_step": int(hcv[0].nbytes)}
        del ad, bd

        # (2) pipelined: HostPipeline overlaps step i+1's uploads and step
        # i-1's download with step i's compute (3 streams, 2 buffer sets)
        pipe = HostPipeline(m, l, n, params, dev)
        for i in range(max(2, args.warmup)):
            pipe.submit(hav, hbv, hcv[i % 2])
        pipe.sync()
        torch.cuda.synchronize()
        h2d, _, d2h = pipe.streams
        # whole-job time from the first upload to the last download; at least
        # 30 products so one pipeline fill/drain does not dominate the average
        pipe_steps = max(args.steps, 30)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(h2d)
        for i in range(pipe_steps):
            pipe.submit(hav, hbv, hcv[i % 2])
        e1.record(d2h)
        pipe.sync()
        torch.cuda.synchronize()
        pip_ms = e0.elapsed_time(e1) / pipe_steps
        ok = all(hashlib.sha256(x.astype("<u8").tobytes()).hexdigest() == want
                 for x in hcv)
        e2e = {"value": bitops / (pip_ms * 1e-3), "unit": UNIT,
               "ms_per_step": pip_ms, "verified_sha256": ok if want else None,
               "steps": pipe_steps,
               "mode": "HostPipeline: per step H2D of A and B from pinned host "
                       "memory, Strassen multiply, D2H of C; copies of "
                       "neighbouring steps overlap compute (3 streams); timed "
                       "from the first upload to the last download",
               "h2d_bytes_per_step": int(hav.nbytes + hbv.nbytes),
               "d2h_bytes_per_step": int(hcv[0].nbytes)}
        if verified is not None and want:
            verified = verified and bool(e2e["verified_sha256"]) and \
                bool(e2e_serial["verified_sha256"])

    if rank != 0:
        if dist_on:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (batched leaf M4RM launch)
    peaks, src = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    props = torch.cuda.get_device_properties(dev)
    nsm = props.multi_processor_count
    smem_peak_gbs = 128.0 * nsm * sm_max * 1e6 / 1e9   # 128 B/clk/SM crossbar
    roofline = None
    if kern_n and args.engine == "m4rm":
        lut_bytes = kern_ops / 64.0      # W/(8k) bytes, k = 8
        ach = lut_bytes / (kern_ms * 1e-3) / 1e9
        roofline = {
            "bound": "smem", "kernel": "k_m4rm (batched Strassen leaves)",
            "achieved": ach, "peak": smem_peak_gbs, "unit": "GB/s",
            "frac": ach / smem_peak_gbs, "traffic": None,
            "peak_source": f"128 B/clk/SM x {nsm} SMs x {sm_max:.0f} MHz "
                           f"(sm_max_mhz from {src}); HBM bound "
                           f"{peaks.get('hbm_gbs')} GB/s never binds here",
        }
    elif kern_n:
        # 0/1 entries through tcgen05 (kind::i8 / kind::f8f6f4 bytes, or
        # kind::mxf4 e2m1 nibbles): 2 ops per MAC, against the dense nominal
        # peak of that operand width (B200_PROFILING.md; no measured 8/4-bit peak)
        ach = 2.0 * kern_ops / (kern_ms * 1e-3) / 1e12
        f4 = args.engine == "tc-f4"
        peak = 9000.0 if f4 else 4500.0
        roofline = {
            "bound": "tensor",
            "kernel": ("k_umma_f4" if f4 else "k_umma") + " (batched Strassen leaves)",
            "achieved": ach, "peak": peak, "unit": "TFLOP/s",
            "frac": ach / peak, "traffic": None,
            "peak_source": ("nominal dense fp4 9 PFLOP/s" if f4 else "nominal dense fp8/int8 4.5 PFLOP/s")
                           + " (B200_PROFILING.md table; frac is 'of nominal': MEASURED_PEAKS has no "
                           "4/8-bit figure). For scale, MEASURED_PEAKS bf16 burst x "
                           + ("4" if f4 else "2") + " (operand-width rate ratio) = "
                           f"{(4 if f4 else 2) * float(peaks.get('bf16_tflops', 0)):.0f} TFLOP/s; "
                           "the higher nominal denominator is the conservative one",
        }
    if roofline is not None:
        roofline.update({
            "kernel_ms_per_step": kern_ms / args.steps,
            "kernel_share_of_step": kern_ms / total_ms if world == 1 else None,
            "kernel_bitops_per_step": kern_ops / args.steps,
        })
        tr = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tr):
            try:
                key = {"m4rm": "k_m4rm", "tc-f4": "k_umma_f4"}.get(args.engine, "k_umma")
                roofline["traffic"] = json.load(open(tr)).get(key)
            except Exception:
                pass
    hbm_bytes = 3.0 * m * g.words_per_row(n) * 8
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        v, thr, rows, dt, reps = cpu_port_sample(m, l, n, w["seed_a"], w["seed_b"])
        cpu = {"value": v, "unit": UNIT, "cores": thr, "kind": "port",
               "sample": f"A[:{rows}] x B ({rows}x{l}x{n}), {reps} runs, mean "
                         f"{dt:.2f} s ({reps * dt:.1f} s total), C port "
                         "of gf2mat mul_strassen (default params) on "
                         f"{thr} host threads"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic: core.random splitmix64 "
                                f"Bernoulli(0.5) bits, seeds {w['seed_a']}/"
                                f"{w['seed_b']}",
        "compute": {"tc-f4": "GF(2) words as u64 (XOR additions); leaf products as "
                             "e2m1 nibbles x e2m1 -> f32 (tcgen05 kind::mxf4, exact "
                             "integer sums), parity of the f32 sum",
                    "tc-i8": "u64 words; leaf products as u8 x u8 -> s32 (kind::i8), parity",
                    "tc-f8": "u64 words; leaf products as e4m3 x e4m3 -> f32 (kind::f8f6f4), parity",
                    "m4rm": "u64 words throughout (XOR of 128-bit Gray-table rows)"}[args.engine],
        "config": {"workload": f"{w['name']}: A,B {m}x{l} . {l}x{n} GF(2), "
                               f"Strassen-Winograd (cutoff {params.cutoff}) "
                               f"over the {args.engine} base case",
                   "m": m, "l": l, "n": n, "cutoff": params.cutoff,
                   "parallelism": "single" if not dist_on else
                   f"rows{world} + NCCL broadcast of B ({args.npanels} panels)",
                   "l2": "flushed between timed steps (512 MiB write)"},
        "verified_sha256": verified,
        "engine": args.engine,
        "gpu_launches": n_launch,
        "gpu_launches_per_step": n_launch / args.steps,
        "clocks": clk,
        "roofline": roofline,
        "hbm_roofline_ms": hbm_bytes / (float(peaks.get("hbm_gbs", 6650)) * 1e9)
        * 1e3,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_serial": e2e_serial,
        "vs_paper_2008_cpu": value / PAPER_2008_CPU,
    }
    emit(line)
    if dist_on:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
