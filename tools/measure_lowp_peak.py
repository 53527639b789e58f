"""Measured low-precision tensor-core peaks on this B200 (roofline
denominators for the tc-f4 / tc-i8 / tc-f8 engines; MEASURED_PEAKS.json has
bf16 only). Writes profiles/measured_peaks_lowp.json.

  * cuBLASLt through torch: MXFP4 (e2m1 x e2m1, UE8M0 block scales, f32 out)
    `torch._scaled_mm`, int8 `torch._int_mm`, fp8 e4m3 `torch._scaled_mm`,
    N^3 at N = 8192 and 16384; burst = best of 20 single calls (CUDA
    events), sustained = back to back for 3 s; 2 ops per MAC.
  * this repo's k_umma_f4 / k_umma (i8, f8) with the epilogue switched off
    (GF2_F4_DBG=2 / GF2_UMMA_DBG=2: operand TMA + MMAs only, timing-only
    knobs) on a direct 8192^3 and on the 7 batched 8192^3 leaves of cfg3,
    timed by the library's kernel timer -- the MMA rate the product kernels
    themselves can reach.

NVML SM clocks are sampled every 5 ms during each timed region.

    python tools/measure_lowp_peak.py [OUT.json]
"""
import json
import os
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "measured_peaks_lowp.json")

MMA_ONLY = r"""
import json, sys, torch
sys.path.insert(0, %(root)r)
import paper_0811_1714_b200 as g
from paper_0811_1714_b200 import _lib
torch.cuda.set_device(0)
g.set_engine(%(engine)r)
out = {}
for name, fn in (("direct_8192", None), ("cfg3_leaves", None)):
    if name == "direct_8192":
        a, b = g.random(8192, 8192, 1), g.random(8192, 8192, 2)
        run = lambda: g.mul_direct(a, b)
    else:
        a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
        run = lambda: g.mul_strassen(a, b)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    best = None
    for _ in range(10):
        _lib.timer_enable(True)
        run()
        ms, ops, n = _lib.timer_read()
        t = 2.0 * ops / (ms * 1e-3) / 1e12
        best = t if best is None or t > best else best
    _lib.timer_enable(False)
    out[name] = best
    del a, b
print(json.dumps(out))
"""


class Clocks:
    def __init__(self):
        self.samples = []
        self._stop = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
            self.nv = pynvml
        except Exception:
            self.nv = None

    def __enter__(self):
        self.samples = []
        self._stop = False
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def _run(self):
        while not self._stop:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            time.sleep(0.005)

    def __exit__(self, *a):
        self._stop = True
        if self.nv:
            self.t.join()

    def median(self):
        s = sorted(self.samples)
        return s[len(s) // 2] if s else None


def burst(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    best = None
    with Clocks() as ck:
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            e1.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None or t < best else best
    return best, ck.median()


def sustained(f, seconds=3.0):
    f()
    torch.cuda.synchronize()
    with Clocks() as ck:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        t0 = time.time()
        e0.record()
        while time.time() - t0 < seconds:
            for _ in range(10):
                f()
            n += 10
            torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
    return e0.elapsed_time(e1) / n, ck.median()


def to_blocked(s):
    r, c = s.shape  # cuBLAS 128x4 tile swizzle for block scales
    return s.view(r // 128, 4, 32, c // 4, 4).permute(0, 3, 2, 1, 4).reshape(-1)


def main():
    torch.cuda.set_device(0)
    res = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "torch": torch.__version__, "cublas": {}}
    one = torch.tensor(1.0, device="cuda")
    for N in (8192, 16384):
        flops = 2.0 * N ** 3
        bits_a = torch.randint(0, 2, (N, N), dtype=torch.uint8, device="cuda")
        bits_b = torch.randint(0, 2, (N, N), dtype=torch.uint8, device="cuda")

        def pack(bits):
            nib = bits * 2  # e2m1 1.0 = 0b0010
            return (nib[:, 0::2] | (nib[:, 1::2] << 4)).contiguous().view(torch.float4_e2m1fn_x2)

        pa, pb = pack(bits_a), pack(bits_b.t().contiguous())
        sa = to_blocked(torch.full((N, N // 32), 127, dtype=torch.uint8, device="cuda")).view(torch.float8_e8m0fnu)
        sb = to_blocked(torch.full((N, N // 32), 127, dtype=torch.uint8, device="cuda")).view(torch.float8_e8m0fnu)
        a8 = bits_a.to(torch.int8)
        b8 = bits_b.to(torch.int8).t().contiguous().t()
        af8 = bits_a.to(torch.float8_e4m3fn)
        bf8 = bits_b.t().contiguous().to(torch.float8_e4m3fn).t()
        try:  # torch >= 2.9 block-scaled API (MXFP4: 1x32 blocks, UE8M0 scales, 32_4_4 swizzle)
            from torch.nn.functional import ScalingType, SwizzleType, scaled_mm

            def mxf4():
                return scaled_mm(pa, pb.t(), sa, ScalingType.BlockWise1x32, sb, ScalingType.BlockWise1x32,
                                 swizzle_a=SwizzleType.SWIZZLE_32_4_4, swizzle_b=SwizzleType.SWIZZLE_32_4_4,
                                 output_dtype=torch.bfloat16)
        except ImportError:
            def mxf4():
                return torch._scaled_mm(pa, pb.t(), scale_a=sa, scale_b=sb, out_dtype=torch.bfloat16)
        cases = {
            "mxf4": mxf4,
            "i8": lambda: torch._int_mm(a8, b8),
            "f8": lambda: torch._scaled_mm(af8, bf8, scale_a=one, scale_b=one, out_dtype=torch.bfloat16),
        }
        for name, f in cases.items():
            try:
                ms, mhz = burst(f)
                ent = {"burst_ms": ms, "burst_tflops": flops / (ms * 1e-3) / 1e12, "burst_sm_mhz": mhz}
                if N == 8192:
                    sms, smhz = sustained(f)
                    ent.update(sustained_ms=sms, sustained_tflops=flops / (sms * 1e-3) / 1e12, sustained_sm_mhz=smhz)
                res["cublas"][f"{name}_{N}"] = ent
            except Exception as e:  # record, keep going
                res["cublas"][f"{name}_{N}"] = {"error": repr(e)[:300]}
            torch.cuda.empty_cache()
        del bits_a, bits_b, pa, pb, a8, b8, af8, bf8
        torch.cuda.empty_cache()
    for engine, key in (("tc-f4", "k_umma_f4_mma_only_tflops"), ("tc-i8", "k_umma_i8_mma_only_tops"),
                        ("tc-f8", "k_umma_f8_mma_only_tflops")):
        env = dict(os.environ, GF2_F4_DBG="2", GF2_UMMA_DBG="2")
        p = subprocess.run([sys.executable, "-c", MMA_ONLY % {"root": ROOT, "engine": engine}], env=env,
                           capture_output=True, text=True, timeout=600)
        try:
            res[key] = json.loads(p.stdout.strip().splitlines()[-1])
        except Exception:
            res[key.replace("tflops", "error").replace("tops", "error")] = (p.stdout + p.stderr)[-600:]

    def best(prefix):
        vals = [v.get("burst_tflops", 0) for k, v in res["cublas"].items() if k.startswith(prefix)]
        return max(vals) if vals else None

    f4 = [best("mxf4_")] + list(res.get("k_umma_f4_mma_only_tflops", {}).values())
    f4 = [x for x in f4 if x]
    res["mxf4_tflops"] = max(f4) if f4 else None
    res["i8_tops"] = max([best("i8_") or 0] + list(res.get("k_umma_i8_mma_only_tops", {}).values()))
    res["f8_tflops"] = max([best("f8_") or 0] + list(res.get("k_umma_f8_mma_only_tflops", {}).values()))
    res["how"] = ("max over cuBLASLt burst (best of 20, N^3 at N=8192/16384, 2 ops/MAC) and this library's "
                  "GEMMs with the epilogue off (GF2_F4_DBG=2 / GF2_UMMA_DBG=2: operand TMA + MMAs) timed by its "
                  "kernel timer, on a direct 8192^3 and on cfg3's 7 batched 8192^3 leaves")
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
