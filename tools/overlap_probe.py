"""Does the pre-GEMM phase (nibble expansions, B transpose) of one multiply
hide behind the leaf GEMM of another? N multiplies on one stream against the
same N alternating between two streams (the persistent GEMMs cannot share
SMs and serialize; everything else may overlap). No L2 flush in either arm.

  python tools/overlap_probe.py [size] [N]
"""
import sys
import torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g  # noqa: E402
from paper_0811_1714_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
try:    # a block freed on one stream must not make the other stream wait for it
    from cuda.bindings import runtime as rt
    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    attr = rt.cudaMemPoolAttr.cudaMemPoolReuseAllowInternalDependencies
    for val in (0, rt.cuuint64_t(0) if hasattr(rt, "cuuint64_t") else 0):
        try:
            err, = rt.cudaMemPoolSetAttribute(pool, attr, val)
            print("pool: ReuseAllowInternalDependencies=0 ->", err)
            break
        except Exception as exc:          # noqa: BLE001
            print("pool attr attempt failed:", exc)
except Exception as exc:                  # noqa: BLE001
    print("pool attribute not set:", exc)
a, b = g.random(n, n, 31), g.random(n, n, 32)
cs = [g.create(n, n) for _ in range(2)]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]


def run(two: bool):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
    for st in streams:
        st.wait_event(e0)
    for i in range(N):
        st = streams[i % 2 if two else 0]
        with torch.cuda.stream(st):
            g.zero_into(cs[i % 2])
            g.addmul(cs[i % 2], a, b)
    for st in streams:
        torch.cuda.current_stream().wait_stream(st)
    e1.record(torch.cuda.current_stream())
    e1.synchronize()
    return e0.elapsed_time(e1) / N


for two in (False, True):
    run(two)
ref = g.mul_strassen(a, b)
for rep in range(3):
    t1, t2 = run(False), run(True)
    ok = bool(g.equal(cs[0], ref)) and bool(g.equal(cs[1], ref))
    print(f"n={n}: one stream {t1:.4f} ms/multiply, two streams {t2:.4f} ms/multiply "
          f"({t2 / t1:.3f}x), results equal: {ok}", flush=True)
_lib.timer_enable(True)
run(True)
torch.cuda.synchronize()
ms, ops, cnt = _lib.timer_read()
print(f"two streams: GEMM launches {cnt}, mean {ms / max(cnt, 1):.4f} ms each")
_lib.timer_enable(True)
run(False)
torch.cuda.synchronize()
ms, ops, cnt = _lib.timer_read()
print(f"one stream: GEMM launches {cnt}, mean {ms / max(cnt, 1):.4f} ms each")
