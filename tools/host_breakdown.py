"""Host-side cost of one small call (design aid): median microseconds of each
piece of mul_m4rm(1024^3) / mul_strassen(4096^3, cutoff 1024) on the host,
with the GPU queue primed so no piece waits on the device."""
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_0811_1714_b200 as g  # noqa: E402
from paper_0811_1714_b200 import _lib  # noqa: E402
from paper_0811_1714_b200.core import BitMatrix, _stream  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
prime = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
a, b = g.random(1024, 1024, 11), g.random(1024, 1024, 12)
c = g.create(1024, 1024)
lib = _lib.lib_cuda()
va, vb, vc = a._view(), b._view(), c._view()
s = _stream()
a2, b2 = g.random(4096, 4096, 21), g.random(4096, 4096, 22)
p2 = g.MulParams(cutoff=1024, k=8)
c2 = g.create(4096, 4096)


def med(fn, reps=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    prime.zero_()                 # ~2.5 ms of queued GPU work
    ts = []
    for i in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        if i % 20 == 19:
            torch.cuda.synchronize()
            prime.zero_()
    torch.cuda.synchronize()
    ts.sort()
    return ts[len(ts) // 2] * 1e6


plan1 = g.M4rmPlan(c, a, b, 8)
rows = [
    ("torch.empty(1024x16 i64)", lambda: torch.empty((1024, 16), dtype=torch.int64, device=dev)),
    ("torch.zeros(1024x16 i64)", lambda: torch.zeros((1024, 16), dtype=torch.int64, device=dev)),
    ("torch.cuda.current_device()", lambda: torch.cuda.current_device()),
    ("BitMatrix(1024,1024,_overwritten)", lambda: BitMatrix(1024, 1024, None, _overwritten=True)),
    ("_stream()", _stream),
    ("a._view()", lambda: a._view()),
    ("lib.gf2_pitch_words", lambda: lib.gf2_pitch_words(1024)),
    ("lib.gf2_version (ctypes floor)", lambda: lib.gf2_version()),
    ("lib.gf2_m4rm(prebuilt views)", lambda: lib.gf2_m4rm(vc, va, vb, 8, 0, s)),
    ("lib.gf2_add (one ewise launch)", lambda: lib.gf2_add(vc, va, vb, s)),
    ("lib.gf2_m4rm accumulate (1 launch + maps)", lambda: lib.gf2_m4rm(vc, va, vb, 8, 1, s)),
    ("g.mul_m4rm(a,b,8)", lambda: g.mul_m4rm(a, b, 8)),
    ("M4rmPlan(c,a,b,8).run()", plan1.run),
    ("lib.gf2_strassen 4096 cutoff 1024", lambda: lib.gf2_strassen(c2._view(), a2._view(), b2._view(), 1024, 8, 0, s)),
    ("g.mul_strassen 4096 cutoff 1024", lambda: g.mul_strassen(a2, b2, p2)),
    ("g.mul_strassen 4096 default", lambda: g.mul_strassen(a2, b2)),
]
for name, fn in rows:
    print(f"{med(fn):8.1f} us  {name}", flush=True)
