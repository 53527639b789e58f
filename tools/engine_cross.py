"""Engine crossover (tuning aid): device time (queue primed, so host
latency is hidden) of Strassen multiplies and single products whose leaves
run on M4RM vs the tc-f4 engine. GF2_TC_MIN_WORK is set per run by the
caller (tools/gpu/cross.sh) -- this prints one line per case.

    GF2_TC_MIN_WORK=1e30 python tools/engine_cross.py   # all M4RM leaves
    GF2_TC_MIN_WORK=1 python tools/engine_cross.py      # all tensor leaves
"""
import json
import os
import sys

import torch

sys.path.insert(0, '.')
import paper_0811_1714_b200 as g  # noqa: E402

torch.cuda.set_device(0)
prime = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        prime.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return min(ts)


cases = [(1024, 0), (1536, 0), (2048, 0), (2560, 0), (3072, 0), (4096, 0),
         (4096, 1024), (4096, 2048), (8192, 1024), (8192, 2048), (8192, 4096), (3000, 512)]
for s, cut in cases:
    a, b = g.random(s, s, 1), g.random(s, s, 2)
    if cut:
        p = g.MulParams(cutoff=cut, k=8)
        us = t(lambda: g.mul_strassen(a, b, p))
    else:
        us = t(lambda: g.mul_strassen(a, b, g.MulParams(cutoff=1 << 20)))  # single product
    print(json.dumps({"min_work": os.environ.get("GF2_TC_MIN_WORK"), "n": s, "cutoff": cut, "us": round(us, 1)}),
          flush=True)
