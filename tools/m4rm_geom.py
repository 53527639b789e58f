"""M4RM geometry probe (tuning aid): one mul_m4rm of the given shape with
GF2_M4RM_GEOM="rpt,nsplit" forced, checked against the C port, timed with
CUDA events (L2 flushed). Run each geometry in its own process.

    GF2_M4RM_GEOM=2,8 python tools/m4rm_geom.py M L N [--window]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_0811_1714_b200 as g  # noqa: E402
from oracle import gf2_port as P  # noqa: E402
from oracle import gf2_oracle as O  # noqa: E402

m, l, n = (int(x) for x in sys.argv[1:4])
torch.cuda.set_device(0)
g.set_engine("m4rm")  # the M4RM kernel itself, whatever the size
a, b = g.random(m, l, 1), g.random(l, n, 2)
c = g.mul_m4rm(a, b, 8)
torch.cuda.synchronize()
P.set_threads(P.max_threads())
want = P.mul_strassen(P.random(m, l, 1), P.random(l, n, 2))
ok = bool((c.to_numpy() == want.words).all())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.mul_m4rm(a, b, 8)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(json.dumps({"geom": os.environ.get("GF2_M4RM_GEOM", "model"), "m": m, "l": l, "n": n,
                  "exact": ok, "us_min": round(min(ts), 2), "us_med": round(sorted(ts)[5], 2)}))
