"""One mul_strassen of an n^3 product at a given cutoff (for ncu captures):
    python tools/strassen_once.py N CUTOFF [REPS]"""
import sys

import torch

sys.path.insert(0, '.')
import paper_0811_1714_b200 as g  # noqa: E402

n, cut = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
torch.cuda.set_device(0)
a, b = g.random(n, n, 21), g.random(n, n, 22)
p = g.MulParams(cutoff=cut, k=8)
for _ in range(reps):
    c = g.mul_strassen(a, b, p)
torch.cuda.synchronize()
print("ok", c.shape)
