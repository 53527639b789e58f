"""Timing probe (design aid): direct tc-f4 product throughput vs the maximum
column-tile width (GF2_F4_BN, read once per process) -- is the MMA cost
linear in N? Run once per width."""
import os, sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
g.set_engine("tc-f4")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a, b = g.random(n, n, 1), g.random(n, n, 2)
g._lib.timer_enable(True)
for _ in range(3): g.mul_direct(a, b)
torch.cuda.synchronize()
g._lib.timer_read()
for _ in range(10): g.mul_direct(a, b)
ms, ops, nl = g._lib.timer_read()
print(f"BN={os.environ.get('GF2_F4_BN','224')} n={n} kernel ms={ms/nl:.3f} TFLOP/s={2*ops/(ms*1e-3)/1e12:.0f}")
