"""One cfg5 addmul (65536^3, C += A.B) for launch-list profiling."""
import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
n = 65536
a, b, c = g.random(n, n, 51), g.random(n, n, 52), g.random(n, n, 53)
g.addmul(c, a, b)          # warm (workspace pool)
torch.cuda.synchronize()
g.addmul(c, a, b)
torch.cuda.synchronize()
print("done")
