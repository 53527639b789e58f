"""One 16384^3 mul_m4rm (k=8) for ncu capture of k_m4rm."""
import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
g.set_engine("m4rm")  # the M4RM kernel itself, not the tensor-core dispatch
a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
c = g.mul_m4rm(a, b, 8)
torch.cuda.synchronize()
print("done")
