import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
a = g.random(65536, 65536, 5)
b = g.transpose(a); torch.cuda.synchronize()
b = g.transpose(a); torch.cuda.synchronize()
print("done")
