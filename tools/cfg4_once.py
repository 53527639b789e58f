"""One cfg4 product (10000x7001 . 7001x12345, p = 0.1) for launch lists."""
import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
from oracle import gf2_oracle as O
torch.cuda.set_device(0)
t = O.bernoulli_threshold(0.1)
a = g.bernoulli(10000, 7001, 41, threshold=t)
b = g.bernoulli(7001, 12345, 42, threshold=t)
for _ in range(2):
    c = g.mul_strassen(a, b)
torch.cuda.synchronize()
print("done")
