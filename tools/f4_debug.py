"""Structured-input probe of a tensor engine (debug aid): identity and
single-entry operands reveal K/N mapping errors without raw accumulators."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
eng = sys.argv[1] if len(sys.argv) > 1 else "tc-f4"
g.set_engine(eng)
rng = np.random.default_rng(1)
M, L, N = 256, 256, 224
Bd = (rng.random((L, N)) < 0.5).astype(np.uint8)
Id = np.eye(M, L, dtype=np.uint8)
C = g.to_dense(g.mul_direct(g.from_dense(Id), g.from_dense(Bd)))
print("identity: C==B", np.array_equal(C, Bd), "frac rows equal", np.mean([np.array_equal(C[i], Bd[i]) for i in range(M)]))
# which B row does C row i equal?
match = []
for i in range(0, M, 1):
    hits = [k for k in range(L) if np.array_equal(C[i], Bd[k])]
    match.append(hits[0] if hits else -1)
print("row map (first 80):", match[:80])
print("zero rows:", int((C.sum(1) == 0).sum()), "C density", C.mean())
# A = ones everywhere, B = single one at (k, j): C column j all = 1, others 0
for k, j in [(0, 0), (1, 0), (2, 5), (63, 31), (64, 32), (200, 100)]:
    A1 = np.ones((M, L), dtype=np.uint8)
    B1 = np.zeros((L, N), dtype=np.uint8); B1[k, j] = 1
    C1 = g.to_dense(g.mul_direct(g.from_dense(A1), g.from_dense(B1)))
    cols = np.nonzero(C1.any(0))[0].tolist()
    rows = int(C1[:, j].sum())
    print(f"ones x e({k},{j}): nonzero cols {cols[:10]} rows-with-1 in col j {rows} total ones {int(C1.sum())}")
# A = e(i,k) (single one), B = ones: C row i all ones
for i, k in [(0, 0), (0, 1), (5, 7), (130, 64), (255, 255)]:
    A2 = np.zeros((M, L), dtype=np.uint8); A2[i, k] = 1
    B2 = np.ones((L, N), dtype=np.uint8)
    C2 = g.to_dense(g.mul_direct(g.from_dense(A2), g.from_dense(B2)))
    print(f"e({i},{k}) x ones: nonzero rows {np.nonzero(C2.any(1))[0].tolist()[:10]} ones {int(C2.sum())} (want {N})")
