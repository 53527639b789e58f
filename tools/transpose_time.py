"""Time the bit-matrix transpose kernels: k_transpose (16384^2, 65536^2) and
the transposing level-0 pre-addition k_combine_t inside a 65536^3 addmul,
with achieved HBM rate (read + write of the packed words)."""
import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


for n in (4096, 16384, 65536):
    a = g.random(n, n, 5)
    t = timed(lambda: g.transpose(a))
    ok = bool(g.equal(g.transpose(g.transpose(a)), a))
    byts = 2 * n * n / 8
    print(f"transpose {n}^2: {t * 1e3:.1f} us, {byts / t / 1e9:.2f} TB/s, involution ok: {ok}", flush=True)
m, n = 10000, 12345
a = g.random(m, n, 6)
t = timed(lambda: g.transpose(a))
print(f"transpose {m}x{n}: {t * 1e3:.1f} us", flush=True)
