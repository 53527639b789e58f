"""PCIe probe (design aid): pinned host<->device bandwidth for the bench's
per-step transfer sizes, raw torch copies vs the gf2_upload/download path."""
import sys, time, json, numpy as np, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
res = {}
def bw(fn, nbytes, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
n = 32 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device='cuda')
res["torch_h2d_32MiB_GBs"] = bw(lambda: d.copy_(h, non_blocking=True), n)
res["torch_d2h_32MiB_GBs"] = bw(lambda: h.copy_(d, non_blocking=True), n)
m = g.create(16384, 16384)
hw = torch.empty((16384, 256), dtype=torch.int64).pin_memory().numpy().view(np.uint64)
s = torch.cuda.current_stream().cuda_stream
lib = g._lib.lib_cuda()
res["gf2_upload_GBs"] = bw(lambda: g._lib.check(lib.gf2_upload(m._view(), hw.ctypes.data, 256, s)), n)
res["gf2_download_GBs"] = bw(lambda: g._lib.check(lib.gf2_download(m._view(), hw.ctypes.data, 256, s)), n)
# bidirectional: H2D on one stream while D2H on another
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n, dtype=torch.uint8, device='cuda')
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
res["bidir_total_GBs"] = bw(both, 2 * n)
print(json.dumps(res, indent=1))
