import torch, time, json
torch.cuda.set_device(0)
res = {}
def timeit(f, iters=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)/iters
N=16384
a8 = torch.randint(0, 2, (N, N), dtype=torch.int8, device='cuda')
b8 = torch.randint(0, 2, (N, N), dtype=torch.int8, device='cuda')
try:
    bt = b8.t().contiguous().t()
    ms = timeit(lambda: torch._int_mm(a8, bt))
    res['int8_int_mm_ms'] = ms; res['int8_TMACs'] = N**3/ms/1e9
    # exactness check small
    c = torch._int_mm(a8[:256], bt)
    ref = (a8[:256].float() @ b8.float())
    res['int8_exact'] = bool(torch.equal(c.float(), ref))
except Exception as e:
    res['int8_err'] = repr(e)[:200]
try:
    af = a8.to(torch.float8_e4m3fn); bf = b8.to(torch.float8_e4m3fn).t().contiguous().t()
    one = torch.tensor(1.0, device='cuda')
    f = lambda: torch._scaled_mm(af, bf, scale_a=one, scale_b=one, out_dtype=torch.float32)
    ms = timeit(f)
    res['fp8_ms'] = ms; res['fp8_TMACs'] = N**3/ms/1e9
    c = torch._scaled_mm(af, bf, scale_a=one, scale_b=one, out_dtype=torch.float32)
    ci = torch._int_mm(a8, b8.t().contiguous().t()) if 'int8_err' not in res else None
    if ci is not None: res['fp8_exact_vs_int8'] = bool(torch.equal(c, ci.float()))
    ones = torch.ones((128, N), device='cuda').to(torch.float8_e4m3fn)
    onesb = torch.ones((N, 128), device='cuda').to(torch.float8_e4m3fn).t().contiguous().t()
    c1 = torch._scaled_mm(ones, onesb, scale_a=one, scale_b=one, out_dtype=torch.float32)
    res['fp8_allones'] = float(c1[0,0]); res['fp8_allones_exact'] = bool((c1 == N).all())
except Exception as e:
    res['fp8_err'] = repr(e)[:300]
try:
    # bf16 for reference
    ab = a8.to(torch.bfloat16); bb = b8.to(torch.bfloat16)
    ms = timeit(lambda: ab @ bb)
    res['bf16_ms'] = ms; res['bf16_TMACs'] = N**3/ms/1e9
except Exception as e:
    res['bf16_err'] = repr(e)[:200]
try:
    # FP4 e2m1 block-scaled (mx) via _scaled_mm if supported
    fp4 = torch.float4_e2m1fn_x2
    # pack: value 1.0 in e2m1 = 0b0010 ; two per byte
    bits_a = torch.randint(0, 2, (N, N), dtype=torch.uint8, device='cuda')
    bits_b = torch.randint(0, 2, (N, N), dtype=torch.uint8, device='cuda')
    def pack(bits):
        nib = bits * 2
        return (nib[:, 0::2] | (nib[:, 1::2] << 4)).contiguous().view(fp4)
    pa = pack(bits_a); pbt = pack(bits_b.t().contiguous())  # (N, N/2) K-major
    sa = torch.full((N, N // 32), 127, dtype=torch.uint8, device='cuda').view(torch.float8_e8m0fnu)
    sb = torch.full((N, N // 32), 127, dtype=torch.uint8, device='cuda').view(torch.float8_e8m0fnu)
    f = lambda: torch._scaled_mm(pa, pbt.t(), scale_a=sa, scale_b=sb, out_dtype=torch.float32)
    c = f()
    ms = timeit(f)
    res['fp4_ms'] = ms; res['fp4_TMACs'] = N**3/ms/1e9
    ref = torch._int_mm(bits_a[:256].to(torch.int8), bits_b.to(torch.int8).t().contiguous().t())
    res['fp4_exact_256rows'] = bool(torch.equal(c[:256], ref.float()))
    res['fp4_maxdiff'] = float((c[:256] - ref.float()).abs().max())
except Exception as e:
    res['fp4_err'] = repr(e)[:400]
print(json.dumps(res, indent=1))
