"""Probe: tensor-core formats for 0/1 GF(2) contraction on B200 (cuBLASLt via torch).
Records rate and exactness (fp32 accumulation of integer sums) -- design input
for the tcgen05 path; not part of the product."""
import json, torch, traceback
torch.cuda.set_device(0)
res = {}
def timeit(f, iters=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters
one = torch.tensor(1.0, device='cuda')
# adversarial fp8 exactness: row of ones vs columns with popcount K-1 (odd), K up to 16384
for K in (4096, 8192, 16384, 32768):
    a = torch.ones((128, K), device='cuda').to(torch.float8_e4m3fn)
    bcols = torch.ones((K, 128), device='cuda')
    bcols[0, ::2] = 0   # even columns: popcount K-1
    b = bcols.to(torch.float8_e4m3fn).t().contiguous().t()
    c = torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.float32)
    want = bcols.sum(0)
    res[f"fp8_adversarial_K{K}"] = bool(torch.equal(c[0], want))
try:
    import inspect
    from torch.nn.functional import ScalingType, SwizzleType
    res['scaled_mm_api'] = str(inspect.signature(torch.nn.functional.scaled_mm))[:300]
    res['ScalingType'] = [x.name for x in ScalingType]
    res['SwizzleType'] = [x.name for x in SwizzleType]
except Exception as e:
    res['api_err'] = repr(e)[:200]
N = 8192
bits_a = torch.randint(0, 2, (N, N), dtype=torch.uint8, device='cuda')
bits_b = torch.randint(0, 2, (N, N), dtype=torch.uint8, device='cuda')
def pack(bits):
    nib = bits * 2   # e2m1 1.0 = 0b0010
    return (nib[:, 0::2] | (nib[:, 1::2] << 4)).contiguous().view(torch.float4_e2m1fn_x2)
pa = pack(bits_a); pb = pack(bits_b.t().contiguous())
def to_blocked(s):
    # cuBLAS 128x4 tile swizzle for block scales (rows multiple of 128, cols multiple of 4)
    r, c = s.shape
    return s.view(r // 128, 4, 32, c // 4, 4).permute(0, 3, 2, 1, 4).reshape(-1)
sa = torch.full((N, N // 32), 127, dtype=torch.uint8, device='cuda')
sb = torch.full((N, N // 32), 127, dtype=torch.uint8, device='cuda')
ref = torch._int_mm(bits_a.to(torch.int8), bits_b.to(torch.int8).t().contiguous().t()).float()
for name, f in [
    ("fp4_mx_blocked", lambda: torch._scaled_mm(pa, pb.t(), scale_a=to_blocked(sa).view(torch.float8_e8m0fnu),
                                                 scale_b=to_blocked(sb).view(torch.float8_e8m0fnu), out_dtype=torch.float32)),
    ("fp4_mx_plain", lambda: torch._scaled_mm(pa, pb.t(), scale_a=sa.view(torch.float8_e8m0fnu),
                                               scale_b=sb.view(torch.float8_e8m0fnu), out_dtype=torch.float32)),
]:
    try:
        c = f()
        res[name + "_exact"] = bool(torch.equal(c, ref))
        res[name + "_maxdiff"] = float((c - ref).abs().max())
        ms = timeit(f)
        res[name + "_TMACs"] = N ** 3 / ms / 1e9
    except Exception as e:
        res[name + "_err"] = "".join(traceback.format_exception_only(e))[-600:]
try:
    from torch.nn.functional import scaled_mm, ScalingType, SwizzleType
    f = lambda: scaled_mm(pa, pb.t(), to_blocked(sa).view(torch.float8_e8m0fnu), ScalingType.BlockWise1x32,
                          to_blocked(sb).view(torch.float8_e8m0fnu), ScalingType.BlockWise1x32,
                          swizzle_a=SwizzleType.SWIZZLE_32_4_4, swizzle_b=SwizzleType.SWIZZLE_32_4_4,
                          output_dtype=torch.float32)
    c = f()
    res["fp4_api2_exact"] = bool(torch.equal(c, ref))
    ms = timeit(f)
    res["fp4_api2_TMACs"] = N ** 3 / ms / 1e9
except Exception as e:
    res["fp4_api2_err"] = "".join(traceback.format_exception_only(e))[-600:]
print(json.dumps(res, indent=1))
