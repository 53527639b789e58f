"""Probe: is FP4 (e2m1, MX block-32 scales = 1.0) tensor-core accumulation exact
for 0/1 operands? Sweeps K, records max error vs the int8 product and the rate.
Design input for a kind::mxf4 engine; not part of the product."""
import json, torch
from torch.nn.functional import scaled_mm, ScalingType, SwizzleType
torch.cuda.set_device(0)
res = {}
def blocked(s):
    r, c = s.shape
    return s.view(r // 128, 4, 32, c // 4, 4).permute(0, 3, 2, 1, 4).reshape(-1)
def pack(bits):
    nib = bits * 2   # e2m1 1.0 = 0b0010
    return (nib[:, 0::2] | (nib[:, 1::2] << 4)).contiguous().view(torch.float4_e2m1fn_x2)
for M, K, dens in [(256, 128, 0.5), (256, 1024, 0.5), (512, 4096, 0.5), (512, 8192, 0.5), (512, 4096, 1.0), (2048, 16384, 0.5)]:
    N = M
    a = (torch.rand(M, K, device='cuda') < dens).to(torch.uint8)
    b = (torch.rand(N, K, device='cuda') < dens).to(torch.uint8)   # b is B^T (K-major)
    ref = (a.float() @ b.float().t())
    sa = torch.full((M, K // 32), 127, dtype=torch.uint8, device='cuda')
    sb = torch.full((N, K // 32), 127, dtype=torch.uint8, device='cuda')
    key = f"M{M}_K{K}_d{dens}"
    try:
        c = scaled_mm(pack(a), pack(b).t(), blocked(sa).view(torch.float8_e8m0fnu), ScalingType.BlockWise1x32,
                      blocked(sb).view(torch.float8_e8m0fnu), ScalingType.BlockWise1x32,
                      swizzle_a=SwizzleType.SWIZZLE_32_4_4, swizzle_b=SwizzleType.SWIZZLE_32_4_4,
                      output_dtype=torch.float32)
        d = (c - ref)
        res[key] = {"exact": bool(torch.equal(c, ref)), "maxdiff": float(d.abs().max()),
                    "nwrong": int((d != 0).sum()), "ref_max": float(ref.max()), "c_max": float(c.max()),
                    "ratio_mean": float((c.sum() / ref.sum())),
                    "parity_exact": bool(torch.equal(c.long() & 1, ref.long() & 1))}
    except Exception as e:
        res[key] = repr(e)[-300:]
print(json.dumps(res, indent=1))
