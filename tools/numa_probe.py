"""NUMA probe (design aid): the GPU's NUMA node, the host's nodes and CPUs,
and pinned H2D / D2H / bidirectional bandwidth with the pinned buffers
first-touched from each node's CPUs (sched_setaffinity before allocation,
so the kernel's default local-allocation policy places the pages)."""
import json
import os
import sys

import torch

sys.path.insert(0, '.')
torch.cuda.set_device(0)
res = {"cpu_count": os.cpu_count(), "affinity": sorted(os.sched_getaffinity(0))}
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(
    torch.cuda.get_device_properties(0), "pci_bus_id") else None
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    bus = pynvml.nvmlDeviceGetPciInfo(h).busId
    bus = bus.decode() if isinstance(bus, bytes) else bus
except Exception as e:  # noqa: BLE001
    res["nvml_err"] = repr(e)[:120]
res["gpu_bus"] = bus
nodes = {}
base = "/sys/devices/system/node"
if os.path.isdir(base):
    for d in sorted(os.listdir(base)):
        if d.startswith("node") and d[4:].isdigit():
            with open(f"{base}/{d}/cpulist") as f:
                nodes[int(d[4:])] = f.read().strip()
res["nodes"] = nodes
if bus:
    b = bus.lower()
    for cand in (b, b[4:] if len(b) > 12 else "0000" + b[-8:]):
        p = f"/sys/bus/pci/devices/{cand}/numa_node"
        if os.path.exists(p):
            res["gpu_numa_node"] = open(p).read().strip()
            break
        p = f"/sys/bus/pci/devices/0000:{cand[-7:]}/numa_node"
        if os.path.exists(p):
            res["gpu_numa_node"] = open(p).read().strip()
            break


def parse(cl):
    out = []
    for part in cl.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


def bw(fn, nbytes, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


n = 64 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
allowed = os.sched_getaffinity(0)
for node, cl in list(nodes.items()) + [("default", None)]:
    cpus = set(parse(cl)) & allowed if cl else allowed
    if not cpus:
        res[f"node{node}"] = "no allowed cpus"
        continue
    os.sched_setaffinity(0, cpus)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    os.sched_setaffinity(0, allowed)

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    res[f"node{node}"] = {
        "h2d_GBs": round(bw(lambda: d.copy_(h, non_blocking=True), n), 1),
        "d2h_GBs": round(bw(lambda: h2.copy_(d2, non_blocking=True), n), 1),
        "bidir_GBs": round(bw(both, 2 * n), 1),
    }
    del h, h2
print(json.dumps(res, indent=1))
