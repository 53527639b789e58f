"""The C ABI from plain C (examples/abi_demo.c): no Python or torch in the
caller -- the boundary a non-Python host (or the reference's maintainers)
would bind."""

import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_abi_from_plain_c(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lib = os.path.join(ROOT, "paper_0811_1714_b200")
    exe = tmp_path / "abi_demo"
    subprocess.run([cc, "-O2", "-Wall", os.path.join(ROOT, "examples", "abi_demo.c"),
                    "-I", os.path.join(ROOT, "include"), "-L", lib, "-lgf2b200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "abi demo OK" in out.stdout
    assert "dimension error reported" in out.stdout


def test_sharded_entry_from_plain_c(tmp_path):
    """gf2_mul_sharded (NCCL loaded at run time) from a C host with its own
    world-size-1 NCCL communicator: K-panel broadcast + multiply against
    gf2_strassen, accumulate, and the missing-communicator error."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None or not os.path.exists("/usr/include/nccl.h"):
        pytest.skip("no C compiler / NCCL headers")
    lib = os.path.join(ROOT, "paper_0811_1714_b200")
    exe = tmp_path / "sharded_demo"
    cuda_inc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "include")
    subprocess.run([cc, "-O2", os.path.join(ROOT, "examples", "sharded_demo.c"),
                    "-I", os.path.join(ROOT, "include"), "-I", cuda_inc, "-L", lib, "-lgf2b200", "-lnccl",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "sharded demo OK" in out.stdout
