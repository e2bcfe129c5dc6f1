"""The opt-in fused next-column step of the binary32 LU (MPIRG_LU_NEXT=1,
lu_f32.cuh next_kernel) against the default two-launch path: identical
factors and pivots, bit for bit, on matrices with and without interchanges and
on sizes that are not multiples of the panel width. The switch is read once
per process, so each mode runs in its own interpreter."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, %r)
from paper_2311_14616_b200 import kernels, lib
L = lib()
out = []
for n, kind in ((1000, "greens"), (777, "randn"), (2048, "randn"), (4096, "greens")):
    a = np.empty(n * n)
    if kind == "randn":
        L.mpirg_gen_normal_matrix(n, n, 1, a.ctypes.data)
    else:
        L.mpirg_gen_greens_operator(n, 800.0, a.ctypes.data)
    d = torch.from_numpy(a).cuda().float()
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    kernels.lu_factor(d, ipiv, n)
    torch.cuda.synchronize()
    h = hashlib.sha256(d.cpu().numpy().tobytes() + ipiv.cpu().numpy().tobytes()).hexdigest()
    out.append(f"{n}:{kind}:{h}")
print(" ".join(out))
"""


def _run(flag):
    env = dict(os.environ, MPIRG_LU_NEXT=flag)
    r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


def test_fused_next_step_is_bitwise_equal(gpulib):
    assert _run("1") == _run("0")
