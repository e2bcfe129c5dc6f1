"""DESIGN 6b: every measurement switch of the binary32 LU selects between
bitwise-identical schedules. Each switch is read once per process, so every
setting factors the same matrices in its own interpreter and the digests of the
packed factors and pivots are compared with the default's. The matrices cover
clean panels (I - aG: whole-panel speculation succeeds), panels with
interchanges (randn) and a size that is not a multiple of the panel width."""
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
    for rep in range(2):  # the second factorization replays the captured graph
        d = torch.from_numpy(a).cuda().float()
        ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
        kernels.lu_factor(d, ipiv, n)
        torch.cuda.synchronize()
        h = hashlib.sha256(d.cpu().numpy().tobytes() + ipiv.cpu().numpy().tobytes()).hexdigest()
        out.append(f"{n}:{kind}:{h}")
print(" ".join(out))
"""

SWITCHES = [
    {"MPIRG_NEXT_CPW": "1"},
    {"MPIRG_NEXT_CPW": "2"},
    {"MPIRG_PANEL_WHOLE": "0"},
    {"MPIRG_PANEL_SPEC": "0"},
    {"MPIRG_PANEL_MAXCS": "8"},
    {"MPIRG_LU_GREEN": "0"},
    {"MPIRG_LU_GRAPH": "0"},
    {"MPIRG_GEMM": "scalar"},
    {"MPIRG_LU_PDL": "0"},
    {"MPIRG_LU_PDL": "2"},
]


def _run(extra):
    env = dict(os.environ, **extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


@pytest.fixture(scope="module")
def default_digests(gpulib):
    d = _run({})
    assert len(d.split()) == 8
    return d


@pytest.mark.parametrize("extra", SWITCHES, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_switch_keeps_factors_and_pivots_bitwise(extra, default_digests):
    assert _run(extra) == default_digests
