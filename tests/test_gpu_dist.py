"""Config 5a on the device: tall panels and the distributed LU schedule.

* Tall panels (taller than one thread-block cluster holds at width nb) are
  factored as 8-column leaves; forced here at small n by capping the cluster
  size (MPIRG_PANEL_MAXCS, read once per process -> subprocess). Factors and
  pivots must equal the compiled reference's lu_inplace bit for bit.
* The distributed LU (paper_2311_14616_b200.dist) with 1-3 ranks. This
  container's GPU box has one GPU, so the ranks are processes sharing it over
  gloo (host-side waits only; no kernel waits on another rank's kernel). The
  factors, pivots, histories and solution must equal the single-GPU path.
"""
import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

pytestmark = pytest.mark.gpu


def _run(code, env_extra, tmp_path):
    env = dict(os.environ, **env_extra)
    env["PYTHONPATH"] = ROOT + os.pathsep + os.path.join(ROOT, "tests")
    r = subprocess.run([sys.executable, "-c", textwrap.dedent(code)], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("prec,n", [(1, 1500), (0, 1100), (1, 777)])
def test_tall_panel_leaves_bitwise(tmp_path, ref, prec, n):
    out = str(tmp_path / "lu.npz")
    _run(f"""
        import numpy as np, torch
        import helpers
        from paper_2311_14616_b200 import kernels
        a = helpers.normal_matrix({n}, 5)
        if {prec} == 1:
            a = helpers.demote_host(a, 1)
        t = torch.from_numpy(np.asfortranarray(a).reshape(-1, order="F").copy()).cuda()
        ipiv = torch.zeros({n}, dtype=torch.int32, device="cuda")
        kernels.lu_factor(t, ipiv, {n})
        np.savez("{out}", lu=t.cpu().numpy(), ipiv=ipiv.cpu().numpy())
        """, {"MPIRG_PANEL_MAXCS": "1"}, tmp_path)
    import helpers
    a = helpers.normal_matrix(n, 5)
    if prec == 1:
        a = helpers.demote_host(a, 1)
    st, lu, ipiv, _, _ = ref.lu(a, prec)
    got = np.load(out)
    assert st == 0
    assert np.array_equal(got["ipiv"], ipiv)
    want = np.asfortranarray(lu).reshape(-1, order="F")
    assert np.array_equal(got["lu"].view(np.uint8), want.view(np.uint8))


WORKER = """
import sys, numpy as np, torch, torch.distributed as dist
import helpers
from paper_2311_14616_b200 import dist as D, mpir
rank, world, port, n, out, la, bc, maxcs = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3],
                                            int(sys.argv[4]), sys.argv[5], sys.argv[6] == "1",
                                            int(sys.argv[7]), sys.argv[8])
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                        world_size=world)
a = helpers.greens(n, 800.0) if rank == 0 else None
b = helpers.normal_vector(n, 0) if rank == 0 else None
rep = D.solve_distributed(a, b, working="double", factor_precision="single",
                          resid_term=False, ce=10.0, litmax=20, nb=16, block_cols=bc,
                          lookahead=la)
if rank == 0:
    f = rep["factorization"]
    np.savez(out, x=rep["x"], rhist=np.array(rep["rhist"]), reason=rep["reason"],
             lu=f.packed_lu().T.copy(), ipiv=f.ipiv())
dist.destroy_process_group()
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,la,bc,maxcs", [(1, True, 32, "16"), (2, True, 32, "16"),
                                                (2, False, 16, "16"), (3, True, 64, "1")])
def test_distributed_solve_equals_single_gpu(tmp_path, world, la, bc, maxcs):
    from helpers import greens, normal_vector
    from paper_2311_14616_b200 import mpir
    n = 640
    out = str(tmp_path / "d.npz")
    port = str(_free_port())
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.path.join(ROOT, "tests"),
               MPIRG_PANEL_MAXCS=maxcs)
    procs = [subprocess.Popen([sys.executable, "-c", WORKER, str(r), str(world), port, str(n),
                               out, "1" if la else "0", str(bc), maxcs], env=env, cwd=ROOT,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    logs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(x[-2000:] for x in logs)
    got = np.load(out)
    f = mpir.Factorization(greens(n, 800.0), factor="single", resid_term=False, nb=16)
    rep = f.solve(normal_vector(n, 0), ce=10.0, litmax=20)
    assert np.array_equal(got["ipiv"], f.ipiv())
    assert np.array_equal(got["lu"].view(np.uint32), f.packed_lu().T.view(np.uint32))
    assert str(got["reason"]) == rep["reason"]
    assert [v.hex() for v in got["rhist"]] == [v.hex() for v in rep["rhist"]]
    assert np.array_equal(got["x"].view(np.uint64), rep["x"].view(np.uint64))
