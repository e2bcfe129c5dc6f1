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


WORKER2 = """
import sys, numpy as np, torch, torch.distributed as dist
import helpers
from paper_2311_14616_b200 import dist as D, mpir
rank, world, port, n, out, bc, kind, backend = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3],
                                                int(sys.argv[4]), sys.argv[5], int(sys.argv[6]),
                                                sys.argv[7], sys.argv[8])
if backend == "nccl":
    torch.cuda.set_device(rank)
dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                        world_size=world)
a = b = None
if rank == 0:
    a = helpers.greens(n, 800.0) if kind == "greens" else helpers.normal_matrix(n, 7)
    b = helpers.normal_vector(n, 0)
df = D.DistributedFactorization(n, D.Comm(), resid_term=False, block_cols=bc)
adev = None
if rank == 0:
    adev = mpir._to_device_working(mpir._colmajor(a), 0)
for rep_i in range(2):  # refactor twice: buffers and streams are reused
    df.refactor(adev if rep_i == 0 else None)
rep = df.solve(b, ce=10.0, litmax=20)
if rank == 0:
    f = df.f
    np.savez(out, x=rep["x"], rhist=np.array(rep["rhist"]), reason=rep["reason"],
             lu=f.packed_lu().T.copy(), ipiv=f.ipiv(), perm=f.pivots())
dist.destroy_process_group()
"""


def _spawn(worker, world, args, env):
    procs = [subprocess.Popen([sys.executable, "-c", worker, str(r), str(world)] + args,
                              env=env, cwd=ROOT, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(world)]
    logs = [p.communicate(timeout=900)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(x[-3000:] for x in logs)


def _check_against_single_gpu(out, n, kind):
    from helpers import greens, normal_matrix, normal_vector
    from paper_2311_14616_b200 import mpir
    got = np.load(out)
    a = greens(n, 800.0) if kind == "greens" else normal_matrix(n, 7)
    f = mpir.Factorization(a, factor="single", resid_term=False)
    rep = f.solve(normal_vector(n, 0), ce=10.0, litmax=20)
    assert np.array_equal(got["ipiv"], f.ipiv())
    assert np.array_equal(got["perm"], f.pivots())
    assert np.array_equal(got["lu"].view(np.uint32), f.packed_lu().T.view(np.uint32))
    assert str(got["reason"]) == rep["reason"]
    assert [v.hex() for v in got["rhist"]] == [v.hex() for v in rep["rhist"]]
    assert np.array_equal(got["x"].view(np.uint64), rep["x"].view(np.uint64))


@pytest.mark.parametrize("world,n,bc,kind", [(1, 1088, 512, "randn"), (2, 1088, 128, "randn"),
                                             (3, 1344, 64, "randn"), (2, 1024, 256, "greens"),
                                             (2, 2112, 512, "randn")])
def test_cpp_driven_paired_lu_equals_single_gpu(tmp_path, world, n, bc, kind):
    """mpirg_dlu_factor, binary32 nb = 64: the single-GPU LU's TMA-fed paired
    schedule on each rank's column runs, panels broadcast through the hook
    (gloo, host-staged: the ranks are processes sharing this box's one GPU and
    only ever wait for each other on the host). Bitwise = the single-GPU path,
    including a pivot-heavy matrix whose row moves cross rank boundaries."""
    out = str(tmp_path / "d.npz")
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.path.join(ROOT, "tests"))
    _spawn(WORKER2, world, [str(_free_port()), str(n), out, str(bc), kind, "gloo"], env)
    _check_against_single_gpu(out, n, kind)


def test_nccl_two_gpus_equals_single_gpu(tmp_path):
    """The product path: two ranks, two GPUs, panels over the library's own
    NCCL communicator. Skipped on boxes with fewer than two GPUs."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    out = str(tmp_path / "d.npz")
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.path.join(ROOT, "tests"))
    _spawn(WORKER2, 2, [str(_free_port()), "2112", out, "512", "randn", "nccl"], env)
    _check_against_single_gpu(out, 2112, "randn")


def test_nccl_single_rank_communicator():
    """NCCL binds at run time and a one-rank communicator broadcasts to itself
    (what a 1-GPU box can exercise of mpirg_comm_*)."""
    import ctypes as C

    import torch
    from paper_2311_14616_b200 import _lib as L
    lib = L.lib()
    assert lib.mpirg_comm_version() >= 20000
    ident = (C.c_char * 128)()
    err = L.mpirg_error()
    L.check(lib.mpirg_comm_unique_id(ident, C.byref(err)), err)
    h = C.c_void_p()
    L.check(lib.mpirg_comm_create(C.byref(h), 1, 0, bytes(ident), 0, C.byref(err)), err)
    t = torch.arange(1024, dtype=torch.uint8, device="cuda")
    st = lib.mpirg_comm_bcast(h, t.data_ptr(), t.numel(), 0,
                              C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert st == 0 and torch.equal(t.cpu(), torch.arange(1024, dtype=torch.uint8))
    lib.mpirg_comm_destroy(h)


def test_batch_solve_devices_slices_in_order():
    """mpir.batch_solve(devices=[...]): one slice per listed GPU (here the same
    GPU twice), reports concatenated in system order and equal to the
    one-device call bit for bit."""
    from helpers import diag_dominant
    from paper_2311_14616_b200 import mpir
    n, count = 192, 7
    a = np.stack([diag_dominant(n, i, float(n)) for i in range(count)])
    b = np.ones((count, n))
    one = mpir.batch_solve(a, b, resid_term=False, ce=10.0, litmax=10)
    two = mpir.batch_solve(a, b, resid_term=False, ce=10.0, litmax=10, devices=[0, 0])
    assert len(two) == count
    for r1, r2 in zip(one, two):
        assert r1["reason"] == r2["reason"] and r1["rhist"] == r2["rhist"]
        assert np.array_equal(r1["x"].view(np.uint64), r2["x"].view(np.uint64))
