"""Config 5a's multi-process schedule on CPU (gloo, world sizes 2 and 3).

Each rank runs paper_2311_14616_b200.dist.factor -- the same ownership,
broadcast, look-ahead and scatter/gather code the GPUs run -- with the
oracle's blocked restatement standing in for the device kernels
(tests/dist_checker.py). Rank 0's gathered factors, pivots and permutation
must equal the compiled reference's lu_inplace bit for bit.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _matrix(kind, n):
    import helpers
    if kind == "greens":
        return helpers.greens(n, 800.0)
    if kind == "normal":
        return helpers.normal_matrix(n, 7)
    a = helpers.normal_matrix(n, 3)
    a[:, n // 3] = 0.0  # exactly zero column -> SingularPivot at a known step
    return a


def _worker(rank, world, port, n, nb, bc, lookahead, kind, prec, out):
    import torch.distributed as dist

    import oracle
    from paper_2311_14616_b200 import dist as D
    from dist_checker import OracleRank
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        orc = oracle.restatement()
        comm = D.Comm()
        dt = torch.float64 if prec == 0 else torch.float32
        local = torch.zeros(n * n, dtype=dt)
        if rank == 0:
            a = _matrix(kind, n)
            st, af, _, _ = orc.demote(a, prec) if prec == 1 else (0, np.asfortranarray(a), 0, 0)
            local.numpy()[:] = np.asfortranarray(af).reshape(-1, order="F")
        ipiv = torch.zeros(n, dtype=torch.int32)
        perm = torch.zeros(n, dtype=torch.int32) if rank == 0 else None
        be = OracleRank(orc, prec, n, world, rank, nb, bc)
        D.scatter_columns(comm, local, local, n, bc)
        sing = D.factor(be, comm, local, ipiv, perm, lookahead=lookahead)
        D.gather_columns(comm, local, local, n, bc)
        if rank == 0:
            np.savez(out, lu=local.numpy(), ipiv=ipiv.numpy(), perm=perm.numpy(), sing=sing)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,nb,bc,lookahead,kind,prec", [
    (2, 200, 16, 32, True, "greens", 1),
    (2, 203, 16, 16, False, "normal", 1),
    (3, 257, 32, 64, True, "normal", 1),
    (2, 150, 16, 32, True, "normal", 0),
    (2, 120, 16, 16, True, "singular", 1),
])
def test_distributed_lu_matches_reference(tmp_path, world, n, nb, bc, lookahead, kind, prec):
    import oracle
    out = str(tmp_path / "r0.npz")
    mp.start_processes(_worker, args=(world, _free_port(), n, nb, bc, lookahead, kind, prec,
                                      out), nprocs=world, join=True, start_method="spawn")
    got = np.load(out)
    chk = oracle.reference() or oracle.restatement()
    a = _matrix(kind, n)
    if prec == 1:
        a = oracle.restatement().demote(a, 1)[1]
    if kind == "singular":
        chk = oracle.restatement()  # keeps ipiv up to the failing column
    st, lu, ipiv, perm, sc = chk.lu(a, prec)
    if kind == "singular":
        assert st == 2 and int(got["sing"]) == sc
        # the reference stops at the zero column; everything before it agrees
        assert np.array_equal(got["ipiv"][:sc], ipiv[:sc])
        return
    assert st == 0 and int(got["sing"]) == -1
    assert np.array_equal(got["ipiv"], ipiv)
    assert np.array_equal(got["perm"], perm)
    dt = np.float64 if prec == 0 else np.float32
    want = np.asfortranarray(lu, dtype=dt).reshape(-1, order="F")
    assert np.array_equal(got["lu"].view(np.uint8), want.view(np.uint8))


def test_ownership_map():
    from paper_2311_14616_b200 import dist as D
    blocks = [D.owned_blocks(1000, 128, 3, r) for r in range(3)]
    cols = sorted(c for bl in blocks for lo, hi in bl for c in range(lo, hi))
    assert cols == list(range(1000))
    assert blocks[1][0] == (128, 256) and blocks[0][-1] == (768, 896)


def _batch_worker(rank, world, port, count, n, out):
    import torch.distributed as dist

    import helpers
    import oracle
    from paper_2311_14616_b200 import dist as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        orc = oracle.restatement()

        def make_slice(lo, hi):
            a = np.stack([helpers.diag_dominant(n, i, float(n)) for i in range(lo, hi)])
            return a, np.ones((hi - lo, n))

        def cpu_stand_in(a, b, **kw):  # the oracle in place of mpir.batch_solve
            reps = []
            for ai, bi in zip(a, b):
                r = orc.ir(0, 1, 0, np.asfortranarray(ai), bi, resid_term=False, ce=10.0,
                           litmax=10)
                reps.append({"x": r["x"], "rhist": list(r["rhist"]), "reason": r["reason"]})
            return reps
        got = D.batch_solve_sliced(make_slice, count, D.Comm(), solver=cpu_stand_in)
        if rank == 0:
            np.savez(out, x=np.stack([g["x"] for g in got]),
                     nr=np.array([len(g["rhist"]) for g in got]))
        else:
            assert got is None
    finally:
        dist.destroy_process_group()


def test_batch_slices_concatenate_in_system_order(tmp_path):
    """Config 5b's multi-rank path (dist.batch_solve_sliced): contiguous slices,
    no collective on the systems, reports gathered to rank 0 in system order.
    The device solver is replaced by the oracle so the plumbing runs under gloo."""
    import helpers
    import oracle
    count, n, world = 5, 48, 2
    out = str(tmp_path / "b.npz")
    mp.start_processes(_batch_worker, args=(world, _free_port(), count, n, out), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out)
    orc = oracle.restatement()
    for i in range(count):
        r = orc.ir(0, 1, 0, np.asfortranarray(helpers.diag_dominant(n, i, float(n))), np.ones(n),
                   resid_term=False, ce=10.0, litmax=10)
        assert np.array_equal(got["x"][i].view(np.uint64), r["x"].view(np.uint64))
        assert got["nr"][i] == len(r["rhist"])


def test_batch_slice_partition():
    from paper_2311_14616_b200 import dist as D
    for count, world in ((4096, 8), (5, 2), (3, 4), (0, 2)):
        parts = [D.batch_slice(count, world, r) for r in range(world)]
        assert parts[0][0] == 0 and parts[-1][1] == count
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        sizes = [hi - lo for lo, hi in parts]
        assert max(sizes) - min(sizes) <= 1
