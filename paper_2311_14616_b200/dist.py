"""Config 5a: the fp32 LU of an N x N system across G ranks (one process per
GPU), then the refinement loop on rank 0.

Layout (B200-first): 1-D block-cyclic columns -- column block b
(``block_cols`` columns) lives on rank b mod G. Every rank holds an n x n
factor buffer (the fp32 N=65536 matrix is 17.2 GB; a B200 has 180 GB), so the
device kernels address owned columns in place and received panels land where
the single-GPU LU would keep them. Per panel p (k0 = p*nb):

* the owner factors the panel (``mpirg_dlu_panel``: one thread-block-cluster
  kernel, or 8-column leaves when the panel is taller than a cluster holds),
* packs rows k0..n-1 of the panel + its pivots + its row moves into one
  message and broadcasts it (NCCL over NVLink; gloo for the CPU tests),
* every rank applies the row moves, U12 = L11^-1 A12 and A22 -= L21 U12 to
  the columns it owns. With look-ahead the owner of panel p+1 first updates
  only that panel's columns, factors it, and leaves the rest of step p to a
  side stream, so the next broadcast starts while step p's update runs.

Row swaps never travel: every rank applies the panel's moves to its own
columns. Factors, pivots and the permutation are bit-identical to the
single-GPU LU for every G (the blocked form keeps the per-element FMA order
of dense_lu.hpp:91-107). The reference has no distributed code; its
single-process ``MPFactorization`` + ``ir_solve_report`` is what rank 0
reproduces.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

PART_ALL, PART_NEXT, PART_REST = 0, 1, 2


# ---------------------------------------------------------------------------
# communication (torch.distributed is the plumbing)
# ---------------------------------------------------------------------------
class Comm:
    """Broadcast / point-to-point over torch.distributed. Under gloo, CUDA
    tensors are staged through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.backend = dist.get_backend(group)

    def _staged(self, t):
        return self.backend == "gloo" and t.is_cuda

    def broadcast(self, t, src):
        if self._staged(t):
            h = t.cpu()
            self.dist.broadcast(h, src, group=self.group)
            t.copy_(h)
        else:
            self.dist.broadcast(t, src, group=self.group)

    def send(self, t, dst):
        self.dist.send(t.cpu() if self._staged(t) else t, dst, group=self.group)

    def recv(self, t, src):
        if self._staged(t):
            h = t.cpu()
            self.dist.recv(h, src, group=self.group)
            t.copy_(h)
        else:
            self.dist.recv(t, src, group=self.group)


class NcclComm:
    """The library's own NCCL communicator (mpirg_comm_*): what the C++-driven
    LU broadcasts its panels over (NCCL over NVLink). The 128-byte unique id is
    made on rank 0 and handed out through torch.distributed (any backend)."""

    def __init__(self, comm: "Comm", device: int):
        import torch
        self.lib = L.lib()
        ident = (C.c_char * 128)()
        err = L.mpirg_error()
        if comm.rank == 0:
            L.check(self.lib.mpirg_comm_unique_id(ident, C.byref(err)), err)
        box = [bytes(ident)]
        comm.dist.broadcast_object_list(box, src=0, group=comm.group)
        self.h = C.c_void_p()
        L.check(self.lib.mpirg_comm_create(C.byref(self.h), comm.size, comm.rank, box[0], device,
                                           C.byref(err)), err)
        torch.cuda.synchronize(device)

    def hook(self):
        """(function pointer, context) for mpirg_dlu_factor."""
        return C.cast(self.lib.mpirg_comm_bcast, C.c_void_p), self.h

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.mpirg_comm_destroy(h)
            self.h = None


def staged_hook(comm: "Comm", device):
    """A broadcast hook over torch.distributed for backends without a device
    data path (gloo in the tests): synchronise the stream, broadcast through
    ``comm`` (host-staged under gloo), synchronise again. Returns (callback
    object -- keep it alive --, context)."""
    import torch

    def cb(_ctx, buf, nbytes, root, stream):
        try:
            torch.cuda.synchronize(device)
            t = _wrap(buf, nbytes, torch.uint8, device)
            comm.broadcast(t, root)
            torch.cuda.synchronize(device)
            return 0
        except Exception:  # pragma: no cover - reported as MPIRG_ERR_NCCL
            import traceback
            traceback.print_exc()
            return 1
    fn = L.BCAST_FN(cb)
    return fn, None


# ---------------------------------------------------------------------------
# the device backend: one rank's share of the LU through the C-ABI
# ---------------------------------------------------------------------------
class CudaRank:
    """mpirg_dlu_* for one rank (the product path; no CPU fallback)."""

    def __init__(self, prec: int, n: int, nranks: int, rank: int, nb: int = 0,
                 block_cols: int = 0, device: int = -1):
        import torch
        if not torch.cuda.is_available():
            raise L.CudaError("no CUDA device available (the B200 path has no CPU fallback)")
        self.torch = torch
        self.lib = L.lib()
        self.h = C.c_void_p()
        err = L.mpirg_error()
        st = self.lib.mpirg_dlu_create(C.byref(self.h), prec, n, nb, nranks, rank, block_cols,
                                       device, C.byref(err))
        L.check(st, err)
        self.n, self.G, self.r = n, nranks, rank
        self.nb = self.lib.mpirg_dlu_nb(self.h)
        self.npanels = self.lib.mpirg_dlu_npanels(self.h)
        self.block_cols = self.lib.mpirg_dlu_block_cols(self.h)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.mpirg_dlu_destroy(h)
            self.h = None

    def _s(self):
        return C.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def _call(self, fn, *args):
        err = L.mpirg_error()
        st = fn(self.h, *args, C.byref(err))
        L.check(st, err)

    @staticmethod
    def _p(t):
        return None if t is None else t.data_ptr()

    def owner(self, p):
        return self.lib.mpirg_dlu_owner(self.h, p)

    def msg_bytes(self, p):
        return self.lib.mpirg_dlu_msg_bytes(self.h, p)

    def new_msg(self, nbytes, like):
        return self.torch.empty(nbytes, dtype=self.torch.uint8, device=like.device)

    def begin(self, perm):
        self._call(self.lib.mpirg_dlu_begin, self._p(perm), self._s())

    def panel(self, a, p, ipiv):
        self._call(self.lib.mpirg_dlu_panel, a.data_ptr(), p, ipiv.data_ptr(), self._s())

    def pack(self, a, p, ipiv, msg):
        self._call(self.lib.mpirg_dlu_pack, a.data_ptr(), p, ipiv.data_ptr(), msg.data_ptr(),
                   self._s())

    def unpack(self, a, p, ipiv, msg):
        self._call(self.lib.mpirg_dlu_unpack, a.data_ptr(), p, ipiv.data_ptr(), msg.data_ptr(),
                   self._s())

    def update(self, a, p, part, perm):
        self._call(self.lib.mpirg_dlu_update, a.data_ptr(), p, part, self._p(perm), self._s())

    def end(self) -> int:
        sc = C.c_int(-1)
        self._call(self.lib.mpirg_dlu_end, self._s(), C.byref(sc))
        return sc.value

    def factor_all(self, a, ipiv, perm, hook) -> int:
        """The whole LU of this rank driven from C++ (mpirg_dlu_factor): the
        panels are broadcast through ``hook`` = (function, context) without a
        Python round trip per panel; binary32 factors run the paired TMA
        schedule of the single-GPU LU on the rank's columns."""
        fn, ctx = hook if hook is not None else (None, None)
        sc = C.c_int(-1)
        self._call(self.lib.mpirg_dlu_factor, a.data_ptr(), ipiv.data_ptr(), self._p(perm),
                   C.cast(fn, C.c_void_p) if fn is not None else None, ctx, self._s(),
                   C.byref(sc))
        return sc.value


# ---------------------------------------------------------------------------
# the schedule (backend-agnostic: CudaRank on GPUs, a CPU checker in tests)
# ---------------------------------------------------------------------------
def owned_blocks(n: int, block_cols: int, nranks: int, rank: int):
    """Global column ranges [c0, c1) owned by ``rank``."""
    nblk = (n + block_cols - 1) // block_cols
    return [(b * block_cols, min(n, (b + 1) * block_cols)) for b in range(rank, nblk, nranks)]


def factor(be, comm, a, ipiv, perm=None, lookahead: bool = True) -> int:
    """This rank's part of the distributed LU. ``a``: the rank's n*n factor
    buffer (column-major, owned blocks filled); ``ipiv``: int32[n] (complete
    on every rank afterwards); ``perm``: int32[n] or None (rank 0). Returns
    the first zero-pivot column this rank saw (-1 = none; rank 0 sees all)."""
    G, r = comm.size, comm.rank
    if lookahead and hasattr(be, "factor_all"):
        hook = None
        if G > 1:
            hook = getattr(comm, "hook", None) or _hook_for(comm, a.device)
            comm.hook = hook  # keeps the callback object alive
        return be.factor_all(a, ipiv, perm, hook)
    msgbuf = be.new_msg(be.msg_bytes(0), a)  # panel 0 is the tallest
    be.begin(perm)
    early = set()
    for p in range(be.npanels):
        owner = be.owner(p)
        msg = msgbuf[: be.msg_bytes(p)]
        if r == owner:
            if p not in early:
                be.panel(a, p, ipiv)
            be.pack(a, p, ipiv, msg)
        if G > 1:
            comm.broadcast(msg, owner)
        if r != owner:
            be.unpack(a, p, ipiv, msg)
        if not lookahead:
            be.update(a, p, PART_ALL, perm)
        elif p + 1 < be.npanels and be.owner(p + 1) == r:
            be.update(a, p, PART_NEXT, perm)
            be.panel(a, p + 1, ipiv)
            early.add(p + 1)
            be.update(a, p, PART_REST, perm)
        else:
            be.update(a, p, PART_REST, perm)
    return be.end()


def _hook_for(comm, device):
    """NCCL through the library's own communicator when the process group runs
    on NCCL; otherwise the host-staged hook."""
    if comm.backend == "nccl":
        comm.native = NcclComm(comm, device.index)
        return comm.native.hook()
    return staged_hook(comm, device)


def scatter_columns(comm, full, local, n: int, block_cols: int):
    """Rank 0's n*n buffer ``full`` -> every rank's owned column blocks of
    ``local`` (rank 0: full is local)."""
    if comm.size == 1:
        return
    nblk = (n + block_cols - 1) // block_cols
    for b in range(nblk):
        q = b % comm.size
        if q == 0:
            continue
        lo, hi = b * block_cols * n, min(n, (b + 1) * block_cols) * n
        if comm.rank == 0:
            comm.send(full[lo:hi], q)
        elif comm.rank == q:
            comm.recv(local[lo:hi], 0)


def gather_columns(comm, local, full, n: int, block_cols: int):
    """Every rank's owned column blocks -> rank 0's n*n buffer ``full``."""
    if comm.size == 1:
        return
    nblk = (n + block_cols - 1) // block_cols
    for b in range(nblk):
        q = b % comm.size
        if q == 0:
            continue
        lo, hi = b * block_cols * n, min(n, (b + 1) * block_cols) * n
        if comm.rank == q:
            comm.send(local[lo:hi], 0)
        elif comm.rank == 0:
            comm.recv(full[lo:hi], q)


# ---------------------------------------------------------------------------
# the end-to-end config 5a solve
# ---------------------------------------------------------------------------
class DistributedFactorization:
    """MPFactorization<TW,TF,TR> whose LU is spread over the ranks of ``comm``
    (one process per GPU). Rank 0 owns the working-precision matrix, the
    gathered factors and the refinement loop, exactly like the single-GPU
    handle; the other ranks hold an n x n factor buffer of which they own the
    column blocks b with b mod G == rank. Buffers are allocated once;
    ``refactor`` and ``solve`` may be called repeatedly (the reference's
    pointer-stable refactor, mp_structures.hpp:155-169)."""

    def __init__(self, n: int, comm=None, *, working="double", factor_precision="single",
                 residual=None, resid_term=False, nb=0, block_cols=0, lookahead=True,
                 device=None):
        import torch

        from . import mpir
        self.torch, self.mpir = torch, mpir
        self.comm = comm or Comm()
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        cfg = mpir.resolve_config(mpir.parse_precision(working),
                                  mpir.parse_precision(factor_precision),
                                  None if residual is None else mpir.parse_precision(residual),
                                  False)
        cfg.resid_term = int(bool(resid_term))
        cfg.device = self.dev.index
        self.cfg, self.n, self.lookahead = cfg, n, lookahead
        self.be = CudaRank(cfg.tf, n, self.comm.size, self.comm.rank, nb=nb,
                           block_cols=block_cols, device=self.dev.index)
        tdt = {L.B64: torch.float64, L.B32: torch.float32, L.B16: torch.int16}[cfg.tf]
        self.f = None
        if self.comm.rank == 0:
            self.f = mpir.Factorization._allocate(n, cfg)
            bufs = [C.c_void_p() for _ in range(4)]
            L.lib().mpirg_factorization_buffers(self.f._h, *[C.byref(x) for x in bufs])
            self.local = _wrap(bufs[0].value, n * n, tdt, self.dev)
            self.ipiv = _wrap(bufs[1].value, n, torch.int32, self.dev)
            self.perm = _wrap(bufs[2].value, n, torch.int32, self.dev)
        else:
            self.local = torch.empty(n * n, dtype=tdt, device=self.dev)
            self.ipiv = torch.zeros(n, dtype=torch.int32, device=self.dev)
            self.perm = None
        self.factor_s = None

    def _agree(self, status: int, column: int = -1, message: str = ""):
        """Every rank learns rank 0's (status, column, message), so an error
        raised on one rank is raised on all of them instead of leaving the
        others blocked in a collective."""
        box = [(status, column, message)]
        self.comm.dist.broadcast_object_list(box, src=0, group=self.comm.group)
        return box[0]

    def refactor(self, a=None, a_on_device=True) -> None:
        """refactor(A): rank 0 passes A (a CUDA tensor of TW in column-major
        order, a pointer-compatible pinned/pageable host array via
        a_on_device=False, or None to refactor the resident copy); the other
        ranks pass nothing. Cast + one-norm on rank 0, scatter of the owned
        column blocks, the distributed LU, gather of the factors to rank 0."""
        import time
        torch, comm = self.torch, self.comm
        t0 = time.perf_counter()
        st, col, msg = 0, -1, ""
        if comm.rank == 0:
            err = L.mpirg_error()
            ptr = None if a is None else (a.data_ptr() if hasattr(a, "data_ptr") else
                                          a.ctypes.data)
            st = L.lib().mpirg_factorization_cast(self.f._h, ptr, 1 if a_on_device else 0,
                                                  C.byref(err))
            col, msg = err.column, err.message.decode(errors="replace")
            self._cast_err = err
        if comm.size > 1:
            st, col, msg = self._agree(st, col, msg)
        if st != 0:
            err = getattr(self, "_cast_err", None) if comm.rank == 0 else None
            if err is None:
                err = L.mpirg_error()
                err.status, err.column, err.message = st, col, msg.encode()[:255]
            L.check(st, err)
        torch.cuda.current_stream(self.dev).synchronize()
        scatter_columns(comm, self.local, self.local, self.n, self.be.block_cols)
        torch.cuda.current_stream(self.dev).synchronize()
        sing = factor(self.be, comm, self.local, self.ipiv, self.perm, lookahead=self.lookahead)
        if comm.size > 1:
            # the first zero pivot column seen by any rank (rank 0 sees all of
            # them in the step messages; this makes every rank agree)
            t = torch.tensor([sing if sing >= 0 else 2 ** 31 - 1], dtype=torch.int64,
                             device=self.dev if comm.backend == "nccl" else "cpu")
            comm.dist.all_reduce(t, op=comm.dist.ReduceOp.MIN, group=comm.group)
            sing = int(t.item())
            sing = -1 if sing == 2 ** 31 - 1 else sing
        torch.cuda.current_stream(self.dev).synchronize()
        gather_columns(comm, self.local, self.local, self.n, self.be.block_cols)
        torch.cuda.current_stream(self.dev).synchronize()
        self.factor_s = time.perf_counter() - t0
        err = L.mpirg_error()
        if comm.rank == 0:
            L.check(L.lib().mpirg_factorization_set_factored(self.f._h, sing, C.byref(err)), err)
        elif 0 <= sing < self.n:
            raise L.SingularPivot("pivot column is exactly zero", sing)

    def solve(self, b=None, *, ce=None, cr=None, rmax=None, litmax=None, tp=None):
        """ir_solve_report on rank 0 (the factors were gathered there); the
        other ranks return None."""
        if self.comm.rank != 0:
            return None
        tp = tp or self.mpir.update_parms(cr, ce, rmax, litmax)
        if hasattr(b, "data_ptr"):
            bdev = b
        else:
            bdev = self.mpir._to_device_working(np.asarray(b, dtype=np.float64).reshape(-1),
                                                self.cfg.tw)
        return self.f._solve_device(bdev, tp)


def solve_distributed(a, b, comm=None, *, working="double", factor_precision="single",
                      residual=None, resid_term=False, ce=10.0, cr=None, rmax=None,
                      litmax=10, nb=0, block_cols=0, lookahead=True, device=None):
    """MPFactorization<TW,TF,TR>(A) + ir_solve_report with the LU spread over
    the ranks of ``comm``. Rank 0 passes A (n x n float64 host array, or a
    device tensor of TW in column-major order) and b; the other ranks pass
    None. Returns the report dict on rank 0 and None elsewhere."""
    import torch

    from . import mpir
    comm = comm or Comm()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    tp = mpir.update_parms(cr, ce, rmax, litmax)
    tw = mpir.parse_precision(working)
    nt = torch.zeros(1, dtype=torch.int64, device=dev)
    adev = None
    if comm.rank == 0:
        if isinstance(a, torch.Tensor):
            adev = a
            nt[0] = int(round(a.numel() ** 0.5))
        else:
            acm = mpir._colmajor(a)
            adev = mpir._to_device_working(acm, tw)
            nt[0] = acm.shape[0]
    comm.broadcast(nt, 0)
    n = int(nt.item())
    df = DistributedFactorization(n, comm, working=working, factor_precision=factor_precision,
                                  residual=residual, resid_term=resid_term, nb=nb,
                                  block_cols=block_cols, lookahead=lookahead, device=dev.index)
    df.refactor(adev)
    rep = df.solve(b, tp=tp)
    if rep is not None:
        rep["factorization"] = df.f
        rep["distributed"] = df
    return rep


# ---------------------------------------------------------------------------
# config 5b: independent systems, one slice per rank, no collective on the
# data path (the results are concatenated on rank 0)
# ---------------------------------------------------------------------------
def batch_slice(count: int, world: int, rank: int):
    """Systems [lo, hi) of ``count`` for ``rank`` (contiguous, sizes differ by
    at most one)."""
    base, rem = divmod(count, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def batch_solve_sliced(make_slice, count: int, comm=None, *, solver=None, **kw):
    """Config 5b over the ranks of ``comm``: rank r solves systems
    batch_slice(count, world, r) -- ``make_slice(lo, hi)`` returns that
    slice's (a, b) -- with ``solver`` (default mpir.batch_solve on the rank's
    GPU; the CPU tests inject a stand-in). No collective touches the systems;
    the per-system reports are gathered to rank 0, which returns the list in
    system order (the other ranks return None)."""
    comm = comm or Comm()
    if solver is None:
        from . import mpir
        solver = mpir.batch_solve
    lo, hi = batch_slice(count, comm.size, comm.rank)
    a, b = make_slice(lo, hi)
    mine = solver(a, b, **kw) if hi > lo else []
    if comm.size == 1:
        return mine
    box = [None] * comm.size if comm.rank == 0 else None
    comm.dist.gather_object(mine, box, dst=0, group=comm.group)
    if comm.rank != 0:
        return None
    return [rep for part in box for rep in part]


_TYPESTR = {"float64": "<f8", "float32": "<f4", "int16": "<i2", "int32": "<i4", "uint8": "|u1"}


def _wrap(ptr: int, numel: int, dtype, device):
    """A torch view of device memory owned by a handle (no copy), via the
    CUDA array interface."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (numel,), "data": (ptr, False), "version": 3,
                                    "typestr": _TYPESTR[str(dtype).split(".")[-1]],
                                    "strides": None}
    return torch.as_tensor(_Arr(), device=device)
