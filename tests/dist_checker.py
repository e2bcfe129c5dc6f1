"""CPU stand-in for one rank of the distributed LU (TEST INFRASTRUCTURE).

Implements the backend interface of paper_2311_14616_b200.dist.factor
(owner / msg_bytes / begin / panel / pack / unpack / update / end) with the
oracle's blocked restatement (oracle/mpir_oracle.c orc_dlu_*), so the
multi-process schedule -- ownership, broadcast order, look-ahead parts,
row-move application, scatter/gather -- runs under gloo on CPU and its
result can be compared bit for bit with the compiled reference's LU.
"""
import numpy as np
import torch


class OracleRank:
    def __init__(self, orc, prec, n, nranks, rank, nb, block_cols):
        assert block_cols & (block_cols - 1) == 0 and block_cols % nb == 0
        self.orc, self.prec, self.n = orc, prec, n
        self.G, self.r, self.nb, self.block_cols = nranks, rank, nb, block_cols
        self.sh = block_cols.bit_length() - 1
        self.npanels = (n + nb - 1) // nb
        self.esz = 8 if prec == 0 else 4
        self.moves = {}
        self.sing = [-1]

    def _geo(self, p):
        k0 = p * self.nb
        return k0, min(self.nb, self.n - k0)

    def owner(self, p):
        return ((p * self.nb) // self.block_cols) % self.G

    def msg_bytes(self, p):
        k0, jb = self._geo(p)
        return 8 + 4 * jb + 8 * 2 * self.nb + self.esz * (self.n - k0) * jb

    def new_msg(self, nbytes, like):
        return torch.zeros(nbytes, dtype=torch.uint8)

    def begin(self, perm):
        if perm is not None:
            perm.copy_(torch.arange(self.n, dtype=torch.int32))

    def _cm(self, a):
        return a.numpy().reshape(self.n, self.n)  # [column, row]

    def panel(self, a, p, ipiv):
        k0, jb = self._geo(p)
        self.moves[p] = self.orc.dlu_panel(self.prec, a.data_ptr(), self.n, k0, jb,
                                           ipiv.numpy(), self.sing)

    def pack(self, a, p, ipiv, msg):
        k0, jb = self._geo(p)
        buf = msg.numpy()
        mv = self.moves[p]
        o = 0
        buf[o:o + 8] = np.array([len(mv), self.sing[0]], dtype=np.int32).view(np.uint8)
        o += 8
        buf[o:o + 4 * jb] = ipiv.numpy()[k0:k0 + jb].view(np.uint8)
        o += 4 * jb
        pad = np.full((2 * self.nb, 2), -1, dtype=np.int32)
        pad[: len(mv)] = mv
        buf[o:o + 16 * self.nb] = pad.reshape(-1).view(np.uint8)
        o += 16 * self.nb
        blk = np.ascontiguousarray(self._cm(a)[k0:k0 + jb, k0:])
        buf[o:] = blk.reshape(-1).view(np.uint8)

    def unpack(self, a, p, ipiv, msg):
        k0, jb = self._geo(p)
        buf = msg.numpy()
        o = 0
        nm, sing = buf[o:o + 8].view(np.int32)
        o += 8
        ipiv.numpy()[k0:k0 + jb] = buf[o:o + 4 * jb].view(np.int32)
        o += 4 * jb
        self.moves[p] = buf[o:o + 16 * self.nb].view(np.int32).reshape(-1, 2)[:nm].copy()
        o += 16 * self.nb
        dt = np.float64 if self.esz == 8 else np.float32
        self._cm(a)[k0:k0 + jb, k0:] = buf[o:].view(dt).reshape(jb, self.n - k0)
        if sing >= 0 and (self.sing[0] < 0 or sing < self.sing[0]):
            self.sing[0] = int(sing)

    def update(self, a, p, part, perm):
        k0, jb = self._geo(p)
        c0 = k0 + jb
        cnext = min(self.n, c0 + self.nb)
        nextmine = p + 1 < self.npanels and ((c0 >> self.sh) % self.G) == self.r
        mv = self.moves[p]
        pm = None if perm is None else perm.numpy()
        args = (self.prec, a.data_ptr(), self.n, k0, jb, mv, self.G, self.r, self.sh)
        if part in (0, 1) and nextmine:
            self.orc.dlu_update(*args, c0, cnext, 0, None)
        if part in (0, 2):
            self.orc.dlu_update(*args, cnext if nextmine else c0, self.n, 1, pm)

    def end(self):
        return self.sing[0]
