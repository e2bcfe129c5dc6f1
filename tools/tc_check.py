"""Debug the TC trailing update against a torch reference (prints mismatch pattern)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_14616_b200 import _lib as L  # noqa: E402

for (n, k0, cb, ce) in [(640, 64, 128, 640), (512, 0, 64, 512)]:
    g = torch.Generator().manual_seed(n + k0)
    a = (torch.randn(n, n, generator=g) * 0.5).half()
    dev = a.clone().cuda()
    err = L.mpirg_error()
    st = L.lib().mpirg_tc_update(n, dev.data_ptr(), k0, cb, ce, None, C.byref(err))
    print("status", st, err.message)
    torch.cuda.synchronize()
    got = dev.cpu()
    c0 = k0 + 64
    prod = a[cb:ce, k0:k0 + 64].double() @ a[k0:k0 + 64, c0:].double()
    want = (a[cb:ce, c0:].float() - prod.float()).half()
    d = (got[cb:ce, c0:].float() - want.float()).abs()
    bad = d > 1e-3 * (want.float().abs() + 1)
    print(n, k0, cb, ce, "exact", (d == 0).float().mean().item(), "bad", bad.float().mean().item())
    idx = bad.nonzero()
    if len(idx):
        cols = idx[:, 0] + cb
        rows = idx[:, 1] + c0
        print(" bad cols range", cols.min().item(), cols.max().item(), "unique cols",
              len(torch.unique(cols)), "rows range", rows.min().item(), rows.max().item(),
              "unique rows", len(torch.unique(rows)))
        print(" rows mod 128 hist", torch.bincount((rows - c0) % 128, minlength=128)[:128].tolist())
        print(" cols mod 256 hist nonzero", torch.nonzero(torch.bincount((cols - cb) % 256, minlength=256)).flatten()[:64].tolist())
        i = idx[0]
        print(" sample got", got[cb + i[0], c0 + i[1]].item(), "want", want[i[0], i[1]].item(),
              "C", a[cb + i[0], c0 + i[1]].item())
    # also: what if D were computed as +L21 U12 or transposed?

def ulp16(x):
    x = np.abs(x.astype(np.float32))
    e = np.floor(np.log2(np.maximum(x, 2.0 ** -14)))
    return 2.0 ** (e - 10)


n, k0, cb, ce = 640, 64, 128, 640
g = torch.Generator().manual_seed(n + k0)
a = (torch.randn(n, n, generator=g) * 0.5).half()
dev = a.clone().cuda()
err = L.mpirg_error()
L.lib().mpirg_tc_update(n, dev.data_ptr(), k0, cb, ce, None, C.byref(err))
torch.cuda.synchronize()
got = dev.cpu()
c0 = k0 + 64
prod = a[cb:ce, k0:k0 + 64].double() @ a[k0:k0 + 64, c0:].double()
exact = a[cb:ce, c0:].double() - prod
want = (a[cb:ce, c0:].float() - prod.float()).half()
tile = got[cb:ce, c0:]
d = (tile.float() - want.float()).abs().numpy()
mag = np.maximum(np.abs(want.float().numpy()), np.abs(tile.float().numpy()))
r = d / ulp16(mag)
print("max diff/ulp", r.max(), "count >1", (r > 1).sum())
for (i, j) in list(zip(*np.nonzero(r > 1)))[:10]:
    print(" got", float(tile[i, j]), "want", float(want[i, j]), "exact", float(exact[i, j]),
          "ulp", float(ulp16(mag)[i, j]))
