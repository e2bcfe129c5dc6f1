"""Residual kernel alone (mpirg_residual_tr on a handle) at n, per MPIRG_RES_RPW;
prints us per pass, GB/s and cycles per column against the DFMA chain latency."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2311_14616_b200 import _lib as L, kernels  # noqa: E402

lib = L.lib()
lat = {}
for prec, name in ((0, "dfma"), (1, "ffma")):
    c = C.c_double(0.0)
    lib.mpirg_fma_latency(prec, C.byref(c))
    lat[name] = c.value
for n in [int(x) for x in sys.argv[1:]] or [4096]:
    a = torch.randn(n * n, dtype=torch.float64, device="cuda")
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    r = torch.empty(n, dtype=torch.float64, device="cuda")
    err = L.mpirg_error()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    ts = []
    for i in range(6):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = lib.mpirg_residual(0, 0, n, a.data_ptr(), x.data_ptr(), b.data_ptr(), r.data_ptr(),
                                None, C.byref(err))
        e1.record()
        torch.cuda.synchronize()
        assert st == 0
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    us = min(ts)
    print(json.dumps({"n": n, "rpw": os.environ.get("MPIRG_RES_RPW", "auto"), "us": round(us, 1),
                      "gbs": round(n * n * 8 / us / 1e3, 1),
                      "cycles_per_column_at_1965MHz": round(us * 1965 / n, 1), **lat}), flush=True)
