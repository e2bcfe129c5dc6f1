"""tcgen05 update (mpirg_tc_gemm) alone at the shapes the recursive LU issues:
TFLOP/s (2 M N K per launch) against MEASURED_PEAKS bf16_tflops, and the HBM
traffic floor of C (4 bytes per element per launch).
usage: python tools/ubench_tc.py [n]"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_14616_b200 import _lib as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
lib = L.lib()
peak = 1627.3
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["bf16_tflops"]
except Exception:
    pass
a = (torch.randn(n, n, device="cuda") * 0.01).half()
err = L.mpirg_error()
shapes = []
h = n // 2
while h >= 64:
    shapes.append((h, n, h, n, 0, h))          # the node update at this level (first block)
    h //= 2
shapes += [(n // 2 + 64, n // 2 + 128, n // 2, n, 0, n // 2 // 64 * 64 // 2),  # inside the U12 solve
           (64, n, 64, n, 0, 64)]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for (r0, r1, cb, ce, k0, K) in shapes:
    if K <= 0 or K % 64 or k0 + K > r0 or k0 + K > cb:
        continue
    ts = []
    for i in range(5):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = lib.mpirg_tc_gemm(n, a.data_ptr(), r0, r1, cb, ce, k0, K, None, C.byref(err))
        e1.record()
        torch.cuda.synchronize()
        assert st == 0, err.message
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    M, N = r1 - r0, ce - cb
    tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12
    print(json.dumps({"M": M, "N": N, "K": K, "ms": round(ms, 4), "tflops": round(tf, 1),
                      "frac_of_bf16_peak": round(tf / peak, 3),
                      "c_traffic_gbs": round(4.0 * M * N / (ms * 1e-3) / 1e9, 1)}), flush=True)
