"""Config 3 in lu_mode=tc against the exact (reference-bitwise) binary16 path:
iteration counts, ||x_tc - x_exact||_inf / ||x||_inf, BASELINE's tolerance
10 eps32 ||x||_inf (relative: 1.19e-6) and the stopping-rule bound of SURVEY 8(d).
usage: python tools/tc_deviation.py [n ...]   (default 1024 2048 4096 8192)"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import greens  # noqa: E402
from paper_2311_14616_b200 import mpir  # noqa: E402

rows = []
for n in [int(x) for x in sys.argv[1:]] or [1024, 2048, 4096, 8192]:
    a = greens(n, 1.0)
    b = np.ones(n)
    kw = dict(working="single", factor="half", resid_term=False)
    exact = mpir.Factorization(a, **kw).solve(b, ce=10.0, litmax=10)
    ftc = mpir.Factorization(a, lu_mode="tc", **kw)
    tc = ftc.solve(b, ce=10.0, litmax=10)
    xe = exact["x"]
    rel = float(np.max(np.abs(tc["x"] - xe)) / np.max(np.abs(xe)))
    eps32 = 2.0 ** -23
    rule = 2 * 1.3 * 10.0 * eps32 * (1.0 + ftc.a_norm1 * np.max(np.abs(xe))) / np.max(np.abs(xe))
    rows.append({"n": n, "iters_exact": len(exact["rhist"]) - 1, "iters_tc": len(tc["rhist"]) - 1,
                 "reason_tc": tc["reason"], "rel_dev": rel, "baseline_tol": 10 * eps32,
                 "meets_baseline_tol": rel <= 10 * eps32, "stopping_rule_bound": float(rule),
                 "rhist_tc": tc["rhist"], "rhist_exact": exact["rhist"],
                 "factor_ms_tc": ftc.last_factor_ms})
    print(json.dumps(rows[-1]), flush=True)
