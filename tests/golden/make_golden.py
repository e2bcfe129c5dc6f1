"""Generate the golden parity vectors from the COMPILED REFERENCE (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py [names...]
Writes tests/golden/<name>.json with, per case: the stop reason, rhist/dhist
(exact doubles), ||A||_1, the underflow flag, and SHA-256 digests of the
pivot vector, the packed LU factors and the solution (exact bytes), plus the
solution itself for small n. The GPU parity tests compare the CUDA path to
these digests bit for bit; the CPU tests check the C restatement against them.

Cases: small shapes of every BASELINE config and of all seven precision
combinations, and the BASELINE configs at full size (cfg1/2a/2b N=4096,
cfg3 N=8192, cfg4 N=16384; the last two take minutes of single-threaded CPU).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2311_14616_b200 import configs  # noqa: E402

COMBOS = [(0, 0, 0), (0, 1, 0), (0, 2, 0), (1, 1, 1), (1, 2, 1), (1, 1, 0), (1, 2, 0)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes(order="F")).hexdigest()


def run_case(impl, cfg: dict, keep_sol: bool) -> dict:
    aw, bw = configs.to_working(cfg, oracle.restatement())
    t0 = time.time()
    rep = impl.ir(cfg["tw"], cfg["tf"], cfg["tr"], aw, bw, on_the_fly=cfg["on_the_fly"],
                  resid_term=cfg["resid_term"], ce=cfg["ce"], litmax=cfg["litmax"],
                  want_packed=True)
    out = {
        "name": cfg["name"], "n": cfg["n"], "tw": cfg["tw"], "tf": cfg["tf"], "tr": cfg["tr"],
        "on_the_fly": cfg["on_the_fly"], "resid_term": cfg["resid_term"], "ce": cfg["ce"],
        "litmax": cfg["litmax"], "status": rep["status"], "reason": rep["reason"],
        "rhist": [float(v).hex() for v in rep["rhist"]],
        "dhist": [float(v).hex() for v in rep["dhist"]],
        "a_norm1": float(rep["a_norm1"]).hex(), "underflow": rep["underflow"],
        "ipiv_sha256": sha(rep["ipiv"]), "packed_sha256": sha(rep["packed"]),
        "sol_sha256": sha(rep["x"]), "seconds": time.time() - t0,
        "generator": "oracle/_ref (unmodified reference headers, GCC -O3 -march=x86-64-v3)",
    }
    if keep_sol:
        out["sol"] = [float(v).hex() for v in rep["x"].astype(np.float64)]
        out["ipiv"] = rep["ipiv"].tolist()
    return out


def cases():
    small = []
    for name, n in (("cfg1", 256), ("cfg2a", 320), ("cfg2b", 320), ("cfg3", 384),
                    ("cfg4", 300), ("cfg1", 1000)):
        small.append((f"{name}_n{n}", configs.config(name, n), True))
    for tw, tf, tr in COMBOS:
        c = configs.config("cfg2a", 200)
        c.update(tw=tw, tf=tf, tr=tr, litmax=20)
        c["name"] = f"combo_{tw}{tf}{tr}_n200"
        small.append((c["name"], c, True))
    full = [(f"{name}_full", configs.config(name), False)
            for name in ("cfg1", "cfg2a", "cfg2b", "cfg3", "cfg4")]
    return small + full


def main(only):
    impl = oracle.reference()
    if impl is None:
        raise SystemExit("the compiled reference (oracle/_ref) is required")
    for key, cfg, keep in cases():
        if only and not any(key.startswith(o) for o in only):
            continue
        path = os.path.join(HERE, key + ".json")
        print("->", key, flush=True)
        res = run_case(impl, cfg, keep)
        with open(path, "w") as f:
            json.dump(res, f, indent=1)
        print(f"   {res['reason']} iters={len(res['rhist']) - 1} {res['seconds']:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
