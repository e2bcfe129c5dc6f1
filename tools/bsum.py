"""One-line summary of bench JSON lines: value, factor, per-kernel ms."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1])
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
        continue
    ks = " ".join(f"{k}={v['ms_per_step']:.2f}" for k, v in d.get("kernels", {}).items())
    print(f"{f}: value={d.get('value'):.5f} factor_ms={d.get('factor_ms', 0):.2f} "
          f"lu_gflops={d.get('lu_gflops', 0):.0f} iters={d.get('iters')} | {ks}")
