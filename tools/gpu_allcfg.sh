# Bench lines for the remaining BASELINE configs (cfg1, cfg2b, cfg3 exact binary16 LU, cfg3 tc, cfg4).
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --config cfg1 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 600 python bench.py --config cfg2b > gpurun_out/bench_cfg2b.json 2> gpurun_out/bench_cfg2b.err
timeout 900 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --config cfg3 --lu-mode tc --no-cpu-baseline > gpurun_out/bench_cfg3tc.json 2> gpurun_out/bench_cfg3tc.err
timeout 900 python bench.py --config cfg4 --no-cpu-baseline --steps 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python - <<'PY'
import json
for c in ("cfg1", "cfg2b", "cfg3", "cfg3tc", "cfg4"):
    try:
        d = json.loads(open(f"gpurun_out/bench_{c}.json").read().strip().splitlines()[-1])
        print(c, round(d["value"] * 1e3, 3), "ms e2e", round(d["e2e"]["value"] * 1e3, 3), d["iters"], d["reason"],
              (d.get("cpu_baseline") or {}).get("value"), d["roofline"]["kernel"], round(d["roofline"]["frac"], 4))
    except Exception as e:
        print(c, "ERR", e)
PY
