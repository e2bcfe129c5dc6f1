set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "trsv or solve or ir or golden or batch or twin or streamed" > gpurun_out/pytest_try6.log 2>&1
tail -3 gpurun_out/pytest_try6.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_try6.json 2>/dev/null
timeout 900 python bench.py --config cfg5a --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_try6_5a.json 2>/dev/null
python - <<'PY'
import json
for f in ("gpurun_out/bench_try6.json", "gpurun_out/bench_try6_5a.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], (d.get("e2e") or {}).get("value"), {k: (round(v["ms_per_step"], 3), round(v.get("frac") or 0, 3)) for k, v in d["kernels"].items() if k.startswith("trsv") or k == "residual"})
PY
