set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "lu or golden or ir or streamed or dist" > gpurun_out/pytest_try3.log 2>&1
tail -3 gpurun_out/pytest_try3.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_try.json 2> gpurun_out/bench_try.err
MPIRG_LU_NEXT=0 timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_try_off.json 2> /dev/null
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --steps 3 --no-e2e > gpurun_out/bench_try4.json 2> gpurun_out/bench_try4.err
MPIRG_LU_TIMELINE=1 timeout 300 python tools/run_lu.py --n 4096 --reps 2 > gpurun_out/timeline.txt 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/bench_try.json", "gpurun_out/bench_try_off.json", "gpurun_out/bench_try4.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d.get("factor_ms"), (d.get("e2e") or {}).get("value"), d["iters"], d["reason"],
              {k: round(v["ms_per_step"], 3) for k, v in d["kernels"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
tail -14 gpurun_out/timeline.txt
