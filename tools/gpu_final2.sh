# Final check of HEAD: parity suite, smoke, default bench line, cfg5b line, reference arm, launch list.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_cfg2a.json 2> gpurun_out/bench_cfg2a.err
timeout 900 python bench.py --config cfg5b --steps 3 --warmup 3 > gpurun_out/bench_cfg5b.json 2> gpurun_out/bench_cfg5b.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
MPIRG_LU_GREEN=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
python - <<'PY'
import json
for f in ("gpurun_out/bench_cfg2a.json", "gpurun_out/bench_cfg5b.json", "gpurun_out/bench_ref.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"))
PY
