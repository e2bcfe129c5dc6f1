set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_streamed.py tests/test_gpu_ir.py -x -q > gpurun_out/pytest_try5.log 2>&1
tail -3 gpurun_out/pytest_try5.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_try_$i.json 2>/dev/null; done
python - <<'PY'
import json
for f in ("gpurun_out/bench_try_1.json", "gpurun_out/bench_try_2.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["e2e"]["value"])
PY
