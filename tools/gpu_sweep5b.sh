set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/pytest_batch.log 2>&1
tail -2 gpurun_out/pytest_batch.log
for w in 8 12 16 24; do
  MPIRG_BATCH_WORKERS=$w timeout 600 python bench.py --config cfg5b --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b5_np_${w}.json 2>/dev/null
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/b5_np_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 4), d["all_ok"])
    except Exception as e:
        print(f, "ERR", e)
PY
