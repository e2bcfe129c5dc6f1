set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/pytest_batch.log 2>&1
tail -3 gpurun_out/pytest_batch.log
timeout 900 python bench.py --config cfg5b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5b.json 2> gpurun_out/bench_cfg5b.err
MPIRG_LU_TIMELINE=1 timeout 300 python tools/run_lu.py --n 4096 --reps 3 > gpurun_out/timeline.txt 2>&1
MPIRG_LU_TIMELINE=1 timeout 300 python tools/run_lu.py --n 16384 --reps 2 --randn 1 > gpurun_out/timeline16k.txt 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_cfg5b.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e'])"
tail -25 gpurun_out/timeline.txt
