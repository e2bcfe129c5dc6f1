set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_new.json 2>gpurun_out/bench_new.err
MPIRG_TRSV=grid timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_grid.json 2>/dev/null
timeout 300 python bench.py --config cfg3 --lu-mode tc --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3.json 2>/dev/null
