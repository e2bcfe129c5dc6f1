set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "lu or golden or ir or dist or batch or tc" > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_new.json 2>gpurun_out/bench_new.err
timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --steps 2 --warmup 1 > gpurun_out/bench_cfg4.json 2>gpurun_out/bench_cfg4.err
MPIRG_LIB=libmpir_gpu_dbg.so timeout 300 python tools/run_lu.py --reps 1 > gpurun_out/panel_dbg.txt 2>&1
