# GPU call: config 5a / 5b bench lines, the full-size 5a test, panel cycle breakdown.
set -x
mkdir -p gpurun_out
free -g | head -2; nproc
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_scale.py -x -q > gpurun_out/pytest_scale.log 2>&1
timeout 900 python bench.py --config cfg5a --steps 2 --warmup 3 > gpurun_out/bench_cfg5a.json 2> gpurun_out/bench_cfg5a.err
timeout 900 python bench.py --config cfg5b --steps 3 --warmup 3 > gpurun_out/bench_cfg5b.json 2> gpurun_out/bench_cfg5b.err
timeout 600 python bench.py --config cfg5b --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_cfg5b.json 2> gpurun_out/bench_ref_cfg5b.err
MPIRG_LIB=libmpir_gpu_dbg.so timeout 300 python tools/run_lu.py --n 4096 --reps 2 > gpurun_out/panel_dbg.txt 2>&1
tail -3 gpurun_out/pytest_scale.log; cat gpurun_out/bench_cfg5a.json gpurun_out/bench_cfg5b.json | cut -c1-600
