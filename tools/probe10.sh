set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "solve or ir or golden or twin or lu" > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_new.json 2>gpurun_out/bench_new.err
MPIRG_LIB=libmpir_gpu_dbg.so timeout 300 python tools/run_solve.py 4096 3 > gpurun_out/trsv_dbg.txt 2>&1
