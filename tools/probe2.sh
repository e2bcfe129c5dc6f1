set -x
timeout 600 python -m pytest tests -m gpu -x -q -k "resid or golden or ir" > gpurun_out/pytest_sub.log 2>&1
for r in 8 16 32; do MPIRG_RES_RPW=$r timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_rpw$r.json 2>/dev/null; done
MPIRG_LIB=libmpir_gpu_dbg.so timeout 300 python tools/run_lu.py --reps 1 > gpurun_out/panel_dbg.txt 2>&1
MPIRG_LIB=libmpir_gpu_dbg.so timeout 300 python tools/run_solve.py 4096 3 > gpurun_out/trsv_dbg.txt 2>&1
tail -3 gpurun_out/pytest_sub.log
