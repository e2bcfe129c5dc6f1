mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py -m gpu -x -q -k "lu or golden" 2>&1 | tail -4
MPIRG_LIB=libmpir_gpu_dbg.so timeout 300 python tools/run_lu.py --n 4096 --reps 1 > gpurun_out/pdbg4096.txt 2>&1
grep panel gpurun_out/pdbg4096.txt | head -3
MPIRG_LU_TIMELINE=1 timeout 300 python tools/run_lu.py --n 4096 --reps 2 > gpurun_out/tl4096.txt 2>&1
grep "chain totals" gpurun_out/tl4096.txt
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b2a.json 2>&1
python tools/bsum.py gpurun_out/b2a.json
