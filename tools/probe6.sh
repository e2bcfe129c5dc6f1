./tools/ubench/diag > gpurun_out/ubench_diag.txt 2>&1
MPIRG_LIB=libmpir_gpu_dbg.so timeout 300 python tools/run_lu.py --reps 1 > gpurun_out/panel_dbg.txt 2>&1
