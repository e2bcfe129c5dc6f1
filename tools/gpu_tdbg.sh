set -x
mkdir -p gpurun_out
MPIRG_LIB=libmpir_gpu_tdbg.so timeout 300 python tools/run_solve.py 4096 1 > gpurun_out/trsv_dbg.txt 2>&1
head -40 gpurun_out/trsv_dbg.txt
