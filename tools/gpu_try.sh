set -x
mkdir -p gpurun_out
timeout 300 python tools/ubench_gemm.py > gpurun_out/ub.txt 2>&1
timeout 600 ncu --set full --import-source on -k regex:gemm_tma -c 1 -o gpurun_out/gemm_tma python tools/ubench_gemm.py 16384,128,128 > gpurun_out/ncu_gemm.log 2>&1
cat gpurun_out/ub.txt
