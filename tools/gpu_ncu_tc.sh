#!/bin/bash
# ncu --set full of the tcgen05 update kernel on the K = 4096 / 2048 / 1024 shapes.
tag=${1:-r02k}
mkdir -p gpurun_out
python tools/ubench_tc.py 8192 > gpurun_out/${tag}_ubench_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 3 -c 3 \
    -o gpurun_out/${tag}_tc_gemm python tools/ubench_tc.py 8192 > gpurun_out/${tag}_ncu_tc.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${tag}_ncu_tc.log
ls -la gpurun_out/${tag}_tc_gemm.ncu-rep
