set -x
mkdir -p gpurun_out
MPIRG_LU_GREEN=0 MPIRG_LU_GRAPH=0 MPIRG_STREAMED_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'trsv_kernel|residual_tma_kernel|cast_norm_kernel' -c 4 \
  -o gpurun_out/full_solve -f python tools/run_solve.py 4096 2 > gpurun_out/ncu_solve.log 2>&1
tail -2 gpurun_out/ncu_solve.log
