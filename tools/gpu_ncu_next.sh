set -x
mkdir -p gpurun_out
MPIRG_LU_GREEN=0 MPIRG_LU_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:next_kernel -s 48 -c 2 -o gpurun_out/next3 -f python tools/run_lu.py --n 4096 --reps 1 > gpurun_out/ncu_next.log 2>&1
MPIRG_LU_GREEN=0 MPIRG_LU_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum,launch__cluster_dim_x,launch__grid_size --clock-control none -k regex:'next_kernel|mt2|gemm_tma' -c 200 --csv --log-file gpurun_out/next_launches.csv python tools/run_lu.py --n 4096 --reps 1 > /dev/null 2>&1
tail -2 gpurun_out/ncu_next.log
