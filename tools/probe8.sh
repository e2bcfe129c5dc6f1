set -x
ncu --set full --clock-control none --import-source on -k regex:lu_gemm_v4 -s 20 -c 1 -o gpurun_out/gemm_v4_n16384 python tools/run_lu.py --n 16384 --reps 1 > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lu_panel2 -s 8 -c 1 -o gpurun_out/panel_spec_n4096 python tools/run_lu.py --n 4096 --reps 1 > gpurun_out/ncu_panel.log 2>&1
tail -3 gpurun_out/ncu_gemm.log gpurun_out/ncu_panel.log
