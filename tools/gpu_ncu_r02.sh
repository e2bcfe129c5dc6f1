#!/bin/bash
# ncu --set full of the round-2 kernels on cfg2a (N = 4096): the first two panel launches
# (whole-panel speculation, clean) and one forward / backward substitution.
tag=${1:-r02v}
mkdir -p gpurun_out
python tools/run_solve.py 4096 2 > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${tag}_plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:lu_panel2_kernel -c 2 \
    -o gpurun_out/${tag}_panel python tools/run_solve.py 4096 2 > gpurun_out/${tag}_ncu_panel.log 2>&1
echo "ncu panel rc=$?"; tail -2 gpurun_out/${tag}_ncu_panel.log
ncu --set full --clock-control none --import-source on -k regex:trsv_kernel -c 2 \
    -o gpurun_out/${tag}_trsv python tools/run_solve.py 4096 2 > gpurun_out/${tag}_ncu_trsv.log 2>&1
echo "ncu trsv rc=$?"; tail -2 gpurun_out/${tag}_ncu_trsv.log
ls -la gpurun_out/${tag}_*.ncu-rep
