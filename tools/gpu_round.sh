# One GPU round: parity suite, smoke, bench lines, ncu launch list of the cfg2a bench,
# and one --set full capture of the panel and trailing-update kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_cfg2a.json 2> gpurun_out/bench_cfg2a.err
timeout 600 python bench.py --config cfg3 --lu-mode tc --no-cpu-baseline > gpurun_out/bench_cfg3tc.json 2> gpurun_out/bench_cfg3tc.err
timeout 900 python bench.py --config cfg4 --no-cpu-baseline --steps 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --config cfg5a --steps 2 --warmup 3 > gpurun_out/bench_cfg5a.json 2> gpurun_out/bench_cfg5a.err
timeout 900 python bench.py --config cfg5b --steps 3 --warmup 3 > gpurun_out/bench_cfg5b.json 2> gpurun_out/bench_cfg5b.err
MPIRG_LU_GREEN=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1
MPIRG_LU_GREEN=0 MPIRG_LU_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'lu_panel2_kernel|gemm_tma_kernel|trsv_kernel|residual_tma_kernel' -s 40 -c 6 \
  -o gpurun_out/full_cfg2a -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; cat gpurun_out/bench_cfg2a.json
