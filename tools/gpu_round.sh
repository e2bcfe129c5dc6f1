#!/bin/bash
# One GPU round: tests, the default bench line, the reference arm, and a launch list of smoke().
# usage (under gpurun): bash tools/gpu_round.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
tail -3 gpurun_out/${tag}_pytest_gpu.log
python bench.py > gpurun_out/${tag}_bench_cfg2a.json 2> gpurun_out/${tag}_bench_cfg2a.err; echo "bench rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke_ncu.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/${tag}_smoke_ncu.log
