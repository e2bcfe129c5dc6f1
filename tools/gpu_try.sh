mkdir -p gpurun_out
MPIRG_LU_TIMELINE=1 timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/b4tl.json 2> gpurun_out/b4tl.err
grep "chain totals" gpurun_out/b4tl.err
MPIRG_LU_GREEN=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1
python tools/launches.py gpurun_out/launches.csv | head -12
