#!/bin/bash
# Full GPU round: every GPU test, then the bench lines of the main configs.
tag=${1:-r02s}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
tail -4 gpurun_out/${tag}_pytest_gpu.log
for cfg in cfg2a cfg4 cfg3 cfg5b; do
  extra=""; [ $cfg = cfg3 ] && extra="--lu-mode tc"
  timeout 1200 python bench.py --config $cfg $extra --no-also --no-cpu-baseline > gpurun_out/${tag}_bench_${cfg}.json 2> gpurun_out/${tag}_bench_${cfg}.err; echo "$cfg rc=$?"
  F=gpurun_out/${tag}_bench_${cfg}.json python - <<'PY'
import json,os
try:
    l=json.load(open(os.environ["F"]))
    print("  value",l["value"],"e2e",(l.get("e2e") or {}).get("value"),"factor_ms",l.get("factor_ms"))
    for k,v in l.get("kernels",{}).items(): print("    ",k,round(v.get("ms_per_step",v.get("ms_summed_over_streams",0)),3),v.get("launches_per_step",v.get("launches")),round(v.get("frac",0) or 0,4))
except Exception as e: print("ERR",e)
PY
done
