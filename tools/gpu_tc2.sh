#!/bin/bash
tag=${1:-r02d}
mkdir -p gpurun_out
timeout 600 python tools/ubench_tc.py > gpurun_out/${tag}_ubench_tc.jsonl 2>&1; echo "ubench rc=$?"; cat gpurun_out/${tag}_ubench_tc.jsonl
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/${tag}_pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/${tag}_pytest_tc.log
for mode in "" "MPIRG_TC_PANEL=f16"; do
env $mode timeout 600 python bench.py --config cfg3 --lu-mode tc --no-cpu-baseline > gpurun_out/${tag}_bench_cfg3tc_${mode:-default}.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/${tag}_bench.err
F=gpurun_out/${tag}_bench_cfg3tc_${mode:-default}.json python - <<'PY'
import json,os
try:
    l=json.load(open(os.environ["F"]))
    print("value",l["value"],"factor_ms",l["factor_ms"],"iters",l["iters"],"profiled_step",l["profiled_step_ms"])
    for k,v in l["kernels"].items(): print("  ",k,round(v["ms_per_step"],3),v.get("launches_per_step"),round(v.get("frac",0),4))
except Exception as e: print("ERR",e)
PY
done
