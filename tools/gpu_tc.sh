#!/bin/bash
tag=${1:-r02c}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/${tag}_pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/${tag}_pytest_tc.log
timeout 600 python tools/tc_deviation.py > gpurun_out/${tag}_tc_deviation.jsonl 2> gpurun_out/${tag}_tc_dev.err; echo "dev rc=$?"; cat gpurun_out/${tag}_tc_deviation.jsonl | cut -c1-400; tail -3 gpurun_out/${tag}_tc_dev.err
timeout 600 python bench.py --config cfg3 --lu-mode tc --no-cpu-baseline > gpurun_out/${tag}_bench_cfg3tc.json 2> gpurun_out/${tag}_bench_cfg3tc.err; echo "bench rc=$?"; tail -3 gpurun_out/${tag}_bench_cfg3tc.err
TAG=$tag python - <<'PY'
import json,os
try:
    l=json.load(open("gpurun_out/%s_bench_cfg3tc.json" % os.environ.get("TAG","r02c")))
    print("value",l["value"],"factor_ms",l["factor_ms"],"iters",l["iters"])
    for k,v in l["kernels"].items(): print("  ",k,round(v["ms_per_step"],3),v.get("launches_per_step"),round(v.get("frac",0),4))
except Exception as e: print("ERR",e)
PY
