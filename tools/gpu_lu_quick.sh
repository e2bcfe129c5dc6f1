#!/bin/bash
# quick LU iteration: LU/golden parity tests, then the cfg2a bench line (no CPU leg)
tag=${1:-r02r}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py tests/test_gpu_ir.py -x -q -k "lu or golden or ir_all" > gpurun_out/${tag}_pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${tag}_pytest_quick.log
timeout 900 python bench.py --no-also --no-cpu-baseline > gpurun_out/${tag}_bench_cfg2a.json 2> gpurun_out/${tag}_bench_cfg2a.err; echo "cfg2a rc=$?"; tail -3 gpurun_out/${tag}_bench_cfg2a.err
F=gpurun_out/${tag}_bench_cfg2a.json python - <<'PY'
import json,os
try:
    l=json.load(open(os.environ["F"]))
    print("value",l["value"],"e2e",l["e2e"]["value"],"factor_ms",l.get("factor_ms"))
    for k,v in l["kernels"].items(): print("  ",k,round(v["ms_per_step"],3),v.get("launches_per_step"),round(v.get("frac",0),4))
except Exception as e: print("ERR",e)
PY
