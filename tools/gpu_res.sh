#!/bin/bash
tag=${1:-r02n}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ir.py tests/test_gpu_golden.py -x -q -k "residual or ir or golden" > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/${tag}_pytest.log
for sp in 1 0; do MPIRG_RES_SPLIT=$sp timeout 300 python tools/ubench_residual.py 1024 4096 8192 16384; done 2>&1 | tee gpurun_out/${tag}_residual_split.txt
timeout 900 python bench.py --no-also --no-cpu-baseline > gpurun_out/${tag}_bench_cfg2a.json 2> gpurun_out/${tag}_bench_cfg2a.err; echo "cfg2a rc=$?"
F=gpurun_out/${tag}_bench_cfg2a.json python - <<'PY'
import json,os
try:
    l=json.load(open(os.environ["F"]))
    print("value",l["value"],"e2e",l["e2e"]["value"],"factor_ms",l["factor_ms"])
    for k,v in l["kernels"].items(): print("  ",k,round(v["ms_per_step"],3),v.get("launches_per_step"),round(v.get("frac",0),4))
except Exception as e: print("ERR",e)
PY
