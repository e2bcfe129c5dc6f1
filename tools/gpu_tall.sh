#!/bin/bash
tag=${1:-r02o}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_golden.py tests/test_gpu_scale.py -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/${tag}_pytest.log
for leaf in 32 8; do
MPIRG_TALL_LEAF=$leaf timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_cfg4_leaf$leaf.json 2> gpurun_out/${tag}_bench_cfg4.err; echo "cfg4 leaf=$leaf rc=$?"
F=gpurun_out/${tag}_bench_cfg4_leaf$leaf.json python - <<'PY'
import json,os
try:
    l=json.load(open(os.environ["F"]))
    print("value",l["value"],"e2e",l["e2e"]["value"],"factor_ms",l["factor_ms"],"lu_gflops",l["lu_gflops"])
    for k,v in l["kernels"].items(): print("  ",k,round(v["ms_per_step"],3),v.get("launches_per_step"),round(v.get("frac",0),4))
except Exception as e: print("ERR",e)
PY
done
