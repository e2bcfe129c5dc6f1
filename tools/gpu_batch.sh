#!/bin/bash
tag=${1:-r02h}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_kernels.py tests/test_cpp_twin.py -x -q > gpurun_out/${tag}_pytest_batch.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/${tag}_pytest_batch.log
for grp in 64 128 256; do
MPIRG_BATCH_GROUP=$grp timeout 900 python bench.py --config cfg5b --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/${tag}_bench_cfg5b_g$grp.json 2> gpurun_out/${tag}_bench_g$grp.err; echo "bench g=$grp rc=$?"; tail -2 gpurun_out/${tag}_bench_g$grp.err
F=gpurun_out/${tag}_bench_cfg5b_g$grp.json python - <<'PY'
import json,os
try:
    l=json.load(open(os.environ["F"]))
    print("value",l["value"],"e2e",l["e2e"]["value"] if l.get("e2e") else None,"all_ok",l["all_ok"],"launches",l["gpu_launches"])
    for k,v in l["kernels"].items(): print("  ",k,round(v["ms_summed_over_streams"],2),v.get("launches"),round(v.get("frac",0),4))
except Exception as e: print("ERR",e)
PY
done
