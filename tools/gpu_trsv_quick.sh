#!/bin/bash
# quick TRSV iteration: block timeline (debug lib), solve-level parity tests, cfg2a bench line
tag=${1:-r02q}
mkdir -p gpurun_out
MPIRG_LIB=libmpir_gpu_dbg.so python tools/run_solve.py 4096 1 > gpurun_out/trsv_timeline.txt 2>&1
grep "^L b=1[0-3] \|^U b=1[0-3] " gpurun_out/trsv_timeline.txt | awk '{print $1,$2,$4,$5,$6,$7,$8,$9,$10,$11,$12}'
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ir.py -x -q -k "solve or trsv or ir or division" > gpurun_out/${tag}_pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${tag}_pytest_quick.log
timeout 900 python bench.py --no-also --no-cpu-baseline > gpurun_out/${tag}_bench_cfg2a.json 2> gpurun_out/${tag}_bench_cfg2a.err; echo "cfg2a rc=$?"
F=gpurun_out/${tag}_bench_cfg2a.json python - <<'PY'
import json,os
try:
    l=json.load(open(os.environ["F"]))
    print("value",l["value"],"e2e",l["e2e"]["value"],"factor_ms",l.get("factor_ms"))
    for k,v in l["kernels"].items(): print("  ",k,round(v["ms_per_step"],3),v.get("launches_per_step"),round(v.get("frac",0),4))
except Exception as e: print("ERR",e)
PY
