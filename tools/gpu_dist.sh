#!/bin/bash
# Distributed-LU round on one GPU: dist tests, then the distributed code path at N=16384
# against the single-GPU path (same workload family).
tag=${1:-r02b}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/${tag}_pytest_dist.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/${tag}_pytest_dist.log
python bench.py --config cfg5a --dist --n 16384 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/${tag}_bench_cfg5a_dist_n16384.json 2> gpurun_out/${tag}_dist.err; echo "dist rc=$?"; tail -3 gpurun_out/${tag}_dist.err
python bench.py --config cfg5a --n 16384 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench_cfg5a_single_n16384.json 2> gpurun_out/${tag}_single.err; echo "single rc=$?"; tail -3 gpurun_out/${tag}_single.err
TAG=$tag python - <<'PY'
import json, os
for f in ("dist","single"):
    try:
        l=json.load(open(f"gpurun_out/%s_bench_cfg5a_%s_n16384.json" % (os.environ["TAG"], f)))
        print(f, "value", l["value"], "factor", l.get("factor_s", l.get("factor_ms")), l.get("checks"))
    except Exception as e:
        print(f, "ERR", e)
PY
