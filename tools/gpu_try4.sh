set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "streamed or golden or abi or twin" > gpurun_out/pytest_try4.log 2>&1
tail -3 gpurun_out/pytest_try4.log
timeout 300 python tools/e2e_probe.py > gpurun_out/probe_graph.txt 2>&1
MPIRG_STREAMED_GRAPH=0 timeout 300 python tools/e2e_probe.py > gpurun_out/probe_nograph.txt 2>&1
MPIRG_LU_TIMELINE=1 timeout 300 python tools/e2e_probe.py > gpurun_out/probe_timeline.txt 2>&1
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_try_$i.json 2>/dev/null; done
MPIRG_STREAMED_GRAPH=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_try_off.json 2>/dev/null
cat gpurun_out/probe_graph.txt gpurun_out/probe_nograph.txt
grep -v "^step" gpurun_out/probe_timeline.txt | tail -6
python - <<'PY'
import json
for f in ("gpurun_out/bench_try_1.json", "gpurun_out/bench_try_2.json", "gpurun_out/bench_try_off.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["e2e"]["value"])
PY
