# Env sweep of panel cluster size / SM partition on cfg2a, plus the cfg5a bench line.
set -x
mkdir -p gpurun_out
for cs in 16 12 8; do for g in 16 24 12; do
  MPIRG_PANEL_MAXCS=$cs MPIRG_LU_GREEN=$g timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/sw_${cs}_${g}.json 2>/dev/null
done; done
timeout 900 python bench.py --config cfg5a --steps 2 --warmup 3 > gpurun_out/bench_cfg5a.json 2> gpurun_out/bench_cfg5a.err
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/sw_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"] * 1e3, 3), round(d["factor_ms"], 3), round(d["kernels"]["panel"]["ms_per_step"], 3))
    except Exception as e:
        print(f, "ERR", e)
PY
tail -3 gpurun_out/bench_cfg5a.err; cut -c1-1500 gpurun_out/bench_cfg5a.json
