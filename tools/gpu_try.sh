mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py tests/test_gpu_ir.py -m gpu -x -q 2>&1 | tail -4
for g in 0 1; do
MPIRG_LU_GRAPH=$g timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b2a_g$g.json 2>&1
MPIRG_LU_GRAPH=$g timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/b4_g$g.json 2>&1
python tools/bsum.py gpurun_out/b2a_g$g.json gpurun_out/b4_g$g.json
done
python -c "
import json
d=json.loads(open('gpurun_out/b2a_g1.json').read().strip().splitlines()[-1]); print('e2e', d['e2e'], 'prof', d['profiled_step_ms'])"
