mkdir -p gpurun_out
timeout 300 python tools/time_refactor.py 4096
MPIRG_STREAMED_H2D=0 timeout 300 python tools/time_refactor.py 4096
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b2a.json 2>&1
python tools/bsum.py gpurun_out/b2a.json
python -c "
import json
d=json.loads(open('gpurun_out/b2a.json').read().strip().splitlines()[-1]); print('e2e', d['e2e'])"
timeout 600 python tools/time_refactor.py 16384
