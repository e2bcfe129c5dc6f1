set -x
mkdir -p gpurun_out
for g in 16 24 32; do
MPIRG_LU_GREEN=$g MPIRG_LU_TIMELINE=1 timeout 300 python tools/run_lu.py --n 4096 --reps 2 > gpurun_out/tl4096_g$g.txt 2>&1
MPIRG_LU_GREEN=$g MPIRG_LU_TIMELINE=1 timeout 300 python tools/run_lu.py --n 16384 --reps 2 --randn 1 > gpurun_out/tl16384_g$g.txt 2>&1
grep -E "partition|chain totals|rror" gpurun_out/tl4096_g$g.txt gpurun_out/tl16384_g$g.txt
done
MPIRG_LU_GREEN=16 timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "lu" 2>&1 | tail -3
