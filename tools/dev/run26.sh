set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_c4_full.py -x -q > $O/t_mixed.log 2>&1; echo "tests rc=$?"
for g in 0 128 256 512; do APX_EN_GROUPS=$g python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/eg_$g.json 2> $O/eg_$g.err; echo "$g rc=$?"; done
