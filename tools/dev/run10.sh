set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_robust.py -x -q > $O/t_mixed.log 2>&1; echo "tests rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_resid.json 2> $O/b_resid.err; echo "rc=$?"
