set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_robust.py tests/test_gpu_c4_full.py -x -q -s > $O/t_mixed.log 2>&1; echo "tests rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b27.json 2> $O/b27.err; echo "rc=$?"
APX_RESID_F16=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b27f.json 2> $O/b27f.err; echo "rc=$?"
