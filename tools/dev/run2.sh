set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_c4_full.py tests/test_gpu_umma.py -x -q -s > $O/t_mixed.log 2>&1; echo "tests rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_resid.json 2> $O/bench_resid.err; echo "resid rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --plan direct > $O/bench_direct.json 2> $O/bench_direct.err; echo "direct rc=$?"
