set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_batch.py tests/test_gpu_errest.py -x -q > $O/t_svd.log 2>&1; echo "tests rc=$?"
python tools/c1_latency.py > $O/c1_lat.txt 2>&1; echo "c1 rc=$?"
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err; echo "c1b rc=$?"
