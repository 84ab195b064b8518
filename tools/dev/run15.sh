set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_mixed.py tests/test_gpu_sharded.py tests/test_gpu_batch.py -x -q > $O/t_svd.log 2>&1; echo "tests rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_resid.json 2> $O/b_resid.err; echo "rc=$?"
python tools/c1_latency.py > $O/c1_lat.txt 2>&1; echo "c1 rc=$?"
APX_CHOL256=1 python tools/c1_latency.py > $O/c1_lat_old.txt 2>&1; echo "c1 rc=$?"
