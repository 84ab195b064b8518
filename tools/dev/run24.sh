set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_mixed.py tests/test_gpu_sharded.py tests/test_gpu_batch.py -x -q > $O/t_chol.log 2>&1; echo "tests rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b24.json 2> $O/b24.err; echo "rc=$?"
APX_CHOL_BARRIER=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b24b.json 2> $O/b24b.err; echo "rc=$?"
python tools/c1_latency.py > $O/c1_lat.txt 2>&1
APX_CHOL_BARRIER=1 python tools/c1_latency.py >> $O/c1_lat.txt 2>&1
