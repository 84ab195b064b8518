set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_batch.py tests/test_gpu_errest.py tests/test_gpu_mixed.py -x -q > $O/t_svd.log 2>&1; echo "tests rc=$?"
for kk in 0 100 300; do APX_QR_KAPPA64=$kk python tools/c1_latency.py > $O/c1_$kk.txt 2>&1; done
APX_QR_KAPPA64=100 timeout 600 python bench.py --config c1 --steps 10 --warmup 3 > $O/bench_c1.json 2> $O/bench_c1.err; echo "c1b rc=$?"
