set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_c4_full.py -x -q -s > $O/t_mixed.log 2>&1; echo "tests rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_resid.json 2> $O/bench_resid.err; echo "resid rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_resid.csv python tools/profile_c4.py --warmup 1 > $O/ncu_l.log 2>&1; echo "ncu rc=$?"
