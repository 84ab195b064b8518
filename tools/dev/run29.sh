set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_circulant.py tests/test_gpu_sharded_circ.py -x -q > $O/t_circ.log 2>&1; echo "tests rc=$?"
python tools/c3_time.py > $O/c3_time.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python tools/profile_c3.py > $O/ncu_c3.log 2>&1
