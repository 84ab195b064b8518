set -u
O=gpurun_out
python tools/c3_time.py > $O/c3_time.txt 2>&1
APX_DA_ROWS=32 python tools/c3_time.py >> $O/c3_time.txt 2>&1
APX_DA_ROWS=32 timeout 600 python -m pytest tests/test_gpu_circulant.py -x -q > $O/t_circ.log 2>&1; echo "tests rc=$?"
APX_DA_ROWS=32 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:big_dA --csv python tools/profile_c3.py > $O/ncu_da.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:big_dA --csv python tools/profile_c3.py >> $O/ncu_da.csv 2>&1
