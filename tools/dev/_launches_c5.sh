set -e
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'cycle|topk|energy|extract|sum_vector|kept|materialize' --log-file gpurun_out/launches_c5.csv python tools/profile_c5.py > gpurun_out/ncu_c5.log 2>&1 || tail -5 gpurun_out/ncu_c5.log
