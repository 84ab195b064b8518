set -e
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'circ|big_dA|fft|topk|sum|kept|gather|transpose|dft|pair|reduce|scale|mag|select' --log-file gpurun_out/launches_c3.csv python tools/profile_c3.py > gpurun_out/ncu_c3.log 2>&1 || tail -5 gpurun_out/ncu_c3.log
