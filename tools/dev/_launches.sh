# launch list of one C4 product (ncu, per-kernel durations); usage: bash tools/_launches.sh TAG
set -e
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python tools/profile_c4.py --warmup 1 > gpurun_out/ncu_$1.log 2>&1 || tail -5 gpurun_out/ncu_$1.log
