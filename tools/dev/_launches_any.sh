# launch list of one product: bash tools/_launches_any.sh TAG SCRIPT
set -e
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python $2 > gpurun_out/ncu_$1.log 2>&1 || tail -5 gpurun_out/ncu_$1.log
