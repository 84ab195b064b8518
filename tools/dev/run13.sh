set -u
O=gpurun_out
for cfg in "0 8" "0 4" "1 8"; do set -- $cfg; APX_B_ORDER=$1 APX_EN_CPS=$2 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/bo_$1_$2.json 2> $O/bo_$1_$2.err; echo "$cfg rc=$?"; done
