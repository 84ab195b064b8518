set -u
O=gpurun_out
for b in 1 2; do for e in 8 4; do APX_B_ORDER=$b APX_EN_CPS=$e python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/bo_${b}_$e.json 2> $O/bo_${b}_$e.err; echo "$b $e rc=$?"; done; done
