set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_mixed.py -x -q -s -k "resid or c4_shape" > $O/t_mixed.log 2>&1; echo "tests rc=$?"
for cfg in 512x4 1024x2 512x2; do
  for ct in 132 148; do
    APX_F16_CFG=$cfg APX_GATHER_CTAS=$ct python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_${cfg}_${ct}.json 2> $O/b_${cfg}_${ct}.err; echo "$cfg $ct rc=$?"
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_resid.csv python tools/profile_c4.py --warmup 1 > $O/ncu_l.log 2>&1; echo "ncu rc=$?"
