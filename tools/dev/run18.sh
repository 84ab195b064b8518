set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_mixed.py -x -q > $O/t_mixed.log 2>&1; echo "tests rc=$?"
for i in 1 2; do python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $O/b18_$i.json 2> $O/b18_$i.err; echo "rc=$?"; done
APX_F16_CFG=1024x2 APX_GATHER_CTAS=148 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $O/b18_3.json 2> $O/b18_3.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cycle_gather_f16 -c 2 --csv python tools/profile_c4.py --warmup 1 > $O/ncu_g18.csv 2>&1
