set -e
python -m pytest tests/test_gpu_mixed.py tests/test_gpu_cycle.py -q -x 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err
python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
print(d['value'], d.get('stages_ms'), d['e2e']['value'], d.get('clocks'))
"
ncu --set full --import-source on --clock-control none -k regex:cycle_right_gather -c 1 -o gpurun_out/gather_v6 python tools/profile_c4.py > gpurun_out/ncu_g6.log 2>&1 || tail -5 gpurun_out/ncu_g6.log
