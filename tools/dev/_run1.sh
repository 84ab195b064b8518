set -e
python -m pytest tests/ -q -x -m gpu 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err
python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
print(d['value'], d.get('stages_ms'), d['e2e']['value'], d.get('clocks'))
"
