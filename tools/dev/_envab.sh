# C4 bench under several environment settings: bash tools/_envab.sh "" "APX_X=1" "APX_X=1 APX_Y=2" ...
for cfg in "$@"; do
  env $cfg python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/envab.json 2> gpurun_out/envab.err || tail -3 gpurun_out/envab.err
  python -c "
import json; d=json.loads(open('gpurun_out/envab.json').read().strip().splitlines()[-1])
print('[$cfg]', round(d['value'],1), {k[:14]: round(v*1000) for k,v in d.get('stages_ms').items()})
"
done
