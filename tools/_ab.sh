# A/B: default library vs $1 (path to an alternative _apx.so), C4 bench stages
set -e
for lib in default $1; do
  if [ "$lib" != default ]; then export APX_LIB=$lib; fi
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$lib', round(d['value'],1), {k[:14]: round(v*1000) for k,v in d.get('stages_ms').items()})
"
done
