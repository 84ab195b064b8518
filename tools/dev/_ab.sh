# A/B: default library vs alternative _apx.so builds (args), C4 bench (value + gather span)
for lib in default "$@"; do
  if [ "$lib" != default ]; then export APX_LIB=$lib; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$lib', round(d['value'],1), 'gather', round(d['stages_ms']['M = A.Bhat (persistent row gather) [hi]']*1000,1))
" 2>/dev/null || echo "$lib failed"
done
