# GPU tests, then the C4 bench at several persistent-gather grid sizes (APX_GATHER_CTAS; 0 = default)
python -m pytest tests/ -m gpu -q -x 2>&1 | tail -2
for g in ${GSWEEP:-0 130 0 130 0}; do
  unset APX_GATHER_CTAS
  if [ $g -gt 0 ]; then export APX_GATHER_CTAS=$g; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$g.json 2> gpurun_out/b_$g.err || tail -3 gpurun_out/b_$g.err
  python -c "
import json; d=json.loads(open('gpurun_out/b_$g.json').read().strip().splitlines()[-1])
print('G=$g', round(d['value'],1), {k[:14]: round(v*1000) for k,v in d.get('stages_ms').items()})
"
done
