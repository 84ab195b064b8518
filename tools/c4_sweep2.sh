#!/bin/bash
# C4 step time against the persistent gather's grid (SMs left to the low-priority chain), same box
cd "$(dirname "$0")/.."
for g in 132 124 128 136 140 144 132; do
  v=$(APX_GATHER_CTAS=$g python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), {k[:10]: round(v*1e3) for k,v in d['stages_ms'].items()})")
  echo "GATHER_CTAS=$g $v"
done
