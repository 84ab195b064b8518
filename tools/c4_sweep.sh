#!/bin/bash
# C4 step time under the plan's tuning knobs (device time only; no CPU leg / e2e)
cd "$(dirname "$0")/.."
for y in 32 64 148; do
  for g in 128 132 136; do
    v=$(APX_Y_SMS=$y APX_GATHER_CTAS=$g python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), {k[:12]: round(v*1e3) for k,v in d['stages_ms'].items()})")
    echo "Y_SMS=$y GATHER_CTAS=$g $v"
  done
done
