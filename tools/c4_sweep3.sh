#!/bin/bash
# C4 step time: W0 = Bm.B behind dA (default) or beside it (APX_W0_EARLY=1), and its SM budget; same box
cd "$(dirname "$0")/.."
run() { v=$(env "$@" python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), {k[:10]: round(v*1e3) for k,v in d['stages_ms'].items()}, 'parity', d.get('parity_vs_oracle'))"); echo "$* $v"; }
run APX_W0_EARLY=0
run APX_W0_EARLY=1
run APX_W0_EARLY=1 APX_W0_SMS=32
run APX_W0_EARLY=1 APX_W0_SMS=64
run APX_W0_EARLY=1 APX_W0_SMS=148
run APX_W0_EARLY=1 APX_W0_SMS=64 APX_GATHER_CTAS=140
run APX_W0_EARLY=1 APX_W0_SMS=64 APX_GATHER_CTAS=144
run APX_W0_EARLY=0
