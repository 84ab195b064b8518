#!/bin/bash
# C4 step time: a 256-thread f16 gather (half the register file, 156 KB of shared memory) on every SM,
# so the low-priority chain's TMA-fed GEMM CTAs can co-reside with it; same box
cd "$(dirname "$0")/.."
run() { v=$(env "$@" python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), {k[:10]: round(v*1e3) for k,v in d['stages_ms'].items()})"); echo "$* $v"; }
run APX_F16_CFG=512x4
run APX_F16_CFG=256x4
run APX_F16_CFG=256x4 APX_GATHER_CTAS=140
run APX_F16_CFG=256x4 APX_GATHER_CTAS=148
run APX_F16_CFG=256x4 APX_GATHER_CTAS=148 APX_W0_EARLY=1 APX_W0_SMS=64
run APX_F16_CFG=512x4 APX_GATHER_CTAS=148
run APX_F16_CFG=256x2 APX_GATHER_CTAS=148
