#!/bin/bash
# One GPU-box pass over every bench config (round-2 evidence): the headline C4 line, the reference
# arm, and the secondary configs with their CPU legs. Outputs under gpurun_out/.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_c4_ref.json 2> $O/bench_c4_ref.err; echo "c4 ref rc=$?"
for c in c1 c2 c3 c5 c5c; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
