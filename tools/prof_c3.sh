#!/bin/bash
# C3 (circulant fp64 n=4096, k=16, order 1) evidence: the bench line, the launch list of one product,
# and one `ncu --set full` capture per kernel of the product. Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
python bench.py --config c3 --steps 20 --warmup 5 > $O/r02e_bench_c3b.json 2> $O/r02e_bench_c3b.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02e_launches_c3.csv \
  python tools/profile_c3.py > $O/ncu_l3.log 2>&1; echo "launches rc=$?"
for k in circ_decompose_r16 circ_left2_r16 big_dA_win circ_right2_r16; do
  ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $O/r02e_c3_$k \
    python tools/profile_c3.py > $O/ncu_$k.log 2>&1; echo "$k rc=$?"
  python tools/ncu_summary.py $O/r02e_c3_$k.ncu-rep "ncu --set full --clock-control none --import-source on -k regex:$k -c 1; command: python tools/profile_c3.py (one C3 product)" > $O/r02e_c3_${k}_ncu.txt 2>&1
  python tools/ncu_lines.py $O/r02e_c3_$k.ncu-rep 15 > $O/r02e_c3_${k}_lines.txt 2>&1
done
