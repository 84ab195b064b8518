#!/bin/bash
# Round-2 profile pass (one GPU): launch lists of one C4 and one C3 product, and `ncu --set full`
# captures of the dominant kernels, summarised into gpurun_out/*.txt (tools/ncu_summary.py).
cd "$(dirname "$0")/.."
O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_c4.csv \
  python tools/profile_c4.py --warmup 1 > $O/ncu_l4.log 2>&1; echo "launches c4 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_c3.csv \
  python tools/profile_c3.py > $O/ncu_l3.log 2>&1; echo "launches c3 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:cycle_right_gather -c 1 -o $O/r02_gather \
  python tools/profile_c4.py --warmup 1 > $O/ncu_g.log 2>&1; echo "gather rc=$?"
python tools/ncu_summary.py $O/r02_gather.ncu-rep "# ncu --set full --clock-control none --import-source on -k regex:cycle_right_gather -c 1; command: python tools/profile_c4.py --warmup 1 (one C4 product, n=8192)" > $O/r02_gather_ncu.txt 2>&1
for k in circ_left2 circ_right2 circ_decompose_rows big_dA; do
  ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $O/r02_$k python tools/profile_c3.py > $O/ncu_$k.log 2>&1
  python tools/ncu_summary.py $O/r02_$k.ncu-rep "# ncu --set full -k regex:$k -c 1; command: python tools/profile_c3.py (one C3 product, fp64 n=4096, k=16, order 1)" > $O/r02_${k}_ncu.txt 2>&1
  echo "$k rc=$?"
done
