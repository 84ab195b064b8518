#!/bin/bash
# Round-2 evidence for the C4 residual plan (one GPU): the headline bench line (with the CPU leg and
# e2e), the reference arm, the all-fp32 plan for A/B, the launch list of one product, and
# `ncu --set full` captures of the f16 gather and of the plan's tcgen05 GEMMs. Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/r02_bench_c4.json 2> $O/r02_bench_c4.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $O/r02_bench_reference.json 2> $O/r02_bench_reference.err; echo "ref rc=$?"
python bench.py --plan direct --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/r02_bench_c4_direct.json 2> $O/r02_bench_c4_direct.err; echo "direct rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_c4.csv \
  python tools/profile_c4.py --warmup 1 > $O/ncu_l4.log 2>&1; echo "launches rc=$?"
ncu --set full --import-source on --clock-control none -k regex:cycle_gather_f16 -c 1 -o $O/r02_gather_f16 \
  python tools/profile_c4.py --warmup 1 > $O/ncu_g.log 2>&1; echo "gather rc=$?"
python tools/ncu_summary.py $O/r02_gather_f16.ncu-rep "ncu --set full --clock-control none --import-source on -k regex:cycle_gather_f16 -c 1; command: python tools/profile_c4.py --warmup 1 (one C4 product, n=8192, residual plan)" > $O/r02_gather_ncu.txt 2>&1
python tools/ncu_lines.py $O/r02_gather_f16.ncu-rep 20 > $O/r02_gather_lines.txt 2>&1
ncu --set full --clock-control none -k regex:gemm_tma_kernel -c 6 -o $O/r02_c4_gemms \
  python tools/profile_c4.py --warmup 0 > $O/ncu_gemm.log 2>&1; echo "gemms rc=$?"
