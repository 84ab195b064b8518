#!/bin/bash
# Round-2 closing evidence (one GPU): the GPU test suite and smoke(), every bench config with its CPU
# leg, the reference arm, launch lists of one C4 / C1 / C5c product, and `ncu --set full` captures of
# the kernels this pass added or changed (fused CholeskyQR2, row-stream energies, f16 gather,
# register four-step FFT passes). Outputs under gpurun_out/.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q > $O/r02c_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -1 $O/r02c_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/r02c_smoke.log 2>&1; echo "smoke rc=$?"
bash tools/measure_all.sh
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02c_launches_c4.csv \
  python tools/profile_c4.py --warmup 1 > /dev/null 2>&1; echo "launches c4 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02c_launches_c1.csv \
  python tools/profile_c1.py > /dev/null 2>&1; echo "launches c1 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02c_launches_c5c.csv \
  python tools/profile_c5c.py > /dev/null 2>&1; echo "launches c5c rc=$?"
cap() {  # name regex script [args]
  local name=$1 rx=$2; shift 2
  ncu --set full --import-source on --clock-control none -k regex:$rx -c 1 -o $O/r02c_$name "$@" > $O/ncu_$name.log 2>&1
  echo "$name rc=$?"
  python tools/ncu_summary.py $O/r02c_$name.ncu-rep "ncu --set full --clock-control none --import-source on -k regex:$rx -c 1; command: $*" > $O/r02c_${name}_ncu.txt 2>&1
}
cap gather_f16 cycle_gather_f16 python tools/profile_c4.py --warmup 1
cap cqr2_c4 cqr2_fused python tools/profile_c4.py --warmup 1
cap energy_rows4 cycle_energy_rows4 python tools/profile_c4.py --warmup 1
cap cqr2_c1 cqr2_fused python tools/profile_c1.py
cap fft4_pass1_r16 fft4_pass1_r16 python tools/profile_c5c.py
cap fft4_pass2_r16 fft4_pass2_r16 python tools/profile_c5c.py
