set -e
rm -f gpurun_out/c3_$1.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:"$2" -c 1 -o gpurun_out/c3_$1 python tools/profile_c3.py > gpurun_out/ncu_c3_$1.log 2>&1 || tail -5 gpurun_out/ncu_c3_$1.log
