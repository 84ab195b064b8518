# ncu --set full of kernels matching REGEX in SCRIPT: bash tools/_prof_any.sh TAG SCRIPT REGEX [COUNT]
set -e
rm -f gpurun_out/$1.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:"$3" -c ${4:-1} -o gpurun_out/$1 python $2 > gpurun_out/ncu_$1.log 2>&1 || tail -5 gpurun_out/ncu_$1.log
