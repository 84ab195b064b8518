# ncu --set full capture of kernels matching $2 in one C4 product; usage: bash tools/_prof.sh TAG REGEX [COUNT]
set -e
rm -f gpurun_out/$1.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:$2 -c ${3:-1} -o gpurun_out/$1 python tools/profile_c4.py --warmup 1 > gpurun_out/ncu_$1.log 2>&1 || tail -5 gpurun_out/ncu_$1.log
