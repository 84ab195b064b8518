set -e
ncu --set full --import-source on --clock-control none -k regex:cholinv64 -c 1 -o gpurun_out/cholinv_v1 python tools/profile_c4.py --warmup 1 > gpurun_out/ncu_ch.log 2>&1 || tail -5 gpurun_out/ncu_ch.log
ncu --set full --import-source on --clock-control none -k regex:apply_x -c 1 -o gpurun_out/applyx_v1 python tools/profile_c4.py --warmup 1 > gpurun_out/ncu_ax.log 2>&1 || tail -5 gpurun_out/ncu_ax.log
