# ncu --set full captures of the non-gather kernels the north star asks evidence for
# (rSVD GEMMs' tensor pipe, the energy pass, the C3 FFT kernels); run after the commands exit 0
set -e
rm -f gpurun_out/ev_*.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:"gemm_tma_kernel|cycle_energy_partial" -c 5 -o gpurun_out/ev_c4 python tools/profile_c4.py --warmup 0 > gpurun_out/ncu_ev_c4.log 2>&1 || tail -3 gpurun_out/ncu_ev_c4.log
ncu --set full --import-source on --clock-control none -k regex:"circ_decompose_rows|circ_left2|circ_right2" -c 3 -o gpurun_out/ev_c3 python tools/profile_c3.py > gpurun_out/ncu_ev_c3.log 2>&1 || tail -3 gpurun_out/ncu_ev_c3.log
