set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_mixed.py -x -q -s -k "resid or c4_shape" > $O/t_mixed.log 2>&1; echo "tests rc=$?"
ncu --set full --import-source on --clock-control none -k regex:cycle_gather_f16 -c 1 -o $O/r02_gather_f16 python tools/profile_c4.py --warmup 1 > $O/ncu_g.log 2>&1; echo "ncu g rc=$?"
ncu --set full --import-source on --clock-control none -k regex:gemm_tma_kernel -c 8 -o $O/r02_c4_gemms python tools/profile_c4.py --warmup 0 > $O/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
