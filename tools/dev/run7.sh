set -u
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_umma.py -x -q > $O/t_umma.log 2>&1; echo "umma rc=$?"
