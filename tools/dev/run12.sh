set -u
O=gpurun_out
python tools/gemm_probe.py > $O/gemm_probe.txt 2>&1
for c in 1 2 4 8; do APX_EN_CPS=$c python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/en_$c.json 2> $O/en_$c.err; echo "$c rc=$?"; done
