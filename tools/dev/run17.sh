set -u
O=gpurun_out
for y in 64 148 296 592; do APX_Y_SMS=$y python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/y_$y.json 2> $O/y_$y.err; echo "$y rc=$?"; done
