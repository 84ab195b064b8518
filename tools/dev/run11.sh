set -u
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "tests rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_resid.json 2> $O/b_resid.err; echo "rc=$?"
