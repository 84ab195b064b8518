set -u
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "gpu tests rc=$?"
python bench.py --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
timeout 600 python tools/conformance.py > $O/conformance.txt 2>&1; echo "conf rc=$?"
