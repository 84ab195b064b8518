# full measurement pass: GPU tests, bench line (with e2e + CPU baseline), launch list, gather capture
set -e
python -m pytest tests/ -m gpu -q -x 2>&1 | tail -2
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -1 gpurun_out/bench_full.json | cut -c1-400
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err || true
tail -1 gpurun_out/bench_ref.json | cut -c1-300
bash tools/_launches.sh $1; python tools/configs_probe.py > gpurun_out/configs_$1.json
bash tools/_prof.sh gather_$1 cycle_right_gather 1
