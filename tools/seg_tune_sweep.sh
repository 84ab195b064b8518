# same-box A/B of the segmented gathers' epilogue / search variant (cycle.cu seg_tune)
for rep in 1 2; do
for t in 0 1; do echo "APX_SEG_TUNE=$t"; APX_SEG_TUNE=$t python bench.py --config c5 --no-cpu-baseline --steps 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['clocks'])"; done
done
for t in 0 1; do echo "APX_SEGH_TUNE=$t"; APX_SEGH_TUNE=$t python tools/seg_f16_probe.py 2>&1 | head -1; done
