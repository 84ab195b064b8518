set -u
O=gpurun_out
run() { name=$1; shift; env "$@" python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/s_$name.json 2> $O/s_$name.err; echo "$name rc=$?"; }
run a_512x4_132_tile APX_F16_CFG=512x4 APX_GATHER_CTAS=132 APX_QW_TILE=1
run b_512x4_132_pers APX_F16_CFG=512x4 APX_GATHER_CTAS=132
run c_512x2_148_tile APX_F16_CFG=512x2 APX_GATHER_CTAS=148 APX_QW_TILE=1
run d_512x2_132_tile APX_F16_CFG=512x2 APX_GATHER_CTAS=132 APX_QW_TILE=1
run e_512x4_140_tile APX_F16_CFG=512x4 APX_GATHER_CTAS=140 APX_QW_TILE=1
run f_512x4_124_tile APX_F16_CFG=512x4 APX_GATHER_CTAS=124 APX_QW_TILE=1
run g_1024x2_148_tile APX_F16_CFG=1024x2 APX_GATHER_CTAS=148 APX_QW_TILE=1
