# GPU box: k_extract lane-group A/B. Entries "lib:lanes" (ESAT_LIB, ESAT_EXTRACT_LANES); parity suites
# first for every lanes value given in $3 (on the default lib), then timing per entry.
# Usage: bash tools/ab_lanes.sh TAG "libA.so:32 libA.so:16 ..." "16 8" ["model:batch ..."]
OUT=gpurun_out/${1:-al}; mkdir -p $OUT
SETS="${4:-resnext50:16384 nasrnn:4096 bert:4096}"
for G in $3; do
  ESAT_EXTRACT_LANES=$G timeout 900 python -m pytest -q -x --timeout 600 -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_scale.py -k "extract or config or scale" > $OUT/pytest_g$G.log 2>&1
  echo "parity lanes=$G: $(tail -1 $OUT/pytest_g$G.log)"
done
for E in $2; do
  V=${E%%:*}; G=${E##*:}
  for mb in $SETS; do
    M=${mb%%:*}; B=${mb##*:}
    ESAT_LIB=$V ESAT_EXTRACT_LANES=$G timeout 300 python bench.py --model $M --batch $B --steps 30 --no-configs --no-mcts --no-cpu-baseline --quick --e2e-steps 3 > $OUT/${V}_${G}_${M}_$B.log 2>&1
    tail -1 $OUT/${V}_${G}_${M}_$B.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V lanes=$G $M $B', round(d['value']), 'step', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms'].items()}, d['parity_vs_reference'])" 2>&1 | tail -1
  done
done
