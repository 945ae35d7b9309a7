# GPU box: k_extract class-group width sweep (ESAT_EXTRACT_GROUP): parity per width, then timing
OUT=gpurun_out/${1:-xg}; mkdir -p $OUT
for G in ${GROUPS_TO_TEST:-8 1 4 16 32}; do
  ESAT_EXTRACT_GROUP=$G timeout 900 python -m pytest -q -x --timeout 600 -p no:cacheprovider tests/test_gpu_parity.py \
    tests/test_gpu_configs.py tests/test_gpu_scale.py -k "extract or config or scale" > $OUT/pytest_g$G.log 2>&1
  echo "G=$G $(tail -1 $OUT/pytest_g$G.log)"
  for m in resnext50 nasrnn bert; do
    for B in 4096 16384; do
      [ $m != resnext50 ] && [ $B = 16384 ] && continue
      ESAT_EXTRACT_GROUP=$G timeout 300 python bench.py --model $m --batch $B --steps 20 --no-configs --no-mcts --no-cpu-baseline > $OUT/g${G}_${m}_$B.log 2>&1
      tail -1 $OUT/g${G}_${m}_$B.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  G=$G $m $B', round(d['value']), d['kernel_ms'], d['parity_vs_reference'])" 2>&1 | tail -1
    done
  done
done
