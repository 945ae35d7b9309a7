# GPU box: k_extract A/B -- parity suites on the default lib, then timing of each ESAT_LIB variant
# (in-tree builds under paper_2410_05534_b200/_lib) on the ResNeXt / NasRNN / BERT leaf sets.
# Usage: bash tools/ab_extract.sh TAG "libA.so libB.so ..."
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
LIBS="$2"; SETS="${3:-resnext50:16384 resnext50:4096 nasrnn:4096 bert:4096}"
[ -n "$NOPARITY" ] || timeout 900 python -m pytest -q -x --timeout 600 -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_scale.py tests/test_gpu_c4.py tests/test_gpu_many_patterns.py > $OUT/pytest_xt.log 2>&1
echo "parity: $(tail -1 $OUT/pytest_xt.log)"
for rep in ${REPS:-1}; do
for V in $LIBS; do
  for mb in $SETS; do
    M=${mb%%:*}; B=${mb##*:}
    ESAT_LIB=$V timeout 300 python bench.py --model $M --batch $B --steps 30 --no-configs --no-mcts --no-cpu-baseline --quick --e2e-steps 3 > $OUT/${V}_${M}_$B.log 2>&1
    tail -1 $OUT/${V}_${M}_$B.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V $M $B', round(d['value']), 'step', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms'].items()}, d['parity_vs_reference'])" 2>&1 | tail -1
  done
done
done
