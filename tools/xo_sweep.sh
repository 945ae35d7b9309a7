# GPU box: k_extract leaf order (ESAT_EXTRACT_ORDER) A/B on the headline batch
OUT=gpurun_out/${1:-xo}; mkdir -p $OUT
for O in 0 1 0 1; do
  for m in resnext50 nasrnn; do
    ESAT_EXTRACT_ORDER=$O timeout 300 python bench.py --model $m --batch 16384 --steps 20 --no-configs --no-mcts --no-cpu-baseline > $OUT/o${O}_$m.log 2>&1
    tail -1 $OUT/o${O}_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('O=$O $m', round(d['value']), round(d['e2e']['value']), d['kernel_ms'], d['parity_vs_reference'])" 2>&1 | tail -1
  done
done
