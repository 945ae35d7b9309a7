# GPU box: headline throughput vs leaves per step (gpurun_out/$1)
OUT=gpurun_out/${1:-bb}
mkdir -p $OUT
for B in 4096 8192 16384; do
  timeout 300 python bench.py --batch $B --steps 30 --no-configs --no-mcts --no-cpu-baseline > $OUT/b$B.log 2>&1
  tail -1 $OUT/b$B.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($B, round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['kernel_ms'], d['parity_vs_reference'])"
done
