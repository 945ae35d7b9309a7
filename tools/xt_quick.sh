# GPU box: extraction parity + timing (gpurun_out/$1)
OUT=gpurun_out/${1:-xq}
mkdir -p $OUT
timeout 900 python -m pytest -q -x --timeout 600 -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_scale.py tests/test_gpu_c4.py > $OUT/pytest_xt.log 2>&1
tail -2 $OUT/pytest_xt.log
for B in 4096 16384; do
  timeout 300 python bench.py --batch $B --steps 30 --no-configs --no-mcts --no-cpu-baseline > $OUT/b$B.log 2>&1
  tail -1 $OUT/b$B.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($B, round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['kernel_ms'], d['parity_vs_reference'])"
done
timeout 300 python bench.py --model nasrnn --batch 4096 --steps 30 --no-configs --no-mcts --no-cpu-baseline > $OUT/nas.log 2>&1
tail -1 $OUT/nas.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nasrnn', round(d['value']), d['kernel_ms'], d['parity_vs_reference'])"
