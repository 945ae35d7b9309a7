OUT=gpurun_out/r24; mkdir -p $OUT
timeout 1200 python -m pytest -q -x --timeout 900 -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_c4.py tests/test_gpu_configs.py tests/test_gpu_apply.py tests/test_dropin_gpu.py tests/test_gpu_mcts_parity.py > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for m in resnext50 nasrnn; do timeout 300 python tools/xt_sizes.py $m > $OUT/xt_$m.log 2>&1; echo "== $m"; grep -v Warn $OUT/xt_$m.log; done
for B in 4096 16384; do timeout 300 python bench.py --batch $B --steps 30 --no-configs --no-mcts --no-cpu-baseline > $OUT/b$B.log 2>&1
  tail -1 $OUT/b$B.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($B, round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['kernel_ms'], d['parity_vs_reference'], d['apply']['kernel_ms'])"; done
