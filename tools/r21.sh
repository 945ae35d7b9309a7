OUT=gpurun_out/r21; mkdir -p $OUT
timeout 1200 python -m pytest -q -x --timeout 900 -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_c4.py tests/test_gpu_apply.py tests/test_mcts.py tests/test_gpu_configs.py > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for B in 4096 16384; do timeout 300 python bench.py --batch $B --steps 30 --no-configs --no-mcts --no-cpu-baseline > $OUT/b$B.log 2>&1
  tail -1 $OUT/b$B.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($B, round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['kernel_ms'], d['parity_vs_reference'])"; done
timeout 300 python bench.py --model nasrnn --batch 4096 --steps 30 --no-configs --no-mcts --no-cpu-baseline > $OUT/nas.log 2>&1
tail -1 $OUT/nas.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nasrnn', round(d['value']), d['kernel_ms'], d['parity_vs_reference'])"
timeout 600 python tools/mcts_profile.py nasrnn 128 32 > $OUT/prof.log 2>&1; head -14 $OUT/prof.log
