# GPU box: apply parity + timing (gpurun_out/$1)
OUT=gpurun_out/${1:-ap}; mkdir -p $OUT
for args in "nasrnn 4096 600" "resnext50 4096 600" "nasrnn 64 30000"; do
  timeout 300 python tools/apply_diff.py $args > $OUT/a.log 2>&1; echo "$args: $(tail -1 $OUT/a.log | cut -c1-220)"; done
timeout 1200 python -m pytest -q -x --timeout 900 -p no:cacheprovider tests/test_gpu_apply.py tests/test_dropin_gpu.py tests/test_mcts.py tests/test_gpu_mcts_parity.py tests/test_gpu_refpatch.py > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 600 python tools/mcts_profile.py nasrnn 128 32 > $OUT/prof.log 2>&1; head -12 $OUT/prof.log
