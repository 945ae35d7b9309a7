# GPU box: k_apply timing + state hashes (tools/apply_diff.py), the explosion replay, apply parity suites
OUT=gpurun_out/${1:-aq}; mkdir -p $OUT
for args in "nasrnn 4096 600" "resnext50 4096 600"; do
  timeout 300 python tools/apply_diff.py $args > $OUT/a.log 2>&1; echo "$args: $(tail -1 $OUT/a.log | cut -c1-200)"; done
timeout 600 python tools/explode_probe.py > $OUT/probe.log 2>&1; tail -3 $OUT/probe.log
timeout 1200 python -m pytest -q -x --timeout 900 -p no:cacheprovider tests/test_gpu_apply.py tests/test_dropin_gpu.py tests/test_gpu_mcts_parity.py tests/test_gpu_snapshot.py > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
