OUT=gpurun_out/${1:-aq}; mkdir -p $OUT
for args in "nasrnn 4096 600" "resnext50 4096 600" "nasrnn 64 30000"; do
  timeout 300 python tools/apply_diff.py $args > $OUT/a.log 2>&1; echo "$args: $(tail -1 $OUT/a.log | cut -c60-190)"; done
ESAT_APPLY_NO_POT=1 timeout 300 python tools/apply_diff.py resnext50 4096 600 > $OUT/a.log 2>&1; echo "nopot resnext: $(tail -1 $OUT/a.log | cut -c60-190)"
timeout 1200 python -m pytest -q -x --timeout 900 -p no:cacheprovider tests/test_gpu_apply.py tests/test_dropin_gpu.py tests/test_gpu_mcts_parity.py > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
