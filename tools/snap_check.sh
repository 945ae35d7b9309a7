OUT=gpurun_out/snap1; mkdir -p $OUT
timeout 900 python -m pytest -q -x --timeout 600 -p no:cacheprovider tests/test_gpu_snapshot.py tests/test_gpu_mcts_parity.py tests/test_dropin_gpu.py > $OUT/pytest.log 2>&1; tail -15 $OUT/pytest.log
timeout 600 python tools/mcts_profile.py nasrnn 128 32 > $OUT/prof_nasrnn.log 2>&1; head -30 $OUT/prof_nasrnn.log
