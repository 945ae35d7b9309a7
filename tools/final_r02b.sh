# GPU box: join/e-match parity suites + smoke after the join SMEM change, then the default bench line
OUT=gpurun_out/${1:-final4}; mkdir -p $OUT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?"
timeout 1200 python -m pytest -q -x --timeout 900 -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_c4.py tests/test_gpu_many_patterns.py tests/test_gpu_mcts_parity.py tests/test_dropin_gpu.py > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
timeout 900 python bench.py > $OUT/bench.log 2>&1; tail -1 $OUT/bench.log > $OUT/bench.json; cut -c1-300 $OUT/bench.json
