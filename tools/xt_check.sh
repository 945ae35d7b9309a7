# GPU box: extraction parity suites + extraction timing per leaf set (logs under gpurun_out/$1)
OUT=gpurun_out/${1:-xt}
mkdir -p $OUT
timeout 900 python -m pytest -q -x --timeout 600 -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_scale.py tests/test_gpu_c4.py tests/test_dropin_gpu.py > $OUT/pytest_xt.log 2>&1
tail -3 $OUT/pytest_xt.log
for m in nasrnn resnext50 bert; do timeout 300 python tools/xt_sizes.py $m > $OUT/xt_sizes_$m.log 2>&1; echo "== $m"; cat $OUT/xt_sizes_$m.log | grep -v Warn; done
