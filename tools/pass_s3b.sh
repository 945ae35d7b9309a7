# GPU box: apply A/B (time + state hash per lib), then the full -m gpu suite on the default lib
OUT=gpurun_out/${1:-s3b}; mkdir -p $OUT
for V in libesat_b200_v1.so libesat_b200_v4.so; do
  for args in "nasrnn 4096 600" "resnext50 4096 600"; do
    ESAT_LIB=$V timeout 300 python tools/apply_diff.py $args > $OUT/a_$V.log 2>&1; echo "$V $args: $(tail -1 $OUT/a_$V.log | cut -c1-220)"; done
done
timeout 2000 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; tail -4 $OUT/pytest_gpu.log
