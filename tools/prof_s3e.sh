# GPU box: ncu --set full (with source) of k_extract on the ResNeXt 16k bench step at HEAD
OUT=gpurun_out/${1:-s3e}; mkdir -p $OUT
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-mcts --quick --e2e-steps 2"
timeout 300 python bench.py $ARGS > $OUT/short.log 2>&1 || { echo "short bench failed"; tail -5 $OUT/short.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k k_extract -s 6 -c 1 -f \
    -o $OUT/full_extract python bench.py $ARGS > $OUT/ncu_full_extract.log 2>&1; echo "full extract $?"
ls -la $OUT
