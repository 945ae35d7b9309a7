# GPU box: the default bench line only -> gpurun_out/$1/bench.json
OUT=gpurun_out/${1:-bo}; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.log 2>&1; tail -1 $OUT/bench.log > $OUT/bench.json; cut -c1-300 $OUT/bench.json
