# GPU box: ncu --set full (with source) of k_extract / k_join / k_ematch / k_rebuild on the ResNeXt 16k
# bench step at HEAD (each only after the same command exited 0 without ncu) -> gpurun_out/$1
OUT=gpurun_out/${1:-s3d}; mkdir -p $OUT
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-mcts --quick --e2e-steps 2"
timeout 300 python bench.py $ARGS > $OUT/short.log 2>&1 || { echo "short bench failed"; tail -5 $OUT/short.log; exit 1; }
tail -1 $OUT/short.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py $ARGS > $OUT/ncu_launches.log 2>&1; echo "launches $?"
for k in extract join ematch rebuild; do
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_${k}" -s 6 -c 1 -f \
      -o $OUT/full_$k python bench.py $ARGS > $OUT/ncu_full_$k.log 2>&1; echo "full $k $?"
done
ls -la $OUT
