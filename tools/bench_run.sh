# GPU box: the default bench line, then the ncu launch list of the headline step (gpurun_out/$1)
OUT=gpurun_out/${1:-bench}
mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.log 2>&1; tail -1 $OUT/bench.log | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-configs --no-mcts --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_bench.log 2>&1
echo "ncu rc $?"; grep -c k_ $OUT/launches.csv
