# GPU box, end of round 2: smoke, the full -m gpu suite, the default bench line, the reference arm and
# the ncu launch list of the short bench (each ncu run after the same command exited 0) -> gpurun_out/$1
OUT=gpurun_out/${1:-final2}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.csv 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?"; tail -1 $OUT/smoke.log
timeout 2000 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.log 2>&1; tail -1 $OUT/bench.log > $OUT/bench.json; cut -c1-400 $OUT/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref.log 2>&1; tail -1 $OUT/ref.log > $OUT/reference_arm.json; cut -c1-300 $OUT/reference_arm.json
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-mcts --quick --e2e-steps 2"
timeout 300 python bench.py $ARGS > $OUT/short.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py $ARGS > $OUT/ncu_launches.log 2>&1; echo "launches $?"
