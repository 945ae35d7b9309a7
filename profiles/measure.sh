#!/usr/bin/env bash
# One measurement pass on a B200 box (run through gpurun from the repo root):
#   bench line, reference arm, ncu launch list, one `ncu --set full` capture per kernel.
# Every ncu command runs only after the same program has exited 0 without ncu.
# Usage: bash profiles/measure.sh TAG      -> gpurun_out/TAG/...
set -u
TAG=${1:-meas}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/smi.csv" 2>&1
timeout 600 python bench.py > "$OUT/bench.log" 2>&1 || { echo "bench failed"; tail -n 20 "$OUT/bench.log"; exit 1; }
tail -n 1 "$OUT/bench.log" > "$OUT/bench.json"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/ref.log" 2>&1
tail -n 1 "$OUT/ref.log" > "$OUT/reference_arm.json"
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-mcts --e2e-steps 2"
timeout 300 python bench.py $ARGS > "$OUT/short.log" 2>&1 || { echo "short bench failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py $ARGS > "$OUT/ncu_launches.log" 2>&1
for k in rebuild ematch join extract; do
    timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_${k}" -s 3 -c 1 -f \
        -o "$OUT/full_$k" python bench.py $ARGS > "$OUT/ncu_full_$k.log" 2>&1
done
ls -la "$OUT"
cat "$OUT/bench.json" | cut -c1-600
