# GPU box: the heaviest MCTS k_apply replayed alone (tools/explode_probe.py), timed, then one
# ncu --set full capture of that launch -> gpurun_out/$1
OUT=gpurun_out/${1:-pe}; mkdir -p $OUT
timeout 600 python tools/explode_probe.py > $OUT/probe.log 2>&1; cat $OUT/probe.log | tail -5
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_apply -c 1 -f \
  -o $OUT/full_explode python tools/explode_probe.py > $OUT/ncu.log 2>&1; echo ncu $?
