# GPU box: k_apply timing vs the heavy-leaf threshold (ESAT_APPLY_HEAVY)
OUT=gpurun_out/${1:-as}; mkdir -p $OUT
for H in ${HS:-256 512 1000000}; do
for args in "nasrnn 4096 600" "resnext50 4096 600"; do
  ESAT_APPLY_HEAVY=$H timeout 300 python tools/apply_diff.py $args > $OUT/a.log 2>&1; echo "H=$H $args: $(tail -1 $OUT/a.log | cut -c1-120)"; done; done
timeout 600 python tools/explode_probe.py > $OUT/probe.log 2>&1; tail -1 $OUT/probe.log
