# GPU box: k_apply leaf order (ESAT_APPLY_ORDER) A/B
OUT=gpurun_out/${1:-ao}; mkdir -p $OUT
for O in 0 1 0 1; do
for args in "nasrnn 4096 600" "resnext50 4096 600"; do
  ESAT_APPLY_ORDER=$O timeout 300 python tools/apply_diff.py $args > $OUT/a.log 2>&1; echo "O=$O $args: $(tail -1 $OUT/a.log | cut -c1-150)"; done; done
