OUT=gpurun_out/r22; mkdir -p $OUT
timeout 300 python tools/apply_diff.py nasrnn 64 30000 > $OUT/ax.log 2>&1; tail -1 $OUT/ax.log | cut -c1-300
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply -s 1 -c 1 -f -o $OUT/full_apply_explode python tools/apply_diff.py nasrnn 64 30000 > $OUT/ncu.log 2>&1; echo ncu $?
