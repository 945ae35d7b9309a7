OUT=gpurun_out/${1:-pa}; mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply -s 1 -c 1 -f -o $OUT/full_apply python tools/apply_diff.py nasrnn 4096 600 > $OUT/ncu.log 2>&1; echo ncu $?
