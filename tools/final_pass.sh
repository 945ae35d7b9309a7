# GPU box: smoke, the full -m gpu suite, then profiles/measure.sh (bench, reference arm, launches, ncu) -> gpurun_out/$1
OUT=gpurun_out/${1:-final}; mkdir -p $OUT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?"; tail -1 $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
bash profiles/measure.sh $1 > $OUT/measure.log 2>&1; tail -2 $OUT/measure.log | cut -c1-300
bash tools/prof_explode.sh $1 > $OUT/explode.log 2>&1; tail -3 $OUT/explode.log
