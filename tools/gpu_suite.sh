# GPU box: the full -m gpu suite, then an MCTS search profile (logs under gpurun_out/$1)
OUT=gpurun_out/${1:-suite}
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
tail -15 $OUT/pytest_gpu.log
timeout 600 python tools/mcts_profile.py nasrnn 128 32 > $OUT/prof_nasrnn.log 2>&1; head -40 $OUT/prof_nasrnn.log
