# GPU box: the default bench line (per_config shows each leaf set's level width and tuned lanes), then -m gpu
OUT=gpurun_out/${1:-s3c}; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.log 2>&1; tail -1 $OUT/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('head', round(d['value']), 'e2e', round(d['e2e']['value']), d['ms_per_step'], d['kernel_ms'], d['extract_lanes'], d['extract_level_width'], d['parity_vs_reference'])
for m,r in d['per_config'].items(): print(m, round(r['value']), r['kernel_ms'], r['extract_lanes'], r['extract_level_width'], r['parity_vs_reference'])"
timeout 2000 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
