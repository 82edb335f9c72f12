#!/bin/bash
# quick GPU iteration: full gpu tests + the C5 sweep bench line (no C2 / configs / CPU legs)
OUT=gpurun_out; mkdir -p $OUT; T=${1:-q}
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gpu_tests_$T.log 2>&1; echo "tests exit $?"; tail -2 $OUT/gpu_tests_$T.log
timeout 600 python bench.py --no-c2 --no-configs --no-cpu-baseline --no-api > $OUT/bench_$T.json 2> $OUT/bench_$T.err; echo "bench exit $?"
python -c "
import json;d=json.loads(open('$OUT/bench_$T.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e']['value']/1e6, 'clocks', d.get('clocks'))"
