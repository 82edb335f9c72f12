#!/bin/bash
# ad-hoc GPU session: GPU test suite + per-instance cycle profile of the C5 sweep
OUT=gpurun_out; mkdir -p $OUT
export PYTHONDONTWRITEBYTECODE=1
T=${1:-diag}
if [[ "${2:-t}" == *t* ]]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:-} > $OUT/gpu_tests_$T.log 2>&1
  echo "gpu tests exit $?"; tail -5 $OUT/gpu_tests_$T.log
fi
if [[ "${2:-t}" == *p* ]]; then
  timeout 600 python scripts/profile_sweep.py 64 > $OUT/profile_sweep_$T.txt 2>&1
  echo "profile exit $?"; cat $OUT/profile_sweep_$T.txt | tail -15
fi
if [[ "${2:-t}" == *b* ]]; then
  timeout 900 python bench.py > $OUT/bench_$T.json 2> $OUT/bench_$T.err
  echo "bench exit $?"; tail -c 300 $OUT/bench_$T.json
fi
