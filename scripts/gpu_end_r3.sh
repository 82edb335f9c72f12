#!/bin/bash
# end-of-session check: GPU tests, smoke, bench (both arms)
OUT=gpurun_out; mkdir -p $OUT; T=${1:-r3e}
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gpu_tests_$T.log 2>&1; echo "tests exit $?"; tail -2 $OUT/gpu_tests_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$T.log 2>&1; echo "smoke exit $?"; tail -1 $OUT/smoke_$T.log
timeout 1200 python bench.py > $OUT/bench_$T.json 2> $OUT/bench_$T.err; echo "bench exit $?"
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$T.json 2> $OUT/bench_ref_$T.err; echo "ref exit $?"
tail -c 300 $OUT/bench_$T.json
