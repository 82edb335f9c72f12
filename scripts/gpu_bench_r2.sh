#!/bin/bash
# round-2 measurement session: bench (both arms), the ncu launch list of the bench
# command, and one ncu --set full capture of the two simulation waves
OUT=gpurun_out; mkdir -p $OUT; T=${1:-r2}
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python bench.py > $OUT/bench_$T.json 2> $OUT/bench_$T.err; echo "bench exit $?"
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$T.json 2> $OUT/bench_ref_$T.err; echo "ref exit $?"
if [[ "${2:-}" == *l* ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_$T.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    --no-configs --no-api > $OUT/bench_ncu_$T.log 2>&1; echo "launches exit $?"
fi
if [[ "${2:-}" == *n* ]]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 2 \
    -f -o $OUT/sim_full_$T python scripts/profile_sweep.py 64 > $OUT/sim_full_$T.log 2>&1
  echo "sim full exit $?"
fi
tail -c 300 $OUT/bench_$T.json; tail -c 300 $OUT/bench_ref_$T.json
