#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (both arms), ncu launch list and
# one `ncu --set full` capture per top kernel. Outputs land in gpurun_out/.
#   gpurun --timeout 3000 -- 'bash scripts/gpu_round.sh [tag] [stages]'
# stages: any of t (tests) s (smoke) b (bench) r (reference arm) l (launch list) f (full ncu)
set -u
TAG=${1:-r01}
STAGES=${2:-tsbrlf}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
nproc > $OUT/nproc_$TAG.txt; lscpu | grep 'Model name' >> $OUT/nproc_$TAG.txt
export PYTHONDONTWRITEBYTECODE=1
if [[ $STAGES == *t* ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gpu_tests_$TAG.log 2>&1
  echo "gpu tests exit $?" >> $OUT/gpu_tests_$TAG.log
  tail -3 $OUT/gpu_tests_$TAG.log
fi
if [[ $STAGES == *s* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
  echo "smoke exit $?" >> $OUT/smoke_$TAG.log; tail -2 $OUT/smoke_$TAG.log
fi
if [[ $STAGES == *b* ]]; then
  timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
  echo "bench exit $?"; tail -c 1500 $OUT/bench_$TAG.json
fi
if [[ $STAGES == *r* ]]; then
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
  echo "ref exit $?"; cat $OUT/bench_ref_$TAG.json | head -c 600
fi
if [[ $STAGES == *l* ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > $OUT/launches_bench_$TAG.log 2>&1
  echo "launch list exit $?"
fi
if [[ $STAGES == *f* ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 2 \
    -f -o $OUT/sim_full_$TAG python scripts/profile_sweep.py 64 > $OUT/sim_full_$TAG.log 2>&1
  echo "sim full exit $?"
  timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:'attention_cost_kernel|attention_forest_kernel|metrics_kernel' -c 3 \
    -f -o $OUT/c2_full_$TAG python scripts/c2_once.py 1 > $OUT/c2_full_$TAG.log 2>&1
  echo "c2 full exit $?"
fi
ls -la $OUT
