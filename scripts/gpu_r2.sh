#!/bin/bash
# Round-2 GPU session: parity tests, smoke, 2-rank (gloo, one GPU) strong-scaling bench,
# and an ncu source-level capture of both simulation waves of the C5 sweep.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_r2.sh TAG [stages]'   stages: t s m n b
set -u
TAG=${1:-r2}
STAGES=${2:-tsmn}
OUT=gpurun_out
mkdir -p $OUT
export PYTHONDONTWRITEBYTECODE=1
if [[ $STAGES == *t* ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gpu_tests_$TAG.log 2>&1
  echo "gpu tests exit $?" >> $OUT/gpu_tests_$TAG.log; tail -3 $OUT/gpu_tests_$TAG.log
fi
if [[ $STAGES == *s* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
  echo "smoke exit $?" >> $OUT/smoke_$TAG.log; tail -2 $OUT/smoke_$TAG.log
fi
if [[ $STAGES == *m* ]]; then
  FS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --scaling strong --steps 3 \
    --warmup 3 --no-c2 --no-configs --no-cpu-baseline > $OUT/bench_2rank_strong_$TAG.json \
    2> $OUT/bench_2rank_strong_$TAG.err
  echo "2-rank strong exit $?"; tail -c 600 $OUT/bench_2rank_strong_$TAG.json
fi
if [[ $STAGES == *b* ]]; then
  timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
  echo "bench exit $?"; tail -c 400 $OUT/bench_$TAG.json
fi
if [[ $STAGES == *n* ]]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 2 \
    -f -o $OUT/sim_full_$TAG python scripts/profile_sweep.py 64 > $OUT/sim_full_$TAG.log 2>&1
  echo "sim full exit $?"
  for k in analytic dense; do
    python scripts/ncu_lines.py $OUT/sim_full_$TAG.ncu-rep 60 "$k" > $OUT/sim_lines_${k}_$TAG.txt 2>&1
  done
fi
ls -la $OUT | tail -20
