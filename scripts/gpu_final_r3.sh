#!/bin/bash
# end-of-round-2 measurement: GPU tests + smoke, bench (both arms), the launch
# list of the bench command, ncu --set full of the MoE wave and (alone) the dense
# wave of the C5 sweep, and of the C2 kernels
OUT=gpurun_out; mkdir -p $OUT; T=${1:-r3}
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gpu_tests_$T.log 2>&1; echo "tests exit $?"; tail -2 $OUT/gpu_tests_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$T.log 2>&1; echo "smoke exit $?"; tail -1 $OUT/smoke_$T.log
timeout 1200 python bench.py > $OUT/bench_$T.json 2> $OUT/bench_$T.err; echo "bench exit $?"
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$T.json 2> $OUT/bench_ref_$T.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_$T.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --no-configs --no-api > $OUT/bench_ncu_$T.log 2>&1; echo "launches exit $?"
FS_FAMILIES=C timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 1 \
  -f -o $OUT/sim_moe_$T python scripts/profile_sweep.py 64 > $OUT/sim_moe_$T.log 2>&1; echo "moe full exit $?"
FS_FAMILIES=AB timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 1 \
  -f -o $OUT/sim_dense_$T python scripts/profile_sweep.py 64 > $OUT/sim_dense_$T.log 2>&1; echo "dense full exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attention -c 2 \
  -f -o $OUT/c2_$T python scripts/c2_once.py 1 > $OUT/c2_$T.log 2>&1; echo "c2 full exit $?"
tail -c 200 $OUT/bench_$T.json
