#!/bin/bash
# MoE wave alone: per-instance cycles, then an ncu source-level capture + per-line summary
OUT=gpurun_out; mkdir -p $OUT; T=${1:-r3}
export PYTHONDONTWRITEBYTECODE=1
FS_FAMILIES=C timeout 300 python scripts/profile_sweep.py 64 > $OUT/moe_cycles_$T.txt 2>&1; echo "cycles exit $?"; cat $OUT/moe_cycles_$T.txt
FS_FAMILIES=C timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 1 \
  -f -o $OUT/sim_moe_$T python scripts/profile_sweep.py 64 > $OUT/sim_moe_$T.log 2>&1; echo "moe full exit $?"
python scripts/ncu_lines.py $OUT/sim_moe_$T.ncu-rep 70 > $OUT/sim_lines_moe_$T.txt 2>&1
python scripts/ncu_report_md.py $OUT/sim_moe_$T.ncu-rep $OUT/sim_moe_$T.md "MoE wave alone" > /dev/null 2>&1
ls -la $OUT | tail
