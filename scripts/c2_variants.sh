#!/bin/bash
# time the g4 C2 kernel in each built variant library (scripts/variants.py build ... SRC=fs_costs.cu)
for v in "$@"; do
  echo "variant $v"
  FS_ENGINE_LIB=paper_2508_03148_b200/lib/variants/$v.so python scripts/c2_time.py ${C2MODE:-g4a} | grep "\"${C2MODE:-g4a}\""
done
