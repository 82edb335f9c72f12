#!/bin/bash
# quick check of a DES-step change: parity subset, sweep timing, dense families, C1/C3
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_trace.py -q -x -p no:cacheprovider 2>&1 | tail -1
python scripts/variants.py _one 64 2>&1 | tail -1
FS_FAMILIES=AB timeout 300 python scripts/profile_sweep.py 64 2>&1 | head -3
python -c "
import json, bench
r = bench.bench_configs(0)
print(json.dumps({k: round(v['ms'], 1) for k, v in r.items() if 'C1' in k or 'C3' in k}))" 2>&1 | tail -1
