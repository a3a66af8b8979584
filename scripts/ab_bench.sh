#!/bin/bash
# A/B of bench.py lines under environment settings: ab_bench.sh CONFIG "ENV1" "ENV2" ...
# (each setting run twice, interleaved; prints ms/step, speedup, clocks)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
cfg=$1; shift
for rep in 1 2; do
  for e in "$@"; do
    env $e timeout 600 python bench.py --config $cfg 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$cfg', '$e', round(d['ms_per_step']*1e3,2), 'us', round(d['speedup_vs_cublas'],3), d['step'].get('sm_budgets'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
