#!/bin/bash
# GPU box: rebuild K1 with different stage counts and probe (diagnostics).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for st in ${STAGES:-2 3 4}; do
  TW_NVCC_EXTRA="-DTW_STAGES=$st" python -m paper_2402_10876_b200._build --force > /dev/null
  echo "stages=$st"
  python scripts/kprobe.py "${SETTINGS:-TW_TN=0}"
done
python -m paper_2402_10876_b200._build --force > /dev/null
