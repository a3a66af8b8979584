#!/bin/bash
# Dev loop on the GPU box: parity tests, kernel timing, stage trace.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
{
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
python scripts/kprof.py --modes ${MODES:-1} --flags ${FLAGS:-0,2} 2>&1 | tail -8
for l in 0 1 2; do python scripts/ktrace.py --layer $l 2>&1 | grep -v "^ cta"; done
} > gpurun_out/dev.txt 2>&1
cat gpurun_out/dev.txt
