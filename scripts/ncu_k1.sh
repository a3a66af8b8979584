#!/bin/bash
# One ncu --set full capture of K1 for each BERT layer (GPU box; 1 GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-dev}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tw_gather_gemm \
   -s ${SKIP:-0} -c ${COUNT:-3} -o gpurun_out/prof_${TAG} -f python scripts/kprof.py --modes 1 --flags 0 --reps 2 > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_${TAG}.log
