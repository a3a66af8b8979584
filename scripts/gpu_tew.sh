#!/bin/bash
# GPU-box helper: TEW parity tests + TEW bench line (K2 tuning loop)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "tew or fuzz" > gpurun_out/pytest_tew.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_tew.txt
tail -3 gpurun_out/pytest_tew.txt
NCU=0 CONFIGS="bert_tew" TAG=${TAG:-k2} bash scripts/gpu_bench.sh > /dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_bert_tew_${TAG:-k2}.json')); print('TEW step', d['ms_per_step'], d['speedup_vs_cublas'], [round(l['us'],1) for l in d['roofline']['layers']])"
