#!/bin/bash
# GPU-box helper (round 2, evidence refresh): group/budget probes, host
# overhead, the VGG sweep, a 2-rank self-launched bench on one GPU, the
# sanitizers, and the per-launch DRAM traffic of the bench configs.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python scripts/group_probe.py > gpurun_out/r2_group_probe.txt 2>&1; echo "group rc=$?"
timeout 900 python scripts/budget_sweep.py > gpurun_out/r2_budget_sweep.txt 2>&1; echo "budget rc=$?"
timeout 600 python scripts/host_overhead.py > gpurun_out/r2_host_overhead.txt 2>&1; echo "host rc=$?"
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_bench_gpus2.json 2> gpurun_out/r2_bench_gpus2.err; echo "gpus2 rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_smoke.py > gpurun_out/r2_sanitize_$tool.txt 2>&1
  echo "sanitize $tool rc=$?"; tail -2 gpurun_out/r2_sanitize_$tool.txt
done
CONFIGS="bert bert_tew big" bash scripts/ncu_traffic.sh
timeout 2400 python scripts/vgg_sweep.py --out gpurun_out/r2_vgg_sweep.json > gpurun_out/r2_vgg_sweep.txt 2>&1; echo "vgg rc=$?"
