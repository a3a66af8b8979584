#!/bin/bash
# GPU-box helper: DRAM bytes per kernel launch for every bench config
# (dram__bytes_read/write; ncu flushes L2 before each launch), for
# profiles/ncu_traffic.json.  Launch lists only -- never a bench value.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in ${CONFIGS:-bert bert_tew bert_tvw big cfg1}; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:"tw_gemm_kernel|tw_residual_kernel" -c 3000 --csv \
      --log-file gpurun_out/traffic_${cfg}.csv python bench.py --config $cfg --steps 3 --warmup 3 > /dev/null 2>&1
  echo "$cfg rc=$?"
done
