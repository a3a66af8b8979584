#!/bin/bash
# GPU-box helper: bench line(s), launch list and one full ncu capture of K1.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
for cfg in ${CONFIGS:-bert}; do
  timeout 600 python bench.py --config $cfg ${BENCH_ARGS:-} > gpurun_out/bench_${cfg}_${TAG}.json 2> gpurun_out/bench_${cfg}_${TAG}.err
  echo "bench $cfg rc=$?"; cat gpurun_out/bench_${cfg}_${TAG}.json; tail -5 gpurun_out/bench_${cfg}_${TAG}.err
done
if [ -n "${NCU:-1}" ] && [ "${NCU:-1}" != "0" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 > /dev/null 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tw_gemm_kernel \
      -s 6 -c 3 -o gpurun_out/prof_${TAG} -f python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_full_${TAG}.log 2>&1
  echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full_${TAG}.log
fi
