#!/bin/bash
# GPU-box helper (round 2): full GPU test suite, every bench config, the
# reference arm, the launch list and one ncu --set full capture of K1.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.txt; tail -3 gpurun_out/r2_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; tail -1 gpurun_out/r2_smoke.txt
for cfg in ${CONFIGS:-bert bert_tew bert_tvw big cfg1}; do
  timeout 600 python bench.py --config $cfg > gpurun_out/r2_bench_${cfg}.json 2> gpurun_out/r2_bench_${cfg}.err
  echo "bench $cfg rc=$?"; tail -c 300 gpurun_out/r2_bench_${cfg}.json; echo
done
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_reference_arm.json 2> gpurun_out/r2_ref.err
echo "ref rc=$?"; tail -c 300 gpurun_out/r2_bench_reference_arm.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2_launches.csv python bench.py --steps 4 --warmup 3 > /dev/null 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tw_gemm_group_kernel \
    -s 12 -c 3 -o gpurun_out/r2_prof_k1 -f python bench.py --steps 4 --warmup 3 > gpurun_out/r2_ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -2 gpurun_out/r2_ncu_full.log
