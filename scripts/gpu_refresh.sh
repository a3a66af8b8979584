#!/bin/bash
# GPU-box helper: every bench config, the reference arm, the launch list and
# full ncu captures of K1 (BERT TW step) and K2 (BERT TEW step).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-final}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1
for cfg in bert bert_tew bert_tvw big cfg1; do
  timeout 600 python bench.py --config $cfg > gpurun_out/bench_${cfg}_${TAG}.json 2> gpurun_out/bench_${cfg}_${TAG}.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference_${TAG}.json 2> gpurun_out/bench_reference_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tw_gemm_kernel \
    -s 6 -c 3 -o gpurun_out/prof_k1_${TAG} -f python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_k1_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tw_residual_kernel \
    -s 3 -c 3 -o gpurun_out/prof_k2_${TAG} -f python bench.py --config bert_tew --steps 3 --warmup 3 > gpurun_out/ncu_k2_${TAG}.log 2>&1
echo done
