#!/bin/bash
# ncu evidence for round 2 (one GPU): the config-1 launch list, and --set full
# captures of the fused SRHT (m = 32 and 4096 of a solve), the DMMA Gram and
# the dataflow Cholesky (k = 1024).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-incremental"
$CMD > gpurun_out/ncu_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_cfg1_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_srht_fused -s 8 -c 1 -o gpurun_out/r02_srht_m32 -f $CMD > gpurun_out/ncu_srht32.log 2>&1
echo "srht m=32 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_srht_fused -s 15 -c 1 -o gpurun_out/r02_srht_m4096 -f $CMD > gpurun_out/ncu_srht4096.log 2>&1
echo "srht m=4096 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_gram_dmma -s 2 -c 2 -o gpurun_out/r02_gram -f $CMD > gpurun_out/ncu_gram.log 2>&1
echo "gram rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_chol_df -s 6 -c 1 -o gpurun_out/r02_chol -f $CMD > gpurun_out/ncu_chol.log 2>&1
echo "chol rc=$?"
SHAPES=2 python tools/gauss64_bench.py > /dev/null 2>&1 && SHAPES=2 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tn_dmma -s 2 -c 1 -o gpurun_out/r02_gauss64 -f python tools/gauss64_bench.py > gpurun_out/ncu_gauss64.log 2>&1
echo "gauss64 rc=$?"
