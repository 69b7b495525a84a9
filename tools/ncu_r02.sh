#!/bin/bash
# ncu evidence for round 2 (one GPU): the config-1 launch list, and --set full
# captures of the DMMA Gram, the dataflow Cholesky and the SRHT pass-1 kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-incremental"
$CMD > gpurun_out/ncu_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_cfg1_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_gram_dmma -s 2 -c 2 -o gpurun_out/r02_gram $CMD > gpurun_out/ncu_gram.log 2>&1
echo "gram rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_chol_df -s 6 -c 1 -o gpurun_out/r02_chol $CMD > gpurun_out/ncu_chol.log 2>&1
echo "chol rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:fwht --log-file gpurun_out/r02_srht_traffic.csv $CMD > gpurun_out/ncu_srht.log 2>&1
echo "srht rc=$?"
