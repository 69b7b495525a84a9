#!/bin/bash
# ncu --set full of the fused SRHT kernel on the config-1 shape (m = 32 and 4096)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export N=65536 D=1024 DT=f64 REPS=2 ADASK_SRHT_FUSED_PF=${ADASK_SRHT_FUSED_PF:-0}
for M in 32 4096; do
  M=$M python tools/srht_one.py > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
  M=$M ncu --set full --clock-control none --import-source on -k regex:k_srht_fused -s 1 -c 1 \
     -o gpurun_out/fused_m$M -f python tools/srht_one.py > gpurun_out/ncu_fused_m$M.log 2>&1
  echo "m=$M rc=$?"
done
