#!/bin/bash
# ncu captures for profiles/ (one GPU; each command first runs clean without ncu):
#   launch list of the default bench (config 1) and --set full of the roofline kernels
set -u
mkdir -p gpurun_out/prof
P=gpurun_out/prof
NCU="ncu --clock-control none"
# config 1 launch list (same command as the bench line, per-launch times)
$NCU --metrics gpu__time_duration.sum -c 600 --csv --log-file $P/cfg1_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-incremental > $P/cfg1_launches.log 2>&1
# config 1 full sets: hess_mult, SRHT passes, Cholesky, Gram
$NCU --set full --import-source on -k regex:"k_hess_tma|k_fwht|k_chol|k_gemm|gemm" -c 10 -o $P/cfg1_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-incremental > $P/cfg1_full.log 2>&1
# config 2 SJLT streamed accumulation at m = 2048 (2^20 x 2048 fp64)
WHICH=sjlt MS=2048 $NCU --set full --import-source on -k regex:k_sjlt_pipe -c 1 -o $P/cfg2_sjlt_full \
  python tools/sketch_probe.py > $P/cfg2.log 2>&1
# config 3 TF32 tcgen05 Gaussian sketch at m = 2048 (2^21 x 4096 fp32)
MS=2048 REPS=1 $NCU --set full --import-source on -k regex:k_gauss_tc -c 1 -o $P/cfg3_tc_full \
  python tools/tc_probe.py > $P/cfg3.log 2>&1
# config 4 block-SRHT passes (2^21-row fp32 block, 1024 columns) at m = 4096 and m = 32768
for M in 4096 32768; do
  M=$M REPS=1 $NCU --set full --import-source on -k regex:"k_fwht_pipe|k_srht_combine" -c 3 -o $P/cfg4_srht_m$M \
    python tools/srht_one.py > $P/cfg4_m$M.log 2>&1
done
ls -la $P
