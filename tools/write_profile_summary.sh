#!/bin/bash
# Regenerate profiles/r01_ncu_full_summary.md from the captures in gpurun_out/prof
set -e
cd /root/repo
{
  echo "# r01 ncu --set full summaries (B200, --clock-control none)"
  echo
  echo "Per-launch values from \`ncu -i <rep> --page raw\` (tools/ncu_summary.py). DRAM % is of ncu's"
  echo "theoretical peak; the bench roofline uses MEASURED_PEAKS.json instead. Absolute durations under"
  echo "ncu are cold-cache and serialised; compare shares, not absolutes, with the bench."
  echo
  echo "## config 1 (bench.py default: ada-PCG, SRHT, fp64, 2^16 x 1024) -- cfg1_full.ncu-rep"
  echo
  python tools/ncu_summary.py gpurun_out/prof/cfg1_full.ncu-rep
  echo
  echo "## config 3 sketch kernel (TF32 tcgen05, m = 2048, n = 2^21, d = 4096) -- cfg3_tc_full.ncu-rep"
  echo
  python tools/ncu_summary.py gpurun_out/prof/cfg3_tc_full.ncu-rep
  echo
  echo "SASS of k_gauss_tc: $(cuobjdump -sass build/adask/gauss_tc.o | grep -oE 'UTC[A-Z]*MMA[.A-Z0-9]*|UTMALDG[.A-Z0-9]*|LDTM' | sort | uniq -c | tr '\n' ';' | tr -s ' ')"
  echo
  echo "## config 2 sketch kernel (SJLT, fp64 2^20 x 2048, m = 2048) -- cfg2_sjlt_full.ncu-rep"
  echo
  python tools/ncu_summary.py gpurun_out/prof/cfg2_sjlt_full.ncu-rep
  echo
  echo "## config 4 sketch kernels (SRHT passes 1 / 2, fp32 2^21-row block, m = 4096) -- cfg4_srht_full.ncu-rep"
  echo
  python tools/ncu_summary.py gpurun_out/prof/cfg4_srht_full.ncu-rep
} > profiles/r01_ncu_full_summary.md
echo wrote profiles/r01_ncu_full_summary.md
