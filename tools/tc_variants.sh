#!/bin/bash
# timing variants of the tcgen05 Gaussian kernel (ADASK_TC_DEBUG bit flags:
# 4 = no S generation, 8 = no A traffic, 16 = 7 Philox rounds, 32 = no
# Box-Muller; ADASK_TC_NOCLUSTER = no multicast)
for v in ${VARIANTS:-0 4 8 12 24 40}; do
  echo "== ADASK_TC_DEBUG=$v"; ADASK_TC_DEBUG=$v MS=${MS:-512,2048} timeout 120 python tools/tc_probe.py 2>&1 | tail -2
done
