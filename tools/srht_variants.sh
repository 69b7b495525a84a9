#!/bin/bash
# SRHT timing at config-1 and config-4 block shapes, pass-1 bit split ADASK_FWHT_B1 variants
for b1 in ${B1S:-default}; do
  if [ "$b1" = default ]; then unset ADASK_FWHT_B1; else export ADASK_FWHT_B1=$b1; fi
  echo "== b1=$b1"; WHICH=srht timeout 120 python tools/sketch_probe.py; WHICH=srht4 timeout 120 python tools/sketch_probe.py
done
