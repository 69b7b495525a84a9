#!/bin/bash
# SRHT timing at config-1 and config-4 block shapes: persistent TMA pipeline vs tile kernels
echo "== tile kernels"; ADASK_FWHT_NOPIPE=1 WHICH=srht timeout 120 python tools/sketch_probe.py; ADASK_FWHT_NOPIPE=1 WHICH=srht4 timeout 120 python tools/sketch_probe.py
echo "== pipe"; WHICH=srht timeout 120 python tools/sketch_probe.py; WHICH=srht4 timeout 120 python tools/sketch_probe.py
