#!/bin/bash
# Cholesky timing: blocked diagonal pivot loop vs the unblocked one
echo "== blocked"; KS=${KS:-256,1024,2048} NOSPIN=1 timeout 200 python tools/chol_probe.py 2>&1 | grep 'chol NB'
echo "== unblocked"; ADASK_CHOL_SLOWDIAG=1 KS=${KS:-256,1024,2048} NOSPIN=1 timeout 200 python tools/chol_probe.py 2>&1 | grep 'chol NB'
