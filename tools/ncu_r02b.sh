#!/bin/bash
# Second set of round-2 `ncu --set full` captures (one GPU), the kernels at the
# sizes of configs 2-4 that the config-1 run of tools/ncu_r02.sh does not reach:
#   * the dense (K-outer) DMMA Gram at config 2's largest sketch (65536 x 2048 fp64),
#   * the Woodbury (K-contiguous) DMMA Gram at m = 1024, d = 2048,
#   * the TF32 tcgen05 Gaussian sketch at config 3 (2^21 x 4096, m = 2048),
#   * one sub-block launch of the fused SRHT and the combine kernel of a
#     config-4 block (2^21 x 1024 fp32, m = 4096),
#   * the streamed SJLT accumulation at config 2 (2^20 x 2048 fp64, m = 2048).
# Each command runs once without ncu first.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on -f"
cat > /tmp/gram_one.py <<'P'
import sys, torch
sys.path.insert(0, ".")
from paper_2104_14101_b200.preconditioner import gram_dev, woodbury_gram_dev
SA = torch.randn(65536, 2048, dtype=torch.float64, device="cuda")
lam = torch.rand(2048, dtype=torch.float64, device="cuda") * 9 + 1
for _ in range(3):
    gram_dev(SA, 1e-6, lam)
for _ in range(3):
    woodbury_gram_dev(SA[:1024], 1e-6, lam)
torch.cuda.synchronize()
print("done")
P
cat > /tmp/sjlt_one.py <<'P'
import sys, torch
sys.path.insert(0, ".")
from paper_2104_14101_b200.embeddings import sjlt_dev
A = torch.randn(1 << 20, 2048, dtype=torch.float64, device="cuda")
for _ in range(3):
    sjlt_dev(A, 2048, 7)
torch.cuda.synchronize()
print("done")
P
python /tmp/gram_one.py > gpurun_out/ncu_b_plain.log 2>&1 || { echo "gram plain failed"; tail -3 gpurun_out/ncu_b_plain.log; }
$NCU -k regex:k_gram_dmma -s 2 -c 1 -o gpurun_out/r02b_gram_dense python /tmp/gram_one.py > gpurun_out/ncu_b_gram.log 2>&1; echo "gram dense rc=$?"
$NCU -k regex:k_gram_dmma -s 5 -c 1 -o gpurun_out/r02b_gram_woodbury python /tmp/gram_one.py >> gpurun_out/ncu_b_gram.log 2>&1; echo "gram woodbury rc=$?"
MS=2048 REPS=1 python tools/tc_probe.py >> gpurun_out/ncu_b_plain.log 2>&1 || echo "tc plain failed"
MS=2048 REPS=1 $NCU -k regex:k_gauss_tc -s 1 -c 1 -o gpurun_out/r02b_gauss_tc python tools/tc_probe.py > gpurun_out/ncu_b_tc.log 2>&1; echo "gauss tc rc=$?"
M=4096 python tools/srht_one.py >> gpurun_out/ncu_b_plain.log 2>&1 || echo "srht plain failed"
M=4096 $NCU -k regex:k_srht_fused -s 11 -c 1 -o gpurun_out/r02b_srht_sub python tools/srht_one.py > gpurun_out/ncu_b_srht.log 2>&1; echo "srht sub-block rc=$?"
M=4096 $NCU -k regex:k_srht_combine -s 1 -c 1 -o gpurun_out/r02b_srht_combine python tools/srht_one.py >> gpurun_out/ncu_b_srht.log 2>&1; echo "srht combine rc=$?"
python /tmp/sjlt_one.py >> gpurun_out/ncu_b_plain.log 2>&1 || { echo "sjlt plain failed"; tail -3 gpurun_out/ncu_b_plain.log; }
$NCU -k regex:k_sjlt_pipe -s 2 -c 1 -o gpurun_out/r02b_sjlt python /tmp/sjlt_one.py > gpurun_out/ncu_b_sjlt.log 2>&1; echo "sjlt rc=$?"
ls -la gpurun_out/*.ncu-rep
