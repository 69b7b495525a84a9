#!/bin/bash
# One GPU-box pass: the GPU test tier, the reference suite through the shim,
# and the bench lines (config 1 default; config 2 with its full-size CPU
# baseline).  Output under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rfE > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
python tools/run_reference_suite.py -- -q -rf 2>&1 | grep -E "passed|failed|FAILED" > gpurun_out/refsuite_summary.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
tail -3 gpurun_out/gputests.log; cat gpurun_out/refsuite_summary.log
