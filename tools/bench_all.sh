#!/bin/bash
# All five BASELINE configs through bench.py (one GPU), JSON lines into gpurun_out/bench/
mkdir -p gpurun_out/bench
for c in 0 1 2 3 4; do
  steps=5; [ $c -ge 2 ] && steps=2
  timeout 1200 python bench.py --config $c --steps $steps --warmup 3 > gpurun_out/bench/cfg$c.log 2>&1
  echo "cfg$c rc=$? $(tail -1 gpurun_out/bench/cfg$c.log | cut -c1-160)"
done
