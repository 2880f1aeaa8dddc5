#!/bin/bash
# Bench every BASELINE config on one GPU plus the reference arm on the
# default config; JSON lines under gpurun_out/r02/.
OUT=gpurun_out/r02
mkdir -p $OUT
nproc > $OUT/nproc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
for c in 3 2 1 5 4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
  echo "bench c$c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_c3.json 2> $OUT/bench_ref_c3.err
echo "ref rc=$?"
timeout 400 python scripts/issue_peak.py > $OUT/issue_peak.log 2>&1
echo "issue peak rc=$?"
