#!/bin/bash
# Bench every BASELINE config on one GPU (+ the reference arm on C2); logs under gpurun_out/.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
for c in 2 1 3 5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "config $c rc=$?"
done
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "config 4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
echo "ref rc=$?"
