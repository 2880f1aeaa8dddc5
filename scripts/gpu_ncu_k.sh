#!/bin/bash
# One full ncu capture of a kernel regex on a given bench config (plain run first).
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-2} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu_plain_${TAG:-x}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_relsky3} -s ${SKIP:-0} -c ${COUNT:-1} \
    -o gpurun_out/prof_${TAG:-x} $CMD > gpurun_out/ncu_full_${TAG:-x}.log 2>&1
echo "full rc=$?"
