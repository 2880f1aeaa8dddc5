#!/bin/bash
# Launch list + one full capture of the dominance kernel (run after the plain
# command exited 0, as the profiling recipe requires).
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-2} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-600} --csv \
    --log-file gpurun_out/launches_c${CFG:-2}.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
$CMD > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_relsky} -s ${SKIP:-8} -c ${COUNT:-3} \
    -o gpurun_out/prof_c${CFG:-2} $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
