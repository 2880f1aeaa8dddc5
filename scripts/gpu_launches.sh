#!/bin/bash
# Launch list (per-kernel device time, serialised) of one bench config.
CFG=${CFG:-3}
OUT=gpurun_out/launch_c$CFG
mkdir -p $OUT
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-200} --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu.log 2>&1
echo "launch list rc=$?"
