#!/bin/bash
# Launch list + full captures for one config (CFG, KREGEX, SKIP, COUNT), each
# ncu run after the same command exited 0 without ncu. Outputs under
# gpurun_out/ncu_c$CFG/ (reports summarized there, then removed).
CFG=${CFG:-3}
OUT=gpurun_out/ncu_c$CFG
mkdir -p $OUT
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -c ${NLAUNCH:-600} --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 300 $CMD > $OUT/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-4} \
    -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
echo "full rc=$?"
python scripts/ncu_summarize.py r02 $OUT/prof.ncu-rep:c$CFG --launches $OUT/launches.csv:c$CFG > $OUT/summary.log 2>&1
cp profiles/r02/ncu_summary.json $OUT/ncu_summary.json 2>/dev/null
for k in $(echo "${KREGEX}" | tr '|' ' '); do
  python scripts/ncu_hot.py $OUT/prof.ncu-rep "$k" 30 > $OUT/hot_$k.txt 2>&1
done
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
rm -f $OUT/prof.ncu-rep
