#!/bin/bash
# Round-2 ncu evidence: launch lists (C2-C5) and full captures of the top
# kernels (C2 dominance + compaction + run merge, C3 streaming passes, C4
# merge + BNL, C5 random partitioner), each ncu run after the same command
# exited 0 without ncu. Summaries under gpurun_out/prof/ (reports removed).
OUT=gpurun_out/prof
mkdir -p $OUT
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 2 3 4 5; do
  CMD="python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 300 $CMD > $OUT/plain_c$c.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -c 800 --csv --log-file $OUT/launches_c$c.csv $CMD > $OUT/ncu_launch_c$c.log 2>&1
  echo "launches c$c rc=$?"
done
full() {  # config regex skip count tag
  CMD="python bench.py --config $1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 300 $CMD > $OUT/plain_full_$5.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c $4 -o $OUT/prof_$5 $CMD > $OUT/ncu_full_$5.log 2>&1
  echo "full $5 rc=$?"
}
full 2 "k_relsky3|k_prefilter|k_dc_|k_merge_runs|onesweep|k_prep" 0 24 c2
full 3 "k_prep_stream|k_prefilter|k_cand_bucket" 3 3 c3
full 4 "k_relsky3|k_bnl2" 0 10 c4
full 5 "k_mt|k_fy|onesweep" 0 12 c5
python scripts/ncu_summarize.py r02 $OUT/prof_c2.ncu-rep:c2 $OUT/prof_c4.ncu-rep:c4 $OUT/prof_c5.ncu-rep:c5 \
    $OUT/prof_c3.ncu-rep:c3:stream --launches $OUT/launches_c2.csv:c2 $OUT/launches_c3.csv:c3 \
    $OUT/launches_c4.csv:c4 $OUT/launches_c5.csv:c5 > $OUT/summary.log 2>&1
cp profiles/r02/ncu_summary.json $OUT/ncu_summary.json
for k in k_relsky3 k_bnl2; do python scripts/ncu_hot.py $OUT/prof_c4.ncu-rep $k 30 > $OUT/hot_c4_$k.txt 2>&1; done
for k in k_prep_stream k_prefilter k_cand_bucket; do python scripts/ncu_hot.py $OUT/prof_c3.ncu-rep $k 30 > $OUT/hot_c3_$k.txt 2>&1; done
for t in c2 c3 c4 c5; do ncu -i $OUT/prof_$t.ncu-rep --page details --csv > $OUT/details_$t.csv 2>/dev/null; done
rm -f $OUT/*.ncu-rep
