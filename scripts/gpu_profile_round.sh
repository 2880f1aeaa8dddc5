#!/bin/bash
# One measurement pass for profiles/<round>: bench lines (all configs + the
# reference arm), launch lists (C2, C3), full ncu captures of the dominance
# kernels (C2, C4) and of the HBM streaming passes (C3); each ncu run only
# after the same command exited 0 without ncu. Then the acceptance suite.
mkdir -p gpurun_out/round
cd "$(dirname "$0")/.."
nproc > gpurun_out/round/nproc.txt
for c in 2 1 3 5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/round/bench_c$c.json 2> gpurun_out/round/bench_c$c.err
  echo "bench c$c rc=$?"
done
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/round/bench_c4.json 2> gpurun_out/round/bench_c4.err
echo "bench c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/round/bench_ref_c2.json 2> gpurun_out/round/bench_ref_c2.err
echo "ref rc=$?"
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 2 3; do
  CMD="python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 300 $CMD > /dev/null 2>&1 && timeout 600 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/round/launches_c$c.csv $CMD > /dev/null 2>&1
  echo "launches c$c rc=$?"
done
CMD2="python bench.py --config 2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_relsky3|k_prefilter" -s 6 -c 4 -o gpurun_out/round/prof_c2 $CMD2 > gpurun_out/round/ncu_c2.log 2>&1
echo "ncu c2 rc=$?"
CMD3="python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_prep_stream|k_cand_bucket|k_prefilter" -s 3 -c 3 -o gpurun_out/round/prof_c3 $CMD3 > gpurun_out/round/ncu_c3.log 2>&1
echo "ncu c3 rc=$?"
CMD4="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $CMD4 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_relsky3|k_bnl2" -s 2 -c 4 -o gpurun_out/round/prof_c4 $CMD4 > gpurun_out/round/ncu_c4.log 2>&1
echo "ncu c4 rc=$?"
timeout 600 python -m pytest tests/test_acceptance.py -q -s > gpurun_out/round/acceptance.log 2>&1
echo "acceptance rc=$?"
# reports are large (gpurun_out travels back only under 64 MiB): summarize
# here, keep the hot-spot listings, drop the reports
python scripts/ncu_summarize.py round gpurun_out/round/prof_c2.ncu-rep:c2 gpurun_out/round/prof_c4.ncu-rep:c4 \
    gpurun_out/round/prof_c3.ncu-rep:c3:stream --launches gpurun_out/round/launches_c2.csv:c2 \
    gpurun_out/round/launches_c3.csv:c3 > gpurun_out/round/ncu_summary.log 2>&1
cp profiles/round/ncu_summary.json gpurun_out/round/ncu_summary.json
for k in k_prep_stream k_cand_bucket k_prefilter; do
  python scripts/ncu_hot.py gpurun_out/round/prof_c3.ncu-rep $k 25 > gpurun_out/round/hot_c3_$k.txt 2>&1
done
for k in k_relsky3 k_bnl2; do
  python scripts/ncu_hot.py gpurun_out/round/prof_c4.ncu-rep $k 25 > gpurun_out/round/hot_c4_$k.txt 2>&1
done
rm -f gpurun_out/round/*.ncu-rep
