#!/bin/bash
# One measurement pass for profiles/<round>: bench lines (all configs + the
# reference arm), the C2 launch list and full ncu captures of the dominance
# kernels (each ncu run only after the same command exited 0 without ncu).
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
CMD2="python bench.py --config 2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $CMD2 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -c 400 --csv --log-file gpurun_out/round/launches_c2.csv $CMD2 > /dev/null 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_relsky3|k_prefilter" -s 6 -c 4 -o gpurun_out/round/prof_c2 $CMD2 > gpurun_out/round/ncu_c2.log 2>&1
echo "ncu c2 rc=$?"
CMD4="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $CMD4 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_relsky3|k_bnl2" -s 2 -c 4 -o gpurun_out/round/prof_c4 $CMD4 > gpurun_out/round/ncu_c4.log 2>&1
echo "ncu c4 rc=$?"
timeout 600 python -m pytest tests/test_acceptance.py -q -s > gpurun_out/round/acceptance.log 2>&1
echo "acceptance rc=$?"
