#!/bin/bash
# Per-SASS-line executed instructions + stall samples of the C3 streaming
# kernels (one launch each), exported as CSV (reports removed).
OUT=gpurun_out/src
mkdir -p $OUT
CMD="python bench.py --config ${CFG:-3} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 900 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:"${KREGEX:-k_prefilter|k_prep_stream}" -s ${SKIP:-2} -c ${COUNT:-2} -o $OUT/prof $CMD > $OUT/ncu.log 2>&1
echo "ncu rc=$?"
for k in $(echo "${KREGEX:-k_prefilter|k_prep_stream}" | tr '|' ' '); do
  ncu -i $OUT/prof.ncu-rep --page source --csv -k regex:$k --print-source sass > $OUT/src_$k.csv 2>/dev/null
done
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
rm -f $OUT/prof.ncu-rep
