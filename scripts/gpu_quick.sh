#!/bin/bash
# Quick GPU round trip after a kernel change: parity subset, then the bench
# on the given configs (device ms per step + phases).
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_full_size.py} -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
for c in ${CFGS:-3 1 2}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline > gpurun_out/quick_c$c.json 2> gpurun_out/quick_c$c.err
  echo "c$c rc=$?"
  python -c "import json; l=json.load(open('gpurun_out/quick_c$c.json')); print('c$c', round(l['ms_per_step'],4), l.get('phase_ms'), l['roofline']['frac'], l['e2e']['value'])"
done
