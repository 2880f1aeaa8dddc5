#!/bin/bash
# A/B of an environment knob on one config: device ms per step, alternating runs
for rep in 1 2 3; do
  for v in "$A" "$B"; do
    r=$(env $v timeout 300 python bench.py --config ${CFG:-2} --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(round(l['ms_per_step'],4), round(l['phase_ms']['local'],4), round(l['phase_ms']['merge'],4))")
    echo "$v $r"
  done
done
