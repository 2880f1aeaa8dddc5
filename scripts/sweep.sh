#!/bin/bash
# parameter sweep of the C2 step (device ms per step, 10 steps)
for v in "SKY_SFS_HEAD=1024" "SKY_SFS_HEAD=2048" "SKY_SFS_HEAD=4096" "SKY_SFS_CHUNK=1024" "SKY_SFS_CHUNK=4096" "SKY_MERGE_HEAD=2048" "SKY_MERGE_HEAD=8192" "SKY_MERGE_HEAD=16384"; do
  r=$(env $v timeout 300 python bench.py --config ${CFG:-2} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(round(l['ms_per_step'],4), {k: round(x,3) for k,x in l['phase_ms'].items()}, l['tests_per_step'])")
  echo "$v $r"
done
