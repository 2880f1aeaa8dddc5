#!/bin/bash
# parameter sweep of one config's step (device ms per step, 20 steps, best of 2)
run() {
  for rep in 1 2; do
    env "$@" timeout 300 python bench.py --config ${CFG:-2} --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(round(l['ms_per_step'],4), {k: round(x,3) for k,x in l['phase_ms'].items()})"
  done
}
for v in "X=0" "SKY_SFS_TILE=128" "SKY_SFS_TILE=64" "SKY_SFS_CHUNK=1024" "SKY_SFS_CHUNK=512" "SKY_GRAIN_ITEMS=8" "SKY_GRAIN_ITEMS=16" "SKY_SFS_TILE=128 SKY_SFS_CHUNK=1024 SKY_GRAIN_ITEMS=8"; do
  echo "== $v"; run $v
done
