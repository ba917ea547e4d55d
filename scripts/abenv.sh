#!/bin/bash
# A/B of environment settings on one build: bash scripts/abenv.sh "" "LM_CARVEOUT=0" ...
mkdir -p gpurun_out/ab
REPS=${REPS:-2}
for r in $(seq $REPS); do
  i=0
  for e in "$@"; do
    i=$((i+1))
    env $e timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab/E$i.$r.json 2> gpurun_out/ab/E$i.$r.err
    python -c "import json; d=json.load(open('gpurun_out/ab/E$i.$r.json')); s=d['stage_ms_per_step']; print('[$e]', $r, round(d['value'],1), round(s['fuse_rev'],2), round(s['fuse_apply'],2), round(s['cull'],2))"
  done
done
