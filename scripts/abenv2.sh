#!/bin/bash
# A/B of environment settings, any stages: STAGES="tri fuse_refresh" bash scripts/abenv2.sh "" "LM_X=1" ...
mkdir -p gpurun_out/ab
REPS=${REPS:-2}
for r in $(seq $REPS); do
  i=0
  for e in "$@"; do
    i=$((i+1))
    env $e timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab/V$i.$r.json 2> gpurun_out/ab/V$i.$r.err
    python -c "
import json; d=json.load(open('gpurun_out/ab/V$i.$r.json')); s=d['stage_ms_per_step']
print('[$e]', $r, round(d['value'],1), ' '.join(k+'='+str(round(s[k],2)) for k in '${STAGES:-fuse_rev fuse_apply}'.split()), d['parity']['final_digest_equal_reference'])"
  done
done
