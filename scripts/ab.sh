#!/bin/bash
# A/B of alternative library builds in one box: bash scripts/ab.sh ab/A.so ab/B.so [reps]
mkdir -p gpurun_out/ab
REPS=${REPS:-3}
for r in $(seq $REPS); do
  for lib in "$@"; do
    n=$(basename $lib .so)
    LM_B200_LIB=$PWD/$lib timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab/$n.$r.json 2> gpurun_out/ab/$n.$r.err
    python -c "import json; d=json.load(open('gpurun_out/ab/$n.$r.json')); s=d['stage_ms_per_step']; print('$n', $r, round(d['value'],1), round(s['fuse_rev'],2), round(s['fuse_apply'],2))"
  done
done
