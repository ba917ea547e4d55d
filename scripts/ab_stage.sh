#!/bin/bash
# A/B of library builds, printing one stage: STAGE=match REPS=2 bash scripts/ab_stage.sh ab/A.so ab/B.so ...
mkdir -p gpurun_out/ab
REPS=${REPS:-2}; STAGE=${STAGE:-match}
for r in $(seq $REPS); do
  for lib in "$@"; do
    n=$(basename $lib .so)
    LM_B200_LIB=$PWD/$lib timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab/$n.$r.json 2> gpurun_out/ab/$n.$r.err
    python -c "import json; d=json.load(open('gpurun_out/ab/$n.$r.json')); s=d['stage_ms_per_step']; print('$n', $r, round(d['value'],1), '$STAGE', round(s['$STAGE'],3), 'parity', d['parity'].get('final_digest_equal_reference'))"
  done
done
