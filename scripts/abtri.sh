#!/bin/bash
# A/B of k_tri slices per neighbour: bash scripts/abtri.sh [reps]
mkdir -p gpurun_out/ab
for r in $(seq ${1:-2}); do
  for s in 1 2 4 8; do
    LM_TRI_SLICES=$s timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab/tri$s.$r.json 2> gpurun_out/ab/tri$s.$r.err
    python -c "import json; d=json.load(open('gpurun_out/ab/tri$s.$r.json')); s=d['stage_ms_per_step']; print('slices $s', $r, round(d['value'],1), 'tri', round(s['tri'],2), 'commit', round(s['commit'],2), d['parity']['final_digest_equal_reference'])"
  done
done
