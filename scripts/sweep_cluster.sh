#!/bin/bash
# bench.py under several forward-apply cluster widths (LM_APPLY_CLUSTER)
mkdir -p gpurun_out/sweep
for c in ${*:-1 4 8 16}; do
  LM_APPLY_CLUSTER=$c timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/sweep/c$c.json 2> gpurun_out/sweep/c$c.err
  python -c "import json; d=json.load(open('gpurun_out/sweep/c$c.json')); print($c, round(d['value'],1), round(d['stage_ms_per_step']['fuse_apply'],1), d['work_per_step']['apply_rounds'])"
done
