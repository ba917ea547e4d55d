#!/bin/bash
# C5 (batched sessions) under several environment settings: bash scripts/c5ab.sh "" "LM_PDL=1"
mkdir -p gpurun_out/c5ab
for e in "$@"; do
  env $e timeout 600 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/c5ab/o.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c5ab/o.json')); print('[$e]', round(d['value'],1))"
done
