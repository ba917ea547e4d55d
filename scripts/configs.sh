#!/bin/bash
# Every BASELINE config through bench.py (C1..C4 single session, C5 batched)
mkdir -p gpurun_out/configs
for w in c1 c3 c4; do
  timeout 900 python bench.py --workload $w --steps 2 --warmup 1 --no-cpu > gpurun_out/configs/$w.json 2> gpurun_out/configs/$w.err
  echo "$w rc=$?"; python -c "import json; d=json.load(open('gpurun_out/configs/$w.json')); print('$w', round(d['value'],1), 'KF/s', round(d['ms_per_keyframe'],3), 'ms/KF', 'e2e', round(d['e2e']['value'],1), d['work_per_step']['created'], d['work_per_step']['merged'])" 2>&1 | tail -1
done
timeout 900 python bench.py --workload c5 --steps 3 --warmup 2 --no-cpu > gpurun_out/configs/c5.json 2> gpurun_out/configs/c5.err
echo "c5 rc=$?"; python -c "import json; d=json.load(open('gpurun_out/configs/c5.json')); print('c5', round(d['value'],1), 'KF/s', round(d['ms_per_step'],1), 'ms/step')" 2>&1 | tail -1
