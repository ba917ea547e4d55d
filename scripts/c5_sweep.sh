#!/bin/bash
# Multi-GPU evidence that fits on one GPU: C5 at 8/16/32/64 sessions on one
# B200 (= each rank's load at G = 8/4/2/1), plus the two-rank rehearsal of the torchrun path on
# one device (LM_BENCH_SAME_DEVICE=1, gloo) for C2 and C5.
#   gpurun --timeout 2400 -- 'bash scripts/c5_sweep.sh <tag>'
set -u
TAG=${1:-c5sweep}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for S in 8 16 32 64; do
  timeout 900 python bench.py --workload c5 --sessions $S --no-cpu --steps 3 --warmup 2 > $OUT/c5_s$S.json 2> $OUT/c5_s$S.err
  python -c "import json; d=json.loads(open('$OUT/c5_s$S.json').read().strip().splitlines()[-1]); print('sessions', $S, round(d['value']), 'KF/s', 'e2e', round((d.get('e2e') or {}).get('value', 0)))"
done
export LM_BENCH_SAME_DEVICE=1 LM_BENCH_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 3 --warmup 2 --no-api > $OUT/rehearsal_c2_2ranks.json 2> $OUT/rehearsal_c2.err; echo "c2 2-rank rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --workload c5 --sessions 16 --steps 3 --warmup 2 > $OUT/rehearsal_c5_2ranks.json 2> $OUT/rehearsal_c5.err; echo "c5 2-rank rc=$?"
tail -c 600 $OUT/rehearsal_c2_2ranks.json; tail -c 400 $OUT/rehearsal_c5_2ranks.json
