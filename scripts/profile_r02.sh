#!/bin/bash
# ncu evidence for round 2: launch list (device-time share) + --set full of the step kernels at a
# steady-state keyframe (C2, keyframe ~150).   gpurun -- 'bash scripts/profile_r02.sh <tag>'
set -u
TAG=${1:-r02prof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --profile-steps 1 > $OUT/launches_bench.log 2>&1; echo "launches rc=$?"
RE='regex:k_match|k_tri$|k_fuse_rev|k_fuse_apply|k_cull|k_fuse_targets|k_fuse_refresh|k_fuse_gather|k_fuse_post|k_commit$'
timeout 1500 ncu --set full --clock-control none --import-source on -k "$RE" --launch-skip 1500 --launch-count 10 \
  -o $OUT/full -f python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --profile-steps 0 > $OUT/full_bench.log 2>&1; echo "full rc=$?"
ls -la $OUT
