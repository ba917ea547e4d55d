#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list and a --set full capture.
#   gpurun --timeout 1500 -- 'bash scripts/gpu_check.sh <tag> [what...]'
# what: tests smoke bench launches full c5 (default: all but c5)
set -u
TAG=${1:-r01}; shift || true
WHAT=${*:-tests smoke bench launches full}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/gpu.txt 2>&1
has() { [[ " $WHAT " == *" $1 "* ]]; }
if has tests; then timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log; fi
if has smoke; then timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log; fi
if has bench; then timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 3000 $OUT/bench.json; tail -5 $OUT/bench.err; fi
if has c5; then timeout 900 python bench.py --workload c5 --no-cpu > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "c5 rc=$?"; tail -c 1500 $OUT/bench_c5.json; tail -5 $OUT/bench_c5.err; fi
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $OUT/launches_bench.log 2>&1; echo "launches rc=$?"
fi
if has full; then
  # steady-state keyframes: skip the first ~100 keyframes' launches, capture the hot kernels
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_match|k_fuse_rev|k_fuse_gather|k_fuse_spec|k_tri|k_fuse_apply' --launch-skip 600 --launch-count 12 \
    -o $OUT/full -f python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $OUT/full_bench.log 2>&1; echo "full rc=$?"
fi
ls -la $OUT
