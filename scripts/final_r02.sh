#!/bin/bash
# Round-2 evidence run: GPU tests, smoke, the default bench line, every BASELINE config, and the
# ncu launch list + --set full capture.   gpurun --timeout 3600 -- 'bash scripts/final_r02.sh <tag>'
set -u
TAG=${1:-r02final}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "reference rc=$?"
for w in c1 c3 c4; do
  timeout 900 python bench.py --workload $w --steps 2 --warmup 1 --no-cpu --no-api > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "$w rc=$?"
done
timeout 900 python bench.py --workload c5 --steps 3 --warmup 2 --no-cpu > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "c5 rc=$?"
bash scripts/profile_r02.sh ${TAG}_prof
ls -la $OUT
