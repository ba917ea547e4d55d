#!/bin/bash
# compute-sanitizer evidence: racecheck + synccheck on small golden workloads,
# memcheck on a C2 prefix.   gpurun --timeout 2400 -- 'bash scripts/sanitize.sh <tag>'
set -u
TAG=${1:-san}; OUT=gpurun_out/$TAG; mkdir -p $OUT
CS="compute-sanitizer --error-exitcode 9 --print-limit 50"
for w in orbit7 line14dup; do
  timeout 1200 $CS --tool racecheck --racecheck-report all python tools/sanitize_run.py $w 8 > $OUT/racecheck_$w.log 2>&1; echo "racecheck $w rc=$?" | tee -a $OUT/summary.txt
  timeout 1200 $CS --tool synccheck python tools/sanitize_run.py $w 8 > $OUT/synccheck_$w.log 2>&1; echo "synccheck $w rc=$?" | tee -a $OUT/summary.txt
done
timeout 1800 $CS --tool memcheck --leak-check full python tools/sanitize_run.py c2 12 > $OUT/memcheck_c2.log 2>&1; echo "memcheck c2 rc=$?" | tee -a $OUT/summary.txt
timeout 1200 $CS --tool initcheck python tools/sanitize_run.py line14dup 8 > $OUT/initcheck_line14dup.log 2>&1; echo "initcheck line14dup rc=$?" | tee -a $OUT/summary.txt
for f in $OUT/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|sanitize_run|Error|error" $f | head -8; done
