for cfg in "--c5-groups 8" "--c5-groups 0" "--c5-groups 2"; do
  timeout 600 python bench.py --workload c5 --sessions 8 --no-cpu --no-e2e --steps 3 --warmup 2 $cfg > /tmp/c5x.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/c5x.json').read().strip().splitlines()[-1]); print('s8 $cfg', round(d['value']))"
done
LM_PDL=0 timeout 600 python bench.py --workload c5 --sessions 8 --no-cpu --no-e2e --steps 3 --warmup 2 --c5-groups 8 > /tmp/c5x.json 2>/dev/null
python -c "import json; d=json.loads(open('/tmp/c5x.json').read().strip().splitlines()[-1]); print('s8 groups8 PDL0', round(d['value']))"
for S in 16 32 64; do
  timeout 600 python bench.py --workload c5 --sessions $S --no-cpu --no-e2e --steps 3 --warmup 2 > /tmp/c5x.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/c5x.json').read().strip().splitlines()[-1]); print('s$S auto', round(d['value']))"
done
