python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for r in 1 2; do python tools/match_time.py 2>&1 | tail -1; done
timeout 900 python bench.py --cpu-budget 1 --no-c3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,1), d['config']['stage_ms_per_step'])"
