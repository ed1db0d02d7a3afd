python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for C in C3 C2 C5; do timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --cpu-budget 0.1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C', round(d['value']/1e6,1), round(d['ms_per_step'],3))"; done
