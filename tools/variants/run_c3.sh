for v in lb16 lb32; do
  echo "== $v"
  APO_LIB=tools/variants/libapo_$v.so python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --cpu-budget 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), round(d['ms_per_step'],3), d['roofline']['achieved'], d['roofline']['share_of_step'])"
done
echo "== current"
python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --cpu-budget 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), round(d['ms_per_step'],3), d['roofline']['achieved'], d['roofline']['share_of_step'])"
