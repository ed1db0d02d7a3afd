for v in ${@}; do
  echo "== $v C4"
  APO_LIB=tools/variants/libapo_$v.so python bench.py --steps 3 --warmup 3 --no-e2e --cpu-budget 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), round(d['ms_per_step'],3))"
done
