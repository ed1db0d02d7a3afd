# usage: run_cfg.sh CONFIG variant...
C=$1; shift
for v in "$@"; do
  echo "== $v $C"
  APO_LIB=tools/variants/libapo_$v.so python bench.py --config $C --steps 3 --warmup 2 --no-e2e --cpu-budget 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), round(d['ms_per_step'],3))"
done
echo "== current $C"
python bench.py --config $C --steps 3 --warmup 2 --no-e2e --cpu-budget 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), round(d['ms_per_step'],3))"
