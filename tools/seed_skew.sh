mkdir -p gpurun_out
for r in 0 1 2 3 4 5 6 7; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --cpu-budget 0.5 --workload-rank $r > gpurun_out/skew_$r.json 2> gpurun_out/skew_$r.err || tail -5 gpurun_out/skew_$r.err
  python -c "
import json; d=json.loads(open('gpurun_out/skew_$r.json').read().strip().splitlines()[-1])
print($r, round(d['ms_per_step'],2), d['config']['stage_ms_per_step'], d['config'].get('traces'))"
done
