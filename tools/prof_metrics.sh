# selected metrics of kernel $1 (regex) in the C4 bench (1 warm-up + 1 timed step)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/plain_m.log 2>&1 && \
ncu --metrics ${2:-gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct} --clock-control none -k regex:$1 --csv --log-file gpurun_out/metrics_$1.csv $CMD > gpurun_out/ncu_m.log 2>&1
echo "rc=$?"
python - "$1" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/metrics_{sys.argv[1]}.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
for r in rows[hi + 1:]:
    if len(r) > 5:
        print(r[h.index("ID")], r[h.index("Kernel Name")][:40], r[h.index("Metric Name")], r[h.index("Metric Value")], r[h.index("Metric Unit")])
PY
