# union build on one GPU: timing + launch list
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 600 python tools/union_build_probe.py 4 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ub4.csv python tools/union_build_probe.py 4 > gpurun_out/ub4.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/ub4.csv')) if len(r)>10]
h=rows[0]; rows=rows[1:]
ki=h.index('Kernel Name'); vi=h.index('Metric Value')
# the last 7 union builds: take launches after the last k_window_sa
last=max(i for i,r in enumerate(rows) if 'k_window_sa' in r[ki])
tail=rows[last+1:]
import collections
agg=collections.OrderedDict()
for r in tail:
    k=r[ki].split('(')[0].replace('void ','').replace('apo::','').replace('(anonymous namespace)::','')[:50]
    a=agg.setdefault(k,[0,0.0]); a[0]+=1; a[1]+=float(r[vi].replace(',',''))
tot=sum(a[1] for a in agg.values())
for k,a in sorted(agg.items(), key=lambda x:-x[1][1])[:25]: print(f"{k:50s} {a[0]//7:4d}/build {a[1]/7/1e3:8.3f} ms")
print('total per build', tot/7/1e3)
PY
