# k_trace_ids A/B under N = 4 union conditions on one GPU
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
for m in 0 1 0 1; do APO_TID_MODE=$m timeout 600 python tools/union_match_probe.py 4 2>&1 | tail -2; done
APO_TID_MODE=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_trace_ids --csv --log-file gpurun_out/tid0.csv python tools/union_match_probe.py 4 > /dev/null 2>&1; echo "ncu0 rc=$?"
APO_TID_MODE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_trace_ids --csv --log-file gpurun_out/tid1.csv python tools/union_match_probe.py 4 > /dev/null 2>&1; echo "ncu1 rc=$?"
for f in gpurun_out/tid0.csv gpurun_out/tid1.csv; do grep -E "k_trace_ids" $f | awk -F'","' '{print $5, $NF}' | tail -3; done
