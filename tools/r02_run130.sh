# launch lists of the N = 1 / N = 4 (union) match on one GPU
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
for N in 1 4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/um$N.csv python tools/union_match_probe.py $N > gpurun_out/um$N.log 2>&1; echo "ncu $N rc=$?"
  python tools/launch_summary.py gpurun_out/um$N.csv | head -32 > gpurun_out/um${N}_summary.txt
done
