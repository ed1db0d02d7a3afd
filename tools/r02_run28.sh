mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rt28.csv python tools/replay_time.py > /dev/null 2>&1; echo "list rc=$?"
python tools/launch_summary.py gpurun_out/launches_rt28.csv | head -24
