mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
CMD="python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/c3_plain.json 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/c3_views.csv $CMD > gpurun_out/c3_ncu.log 2>&1; echo "ncu rc=$?"
python tools/c3_views.py gpurun_out/c3_views.csv 3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv $CMD > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/c3_launches.csv | head -25
