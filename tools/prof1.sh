# launch list + one full ncu capture of the top kernel (C4 bench, 1 step)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 70 -c 2 -o gpurun_out/prof_onesweep $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
cat gpurun_out/plain.log
