mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 40 -c 2 -o gpurun_out/prof_onesweep2 $CMD > gpurun_out/ncu_full2.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full2.log
