mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/pf_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_c4.csv $CMD > gpurun_out/pf_list.log 2>&1
echo "list rc=$?"
$CMD > gpurun_out/pf_plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_window_sa|k_onesweep" -s 2 -c 3 -o gpurun_out/r01_full $CMD > gpurun_out/pf_full.log 2>&1
echo "full rc=$?"
