CMD="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/pf_plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_window_sa -s 0 -c 1 -o gpurun_out/r01_k9 $CMD > gpurun_out/pf_k9.log 2>&1
echo "k9 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 84 -c 1 -o gpurun_out/r01_k1 $CMD > gpurun_out/pf_k1.log 2>&1
echo "k1 rc=$?"
