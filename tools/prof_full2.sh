# ncu --set full of K9 (first launch) -- one tool per gpurun call
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/plain_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_window_sa -s 0 -c 1 -o gpurun_out/r01_k9_full $CMD > gpurun_out/ncu_f1.log 2>&1
echo "k9 rc=$?"
