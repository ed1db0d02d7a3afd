# one ncu --set full capture of kernel $1 (launch index skip $2) in the C4 bench
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/plain_k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$1 -s ${2:-0} -c 1 -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_k.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_k.log
