# one ncu --set full capture of the kernel whose DEMANGLED name matches regex $1 (skip $2 launches)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-c3 --cpu-budget 0.1"
NAME=${3:-$1}
$CMD > gpurun_out/plain_k.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$1" -s ${2:-0} -c 1 -o "gpurun_out/prof_$NAME" $CMD > gpurun_out/ncu_k.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_k.log
